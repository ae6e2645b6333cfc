"""CPU: the bench.py JSON-line contract, checked on the committed round record
(profiles/r02_bench_default_final.json, written by `python bench.py` on a B200) and
on a live `--impl reference` line (the fp64 oracle arm runs on the host)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
RECORD = os.path.join(ROOT, "profiles", "r02_bench_default_final.json")

BASE_KEYS = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config")


def _last_json_line(text):
    return json.loads([ln for ln in text.strip().splitlines() if ln.startswith("{")][-1])


def test_recorded_line_has_the_contract_keys():
    d = _last_json_line(open(RECORD).read())
    for k in BASE_KEYS + ("roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["scaling"] in ("weak", "strong") and d["higher_is_better"] is True
    assert d["config"]["workload"].startswith("C1:") and "l2" in d["config"]
    r = d["roofline"]
    assert r["bound"] == "tensor" and r["unit"] == "TFLOP/s"
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    # achieved = algorithmic FLOP of one Refresh launch / its mean CUDA-event time
    k = d["kernels"]["refresh"]
    assert abs(k["TFLOP/s"] - k["flop_per_launch"] / (k["us"] * 1e-6) / 1e12) < 1e-6 * k["TFLOP/s"]
    assert k["flop_per_launch"] == 4 * 32 * 1024 ** 2 * 128 * 16        # 4 H L^2 D per request, 16 requests
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    e = d["e2e"]
    assert e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0 and 0 < e["value"] < d["value"]
    assert d["gpu_launches"] > 0
    c = d["clocks"]
    assert not set(c["reasons"]) & {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}
    for cfg in ("C2", "C3", "C4"):
        assert cfg in d["configs"] and d["configs"][cfg]["ms_per_step"] > 0


def test_reference_arm_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "0"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    d = _last_json_line(out.stdout)
    for k in BASE_KEYS + ("cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["cpu_baseline"]["kind"] == "oracle"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"] > 0
