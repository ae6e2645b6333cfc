"""Summarise ncu captures into profiles/ (run here, after gpurun brought the reports back).

    python scripts/summarize_ncu.py gpurun_out C1 r01
writes profiles/ncu_traffic.json (dram bytes per launch, read by bench.py) and
profiles/<round>_ncu_<cfg>.md (key metrics per kernel + launch-list shares).
"""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
src, cfg, rnd = sys.argv[1], sys.argv[2], sys.argv[3]
KERNELS = {"refresh": "refresh_tc2", "reuse": "reuse_tc", "select": "select_heads", "lm_head": "lmhead"}
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
           "launch__registers_per_thread", "sm__cycles_elapsed.avg.per_second",
           "sm__warps_active.avg.pct_of_peak_sustained_active"]
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    return {h: (v, u) for h, u, v in zip(rows[0], rows[1], rows[2])}


path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
traffic = json.load(open(path)) if os.path.exists(path) else {}
lines = [f"# ncu summary, {rnd}, config {cfg}", "",
         "`ncu --set full --clock-control none` on one launch of each kernel (scripts/profile.sh, "
         "scripts/kbench.py); traffic = dram__bytes_read.sum + dram__bytes_write.sum of that launch.", ""]
for name, k in KERNELS.items():
    rep = os.path.join(src, f"prof_{cfg}_{k}.ncu-rep")
    if not os.path.exists(rep) and name == "lm_head":
        rep = os.path.join(src, "prof_N4_lmhead.ncu-rep")
    if not os.path.exists(rep):
        continue
    m = raw(rep)
    b = sum(float(m[x][0].replace(",", "")) * UNIT.get(m[x][1], 1) for x in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
    traffic.setdefault(cfg, {})[name] = {"kernel": k, "dram_bytes_per_launch": b, "round": rnd,
                                         "duration_us_under_ncu": float(m["gpu__time_duration.sum"][0].replace(",", "")) *
                                         {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(
                                             m["gpu__time_duration.sum"][1], 1.0)}
    lines.append(f"## {name} (`{k}`)")
    for x in METRICS:
        if x in m:
            lines.append(f"- {x} = {m[x][0]} {m[x][1]}")
    lines.append(f"- traffic (read + write) = {b / 1e6:.1f} MB per launch")
    lines.append("")
# launch list shares
ll = os.path.join(src, f"launches_{cfg}.csv")
if os.path.exists(ll):
    rows = [r for r in csv.reader(open(ll)) if len(r) > 14 and r[12] == "gpu__time_duration.sum"]
    tot = {}
    for r in rows:
        name = r[4].split("(")[0].replace("void ", "")
        tot[name] = tot.get(name, 0.0) + float(r[14].replace(",", ""))
    ours = {k: v for k, v in tot.items() if "dllm" in k}
    s = sum(ours.values())
    lines.append("## launch list (cold-cache, serialised; shares of our kernels)")
    for k, v in sorted(ours.items(), key=lambda x: -x[1]):
        lines.append(f"- {k}: {v / 1e3:.1f} us total, {100 * v / s:.1f}%")
json.dump(traffic, open(path, "w"), indent=1)
open(os.path.join(ROOT, "profiles", f"{rnd}_ncu_{cfg}.md"), "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
