#!/usr/bin/env python
"""Benchmark of the Head-Centric Sparse Attention hot path (one JSON line).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C1] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...     (one process per GPU, NCCL)

A step = one pass of the whole hot path over one batch:
dllm_refresh_attn (Eq. 3 + importance) -> dllm_select_heads (Eq. 6 + TopK) ->
dllm_reuse_sparse_attn (Eq. 4), through the C-ABI.  At N=1 the batch is
BASELINE.json configs[1] (C1, LLaDA-8B layer shape: 16 requests, 32 heads,
D=128, L=1024, block 32, keep 0.25).  At N>1 every rank runs its LPT shard of
an N-times-replicated batch (weak scaling: 16 requests per GPU); there is no
collective on the data path (requests are independent).  The NCCL all-gather
of the per-request outputs is timed separately (`allgather_ms`).

value  = requests/s over all ranks = (requests per step * K) / max-over-ranks
         device time of the K steps (CUDA events on the launch stream; L2
         flushed before every step by a 512 MiB write outside the events).
e2e    = the same metric through the public API with HOST buffers: every step
         copies its inputs from pinned host memory to the device, runs the
         three calls and copies the results back (all inside the events).
roofline = the dominant kernel (Refresh, tensor-bound) against the measured
         bf16 peak in MEASURED_PEAKS.json; Reuse / select are reported in
         `kernels` against the measured HBM copy bandwidth.
cpu_baseline = the fp64 oracle (oracle/) timed on this host's cores on a
         bounded sample of the same workload (rank 0, N=1 only).
--impl reference runs that oracle as the reference arm (BASELINE has no
         runnable reference implementation: the paper ships no code).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Reuse sparse-attn HBM GB/s and Refresh TFLOPS vs peak; requests/s at 1/2/4/8 B200"
UNIT = "requests/s"


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return pk["bf16_tflops"], pk.get("bf16_tflops_sustained"), pk["hbm_gbs"], "measured"
    except Exception:
        return 1590.0, 1400.0, 6650.0, "fallback"


def workload_desc(wl, n):
    mix = "" if wl.refresh_mask is None else \
        f" ({sum(wl.refresh_mask)} Refresh+select+Reuse, {wl.num_requests - sum(wl.refresh_mask)} Reuse-only)"
    return (f"{wl.name}: {wl.num_requests} requests/GPU{mix} x {n} GPU, H={wl.num_heads}, H_kv={wl.num_kv_heads}, "
            f"D={wl.head_dim}, L={min(wl.seq_len)}..{max(wl.seq_len)}, blk={wl.blk[0]}, r={wl.keep_ratio}, "
            f"w={wl.pool_window}, page={wl.page_size}")


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """SM clocks, power and throttle reasons sampled through NVML every ~2 ms while
    the timed region runs (samples taken before the region starts are dropped).
    The timed region of a default run is only a few ms, so `extend(fn, seconds)`
    keeps replaying the same step afterwards, untimed, and records the clocks the
    workload settles at under the power cap (reported separately)."""

    def __init__(self, index: int):
        self.index, self.samples, self._stop = index, [], threading.Event()
        self._phase = None
        self._t = threading.Thread(target=self._run, daemon=True)
        self._ready = threading.Event()

    def _run(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            names = {"hw_slowdown": pynvml.nvmlClocksEventReasonHwSlowdown,
                     "hw_thermal_slowdown": pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                     "sw_thermal_slowdown": pynvml.nvmlClocksEventReasonSwThermalSlowdown,
                     "sw_power_cap": pynvml.nvmlClocksEventReasonSwPowerCap}
            self._ready.set()
            while not self._stop.is_set():
                ph = self._phase
                if ph is not None:
                    sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                    rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                    try:
                        pw = pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0
                    except Exception:
                        pw = None
                    self.samples.append((ph, sm, mx, sorted(k for k, v in names.items() if rs & v), pw))
                self._stop.wait(0.002)
        except Exception as e:  # pragma: no cover
            self.samples.append(("region", None, None, [f"nvml-error: {e}"], None))
            self._ready.set()

    def __enter__(self):
        self._t.start()
        self._ready.wait(timeout=30)
        self._phase = "region"
        return self

    def __exit__(self, *a):
        self._phase = None

    def extend(self, fn, seconds: float = 0.2):
        """Replay `fn` (one untimed step, device-synchronised by the caller's loop)
        for about `seconds` with sampling on, then stop the sampler."""
        import torch
        self._phase = "extended"
        t0 = time.perf_counter()
        while time.perf_counter() - t0 < seconds:
            fn()
            torch.cuda.synchronize()
        self._phase = None
        self._stop.set()
        self._t.join(timeout=10)

    def close(self):
        self._phase = None
        self._stop.set()
        self._t.join(timeout=10)

    @staticmethod
    def _summ(rows):
        sm = [r[1] for r in rows if r[1] is not None]
        mx = [r[2] for r in rows if r[2] is not None]
        pw = [r[4] for r in rows if r[4] is not None]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted({x for r in rows for x in r[3]}), "samples": len(rows),
                "power_w": statistics.median(pw) if pw else None}

    def summary(self):
        out = self._summ([r for r in self.samples if r[0] == "region"])
        ext = [r for r in self.samples if r[0] == "extended"]
        if ext:
            out["under_load_extended"] = self._summ(ext)
        return out


# ----------------------------------------------------------------------------- oracle (CPU) timing
def cpu_oracle_rate(wl, budget_s: float = 12.0, max_requests: int | None = None):
    """The fp64 oracle as it stands, on a bounded sample of the workload's
    requests (whole requests: Refresh + importance + select + Reuse, all heads;
    in a mixed batch the Refresh requests run Refresh + select and the
    reuse-only requests run Reuse alone on the same index lists as the GPU arm).  Returns (requests/s, requests timed, seconds, threads).
    For a mixed batch the rate is the batch's request count over the batch time
    extrapolated from the per-kind mean request times of the sample."""
    import torch

    import oracle as O
    from paper_2512_17077_b200 import synth
    cores = len(os.sched_getaffinity(0))
    torch.set_num_threads(cores)
    mask = wl.refresh_mask or [True] * wl.num_requests
    kinds = sorted(set(mask), reverse=True)
    order = [[b for b in range(wl.num_requests) if mask[b] == kd] for kd in kinds]
    per_kind = {}
    done, t_total = 0, 0.0
    for kd, reqs in zip(kinds, order):
        t_kind, n_kind = 0.0, 0
        # whole passes over the requests until the time budget is spent (C1 has only
        # 16 requests: a single pass is ~3 s of oracle time)
        for b in (reqs * 8 if max_requests is None else reqs):
            if max_requests is not None and done >= max_requests:
                break
            q, K, V, qb = (t.double().numpy() for t in synth.request_tensors(wl, b))
            bs, be, L = wl.blk_start[b], wl.blk_end[b], wl.seq_len[b]
            if not kd:
                k = O.keep_count(wl.keep_ratio, L - (be - bs))
                sel = synth.indices(synth.subset(wl, [b]), [k])[0]
            t0 = time.perf_counter()
            if kd:
                O.attention_dense(q, K, V)
                raw = O.raw_scores(q[bs:be], K)
                sel = O.select_batch([raw], [L], [bs], [be], wl.keep_ratio, wl.pool_window)[0]
            if not kd or wl.refresh_mask is None:
                # mixed (C3) batches: Refresh requests stop at select, as on the GPU leg
                O.attention_with_cache(qb, K, V, bs, be, sel)
            dt = time.perf_counter() - t0
            t_kind += dt
            t_total += dt
            n_kind += 1
            done += 1
            if t_kind >= budget_s / len(kinds):
                break
        if n_kind:
            per_kind[kd] = t_kind / n_kind
    if len(kinds) == 1:
        return done / t_total, done, t_total, cores
    t_batch = sum(per_kind.get(kd, 0.0) * len(reqs) for kd, reqs in zip(kinds, order))
    return wl.num_requests / t_batch, done, t_total, cores


# ----------------------------------------------------------------------------- ncu traffic
def ncu_traffic(kernel: str, cfg: str):
    """dram read+write bytes per launch from the committed `ncu --set full`
    summary (profiles/ncu_traffic.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            d = json.load(f)
        e = d.get(cfg, {}).get(kernel)
        return None if e is None else e.get("dram_bytes_per_launch")
    except Exception:
        return None


# ----------------------------------------------------------------------------- reference arm
def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2512_17077_b200 import synth
    wl = synth.config(args.config)
    rates = []
    for _ in range(args.warmup):
        cpu_oracle_rate(wl, budget_s=0.0, max_requests=1)
    t0 = time.perf_counter()
    n_req = 0
    for _ in range(args.steps):
        r, n, t, cores = cpu_oracle_rate(wl, budget_s=0.0, max_requests=1)
        rates.append(r)
        n_req += n
    wall = time.perf_counter() - t0
    value = n_req / wall
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * wall / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_desc(wl, 1), "sample": "1 request (all heads) per step"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": len(os.sched_getaffinity(0)), "kind": "oracle",
                             "sample": f"{args.steps} steps x 1 request of {wl.name} (Refresh+select+Reuse, all heads)"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- our arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C1")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-graph", action="store_true", help="time eager launches instead of a CUDA graph replay")
    ap.add_argument("--no-mixed", action="store_true",
                    help="C3: separate Refresh and Reuse launches instead of one mixed launch")
    ap.add_argument("--fused-select", action="store_true",
                    help="dllm_refresh_select_attn (select fused into the Refresh kernel when the library is built "
                         "with DLLM_TC2_FUSEDSEL=1) instead of dllm_refresh_attn + dllm_select_heads")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    from paper_2512_17077_b200 import lib, shard, synth

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    tf_peak, tf_sust, hbm_peak, peak_src = load_peaks()

    base = synth.config(args.config)
    glob = synth.replicate(base, world)
    k_glob = [lib.keep_count(glob.keep_ratio, L - (e - s)) for L, s, e in zip(glob.seq_len, glob.blk_start, glob.blk_end)]
    costs = [shard.request_cost(L, e - s, glob.num_heads, glob.num_kv_heads, glob.head_dim, k)
             for L, s, e, k in zip(glob.seq_len, glob.blk_start, glob.blk_end, k_glob)]
    parts = shard.lpt_partition(costs, world)
    wl = synth.subset(glob, parts[rank])
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device=dev)

    # A step runs Refresh -> select -> Reuse for every request (C1/C2/C4: the whole
    # hot path over the batch), except in a mixed (burst) batch (C3: refresh_mask,
    # SURVEY §8(d)): there the Refresh requests run Refresh + select (their block
    # output is the dense one; the new index lists serve their next Reuse steps)
    # and the others run Reuse alone with the index lists of an earlier selection
    # (generated once, outside the timed region).
    def make_part(sub, refresh):
        bt = synth.make_batch(sub)
        pp = lib.Problem(sub.seq_len, sub.blk_start, sub.blk_end, num_heads=sub.num_heads,
                         num_kv_heads=sub.num_kv_heads, head_dim=sub.head_dim, keep_ratio=sub.keep_ratio,
                         pool_window=sub.pool_window, page_size=sub.page_size, block_table=bt.block_table.to(dev))
        tens = [t.to(dev) for t in (bt.q, bt.q_blk, bt.k_cache, bt.v_cache)]
        bf = lib.alloc_buffers(pp, device=dev)
        if not refresh:
            kk = pp.layout()[0]
            flat = np.concatenate([x.reshape(-1) for x in synth.indices(sub, kk)]).astype(np.int32)
            if flat.size:
                bf.idx[:flat.size].copy_(torch.from_numpy(flat))
        return {"wl": sub, "batch": bt, "p": pp, "t": tens, "buf": bf, "refresh": refresh, "reuse": True}

    def make_part_shared(shared, dk, dv, reqs, refresh):
        # a phase of a mixed batch: its own problem (block-table rows of its requests)
        # over the batch's ONE paged cache
        sub = synth.subset(wl, reqs)
        pp = lib.Problem(sub.seq_len, sub.blk_start, sub.blk_end, num_heads=sub.num_heads,
                         num_kv_heads=sub.num_kv_heads, head_dim=sub.head_dim, keep_ratio=sub.keep_ratio,
                         pool_window=sub.pool_window, page_size=sub.page_size,
                         block_table=shared.block_table[reqs].contiguous().to(dev))
        q = torch.cat([shared.q_req(b) for b in reqs])
        qb = torch.cat([shared.q_blk_req(b) for b in reqs])
        bf = lib.alloc_buffers(pp, device=dev)
        if not refresh:
            kk = pp.layout()[0]
            flat = np.concatenate([x.reshape(-1) for x in synth.indices(sub, kk)]).astype(np.int32)
            if flat.size:
                bf.idx[:flat.size].copy_(torch.from_numpy(flat))
        host = {"q": q, "q_blk": qb, "k_cache": shared.k_cache, "v_cache": shared.v_cache}
        return {"wl": sub, "host": host, "p": pp, "t": [q.to(dev), qb.to(dev), dk, dv], "buf": bf,
                "refresh": refresh, "reuse": not refresh}

    mixed = False
    if wl.refresh_mask is None:
        parts_local = [make_part(wl, True)]
    else:
        ri = [i for i, m in enumerate(wl.refresh_mask) if m]
        ui = [i for i, m in enumerate(wl.refresh_mask) if not m]
        shared = synth.make_batch(wl)
        dk, dv = shared.k_cache.to(dev), shared.v_cache.to(dev)
        parts_local = ([make_part_shared(shared, dk, dv, ri, True)] if ri else []) + \
                      ([make_part_shared(shared, dk, dv, ui, False)] if ui else [])
        # both phases in ONE launch (dllm_mixed_attn, next row N3) unless disabled
        mixed = len(parts_local) == 2 and not args.no_mixed
    for pt in parts_local:
        if "host" not in pt:
            bt = pt["batch"]
            pt["host"] = {"q": bt.q, "q_blk": bt.q_blk, "k_cache": bt.k_cache, "v_cache": bt.v_cache}

    fused = args.fused_select   # dllm_refresh_select_attn (one call; fused only in a DLLM_TC2_FUSEDSEL=1 build)
    fused_in_kernel = fused and "select_in_refresh=on" in lib.version()

    def step(ev=None):
        stream = torch.cuda.current_stream(dev)   # the capture stream while a graph is recorded
        if mixed:
            pr, pu = parts_local
            q, _, kc, vc = pr["t"]
            qb = pu["t"][1]
            if ev is not None:
                ev[0].record(stream)
            if fused:
                lib.mixed_select_attn(pr["p"], q, pr["buf"].out, pr["buf"].scores, pr["buf"].idx, pu["p"], qb,
                                      pu["buf"].idx, pu["buf"].out_blk, kc, vc, stream)
            else:
                lib.mixed_attn(pr["p"], q, pr["buf"].out, pr["buf"].scores, pu["p"], qb, pu["buf"].idx,
                               pu["buf"].out_blk, kc, vc, stream)
            if ev is not None:
                ev[1].record(stream)
            if not fused:
                lib.select_heads(pr["p"], pr["buf"].scores, pr["buf"].idx, stream)
            if ev is not None:
                ev[2].record(stream)
                ev[3].record(stream)
            return
        if ev is not None:
            ev[0].record(stream)
        for pt in parts_local:
            if pt["refresh"]:
                q, qb, kc, vc = pt["t"]
                if fused:
                    lib.refresh_select_attn(pt["p"], q, kc, vc, pt["buf"].out, pt["buf"].scores, pt["buf"].idx, stream)
                else:
                    lib.refresh_attn(pt["p"], q, kc, vc, pt["buf"].out, pt["buf"].scores, stream)
        if ev is not None:
            ev[1].record(stream)
        for pt in parts_local:
            if pt["refresh"] and not fused:
                lib.select_heads(pt["p"], pt["buf"].scores, pt["buf"].idx, stream)
        if ev is not None:
            ev[2].record(stream)
        for pt in parts_local:
            if pt["reuse"]:
                q, qb, kc, vc = pt["t"]
                lib.reuse_sparse_attn(pt["p"], qb, kc, vc, pt["buf"].idx, pt["buf"].out_blk, stream)
        if ev is not None:
            ev[3].record(stream)

    for _ in range(args.warmup):
        flush.zero_()
        step()
    torch.cuda.synchronize(dev)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    clk = ClockSampler(local_rank)
    with clk:
        for i in range(args.steps):
            flush.zero_()
            step(evs[i])
        torch.cuda.synchronize(dev)
    clk.close()
    if world > 1:
        dist.barrier()
    t_ref = [evs[i][0].elapsed_time(evs[i][1]) * 1e-3 for i in range(args.steps)]
    t_sel = [evs[i][1].elapsed_time(evs[i][2]) * 1e-3 for i in range(args.steps)]
    t_reu = [evs[i][2].elapsed_time(evs[i][3]) * 1e-3 for i in range(args.steps)]
    t_step = [evs[i][0].elapsed_time(evs[i][3]) * 1e-3 for i in range(args.steps)]
    total_eager = sum(t_step)
    total = total_eager
    launch_mode = "eager"
    if not args.no_graph:
        # the step's launches captured once in a CUDA graph (requests/s
        # without launch gaps); each replay is one full step on the same buffers
        g = torch.cuda.CUDAGraph()
        cs = torch.cuda.Stream(dev)
        cs.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(cs):
            step()   # warm the capture stream
        torch.cuda.current_stream(dev).wait_stream(cs)
        torch.cuda.synchronize(dev)
        with torch.cuda.graph(g, stream=cs):
            step()
        for _ in range(args.warmup):
            flush.zero_()
            g.replay()
        torch.cuda.synchronize(dev)
        gev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(args.steps)]
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        clk = ClockSampler(local_rank)
        with clk:
            for i in range(args.steps):
                flush.zero_()
                gev[i][0].record(stream)
                g.replay()
                gev[i][1].record(stream)
            torch.cuda.synchronize(dev)
        clk.extend(g.replay, 0.25)
        if world > 1:
            dist.barrier()
        total = sum(gev[i][0].elapsed_time(gev[i][1]) * 1e-3 for i in range(args.steps))
        launch_mode = "cuda_graph"
    tt = torch.tensor([total], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    total_max = float(tt.item())
    reqs_per_step = glob.num_requests
    value = reqs_per_step * args.steps / total_max

    # ---- algorithmic work per launch
    H, Hk, D = wl.num_heads, wl.num_kv_heads, wl.head_dim
    g = H // Hk
    flops_refresh = 0.0
    reuse_bytes = reuse_logical = select_bytes = 0
    total_idx_all = rows_all = 0
    for pt in parts_local:
        sub = pt["wl"]
        kk, total_idx, rows, blk_rows = pt["p"].layout()
        idx_host = pt["buf"].idx[:total_idx].cpu().numpy()
        uniq_rows, off = 0, 0
        for b in range(sub.num_requests):
            rows_b = idx_host[off:off + H * kk[b]].reshape(H, kk[b])
            off += H * kk[b]
            for kv in range(Hk):
                uniq_rows += len(np.unique(rows_b[kv * g:(kv + 1) * g])) + sub.blk[b]
        if pt["reuse"]:
            reuse_bytes += uniq_rows * 2 * D * 2 + 2 * blk_rows * H * D * 2 + 4 * total_idx
            reuse_logical += sum(H * (sub.blk[b] + kk[b]) for b in range(sub.num_requests)) * 2 * D * 2 + \
                2 * blk_rows * H * D * 2 + 4 * total_idx
        if pt["refresh"]:
            flops_refresh += sum(4.0 * H * L * L * D for L in sub.seq_len)
            select_bytes += 4 * H * rows + 4 * total_idx
        total_idx_all += total_idx
        rows_all += rows
    a_ref = flops_refresh / statistics.mean(t_ref) / 1e12 if flops_refresh else 0.0
    a_reu = reuse_bytes / statistics.mean(t_reu) / 1e9 if reuse_bytes and not mixed else 0.0
    a_sel = select_bytes / statistics.mean(t_sel) / 1e9 if select_bytes and not fused else 0.0
    main_part = parts_local[0]
    buf = main_part["buf"]
    q, qb, kc, vc = main_part["t"]
    p = main_part["p"]
    k, total_idx, rows, blk_rows = p.layout()

    # ---- all-gather of per-request outputs (NCCL), timed separately
    allgather_ms = None
    if world > 1 and len(parts_local) == 1:
        counts_rows = [sum(glob.seq_len[i] for i in parts[r]) for r in range(world)]
        counts_blk = [sum(glob.blk[i] for i in parts[r]) for r in range(world)]
        for _ in range(2):
            shard.allgather_outputs(buf.out, counts_rows)
            shard.allgather_outputs(buf.out_blk, counts_blk)
        torch.cuda.synchronize(dev)
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        shard.allgather_outputs(buf.out, counts_rows)
        shard.allgather_outputs(buf.out_blk, counts_blk)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        ag = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
        dist.all_reduce(ag, op=dist.ReduceOp.MAX)
        allgather_ms = float(ag.item())

    # ---- end to end through the public API with host buffers
    pin = lambda t: t.pin_memory()  # noqa: E731
    h_in, d_in, h_out, d_out = [], [], [], []
    seen = set()

    def add_in(host, dev_t):
        if id(dev_t) not in seen:    # a mixed batch's phases share one cache: copied once
            seen.add(id(dev_t))
            h_in.append(pin(host))
            d_in.append(dev_t)

    for pt in parts_local:
        ht, tb, (_, tidx, _, _) = pt["host"], pt["buf"], pt["p"].layout()
        add_in(ht["k_cache"], pt["t"][2])
        add_in(ht["v_cache"], pt["t"][3])
        if pt["reuse"]:
            add_in(ht["q_blk"], pt["t"][1])
            d_out.append(tb.out_blk)
        if pt["refresh"]:
            add_in(ht["q"], pt["t"][0])
            d_out += [tb.out, tb.idx[:max(tidx, 1)]]
        else:
            # reuse-only requests bring the index lists of their earlier selection
            h_in.append(tb.idx[:max(tidx, 1)].cpu().pin_memory())
            d_in.append(tb.idx[:max(tidx, 1)])
    h_out = [torch.empty(t.shape, dtype=t.dtype).pin_memory() for t in d_out]
    h2d = sum(t.numel() * t.element_size() for t in h_in)
    d2h = sum(t.numel() * t.element_size() for t in h_out)

    # Steps are pipelined the way a serving loop runs them: step i's results go back
    # to the host on a second stream (the D2H copy engine) while step i+1's inputs
    # come in on the compute stream (the H2D engine); step i+1's kernels wait for
    # both (its inputs, and the read-out of the output buffers they overwrite).
    d2h_stream = torch.cuda.Stream(dev)
    d2h_done = [None]

    def e2e_step():
        for d, h in zip(d_in, h_in):
            d.copy_(h, non_blocking=True)
        if d2h_done[0] is not None:
            stream.wait_event(d2h_done[0])
        step()
        computed = torch.cuda.Event()
        computed.record(stream)
        d2h_stream.wait_event(computed)
        with torch.cuda.stream(d2h_stream):
            for h, d in zip(h_out, d_out):
                h.copy_(d, non_blocking=True)
        d2h_done[0] = torch.cuda.Event()
        d2h_done[0].record(d2h_stream)

    e2e_step()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.e2e_steps):
        e2e_step()
    stream.wait_event(d2h_done[0])      # the last step's results are on the host
    e1.record(stream)
    torch.cuda.synchronize(dev)
    te = torch.tensor([e0.elapsed_time(e1) * 1e-3], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = reqs_per_step * args.e2e_steps / float(te.item())

    # ---- CPU oracle baseline (rank 0, N=1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        r, n, t, cores = cpu_oracle_rate(base, budget_s=12.0)
        what = ("Refresh+importance+select+Reuse" if base.refresh_mask is None else
                "mixed: Refresh+importance+select for Refresh requests, Reuse for the rest, batch time "
                "extrapolated from per-kind means")
        cpu = {"value": r, "unit": UNIT, "cores": cores, "kind": "oracle",
               "sample": f"{n} request passes over the {base.num_requests} {base.name} requests ({what}, "
                         f"all heads, fp64 numpy), {t:.1f} s"}

    if rank == 0:
        clocks = clk.summary()
        traffic = ncu_traffic("refresh", args.config)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * total_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": workload_desc(base, world), "global_requests": reqs_per_step,
                       "parallelism": f"request-sharded dp{world} (LPT), no data-path collective",
                       "l2": "flushed before every step (512 MiB write, outside the step events)",
                       "seed": synth.base_seed()},
            "roofline": ({"bound": "tensor", "kernel": ("dllm_refresh_select_attn (tcgen05 Refresh + select in one "
                                                        "call: FLOP of Refresh only / time of both)") if fused else
                          "dllm_refresh_attn (tcgen05)", "achieved": a_ref,
                          "peak": tf_peak, "unit": "TFLOP/s", "frac": a_ref / tf_peak, "traffic": traffic,
                          "peak_source": f"{peak_src} bf16 burst (MEASURED_PEAKS.json)",
                          "frac_of_sustained": (a_ref / tf_sust) if tf_sust else None} if not mixed else
                         {"bound": "tensor+hbm", "kernel": "dllm_mixed_attn (Refresh + Reuse, one launch)",
                          "achieved": a_ref, "peak": tf_peak, "unit": "TFLOP/s (Refresh FLOP / launch time)",
                          "frac": (flops_refresh / (tf_peak * 1e12) + reuse_bytes / (hbm_peak * 1e9))
                          / statistics.mean(t_ref),
                          "frac_definition": "additive roofline time (Refresh FLOP / bf16 peak + Reuse unique "
                                             "bytes / HBM peak) / measured launch time", "traffic": None,
                          "peak_source": f"{peak_src} (MEASURED_PEAKS.json)"}),
            "kernels": ({
                "mixed": {"us": 1e6 * statistics.mean(t_ref), "refresh_flop": flops_refresh,
                          "reuse_bytes_unique": reuse_bytes, "reuse_bytes_logical": reuse_logical,
                          "roofline_us": 1e6 * (flops_refresh / (tf_peak * 1e12) + reuse_bytes / (hbm_peak * 1e9))},
                "select": ({"in_one_call_with": "Refresh (timed with it)", "fused_in_kernel": fused_in_kernel,
                            "bytes_per_launch": select_bytes}
                           if fused else {"us": 1e6 * statistics.mean(t_sel), "GB/s": a_sel, "frac": a_sel / hbm_peak,
                                          "bytes_per_launch": select_bytes})} if mixed else {
                "refresh": {"us": 1e6 * statistics.mean(t_ref), "TFLOP/s": a_ref, "frac": a_ref / tf_peak,
                            "flop_per_launch": flops_refresh},
                "select": ({"in_one_call_with": "Refresh (timed with it)", "fused_in_kernel": fused_in_kernel,
                            "bytes_per_launch": select_bytes}
                           if fused else {"us": 1e6 * statistics.mean(t_sel), "GB/s": a_sel, "frac": a_sel / hbm_peak,
                                          "bytes_per_launch": select_bytes}),
                "reuse": {"us": 1e6 * statistics.mean(t_reu), "GB/s": a_reu, "frac": a_reu / hbm_peak,
                          "bytes_per_launch_unique": reuse_bytes, "bytes_per_launch_logical": reuse_logical,
                          "GB/s_logical": reuse_logical / statistics.mean(t_reu) / 1e9, "bound": "hbm",
                          "peak": hbm_peak},
                "block_cycle_us": (1e6 * (statistics.mean(t_ref) + statistics.mean(t_sel) + 31 * statistics.mean(t_reu))
                                   if len(parts_local) == 1 and parts_local[0]["refresh"] else None),
            }),
            "launch_mode": launch_mode,
            "ms_per_step_eager": 1e3 * total_eager / args.steps,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "steps": args.e2e_steps, "pipelining": "D2H of step i on a second stream beside the H2D of step i+1"},
            "select_fused": fused_in_kernel,
            "gpu_launches": ((1 if fused_in_kernel else 2) if mixed else
                             sum(((1 if fused_in_kernel else 2) * pt["refresh"] + pt["reuse"]) * ((pt["wl"].num_requests + 255) // 256)
                                                 for pt in parts_local)) * args.steps,
            "clocks": clocks,
            "cpu_baseline": cpu,
            "allgather_ms": allgather_ms,
            "lib": lib.version(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
