#!/usr/bin/env python
"""Benchmark of the Head-Centric Sparse Attention hot path (one JSON line).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C1] [--scaling weak|strong]
                    [--impl ours|reference] [--no-configs]
    torchrun --nproc-per-node N bench.py --gpus N ...     (one process per GPU, NCCL)

A step = one pass of the whole hot path over one batch:
dllm_refresh_attn (Eq. 3 + importance) -> dllm_select_heads (Eq. 6 + TopK) ->
dllm_reuse_sparse_attn (Eq. 4), through the C-ABI; for the mixed burst batch
(C3) the Refresh requests run Refresh + select and the others Reuse, in one
launch (dllm_mixed_attn) + the select.  `value` is measured on --config (default
C1, BASELINE.json configs[1], LLaDA-8B layer shape on 1 B200).

Multi-GPU: requests are independent, so the batch is LPT-partitioned over the
ranks with no collective on the data path.  --scaling weak (default): every rank
holds a C-sized shard of an N-times replicated batch; --scaling strong: the
config's own batch is partitioned (C3: 256 requests over 8 GPUs = 32 each).  The
NCCL all-gather of the per-request outputs (Refresh rows, new index lists,
Reuse rows) is timed separately: serial, and overlapped with the next step's
compute on a side stream.

value  = requests/s over all ranks = (requests per step * K) / max-over-ranks
         device time of the K steps (CUDA graph replay of the step; CUDA events on
         the launch stream; L2 flushed before every step by a 512 MiB write
         outside the events).
kernels = per-kernel CUDA-event times of eager launches (one kernel between two
         events, L2 flushed before each), against the measured peaks; Reuse also
         "in stream": a CUDA graph of 31 back-to-back Reuse launches (the Reuse
         steps of one block cycle) rotating over 3 input sets so
         that no launch finds its K/V in L2, per-launch time = graph time / 31.
configs = the same sub-results for the other BASELINE configs (N=1 only):
         C2 (Dream GQA), C3 (burst mix), C4 (r = 0.25), and the N4 LM head.
e2e    = the same metric through the public API with HOST buffers: every step
         copies its inputs from pinned host memory to the device, runs the calls
         and copies the results back (pipelined as a serving loop would).
cpu_baseline = the fp64 oracle (oracle/) timed on this host's cores on a
         bounded sample of the same workload (rank 0, N=1 only).
--impl reference runs that oracle as the reference arm (the paper ships no code).
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
BLOCK_CYCLE_REUSE = 31   # Reuse steps per Refresh (gen 256 / steps 256 / block 32)


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return pk["bf16_tflops"], pk.get("bf16_tflops_sustained"), pk["hbm_gbs"], "measured"
    except Exception:
        return 1590.0, 1400.0, 6650.0, "fallback"


def workload_desc(wl, n, scaling):
    mix = "" if wl.refresh_mask is None else \
        f" ({sum(wl.refresh_mask)} Refresh+select, {wl.num_requests - sum(wl.refresh_mask)} Reuse-only)"
    per = "requests/GPU" if scaling == "weak" else "requests in total"
    return (f"{wl.name}: {wl.num_requests} {per}{mix} x {n} GPU, H={wl.num_heads}, H_kv={wl.num_kv_heads}, "
            f"D={wl.head_dim}, L={min(wl.seq_len)}..{max(wl.seq_len)}, blk={wl.blk[0]}, r={wl.keep_ratio}, "
            f"w={wl.pool_window}, page={wl.page_size}")


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """SM clocks, power and throttle reasons sampled through NVML every ~2 ms while
    the timed region runs.  The timed region of a default run is short, so
    `extend(fn, seconds)` keeps replaying the same step afterwards, untimed, and
    records the clocks the workload settles at under the power cap (separately)."""

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
def cpu_oracle_rate(wl, budget_s: float = 12.0, max_requests: int | None = None, time_inputs: bool = False):
    """The fp64 oracle as it stands, on a bounded sample of the workload's requests
    (whole requests: Refresh + importance + select + Reuse, all heads; in a mixed
    batch the Refresh requests run Refresh + select and the Reuse-only requests
    Reuse on generated index lists).  Input generation is outside the timed region
    unless time_inputs.  Returns (requests/s, requests timed, seconds, threads).
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
        for b in (reqs * 8 if max_requests is None else reqs):
            if max_requests is not None and done >= max_requests:
                break
            q, K, V, qb = (t.double().numpy() for t in synth.request_tensors(wl, b))
            bs, be, L = wl.blk_start[b], wl.blk_end[b], wl.seq_len[b]
            sel = None
            if not kd:
                k = O.keep_count(wl.keep_ratio, L - (be - bs))
                sel = synth.indices(synth.subset(wl, [b]), [k])[0]
            t0 = time.perf_counter()
            if kd:
                O.attention_dense(q, K, V)
                raw = O.raw_scores(q[bs:be], K)
                sel = O.select_batch([raw], [L], [bs], [be], wl.keep_ratio, wl.pool_window)[0]
            if not kd or wl.refresh_mask is None:
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
    for _ in range(args.warmup):
        cpu_oracle_rate(wl, budget_s=0.0, max_requests=1)
    n_req, t_oracle = 0, 0.0
    for _ in range(args.steps):
        # the oracle alone is timed (inputs are generated outside the measured region)
        r, n, t, cores = cpu_oracle_rate(wl, budget_s=0.0, max_requests=1)
        n_req += n
        t_oracle += t
    value = n_req / t_oracle
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t_oracle / args.steps,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": workload_desc(wl, 1, args.scaling), "sample": "1 request (all heads) per step"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": len(os.sched_getaffinity(0)), "kind": "oracle",
                             "sample": f"{args.steps} steps x 1 request of {wl.name} (Refresh+select+Reuse, all "
                                       "heads; oracle time only, input generation excluded)"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- one config on this rank
class Step:
    """The batch of this rank (an LPT shard of `glob`), its problems / buffers and
    the step closure."""

    def __init__(self, glob, parts, rank, dev, lib, synth, select="heads"):
        import torch
        self.select = select   # "heads" (Eq. 6 per query head) or "groups" (N2: one set per KV group)
        self.torch, self.lib, self.synth, self.dev = torch, lib, synth, dev
        self.glob, self.parts, self.rank = glob, parts, rank
        wl = synth.subset(glob, parts[rank])
        self.wl = wl
        self.pieces = []
        if wl.refresh_mask is None:
            self.pieces = [self._make_piece(wl, True, True)]
        else:
            ri = [i for i, m in enumerate(wl.refresh_mask) if m]
            ui = [i for i, m in enumerate(wl.refresh_mask) if not m]
            shared = synth.make_batch(wl)
            dk, dv = shared.k_cache.to(dev), shared.v_cache.to(dev)
            if ri:
                self.pieces.append(self._make_shared(shared, dk, dv, ri, True))
            if ui:
                self.pieces.append(self._make_shared(shared, dk, dv, ui, False))
        # both phases of a mixed batch in ONE launch (dllm_mixed_attn, next row N3)
        self.mixed = len(self.pieces) == 2

    def _problem(self, sub, block_table):
        return self.lib.Problem(sub.seq_len, sub.blk_start, sub.blk_end, num_heads=sub.num_heads,
                                num_kv_heads=sub.num_kv_heads, head_dim=sub.head_dim, keep_ratio=sub.keep_ratio,
                                pool_window=sub.pool_window, page_size=sub.page_size,
                                block_table=block_table.contiguous().to(self.dev))

    def _prefill_idx(self, sub, pp, bf):
        # Reuse-only requests bring the index lists of an earlier selection
        kk = pp.layout()[0]
        flat = np.concatenate([x.reshape(-1) for x in self.synth.indices(sub, kk)]).astype(np.int32)
        if flat.size:
            bf.idx[:flat.size].copy_(self.torch.from_numpy(flat))

    def _make_piece(self, sub, refresh, reuse):
        bt = self.synth.make_batch(sub)
        pp = self._problem(sub, bt.block_table)
        tens = [t.to(self.dev) for t in (bt.q, bt.q_blk, bt.k_cache, bt.v_cache)]
        bf = self.lib.alloc_buffers(pp, device=self.dev)
        if not refresh:
            self._prefill_idx(sub, pp, bf)
        host = {"q": bt.q, "q_blk": bt.q_blk, "k_cache": bt.k_cache, "v_cache": bt.v_cache}
        return {"wl": sub, "p": pp, "t": tens, "buf": bf, "refresh": refresh, "reuse": reuse, "host": host}

    def _make_shared(self, shared, dk, dv, reqs, refresh):
        # a phase of a mixed batch: its own problem (block-table rows of its requests)
        # over the batch's ONE paged cache
        sub = self.synth.subset(self.wl, reqs)
        pp = self._problem(sub, shared.block_table[reqs])
        q = self.torch.cat([shared.q_req(b) for b in reqs])
        qb = self.torch.cat([shared.q_blk_req(b) for b in reqs])
        bf = self.lib.alloc_buffers(pp, device=self.dev)
        if not refresh:
            self._prefill_idx(sub, pp, bf)
        host = {"q": q, "q_blk": qb, "k_cache": shared.k_cache, "v_cache": shared.v_cache}
        return {"wl": sub, "p": pp, "t": [q.to(self.dev), qb.to(self.dev), dk, dv], "buf": bf, "refresh": refresh,
                "reuse": not refresh, "host": host}

    def step(self, ev=None, bufs=None):
        """One step on the current stream; ev = 4 events around Refresh / select /
        Reuse (or the mixed launch / select); bufs overrides the output buffers."""
        lib = self.lib
        stream = self.torch.cuda.current_stream(self.dev)
        bufs = bufs or [pc["buf"] for pc in self.pieces]
        rec = (lambda i: ev[i].record(stream)) if ev is not None else (lambda i: None)
        if self.mixed:
            (pr, pu), (br, bu) = self.pieces, bufs
            q, _, kc, vc = pr["t"]
            rec(0)
            lib.mixed_attn(pr["p"], q, br.out, br.scores, pu["p"], pu["t"][1], bu.idx, bu.out_blk, kc, vc, stream)
            rec(1)
            lib.select_heads(pr["p"], br.scores, br.idx, stream)
            rec(2)
            rec(3)
            return
        rec(0)
        for pc, bf in zip(self.pieces, bufs):
            if pc["refresh"]:
                q, qb, kc, vc = pc["t"]
                lib.refresh_attn(pc["p"], q, kc, vc, bf.out, bf.scores, stream)
        rec(1)
        for pc, bf in zip(self.pieces, bufs):
            if pc["refresh"]:
                (lib.select_groups if self.select == "groups" else lib.select_heads)(pc["p"], bf.scores, bf.idx,
                                                                                    stream)
        rec(2)
        for pc, bf in zip(self.pieces, bufs):
            if pc["reuse"]:
                q, qb, kc, vc = pc["t"]
                # one set per KV group: the group kernel gathers each group's rows once
                (lib.reuse_group_sets if self.select == "groups" else lib.reuse_sparse_attn)(
                    pc["p"], qb, kc, vc, bf.idx, bf.out_blk, stream)
        rec(3)

    def algorithmic(self):
        """Refresh FLOPs, Reuse unique / logical bytes and select bytes of one step
        (DESIGN.md §6); unique rows are counted from the index lists in use."""
        flops = 0.0
        reuse_u = reuse_l = sel = 0
        for pc in self.pieces:
            sub = pc["wl"]
            H, Hk, D = sub.num_heads, sub.num_kv_heads, sub.head_dim
            g = H // Hk
            kk, total_idx, rows, blk_rows = pc["p"].layout()
            idx_host = pc["buf"].idx[:total_idx].cpu().numpy()
            uniq, off = 0, 0
            for b in range(sub.num_requests):
                rb = idx_host[off:off + H * kk[b]].reshape(H, kk[b])
                off += H * kk[b]
                for kv in range(Hk):
                    uniq += len(np.unique(rb[kv * g:(kv + 1) * g])) + sub.blk[b]
            if pc["reuse"]:
                extra = 2 * blk_rows * H * D * 2 + 4 * total_idx
                reuse_u += uniq * 2 * D * 2 + extra
                reuse_l += sum(H * (sub.blk[b] + kk[b]) for b in range(sub.num_requests)) * 2 * D * 2 + extra
            if pc["refresh"]:
                flops += sum(4.0 * H * L * L * D for L in sub.seq_len)
                sel += 4 * H * rows + 4 * total_idx
        return flops, reuse_u, reuse_l, sel


def time_eager(st, steps, warmup, flush):
    """Per-kernel CUDA-event times (s) of eager steps, L2 flushed before each."""
    torch = st.torch
    for _ in range(warmup):
        flush.zero_()
        st.step()
    torch.cuda.synchronize(st.dev)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(steps)]
    for i in range(steps):
        flush.zero_()
        st.step(evs[i])
    torch.cuda.synchronize(st.dev)
    el = lambda i, a, b: evs[i][a].elapsed_time(evs[i][b]) * 1e-3  # noqa: E731
    return ([el(i, 0, 1) for i in range(steps)], [el(i, 1, 2) for i in range(steps)],
            [el(i, 2, 3) for i in range(steps)], [el(i, 0, 3) for i in range(steps)])


def capture_graph(st):
    torch = st.torch
    g = torch.cuda.CUDAGraph()
    cs = torch.cuda.Stream(st.dev)
    cs.wait_stream(torch.cuda.current_stream(st.dev))
    with torch.cuda.stream(cs):
        st.step()   # warm the capture stream
    torch.cuda.current_stream(st.dev).wait_stream(cs)
    torch.cuda.synchronize(st.dev)
    with torch.cuda.graph(g, stream=cs):
        st.step()
    return g


def time_graph(st, g, steps, warmup, flush, clk=None, dist=None):
    torch = st.torch
    stream = torch.cuda.current_stream(st.dev)
    for _ in range(warmup):
        flush.zero_()
        g.replay()
    torch.cuda.synchronize(st.dev)
    gev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(steps)]
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize(st.dev)
    if clk is not None:
        clk.__enter__()
    for i in range(steps):
        flush.zero_()
        gev[i][0].record(stream)
        g.replay()
        gev[i][1].record(stream)
    torch.cuda.synchronize(st.dev)
    if clk is not None:
        clk.__exit__()
        clk.extend(g.replay, 0.25)
    if dist is not None:
        dist.barrier()
    return sum(gev[i][0].elapsed_time(gev[i][1]) * 1e-3 for i in range(steps))


def reuse_in_stream(st, reps=BLOCK_CYCLE_REUSE, iters=5):
    """Reuse per-launch time in a stream of back-to-back launches: one CUDA graph of
    `reps` launches rotating over independent input sets (3 when the step's unique
    Reuse bytes are below 4x L2, else the step's own set), so launch latency
    overlaps the previous launch (PDL) but no launch finds its rows in L2."""
    import torch
    lib, synth, dev = st.lib, st.synth, st.dev
    pc = st.pieces[0]
    sets = [(pc["p"], pc["t"][1], pc["t"][2], pc["t"][3], pc["buf"])]
    base = st.wl
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    nsets = 3 if st.algorithmic()[1] < 4 * l2 else 1
    for s in range(1, nsets):
        wl = synth.replicate(base, nsets)   # replica s: the same shapes, its own values
        sub = synth.subset(wl, list(range(s * base.num_requests, (s + 1) * base.num_requests)))
        bt = synth.make_batch(sub)
        pp = lib.Problem(sub.seq_len, sub.blk_start, sub.blk_end, num_heads=sub.num_heads,
                         num_kv_heads=sub.num_kv_heads, head_dim=sub.head_dim, keep_ratio=sub.keep_ratio,
                         pool_window=sub.pool_window, page_size=sub.page_size, block_table=bt.block_table.to(dev))
        bf = lib.alloc_buffers(pp, device=dev)
        kk = pp.layout()[0]
        mode = "shared" if st.select == "groups" else "random"
        flat = np.concatenate([x.reshape(-1) for x in synth.indices(sub, kk, mode=mode)]).astype(np.int32)
        bf.idx[:flat.size].copy_(torch.from_numpy(flat))
        sets.append((pp, bt.q_blk.to(dev), bt.k_cache.to(dev), bt.v_cache.to(dev), bf))
    reuse = lib.reuse_group_sets if st.select == "groups" else lib.reuse_sparse_attn
    cs = torch.cuda.Stream(dev)

    def launches():
        for i in range(reps):
            pp, qb, kc, vc, bf = sets[i % nsets]
            reuse(pp, qb, kc, vc, bf.idx, bf.out_blk, cs)

    cs.wait_stream(torch.cuda.current_stream(dev))
    with torch.cuda.stream(cs):
        launches()
    torch.cuda.synchronize(dev)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=cs):
        launches()
    flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device=dev)
    ts = []
    stream = torch.cuda.current_stream(dev)
    for it in range(iters + 2):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        g.replay()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        if it >= 2:
            ts.append(e0.elapsed_time(e1) * 1e-3 / reps)
    return statistics.median(ts)


def select_in_stream(st, reps=BLOCK_CYCLE_REUSE, iters=5):
    """Select per-launch time in a stream: one CUDA graph of `reps` back-to-back
    launches over the step's own raw scores (L2-resident after the first launch, as
    when select directly follows the Refresh that wrote them), so launch latency
    overlaps the previous launch (PDL) -- the event-timed floor of one launch on
    this box is ~5-6 us (profiles/r02_flush_modes.log: an empty fill)."""
    import torch
    lib, dev = st.lib, st.dev
    pc = st.pieces[0]
    sel = lib.select_groups if st.select == "groups" else lib.select_heads
    cs = torch.cuda.Stream(dev)

    def launches():
        for _ in range(reps):
            sel(pc["p"], pc["buf"].scores, pc["buf"].idx, cs)

    cs.wait_stream(torch.cuda.current_stream(dev))
    with torch.cuda.stream(cs):
        launches()
    torch.cuda.synchronize(dev)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=cs):
        launches()
    flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device=dev)
    ts = []
    stream = torch.cuda.current_stream(dev)
    for it in range(iters + 2):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        g.replay()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        if it >= 2:
            ts.append(e0.elapsed_time(e1) * 1e-3 / reps)
    return statistics.median(ts)


def lm_head_result(dev, lib, synth, tf_peak, iters=10):
    """N4: dllm_lm_head_argmax at the LLaDA-8B LM head (2,048 x 4,096 x 126,464)."""
    import torch
    f = synth.LM_HEAD_FULL
    n, d, v = f["n_tok"], f["d_model"], f["vocab"]
    h, w = synth.lm_head_inputs(n, d, v, "realistic")
    h, w = h.to(dev), w.to(dev)
    ids = torch.empty(n, dtype=torch.int32, device=dev)
    ws = torch.empty(lib.lm_head_workspace_bytes(n, v, f["max_num_logits"]), dtype=torch.uint8, device=dev)
    for _ in range(3):
        lib.lm_head_argmax(h, w, ids, f["max_num_logits"], ws)
    torch.cuda.synchronize(dev)
    ts = []
    for _ in range(iters):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        lib.lm_head_argmax(h, w, ids, f["max_num_logits"], ws)
        e1.record()
        torch.cuda.synchronize(dev)
        ts.append(e0.elapsed_time(e1) * 1e-3)
    t = statistics.median(ts)
    flop = 2.0 * n * d * v
    return {"kernel": "dllm_lm_head_argmax (tcgen05 GEMM + fused argmax)", "shape": [n, d, v],
            "max_num_logits": f["max_num_logits"], "us": t * 1e6, "TFLOP/s": flop / t / 1e12,
            "frac": flop / t / 1e12 / tf_peak, "bound": "tensor", "weight_bytes": v * d * 2,
            "note": "weight (1.04 GB) larger than L2: no flush needed"}


def kernels_result(st, t_ref, t_sel, t_reu, tf_peak, hbm_peak, reuse_stream_s=None, select_stream_s=None):
    flops, reuse_u, reuse_l, sel = st.algorithmic()
    m = statistics.mean
    if st.mixed:
        t_roof = flops / (tf_peak * 1e12) + reuse_u / (hbm_peak * 1e9)
        return {
            "mixed": {"us": 1e6 * m(t_ref), "refresh_flop": flops, "reuse_bytes_unique": reuse_u,
                      "reuse_bytes_logical": reuse_l, "roofline_us": 1e6 * t_roof, "frac": t_roof / m(t_ref),
                      "frac_definition": "additive roofline time (Refresh FLOP / bf16 peak + Reuse unique bytes / "
                                         "HBM peak) / measured launch time"},
            "select": {"us": 1e6 * m(t_sel), "GB/s": sel / m(t_sel) / 1e9, "frac": sel / m(t_sel) / 1e9 / hbm_peak,
                       "bytes_per_launch": sel},
        }, flops, reuse_u
    a_ref = flops / m(t_ref) / 1e12
    out = {
        "refresh": {"us": 1e6 * m(t_ref), "TFLOP/s": a_ref, "frac": a_ref / tf_peak, "flop_per_launch": flops,
                    "bound": "tensor", "peak": tf_peak},
        "select": {"us": 1e6 * m(t_sel), "GB/s": sel / m(t_sel) / 1e9, "frac": sel / m(t_sel) / 1e9 / hbm_peak,
                   "bytes_per_launch": sel, "bound": "hbm (latency at these sizes)"},
        "reuse": {"us": 1e6 * m(t_reu), "GB/s": reuse_u / m(t_reu) / 1e9, "frac": reuse_u / m(t_reu) / 1e9 / hbm_peak,
                  "bytes_per_launch_unique": reuse_u, "bytes_per_launch_logical": reuse_l,
                  "GB/s_logical": reuse_l / m(t_reu) / 1e9, "bound": "hbm", "peak": hbm_peak,
                  "timing": "one launch between two CUDA events, L2 flushed before it"},
        "block_cycle_us": 1e6 * (m(t_ref) + m(t_sel) + BLOCK_CYCLE_REUSE * m(t_reu)),
    }
    if reuse_stream_s is not None:
        out["reuse"].update({
            "us_in_stream": 1e6 * reuse_stream_s, "GB/s_in_stream": reuse_u / reuse_stream_s / 1e9,
            "frac_in_stream": reuse_u / reuse_stream_s / 1e9 / hbm_peak,
            "in_stream_timing": f"CUDA graph of {BLOCK_CYCLE_REUSE} back-to-back launches over 3 rotating input "
                                "sets (no L2 reuse), graph time / launches"})
        out["block_cycle_us_in_stream"] = 1e6 * (m(t_ref) + m(t_sel) + BLOCK_CYCLE_REUSE * reuse_stream_s)
    if select_stream_s is not None:
        out["select"].update({
            "us_in_stream": 1e6 * select_stream_s, "GB/s_in_stream": sel / select_stream_s / 1e9,
            "in_stream_timing": f"CUDA graph of {BLOCK_CYCLE_REUSE} back-to-back launches over the step's scores "
                                "(L2-resident after the first, as after the Refresh that writes them), graph time / "
                                "launches; a single event-timed launch carries a ~5-6 us floor on this box"})
    return out, flops, reuse_u


def config_result(cfg_name, dev, lib, synth, shard, tf_peak, hbm_peak, steps, warmup, flush, select="heads"):
    """A sub-result for `configs`: one GPU, the whole config batch."""
    wl = synth.config(cfg_name)
    st = Step(wl, [list(range(wl.num_requests))], 0, dev, lib, synth, select)
    t_ref, t_sel, t_reu, t_step = time_eager(st, steps, warmup, flush)
    g = capture_graph(st)
    total = time_graph(st, g, steps, warmup, flush)
    rs = None if st.mixed else reuse_in_stream(st)
    ss = None if st.mixed else select_in_stream(st)
    kern, flops, reuse_u = kernels_result(st, t_ref, t_sel, t_reu, tf_peak, hbm_peak, rs, ss)
    del g
    return {"workload": workload_desc(wl, 1, "weak") + ("" if select == "heads" else
                                                       ", selection: one set per KV group (dllm_select_groups),"
                                                       " Reuse dllm_reuse_group_sets"),
            "requests_per_s": wl.num_requests * steps / total,
            "ms_per_step": 1e3 * total / steps, "launch_mode": "cuda_graph", "kernels": kern}


# ----------------------------------------------------------------------------- our arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C1")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="skip the C2/C3/C4/N4 sub-results (N=1 only anyway)")
    ap.add_argument("--config-steps", type=int, default=5)
    ap.add_argument("--no-in-stream", action="store_true", help="skip the in-stream Reuse timing (ncu launch lists)")
    ap.add_argument("--e2e-steps", type=int, default=5)
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
    backend = os.environ.get("DLLM_BENCH_BACKEND", "nccl")   # gloo: dev check of the multi-rank logic on 1 GPU
    if world > 1:
        torch.cuda.set_device(local_rank if backend == "nccl" else 0)
        dist.init_process_group(backend, **({"device_id": torch.device("cuda", local_rank)}
                                            if backend == "nccl" else {}))
    dev = torch.device("cuda", local_rank if backend == "nccl" else 0)
    torch.cuda.set_device(dev)
    tf_peak, tf_sust, hbm_peak, peak_src = load_peaks()

    base = synth.config(args.config)
    glob = synth.replicate(base, world) if args.scaling == "weak" else base
    k_glob = [lib.keep_count(glob.keep_ratio, L - (e - s)) for L, s, e in zip(glob.seq_len, glob.blk_start, glob.blk_end)]
    costs = shard.workload_costs(glob, k_glob)
    parts = shard.lpt_partition(costs, world)
    st = Step(glob, parts, rank, dev, lib, synth)
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device=dev)

    # ---- eager per-kernel times, then the graph-replayed step (the `value`)
    t_ref, t_sel, t_reu, t_step = time_eager(st, args.steps, args.warmup, flush)
    total_eager = sum(t_step)
    g = capture_graph(st)
    clk = ClockSampler(local_rank)
    total = time_graph(st, g, args.steps, args.warmup, flush, clk, dist if world > 1 else None)
    tt = torch.tensor([total], dtype=torch.float64, device=dev if backend == "nccl" else "cpu")
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    total_max = float(tt.item())
    reqs_per_step = glob.num_requests
    value = reqs_per_step * args.steps / total_max
    in_stream = rank == 0 and world == 1 and not st.mixed and not args.no_in_stream
    rs = reuse_in_stream(st) if in_stream else None
    ss = select_in_stream(st) if in_stream else None
    kern, flops, reuse_u = kernels_result(st, t_ref, t_sel, t_reu, tf_peak, hbm_peak, rs, ss)

    # ---- multi-GPU: all-gather of the per-request outputs (serial and overlapped)
    gather = None
    if world > 1:
        gather = gather_times(st, dist, shard, backend, g, flush, args)

    # ---- end to end through the public API with host buffers
    e2e = e2e_result(st, args, dist if world > 1 else None, backend)

    # ---- CPU oracle baseline and the other configs (rank 0, N=1 only)
    cpu = None
    configs = None
    if rank == 0 and world == 1:
        if not args.no_cpu_baseline:
            r, n, t, cores = cpu_oracle_rate(base, budget_s=12.0)
            what = ("Refresh+importance+select+Reuse" if base.refresh_mask is None else
                    "mixed: Refresh+importance+select for Refresh requests, Reuse for the rest, batch time "
                    "extrapolated from per-kind means")
            cpu = {"value": r, "unit": UNIT, "cores": cores, "kind": "oracle",
                   "sample": f"{n} request passes over the {base.num_requests} {base.name} requests ({what}, "
                             f"all heads, fp64 numpy), {t:.1f} s"}
        if not args.no_configs:
            del g
            configs = {}
            for c in [x for x in ("C1", "C2", "C3", "C4") if x != args.config]:
                try:
                    configs[c] = config_result(c, dev, lib, synth, shard, tf_peak, hbm_peak, args.config_steps, 3,
                                               flush)
                except Exception as e:   # a sub-result must not lose the main line
                    configs[c] = {"error": repr(e)}
                torch.cuda.empty_cache()
            try:   # next row N2: the Dream GQA shape with one index set per KV group
                configs["C2_groups"] = config_result("C2", dev, lib, synth, shard, tf_peak, hbm_peak,
                                                     args.config_steps, 3, flush, select="groups")
            except Exception as e:
                configs["C2_groups"] = {"error": repr(e)}
            torch.cuda.empty_cache()
            try:
                configs["N4_lm_head"] = lm_head_result(dev, lib, synth, tf_peak)
            except Exception as e:
                configs["N4_lm_head"] = {"error": repr(e)}

    if rank == 0:
        clocks = clk.summary()
        if st.mixed:
            km = kern["mixed"]
            roof = {"bound": "tensor+hbm", "kernel": "dllm_mixed_attn (Refresh + Reuse, one launch)",
                    "achieved": flops / (km["us"] * 1e-6) / 1e12, "peak": tf_peak,
                    "unit": "TFLOP/s (Refresh FLOP / launch time)", "frac": km["frac"],
                    "frac_definition": km["frac_definition"], "traffic": None,
                    "peak_source": f"{peak_src} (MEASURED_PEAKS.json)"}
        else:
            kr = kern["refresh"]
            roof = {"bound": "tensor", "kernel": "dllm_refresh_attn (tcgen05)", "achieved": kr["TFLOP/s"],
                    "peak": tf_peak, "unit": "TFLOP/s", "frac": kr["frac"],
                    "traffic": ncu_traffic("refresh", args.config),
                    "peak_source": f"{peak_src} bf16 burst (MEASURED_PEAKS.json)",
                    "frac_of_sustained": (kr["TFLOP/s"] / tf_sust) if tf_sust else None,
                    "traffic_note": "ncu DRAM bytes per launch (profiles/ncu_traffic.json); the algorithmic bytes "
                                    "(Q + K + V + O once, + scores) are ~0.54 GB at C1: the LPT unit order "
                                    "(importance pairs first) reads each (request, KV head)'s K/V a second time "
                                    "(request-major order: 518 MB, 1.5-2% slower); DRAM ~35% of peak in this "
                                    "tensor-bound kernel (DESIGN.md §6)"}
        n_launch = 2 if st.mixed else sum(((2 if pc["refresh"] else 0) + (1 if pc["reuse"] else 0)) *
                                          ((pc["wl"].num_requests + 255) // 256) for pc in st.pieces)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * total_max / args.steps, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": workload_desc(base, world, args.scaling), "global_requests": reqs_per_step,
                       "parallelism": f"request-sharded dp{world} (LPT), no data-path collective",
                       "l2": "flushed before every step (512 MiB write, outside the step events)",
                       "seed": synth.base_seed()},
            "roofline": roof,
            "kernels": kern,
            "launch_mode": "cuda_graph",
            "ms_per_step_eager": 1e3 * total_eager / args.steps,
            "e2e": e2e,
            "gpu_launches": n_launch * args.steps,
            "clocks": clocks,
            "cpu_baseline": cpu,
            "allgather": gather,
            "configs": configs,
            "lib": lib.version(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def _step_outputs(st, bufs=None):
    """This rank's per-request outputs of one step, each the concatenation over its
    requests (ascending): Refresh rows, new index lists (Refresh requests) and Reuse
    rows; plus the per-global-request sizes of each (0 for requests without it)."""
    n = st.glob.num_requests
    sizes = {"out": [0] * n, "idx": [0] * n, "out_blk": [0] * n}
    mine = st.parts[st.rank]
    tensors = {"out": [], "idx": [], "out_blk": []}
    bufs = bufs or [pc["buf"] for pc in st.pieces]
    for pc, bf in zip(st.pieces, bufs):
        sub = pc["wl"]
        kk, total_idx, rows, blk_rows = pc["p"].layout()
        H = sub.num_heads
        gids = [mine[i] for i in range(len(mine)) if
                (st.wl.refresh_mask is None or st.wl.refresh_mask[i] == pc["refresh"])]
        if pc["refresh"]:
            tensors["out"].append(bf.out[:rows])
            tensors["idx"].append(bf.idx[:total_idx])
            for j, gi in enumerate(gids):
                sizes["out"][gi] = sub.seq_len[j]
                sizes["idx"][gi] = H * kk[j]
        if pc["reuse"]:
            tensors["out_blk"].append(bf.out_blk[:blk_rows])
            for j, gi in enumerate(gids):
                sizes["out_blk"][gi] = sub.blk[j]
    # every rank computes every rank's sizes (shapes are known from the workload)
    for name in sizes:
        for r, part in enumerate(st.parts):
            if r == st.rank:
                continue
            sub_r = st.synth.subset(st.glob, part)
            for j, gi in enumerate(part):
                m = None if st.glob.refresh_mask is None else st.glob.refresh_mask[gi]
                blk = sub_r.blk[j]
                L = sub_r.seq_len[j]
                k = st.lib.keep_count(st.glob.keep_ratio, L - blk)
                if name == "out" and m is not False:
                    sizes[name][gi] = L
                elif name == "idx" and m is not False:
                    sizes[name][gi] = st.glob.num_heads * k
                elif name == "out_blk" and m is not True:
                    sizes[name][gi] = blk
    torch = st.torch
    cat = {k: (torch.cat(v) if v else None) for k, v in tensors.items()}
    return cat, sizes


def gather_times(st, dist, shard, backend, g, flush, args):
    """NCCL all-gather of one step's per-request outputs to every rank: serial time
    (gather alone) and the per-step time when step i's gather overlaps step i+1's
    compute on a side stream (max over ranks)."""
    torch = st.torch
    dev = st.dev
    outs, sizes = _step_outputs(st)
    counts = {k: [sum(sizes[k][i] for i in p) for p in st.parts] for k in sizes}

    def gather_all():
        res = {}
        for k, t in outs.items():
            if sum(counts[k]) == 0:
                continue
            loc = t if t is not None else torch.zeros((0,), device=dev)
            if backend != "nccl":
                loc = loc.cpu()
            if loc.dim() > 1:
                loc = loc.reshape(loc.shape[0], -1)
            res[k] = shard.allgather_outputs(loc, counts[k])
        return res

    for _ in range(2):
        gather_all()
    torch.cuda.synchronize(dev)
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    gathered = gather_all()
    e1.record()
    torch.cuda.synchronize(dev)
    serial_ms = e0.elapsed_time(e1)
    # overlapped: the gather of step i (side stream) beside the compute of step i+1
    side = torch.cuda.Stream(dev)
    steps = max(3, min(args.steps, 10))
    dist.barrier()
    torch.cuda.synchronize(dev)
    e0.record()
    for _ in range(steps):
        done = torch.cuda.Event()
        g.replay()
        done.record()
        side.wait_event(done)
        with torch.cuda.stream(side):
            gather_all()
    torch.cuda.current_stream(dev).wait_stream(side)
    e1.record()
    torch.cuda.synchronize(dev)
    ovl_ms = e0.elapsed_time(e1) / steps
    t = torch.tensor([serial_ms, ovl_ms], dtype=torch.float64)
    if backend == "nccl":
        t = t.to(dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    # reassembly check: every rank holds the global outputs in request order
    n_ok = 0
    for k, gt in gathered.items():
        per_req = shard.reassemble(gt, st.parts, sizes[k])
        n_ok += sum(1 for x in per_req if x is not None)
    nbytes = {k: sum(counts[k]) * (outs[k][0].numel() * outs[k].element_size() if outs[k] is not None and
                                   outs[k].shape[0] else 0) for k in counts}
    return {"serial_ms": float(t[0]), "overlapped_ms_per_step": float(t[1]),
            "gathered": sorted(gathered), "bytes_gathered_per_rank": int(sum(nbytes.values())),
            "backend": backend, "requests_reassembled": n_ok,
            "note": "serial: all outputs of one step gathered alone; overlapped: per-step time with step i's "
                    "gather on a side stream beside step i+1's graph replay"}


def e2e_result(st, args, dist, backend):
    """The metric through the public API from pinned HOST buffers: each step copies
    its inputs to the device and its outputs back, pipelined the way a serving loop
    runs them (step i's read-back on a second stream beside step i+1's input copy)."""
    torch = st.torch
    dev = st.dev
    stream = torch.cuda.current_stream(dev)
    h_in, d_in, d_out = [], [], []
    seen = set()

    def add_in(host, dev_t):
        if id(dev_t) not in seen:    # a mixed batch's phases share one cache: copied once
            seen.add(id(dev_t))
            h_in.append(host.pin_memory())
            d_in.append(dev_t)

    for pc in st.pieces:
        ht, tb, (_, tidx, _, _) = pc["host"], pc["buf"], pc["p"].layout()
        add_in(ht["k_cache"], pc["t"][2])
        add_in(ht["v_cache"], pc["t"][3])
        if pc["reuse"]:
            add_in(ht["q_blk"], pc["t"][1])
            d_out.append(tb.out_blk)
        if pc["refresh"]:
            add_in(ht["q"], pc["t"][0])
            d_out += [tb.out, tb.idx[:max(tidx, 1)]]
        else:
            h_in.append(tb.idx[:max(tidx, 1)].cpu().pin_memory())
            d_in.append(tb.idx[:max(tidx, 1)])
    h_out = [torch.empty(t.shape, dtype=t.dtype).pin_memory() for t in d_out]
    h2d = sum(t.numel() * t.element_size() for t in h_in)
    d2h = sum(t.numel() * t.element_size() for t in h_out)
    d2h_stream = torch.cuda.Stream(dev)
    d2h_done = [None]

    def e2e_step():
        for d, h in zip(d_in, h_in):
            d.copy_(h, non_blocking=True)
        if d2h_done[0] is not None:
            stream.wait_event(d2h_done[0])
        st.step()
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
    if dist is not None:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.e2e_steps):
        e2e_step()
    stream.wait_event(d2h_done[0])      # the last step's results are on the host
    e1.record(stream)
    torch.cuda.synchronize(dev)
    te = torch.tensor([e0.elapsed_time(e1) * 1e-3], dtype=torch.float64)
    if dist is not None:
        if backend == "nccl":
            te = te.to(dev)
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    return {"value": st.glob.num_requests * args.e2e_steps / float(te.item()), "unit": UNIT,
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "steps": args.e2e_steps,
            "pipelining": "D2H of step i on a second stream beside the H2D of step i+1"}


if __name__ == "__main__":
    main()
