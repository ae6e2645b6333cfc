"""Per-kernel timing on one config (dev tool; bench.py is the contract).

    python scripts/kbench.py C1 [--iters 20] [--impl mma|tc]
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_17077_b200 import lib, synth  # noqa: E402


def reuse_unique_bytes(wl, k, idx_flat):
    g = wl.num_heads // wl.num_kv_heads
    D = wl.head_dim
    total, logical, off = 0, 0, 0
    for b in range(wl.num_requests):
        kb = k[b]
        rows = idx_flat[off:off + wl.num_heads * kb].reshape(wl.num_heads, kb)
        off += wl.num_heads * kb
        blk = wl.blk_end[b] - wl.blk_start[b]
        for kv in range(wl.num_kv_heads):
            u = np.unique(rows[kv * g:(kv + 1) * g])
            total += (len(u) + blk) * 2 * D * 2
        logical += wl.num_heads * (kb + blk) * 2 * D * 2
    extra = sum(wl.blk) * wl.num_heads * D * 2 * 2 + len(idx_flat) * 4
    return total + extra, logical + extra


def _with_env(k, v, f):
    os.environ[k] = v
    try:
        f()
    finally:
        del os.environ[k]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cfg", nargs="?", default="C1")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--r", type=float, default=None)
    args = ap.parse_args()
    wl = synth.config(args.cfg, keep_ratio=args.r)
    batch = synth.make_batch(wl)
    bt = batch.block_table.cuda()
    p = lib.Problem(wl.seq_len, wl.blk_start, wl.blk_end, num_heads=wl.num_heads, num_kv_heads=wl.num_kv_heads,
                    head_dim=wl.head_dim, keep_ratio=wl.keep_ratio, pool_window=wl.pool_window,
                    page_size=wl.page_size, block_table=bt)
    q, qb, kc, vc = batch.q.cuda(), batch.q_blk.cuda(), batch.k_cache.cuda(), batch.v_cache.cuda()
    buf = lib.alloc_buffers(p)
    gidx = torch.empty_like(buf.idx)   # one set per KV group (select_groups), for the group kernel
    flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    fns = {
        "refresh": lambda: lib.refresh_attn(p, q, kc, vc, buf.out, buf.scores),
        "select": lambda: lib.select_heads(p, buf.scores, buf.idx),
        "reuse": lambda: lib.reuse_sparse_attn(p, qb, kc, vc, buf.idx, buf.out_blk),
        "reuse_union": lambda: _with_env("DLLM_REUSE_IMPL", "union",
                                         lambda: lib.reuse_sparse_attn(p, qb, kc, vc, buf.idx, buf.out_blk)),
        "select_groups": lambda: lib.select_groups(p, buf.scores, gidx),
        "reuse_group_sets": lambda: lib.reuse_group_sets(p, qb, kc, vc, gidx, buf.out_blk),
        "reuse_per_head_on_group_sets": lambda: lib.reuse_sparse_attn(p, qb, kc, vc, gidx, buf.out_blk),
        "refresh_select": lambda: lib.refresh_select_attn(p, q, kc, vc, buf.out, buf.scores, buf.idx),
    }
    k_, total_idx_, _, _ = p.layout()
    kp = torch.empty((max(total_idx_, 1), wl.head_dim), dtype=torch.bfloat16, device="cuda")
    vp = torch.empty_like(kp)
    fns["pack"] = lambda: lib.pack_kv(p, kc, vc, buf.idx, kp, vp)
    fns["reuse_packed"] = lambda: lib.reuse_packed(p, qb, kc, vc, kp, vp, buf.out_blk)
    for f in fns.values():
        f()
    torch.cuda.synchronize()
    res = {}
    for name, f in fns.items():
        ts = []
        for _ in range(args.iters):
            flush.zero_()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            f()
            e.record()
            torch.cuda.synchronize()
            ts.append(s.elapsed_time(e) * 1e-3)
        res[name] = (np.median(ts), np.min(ts))
    k, total_idx, rows, _ = p.layout()
    flops = sum(4 * wl.num_heads * L * L * wl.head_dim for L in wl.seq_len)
    ub, lb = reuse_unique_bytes(wl, k, buf.idx.cpu().numpy()[:total_idx])
    sel_bytes = 4 * wl.num_heads * rows + 4 * total_idx
    t = res["refresh"][0]
    print(f"{args.cfg} refresh: {t*1e6:.1f} us  {flops/t/1e12:.1f} TFLOP/s (min {res['refresh'][1]*1e6:.1f})")
    t = res["select"][0]
    print(f"{args.cfg} select : {t*1e6:.1f} us  {sel_bytes/t/1e9:.1f} GB/s")
    t = res["refresh_select"][0]
    print(f"{args.cfg} refresh+select fused: {t*1e6:.1f} us  {flops/t/1e12:.1f} TFLOP/s (Refresh FLOP; min "
          f"{res['refresh_select'][1]*1e6:.1f})")
    t = res["reuse"][0]
    print(f"{args.cfg} reuse  : {t*1e6:.1f} us  {ub/t/1e9:.1f} GB/s unique ({lb/t/1e9:.1f} logical), "
          f"unique {ub/1e6:.1f} MB")
    t = res["reuse_union"][0]
    print(f"{args.cfg} reuse (union of up to 4 heads' sets, DLLM_REUSE_IMPL=union): {t*1e6:.1f} us  "
          f"{ub/t/1e9:.1f} GB/s unique")
    gub, glb = reuse_unique_bytes(wl, k, gidx.cpu().numpy()[:total_idx])
    t = res["select_groups"][0]
    print(f"{args.cfg} select_groups: {t*1e6:.1f} us")
    for name in ("reuse_group_sets", "reuse_per_head_on_group_sets"):
        t = res[name][0]
        print(f"{args.cfg} {name}: {t*1e6:.1f} us  {gub/t/1e9:.1f} GB/s unique ({glb/t/1e9:.1f} logical), "
              f"unique {gub/1e6:.1f} MB (min {res[name][1]*1e6:.1f})")
    t = res["pack"][0]
    pb = 2 * 2 * total_idx * wl.head_dim * 2
    print(f"{args.cfg} pack   : {t*1e6:.1f} us  {pb/t/1e9:.1f} GB/s (read+write {pb/1e6:.1f} MB)")
    t = res["reuse_packed"][0]
    print(f"{args.cfg} reuse_packed: {t*1e6:.1f} us  {lb/t/1e9:.1f} GB/s logical")
    print(lib.version())


if __name__ == "__main__":
    main()
