"""Dev A/B: how the L2 flush before a timed launch changes the HBM-bound kernels.

    python scripts/flush_ab.py C1 [--iters 20]

"write": the bench's flush (512 MiB zero_) leaves ~L2-size DIRTY lines, so the
timed kernel's first reads evict them and pay their write-back;
"write+read": the same write, then a read of a separate 384 MiB buffer, so the
L2 holds only clean lines of that buffer (still none of the kernel's inputs);
"hot": no flush (inputs partly L2-resident) -- context only.
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_17077_b200 import lib, synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cfg", nargs="?", default="C1")
    ap.add_argument("--iters", type=int, default=20)
    args = ap.parse_args()
    wl = synth.config(args.cfg)
    batch = synth.make_batch(wl)
    bt = batch.block_table.cuda()
    p = lib.Problem(wl.seq_len, wl.blk_start, wl.blk_end, num_heads=wl.num_heads, num_kv_heads=wl.num_kv_heads,
                    head_dim=wl.head_dim, keep_ratio=wl.keep_ratio, pool_window=wl.pool_window,
                    page_size=wl.page_size, block_table=bt)
    q, qb, kc, vc = batch.q.cuda(), batch.q_blk.cuda(), batch.k_cache.cuda(), batch.v_cache.cuda()
    buf = lib.alloc_buffers(p)
    lib.refresh_attn(p, q, kc, vc, buf.out, buf.scores)
    lib.select_heads(p, buf.scores, buf.idx)
    n82 = 82 * 1024 * 1024 // 2
    src = torch.randn(n82, dtype=torch.bfloat16, device="cuda")
    dst = torch.empty(64, dtype=torch.float32, device="cuda")
    wflush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    rflush = torch.ones(384 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    fns = {
        "reuse": lambda: lib.reuse_sparse_attn(p, qb, kc, vc, buf.idx, buf.out_blk),
        "select": lambda: lib.select_heads(p, buf.scores, buf.idx),
        "refresh": lambda: lib.refresh_attn(p, q, kc, vc, buf.out, buf.scores),
        "torch_sum_82MB": lambda: src.view(-1, 4096).sum(dim=0),
        "empty_fill_64B": lambda: dst.zero_(),
    }
    modes = {
        "write": lambda: wflush.zero_(),
        "write+read": lambda: (wflush.zero_(), rflush.sum()),
        "hot": lambda: None,
    }
    for f in fns.values():
        f()
    torch.cuda.synchronize()
    for name, f in fns.items():
        for mname, m in modes.items():
            ts = []
            for _ in range(args.iters):
                m()
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                f()
                e.record()
                torch.cuda.synchronize()
                ts.append(s.elapsed_time(e) * 1e3)
            print(f"{args.cfg} {name:16s} flush={mname:10s} median {np.median(ts):8.1f} us  min {np.min(ts):8.1f}")


if __name__ == "__main__":
    main()
