"""Dev: CUDA-event time of the Reuse launch alone (L2 flushed before each), for A/B of builds.

    DLLM_LIB=paper_2512_17077_b200/libdllm_<tag>.so python scripts/reuse_time.py C1 [iters]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_17077_b200 import lib, synth  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C1"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 30
wl = synth.config(cfg)
b = synth.make_batch(wl)
p = lib.Problem(wl.seq_len, wl.blk_start, wl.blk_end, num_heads=wl.num_heads, num_kv_heads=wl.num_kv_heads,
                head_dim=wl.head_dim, keep_ratio=wl.keep_ratio, pool_window=wl.pool_window, page_size=wl.page_size,
                block_table=b.block_table.cuda())
q, qb, kc, vc = b.q.cuda(), b.q_blk.cuda(), b.k_cache.cuda(), b.v_cache.cuda()
buf = lib.alloc_buffers(p)
lib.refresh_attn(p, q, kc, vc, buf.out, buf.scores)
lib.select_heads(p, buf.scores, buf.idx)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for _ in range(3):
    lib.reuse_sparse_attn(p, qb, kc, vc, buf.idx, buf.out_blk)
torch.cuda.synchronize()
ts = []
for _ in range(iters):
    flush.zero_()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    lib.reuse_sparse_attn(p, qb, kc, vc, buf.idx, buf.out_blk)
    e.record()
    torch.cuda.synchronize()
    ts.append(s.elapsed_time(e) * 1e-3)
t = float(np.median(ts))
print(f"{os.path.basename(os.environ.get('DLLM_LIB', 'libdllm.so'))} {cfg} reuse {t * 1e6:.1f} us (min {min(ts) * 1e6:.1f})")
