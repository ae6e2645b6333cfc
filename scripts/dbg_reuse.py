import os, sys, time
sys.path.insert(0, os.getcwd())
import torch, numpy as np
from paper_2512_17077_b200 import lib, synth
from tests._util import problem_of, to_dev, join_idx, oracle_keep_counts
for cfg, n, ws in [("C0", None, True), ("C1", 4, False), ("C1", 4, True), ("C2", 2, True), ("C3", 6, True), ("C1", None, True)]:
    wl = synth.config(cfg, num_requests=n)
    batch = synth.make_batch(wl)
    p = problem_of(batch)
    if not ws:
        p = lib.Problem(wl.seq_len, wl.blk_start, wl.blk_end, num_heads=wl.num_heads, num_kv_heads=wl.num_kv_heads,
                        head_dim=wl.head_dim, keep_ratio=wl.keep_ratio, pool_window=wl.pool_window,
                        page_size=wl.page_size, block_table=batch.block_table.cuda(), workspace=None)
    k = oracle_keep_counts(wl)
    idx = torch.from_numpy(join_idx(synth.indices(wl, k))).cuda()
    q, qb, kc, vc = to_dev(batch)
    out = torch.zeros((sum(wl.blk), wl.num_heads, wl.head_dim), dtype=torch.bfloat16, device="cuda")
    print(cfg, n, "ws" if ws else "nows", flush=True)
    lib.reuse_sparse_attn(p, qb, kc, vc, idx, out)
    torch.cuda.synchronize()
    print("  ok, finite:", bool(torch.isfinite(out.float()).all()), flush=True)
