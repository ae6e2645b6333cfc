"""Sanitizer tier: one pass of every kernel of the path on small
configs, meant to run under compute-sanitizer (memcheck / racecheck / synccheck):

    compute-sanitizer --tool memcheck python scripts/sanitize.py

Refresh (tcgen05) -> select -> Reuse (tcgen05) on C0 (mma.sync paths, D = 16),
2-request C1 and C2 (GQA) batches, one mixed launch on a 12-request burst mix, the
uniform select, the pack + packed Reuse, and a small LM-head argmax."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_17077_b200 import lib, synth  # noqa: E402


def problem(wl, bt):
    return lib.Problem(wl.seq_len, wl.blk_start, wl.blk_end, num_heads=wl.num_heads, num_kv_heads=wl.num_kv_heads,
                       head_dim=wl.head_dim, keep_ratio=wl.keep_ratio, pool_window=wl.pool_window,
                       page_size=wl.page_size, block_table=bt.contiguous().cuda())


def hot_path(cfg, n):
    wl = synth.config(cfg, num_requests=n)
    b = synth.make_batch(wl)
    p = problem(wl, b.block_table)
    q, qb, kc, vc = b.q.cuda(), b.q_blk.cuda(), b.k_cache.cuda(), b.v_cache.cuda()
    buf = lib.alloc_buffers(p)
    lib.refresh_attn(p, q, kc, vc, buf.out, buf.scores)
    lib.select_heads(p, buf.scores, buf.idx)
    lib.reuse_sparse_attn(p, qb, kc, vc, buf.idx, buf.out_blk)
    lib.select_global(p, buf.scores, buf.idx)
    _, total_idx, _, _ = p.layout()
    kp = torch.empty((max(total_idx, 1), wl.head_dim), dtype=torch.bfloat16, device="cuda")
    vp = torch.empty_like(kp)
    lib.pack_kv(p, kc, vc, buf.idx, kp, vp)
    lib.reuse_packed(p, qb, kc, vc, kp, vp, buf.out_blk)
    torch.cuda.synchronize()
    print(f"{cfg} x{wl.num_requests}: ok", flush=True)


def mixed(n):
    wl = synth.config("C3", num_requests=n)
    b = synth.make_batch(wl)
    ri = [i for i in range(n) if i % 4 == 0]
    ui = [i for i in range(n) if i % 4]
    pr, pu = problem(synth.subset(wl, ri), b.block_table[ri]), problem(synth.subset(wl, ui), b.block_table[ui])
    br, bu = lib.alloc_buffers(pr), lib.alloc_buffers(pu)
    ku = pu.layout()[0]
    flat = np.concatenate([x.reshape(-1) for x in synth.indices(synth.subset(wl, ui), ku)]).astype(np.int32)
    bu.idx[:flat.size].copy_(torch.from_numpy(flat))
    q = torch.cat([b.q_req(i) for i in ri]).cuda()
    qb = torch.cat([b.q_blk_req(i) for i in ui]).cuda()
    lib.mixed_attn(pr, q, br.out, br.scores, pu, qb, bu.idx, bu.out_blk, b.k_cache.cuda(), b.v_cache.cuda())
    lib.select_heads(pr, br.scores, br.idx)
    torch.cuda.synchronize()
    print(f"C3 mixed x{n}: ok", flush=True)


def reuse_only(cfg, n):
    wl = synth.config(cfg, num_requests=n)
    b = synth.make_batch(wl)
    p = problem(wl, b.block_table)
    k = p.layout()[0]
    idx = torch.from_numpy(np.concatenate([x.reshape(-1) for x in synth.indices(wl, k)]).astype(np.int32)).cuda()
    buf = lib.alloc_buffers(p)
    lib.reuse_sparse_attn(p, b.q_blk.cuda(), b.k_cache.cuda(), b.v_cache.cuda(), idx, buf.out_blk)
    torch.cuda.synchronize()
    print(f"reuse {cfg} x{wl.num_requests}: ok", flush=True)


def select_only(cfg, n):
    wl = synth.config(cfg, num_requests=n)
    p = problem(wl, torch.zeros((wl.num_requests, 64), dtype=torch.int32))
    sc = torch.from_numpy(np.concatenate([s.reshape(-1) for s in synth.scores(wl, mode="normal")])).cuda()
    buf = lib.alloc_buffers(p)
    lib.select_heads(p, sc, buf.idx)
    lib.select_global(p, sc, buf.idx)
    torch.cuda.synchronize()
    print(f"select {cfg} x{wl.num_requests}: ok", flush=True)


def lm_head():
    h, w = synth.lm_head_inputs(200, 256, 3000, "realistic")
    ids = torch.empty(200, dtype=torch.int32, device="cuda")
    lib.lm_head_argmax(h.cuda(), w.cuda(), ids, max_num_logits=128)
    torch.cuda.synchronize()
    print("lm_head: ok", flush=True)


if __name__ == "__main__":
    which = sys.argv[1:] or ["C0", "C1", "C2", "C3", "lm"]
    if "C0" in which:
        hot_path("C0", None)
    if "C1" in which:
        hot_path("C1", 2)
    if "C2" in which:
        hot_path("C2", 2)
    if "C3" in which:
        mixed(12)
    if "lm" in which:
        lm_head()
    if "select" in which:
        select_only("C1", 2)
        select_only("C3", 12)
    if "reuse" in which:
        reuse_only("C1", 2)
        reuse_only("C2", 2)
