"""GPU, two ranks: the batch LPT-partitioned over two
processes that share cuda:0, each running its shard through libdllm, the
per-request outputs all-gathered with gloo on the CPU and reassembled in request
order (shard.reassemble) — bit-identical to one process running the whole batch.
Requests are independent (each carries its own lengths and KV), so
sharding must not change a single bit."""
import os
import socket

import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _outputs(lib, synth, wl, dev):
    """Refresh rows, index lists (Refresh requests) and Reuse rows of one step, as
    per-request CPU tensors in wl's request order.  Mixed batches (refresh_mask):
    Refresh + select for the Refresh requests and Reuse (on generated index lists)
    for the others, in one dllm_mixed_attn launch."""
    batch = synth.make_batch(wl)
    B, H = wl.num_requests, wl.num_heads

    def problem(sub, bt):
        return lib.Problem(sub.seq_len, sub.blk_start, sub.blk_end, num_heads=H, num_kv_heads=sub.num_kv_heads,
                           head_dim=sub.head_dim, keep_ratio=sub.keep_ratio, pool_window=sub.pool_window,
                           page_size=sub.page_size, block_table=bt.contiguous().to(dev))

    res = {"out": [torch.zeros(0)] * B, "idx": [torch.zeros(0, dtype=torch.int32)] * B,
           "out_blk": [torch.zeros(0)] * B}
    kc, vc = batch.k_cache.to(dev), batch.v_cache.to(dev)
    if wl.refresh_mask is None:
        p = problem(wl, batch.block_table)
        buf = lib.alloc_buffers(p, device=dev)
        lib.refresh_attn(p, batch.q.to(dev), kc, vc, buf.out, buf.scores)
        lib.select_heads(p, buf.scores, buf.idx)
        lib.reuse_sparse_attn(p, batch.q_blk.to(dev), kc, vc, buf.idx, buf.out_blk)
        torch.cuda.synchronize(dev)
        k, total_idx, _, _ = p.layout()
        out, idx, ob = buf.out.cpu(), buf.idx[:total_idx].cpu(), buf.out_blk.cpu()
        oi = ii = 0
        for b in range(B):
            L, blk = wl.seq_len[b], wl.blk[b]
            res["out"][b] = out[batch.cu_seqlens[b]:batch.cu_seqlens[b] + L]
            res["idx"][b] = idx[ii:ii + H * k[b]]
            res["out_blk"][b] = ob[batch.cu_blk[b]:batch.cu_blk[b] + blk]
            ii += H * k[b]
        return res
    ri = [i for i, m in enumerate(wl.refresh_mask) if m]
    ui = [i for i, m in enumerate(wl.refresh_mask) if not m]
    import numpy as np
    pr = pu = br = bu = None
    if ri:
        sr = synth.subset(wl, ri)
        pr = problem(sr, batch.block_table[ri])
        br = lib.alloc_buffers(pr, device=dev)
        q = torch.cat([batch.q_req(b) for b in ri]).to(dev)
    if ui:
        su = synth.subset(wl, ui)
        pu = problem(su, batch.block_table[ui])
        bu = lib.alloc_buffers(pu, device=dev)
        ku = pu.layout()[0]
        flat = np.concatenate([x.reshape(-1) for x in synth.indices(su, ku)]).astype(np.int32)
        bu.idx[:flat.size].copy_(torch.from_numpy(flat))
        qb = torch.cat([batch.q_blk_req(b) for b in ui]).to(dev)
    if ri and ui:
        lib.mixed_attn(pr, q, br.out, br.scores, pu, qb, bu.idx, bu.out_blk, kc, vc)
    elif ri:
        lib.refresh_attn(pr, q, kc, vc, br.out, br.scores)
    else:
        lib.reuse_sparse_attn(pu, qb, kc, vc, bu.idx, bu.out_blk)
    if ri:
        lib.select_heads(pr, br.scores, br.idx)
    torch.cuda.synchronize(dev)
    if ri:
        kr, tr, _, _ = pr.layout()
        out, idx = br.out.cpu(), br.idx[:tr].cpu()
        o = i = 0
        for j, b in enumerate(ri):
            L = wl.seq_len[b]
            res["out"][b] = out[o:o + L]
            res["idx"][b] = idx[i:i + H * kr[j]]
            o += L
            i += H * kr[j]
    if ui:
        ob = bu.out_blk.cpu()
        o = 0
        for b in ui:
            res["out_blk"][b] = ob[o:o + wl.blk[b]]
            o += wl.blk[b]
    return res


def _worker(rank, world, port, cfg, n, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    # one Reuse kernel for every batch size (the library picks mma.sync for small
    # batches: a shard and the whole batch could otherwise round differently)
    os.environ["DLLM_REUSE_IMPL"] = "tc"
    import torch.distributed as dist

    from paper_2512_17077_b200 import lib, shard, synth
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        _run_rank(rank, world, cfg, n, q, dist, lib, shard, synth)
    except Exception:   # report instead of leaving the parent waiting
        import traceback
        q.put((rank, "error: " + traceback.format_exc(), None))
    finally:
        dist.destroy_process_group()


def _run_rank(rank, world, cfg, n, q, dist, lib, shard, synth):
    if True:
        dev = torch.device("cuda", 0)
        torch.cuda.set_device(dev)
        glob = synth.config(cfg, num_requests=n)
        if glob.refresh_mask is not None:
            glob.refresh_mask = [i % 4 == 0 for i in range(n)]   # a burst mix in the truncated batch
        k = [lib.keep_count(glob.keep_ratio, L - (e - s)) for L, s, e in zip(glob.seq_len, glob.blk_start,
                                                                            glob.blk_end)]
        parts = shard.lpt_partition(shard.workload_costs(glob, k), world)
        mine = parts[rank]
        local = _outputs(lib, synth, synth.subset(glob, mine), dev)
        ref_all = _outputs(lib, synth, glob, dev) if rank == 0 else None
        ok = True
        for name in ("out", "idx", "out_blk"):
            sizes = [0] * glob.num_requests
            for r, p in enumerate(parts):
                sub_r = synth.subset(glob, p)
                for j, gi in enumerate(p):
                    m = None if glob.refresh_mask is None else glob.refresh_mask[gi]
                    L, blk = sub_r.seq_len[j], sub_r.blk[j]
                    if name == "out":
                        sizes[gi] = L if m is not False else 0
                    elif name == "idx":
                        sizes[gi] = glob.num_heads * k[gi] if m is not False else 0
                    else:
                        sizes[gi] = blk if m is not True else 0
            mine_t = [local[name][j] for j in range(len(mine)) if local[name][j].numel() > 0]
            # every rank contributes [rows, width] of one dtype, even with no rows of its own
            width, dtype = (1, torch.int32) if name == "idx" else (glob.num_heads * glob.head_dim, torch.bfloat16)
            cat = torch.cat([t.reshape(-1, width) for t in mine_t]) if mine_t else torch.zeros((0, width), dtype=dtype)
            counts = [sum(sizes[i] for i in p) for p in parts]
            gathered = shard.allgather_outputs(cat.contiguous(), counts)
            per_req = shard.reassemble(gathered, parts, sizes)
            if rank == 0:
                ref = ref_all[name]
                for b in range(glob.num_requests):
                    a = per_req[b].reshape(-1)
                    r_ = ref[b].reshape(-1)
                    if a.numel() != r_.numel() or not torch.equal(a.view(torch.int16) if a.dtype == torch.bfloat16
                                                                  else a, r_.view(torch.int16)
                                                                  if r_.dtype == torch.bfloat16 else r_):
                        ok = False
        q.put((rank, ok, [len(p) for p in parts]))


@pytest.mark.parametrize("cfg,n", [("C1", 6), ("C3", 12)])
def test_two_ranks_reassemble_bit_identical(cfg, n):
    assert torch.cuda.is_available()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, cfg, n, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict((r, (ok, sizes)) for r, ok, sizes in (q.get(timeout=300) for _ in procs))
    for p in procs:
        p.join(timeout=120)
    for r in res:
        assert not (isinstance(res[r][0], str) and res[r][0].startswith("error")), res[r][0]
    assert all(res[r][1] == res[0][1] for r in res) and min(res[0][1]) >= 1, res
    assert res[0][0], f"{cfg}: reassembled two-rank outputs differ from the single-process run"
