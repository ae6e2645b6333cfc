"""GPU parity for the single-launch mixed-phase batch (next row N3,
dllm_mixed_attn): one launch computes Refresh for some
requests and Reuse for the others over ONE paged cache.  Its outputs must be
bit-identical to the two separate calls (same kernels, same arithmetic) and
match the fp64 oracle within the north_star tolerances."""
import os

import numpy as np
import pytest
import torch

import oracle as O
from paper_2512_17077_b200 import synth
from tests._util import assert_close, f64, join_idx

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def L():
    from paper_2512_17077_b200 import lib
    return lib


def _split(L, wl, batch, ri, ui):
    dev = "cuda"

    def prob(reqs):
        sub = synth.subset(wl, reqs)
        bt = batch.block_table[reqs].contiguous().to(dev) if reqs else torch.zeros((0, batch.block_table.shape[1]),
                                                                                   dtype=torch.int32, device=dev)
        return sub, L.Problem(sub.seq_len, sub.blk_start, sub.blk_end, num_heads=wl.num_heads,
                              num_kv_heads=wl.num_kv_heads, head_dim=wl.head_dim, keep_ratio=wl.keep_ratio,
                              pool_window=wl.pool_window, page_size=wl.page_size, block_table=bt)

    sr, pr = prob(ri)
    su, pu = prob(ui)
    q = torch.cat([batch.q_req(b) for b in ri]).to(dev) if ri else torch.zeros((1, wl.num_heads, wl.head_dim),
                                                                              dtype=torch.bfloat16, device=dev)
    qb = torch.cat([batch.q_blk_req(b) for b in ui]).to(dev) if ui else torch.zeros((1, wl.num_heads, wl.head_dim),
                                                                                   dtype=torch.bfloat16, device=dev)
    ku = pu.layout()[0] if ui else []
    idx_list = synth.indices(su, ku) if ui else []
    flat = join_idx(idx_list)
    idx = torch.from_numpy(flat).to(dev) if flat.size else torch.zeros(1, dtype=torch.int32, device=dev)
    return sr, pr, su, pu, q, qb, idx, idx_list


def _outputs(wl, pr, pu, q):
    rows = pr.layout()[2] if pr.num_requests else 1
    blk_rows = pu.layout()[3] if pu.num_requests else 1
    out = torch.full((max(rows, 1), wl.num_heads, wl.head_dim), float("nan"), dtype=torch.bfloat16, device="cuda")
    sc = torch.full((max(wl.num_heads * rows, 1),), float("nan"), dtype=torch.float32, device="cuda")
    ob = torch.full((max(blk_rows, 1), wl.num_heads, wl.head_dim), float("nan"), dtype=torch.bfloat16, device="cuda")
    return out, sc, ob


def _mixed_vs_separate(L, wl, ri, ui, check_oracle=()):
    # the mixed launch runs the tcgen05 Reuse body: compare with the tcgen05 kernel
    # (dllm_reuse_sparse_attn would pick the mma.sync kernel for small batches)
    os.environ["DLLM_REUSE_IMPL"] = "tc"
    try:
        _mixed_vs_separate_tc(L, wl, ri, ui, check_oracle)
    finally:
        del os.environ["DLLM_REUSE_IMPL"]


def _mixed_vs_separate_tc(L, wl, ri, ui, check_oracle=()):
    batch = synth.make_batch(wl)
    kc, vc = batch.k_cache.cuda(), batch.v_cache.cuda()
    sr, pr, su, pu, q, qb, idx, idx_list = _split(L, wl, batch, ri, ui)
    out_m, sc_m, ob_m = _outputs(wl, pr, pu, q)
    L.mixed_attn(pr, q, out_m, sc_m, pu, qb, idx, ob_m, kc, vc)
    out_s, sc_s, ob_s = _outputs(wl, pr, pu, q)
    if ri:
        L.refresh_attn(pr, q, kc, vc, out_s, sc_s)
    if ui:
        L.reuse_sparse_attn(pu, qb, kc, vc, idx, ob_s)
    torch.cuda.synchronize()
    if ri:
        assert torch.equal(out_m.view(torch.int16), out_s.view(torch.int16))
        assert torch.equal(sc_m.view(torch.int32), sc_s.view(torch.int32))
    if ui:
        assert torch.equal(ob_m.view(torch.int16), ob_s.view(torch.int16))
    # oracle on a few requests of each phase
    got_o, got_b = out_m.float().cpu().numpy(), ob_m.float().cpu().numpy()
    cu_r = np.concatenate([[0], np.cumsum([wl.seq_len[b] for b in ri])]).astype(int)
    cu_u = np.concatenate([[0], np.cumsum([wl.blk[b] for b in ui])]).astype(int)
    for j, b in enumerate(ri):
        if j in check_oracle:
            ref = O.attention_dense(f64(batch.q_req(b)), f64(batch.k_logical(b)), f64(batch.v_logical(b)))
            assert_close(got_o[cu_r[j]:cu_r[j + 1]], ref, f"mixed refresh req {b}")
    for j, b in enumerate(ui):
        if j in check_oracle:
            ref = O.attention_with_cache(f64(batch.q_blk_req(b)), f64(batch.k_logical(b)), f64(batch.v_logical(b)),
                                         wl.blk_start[b], wl.blk_end[b], idx_list[j])
            assert_close(got_b[cu_u[j]:cu_u[j + 1]], ref, f"mixed reuse req {b}")


@pytest.mark.parametrize("n,every", [(24, 6), (40, 4), (12, 2)])
def test_mixed_c3_shape_bit_identical_to_separate(L, n, every):
    wl = synth.config("C3", num_requests=n)
    ri = [i for i in range(n) if i % every == 0]
    ui = [i for i in range(n) if i % every != 0]
    _mixed_vs_separate(L, wl, ri, ui, check_oracle=(0, 1))


def test_mixed_gqa_shape(L):
    wl = synth.config("C2", num_requests=6)
    _mixed_vs_separate(L, wl, [0, 3], [1, 2, 4, 5], check_oracle=(0,))


def test_mixed_one_phase_empty_falls_back(L):
    wl = synth.config("C1", num_requests=3)
    _mixed_vs_separate(L, wl, [0, 1, 2], [], check_oracle=(0,))
    _mixed_vs_separate(L, wl, [], [0, 1, 2], check_oracle=(0,))


def test_mixed_realistic_c3_full_step(L):
    # the C3 burst batch itself: 8 Refresh + 248 Reuse requests, sampled oracle checks
    wl = synth.config("C3")
    ri = [i for i, m in enumerate(wl.refresh_mask) if m]
    ui = [i for i, m in enumerate(wl.refresh_mask) if not m]
    _mixed_vs_separate(L, wl, ri, ui, check_oracle=(0, 247))
