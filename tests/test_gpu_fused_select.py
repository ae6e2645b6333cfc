"""GPU parity for the select fused into the Refresh kernel (next row N1, second
half; dllm_refresh_select_attn / dllm_mixed_select_attn).  The selection of
Eq. 6 + TopK (§4.5) runs in the tcgen05 Refresh kernel's
epilogue warpgroup; the result must be bit-identical to dllm_refresh_attn +
dllm_select_heads (out, scores AND idx), and, on exact-integer inputs, equal
to the fp64 oracle's selection index for index.  (The default library build
runs the two kernels behind this call; a DLLM_TC2_FUSEDSEL=1 build runs the
select inside the Refresh kernel -- both must pass these tests.)"""
import numpy as np
import pytest
import torch

import oracle as O
from paper_2512_17077_b200 import synth
from tests._util import f64, join_idx, problem_of, to_dev
from tests.test_gpu_parity import EDGE

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def L():
    assert torch.cuda.is_available(), "GPU tests need a B200"
    from paper_2512_17077_b200 import lib
    return lib


def _bufs(wl, p):
    k, total_idx, rows, blk_rows = p.layout()
    out = torch.full((max(rows, 1), wl.num_heads, wl.head_dim), float("nan"), dtype=torch.bfloat16, device="cuda")
    sc = torch.full((max(wl.num_heads * rows, 1),), float("nan"), dtype=torch.float32, device="cuda")
    idx = torch.full((max(total_idx, 1),), -7, dtype=torch.int32, device="cuda")
    return out, sc, idx, total_idx


def _fused_vs_separate(L, batch):
    wl = batch.wl
    p = problem_of(batch)
    q, q_blk, kc, vc = to_dev(batch)
    out_f, sc_f, idx_f, n_idx = _bufs(wl, p)
    L.refresh_select_attn(p, q, kc, vc, out_f, sc_f, idx_f)
    out_s, sc_s, idx_s, _ = _bufs(wl, p)
    L.refresh_attn(p, q, kc, vc, out_s, sc_s)
    L.select_heads(p, sc_s, idx_s)
    torch.cuda.synchronize()
    assert torch.equal(out_f.view(torch.int16), out_s.view(torch.int16))
    assert torch.equal(sc_f.view(torch.int32), sc_s.view(torch.int32))
    assert torch.equal(idx_f[:n_idx], idx_s[:n_idx])
    return idx_f.cpu().numpy()[:n_idx]


def _oracle_sel(batch):
    wl = batch.wl
    return join_idx([O.select_heads(f64(batch.q_req(b))[wl.blk_start[b]:wl.blk_end[b]], f64(batch.k_logical(b)),
                                    wl.seq_len[b], wl.blk_start[b], wl.blk_end[b], wl.keep_ratio, wl.pool_window)
                     for b in range(wl.num_requests)])


@pytest.mark.parametrize("cfg,n", [("C0", None), ("C1", 3), ("C2", 2), ("C3", 4), ("C4", 1)])
def test_fused_select_exact_matches_oracle(L, cfg, n):
    batch = synth.make_batch(synth.config(cfg, num_requests=n, kind="exact"))
    got = _fused_vs_separate(L, batch)
    assert np.array_equal(got, _oracle_sel(batch))


@pytest.mark.parametrize("cfg,n", [("C1", None), ("C2", 8), ("C3", 16)])
def test_fused_select_realistic_bit_identical(L, cfg, n):
    _fused_vs_separate(L, synth.make_batch(synth.config(cfg, num_requests=n)))


@pytest.mark.parametrize("name", sorted(EDGE))
def test_fused_select_edges(L, name):
    # includes n_ctx > 4096 (long_8k: falls back to the select launch), k = 0, w = 1 / 5,
    # D < 64 (mma.sync Refresh + select launch), blocks straddling Q tiles
    wl = synth.Workload(**{**EDGE[name].__dict__, "kind": "exact"})
    batch = synth.make_batch(wl)
    got = _fused_vs_separate(L, batch)
    assert np.array_equal(got, _oracle_sel(batch))


def test_mixed_select_bit_identical(L):
    from tests.test_gpu_mixed import _outputs, _split
    wl = synth.config("C3", num_requests=24)
    batch = synth.make_batch(wl)
    kc, vc = batch.k_cache.cuda(), batch.v_cache.cuda()
    ri = [i for i in range(24) if i % 4 == 0]
    ui = [i for i in range(24) if i % 4 != 0]
    sr, pr, su, pu, q, qb, idx, idx_list = _split(L, wl, batch, ri, ui)
    n_idx = pr.layout()[1]
    out_m, sc_m, ob_m = _outputs(wl, pr, pu, q)
    sel_m = torch.full((max(n_idx, 1),), -7, dtype=torch.int32, device="cuda")
    L.mixed_select_attn(pr, q, out_m, sc_m, sel_m, pu, qb, idx, ob_m, kc, vc)
    out_s, sc_s, ob_s = _outputs(wl, pr, pu, q)
    sel_s = torch.full((max(n_idx, 1),), -7, dtype=torch.int32, device="cuda")
    L.mixed_attn(pr, q, out_s, sc_s, pu, qb, idx, ob_s, kc, vc)
    L.select_heads(pr, sc_s, sel_s)
    torch.cuda.synchronize()
    assert torch.equal(out_m.view(torch.int16), out_s.view(torch.int16))
    assert torch.equal(sc_m.view(torch.int32), sc_s.view(torch.int32))
    assert torch.equal(ob_m.view(torch.int16), ob_s.view(torch.int16))
    assert torch.equal(sel_m[:n_idx], sel_s[:n_idx])
