"""GPU parity: the CUDA path through the C-ABI vs the fp64 oracle on the same
seeded inputs (``-m gpu``).

Contract (BASELINE.json north_star):
  * selection indices bit-exact — (i) on generated fp32 score tensors fed to
    both sides, (ii) end to end Refresh -> select on exact-integer Q/K,
    (iii) on realistic inputs a valid top-k of the oracle's fp64 scores up to
    the fp32 rounding bound;
  * attention outputs within max-abs 1e-2 and mean-abs 1e-3 of the oracle.
"""
import math

import os

import numpy as np
import pytest
import torch

import oracle as O
from paper_2512_17077_b200 import synth
from tests._util import (assert_close, f64, join_idx, join_scores, oracle_keep_counts, problem_of, split_idx,
                         split_scores, to_dev)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def L():
    assert torch.cuda.is_available(), "GPU tests need a B200"
    from paper_2512_17077_b200 import lib
    return lib


def custom(name, L_, bs, be, H=4, Hk=2, D=128, r=0.25, w=3, P=64, kind="realistic"):
    return synth.Workload(name, H, Hk, D, list(L_), list(bs), list(be), r, w, P, kind)


EDGE = {
    "single_token": custom("e_single", [1], [0], [1], H=2, Hk=2, D=64),
    "block_whole_seq": custom("e_whole", [40], [0], [40], H=2, Hk=1, D=64),
    "block_first": custom("e_first", [64], [0], [8], H=2, Hk=2, D=16, P=16),
    "block_last": custom("e_last", [64], [56], [64], H=2, Hk=2, D=16, P=16),
    "ragged_straddle": custom("e_strad", [100, 77], [60, 10], [70, 42], H=4, Hk=4, D=128),
    "blk128_straddle": custom("e_b128", [300], [100], [228], H=2, Hk=1, D=128),
    "blk1_mid": custom("e_blk1", [513], [200], [201], H=4, Hk=2, D=64, P=256),
    "gqa_d32_p16": custom("e_gqa", [130, 257, 64], [64, 225, 0], [96, 257, 32], H=8, Hk=2, D=32, P=16),
    "r1_dense": custom("e_r1", [192], [96], [128], H=2, Hk=2, D=128, r=1.0),
    "tiny_r_w5": custom("e_tiny", [333], [300], [332], H=3, Hk=1, D=64, r=0.001, w=5),
    "w1": custom("e_w1", [129], [64], [96], H=2, Hk=2, D=128, w=1),
    "p16_d128": custom("e_p16", [300, 77], [250, 40], [282, 72], H=4, Hk=2, D=128, P=16),
    "p1024_d64": custom("e_p1024", [1500], [1400], [1432], H=2, Hk=1, D=64, P=1024),
    "long_8k": custom("e_long", [8192], [8000], [8032], H=2, Hk=1, D=128, r=0.1),
    "gqa_mixed_lengths": custom("e_gqamix", [640, 129, 1025, 64], [608, 0, 993, 32], [640, 32, 1025, 64],
                                H=6, Hk=2, D=128),
}


def _run_refresh(L, batch, with_scores=True):
    p = problem_of(batch)
    q, q_blk, kc, vc = to_dev(batch)
    k, total_idx, rows, blk_rows = p.layout()
    wl = batch.wl
    out = torch.full((rows, wl.num_heads, wl.head_dim), float("nan"), dtype=torch.bfloat16, device="cuda")
    sc = torch.full((wl.num_heads * rows,), float("nan"), dtype=torch.float32, device="cuda") if with_scores else None
    L.refresh_attn(p, q, kc, vc, out, sc)
    torch.cuda.synchronize()
    return p, out.float().cpu().numpy(), (sc.cpu().numpy() if with_scores else None)


def _run_select(L, p, scores_flat):
    k, total_idx, rows, blk_rows = p.layout()
    idx = torch.full((max(total_idx, 1),), -7, dtype=torch.int32, device="cuda")
    L.select_heads(p, torch.from_numpy(np.ascontiguousarray(scores_flat, dtype=np.float32)).cuda(), idx)
    torch.cuda.synchronize()
    return k, idx.cpu().numpy()[:total_idx]


def _run_reuse(L, batch, p, idx_flat):
    q, q_blk, kc, vc = to_dev(batch)
    k, total_idx, rows, blk_rows = p.layout()
    wl = batch.wl
    out = torch.full((blk_rows, wl.num_heads, wl.head_dim), float("nan"), dtype=torch.bfloat16, device="cuda")
    idx = torch.from_numpy(np.ascontiguousarray(idx_flat, dtype=np.int32)).cuda() if len(idx_flat) else \
        torch.zeros(1, dtype=torch.int32, device="cuda")
    L.reuse_sparse_attn(p, q_blk, kc, vc, idx, out)
    torch.cuda.synchronize()
    return out.float().cpu().numpy()


def _oracle_refresh(batch, b):
    wl = batch.wl
    q, K, V = f64(batch.q_req(b)), f64(batch.k_logical(b)), f64(batch.v_logical(b))
    return O.attention_dense(q, K, V), O.raw_scores(q[wl.blk_start[b]:wl.blk_end[b]], K)


def _check_refresh(batch, out, scores, requests=None):
    wl = batch.wl
    sc = split_scores(scores, wl) if scores is not None else None
    for b in (range(wl.num_requests) if requests is None else requests):
        o_ref, raw_ref = _oracle_refresh(batch, b)
        c0, c1 = batch.cu_seqlens[b], batch.cu_seqlens[b + 1]
        assert_close(out[c0:c1], o_ref, f"{wl.name} refresh out req {b}")
        if sc is not None:
            # fp32 tensor-core accumulation vs fp64: |err| <= D * 2^-22 * sum|q k|
            q, K = f64(batch.q_req(b)), f64(batch.k_logical(b))
            qb = np.abs(q[wl.blk_start[b]:wl.blk_end[b]])
            bound = wl.head_dim * 2.0 ** -22 * np.stack(
                [(qb[:, h] @ np.abs(K[:, h // (wl.num_heads // wl.num_kv_heads)]).T).max(axis=0)
                 for h in range(wl.num_heads)]) + 1e-6
            err = np.abs(sc[b] - raw_ref)
            assert (err <= bound).all(), f"{wl.name} scores req {b}: max err {err.max():.3e}"


# ------------------------------------------------------------------ select (i)
SELECT_CASES = [("C0", None, None), ("C1", None, None), ("C2", None, None), ("C3", None, 24),
                ("C4", 0.05, 3), ("C4", 0.5, 3), ("C4", 1.0, 2)]


@pytest.mark.parametrize("mode", ["ties", "normal", "wide"])
@pytest.mark.parametrize("cfg,r,n", SELECT_CASES)
def test_select_bitexact_on_generated_scores(L, cfg, r, n, mode):
    wl = synth.config(cfg, keep_ratio=r, num_requests=n)
    batch_bt = torch.zeros((wl.num_requests, 1), dtype=torch.int32)
    p = L.Problem(wl.seq_len, wl.blk_start, wl.blk_end, num_heads=wl.num_heads, num_kv_heads=wl.num_kv_heads,
                  head_dim=wl.head_dim, keep_ratio=wl.keep_ratio, pool_window=wl.pool_window,
                  page_size=1024, block_table=batch_bt.cuda(), pages_per_req=8)
    sc = synth.scores(wl, mode=mode)
    k, got = _run_select(L, p, join_scores(sc))
    assert k == oracle_keep_counts(wl)
    ref = O.select_batch([s.astype(np.float64) for s in sc], wl.seq_len, wl.blk_start, wl.blk_end,
                         wl.keep_ratio, wl.pool_window)
    assert np.array_equal(got, join_idx(ref)), f"{cfg}/{mode}: selection differs"


@pytest.mark.parametrize("w", [1, 5, 7])
def test_select_windows(L, w):
    wl = synth.config("C1", num_requests=4)
    wl.pool_window = w
    p = L.Problem(wl.seq_len, wl.blk_start, wl.blk_end, num_heads=32, num_kv_heads=32, head_dim=128,
                  keep_ratio=0.25, pool_window=w, page_size=64,
                  block_table=torch.zeros((4, 16), dtype=torch.int32).cuda())
    sc = synth.scores(wl, mode="ties")
    k, got = _run_select(L, p, join_scores(sc))
    ref = O.select_batch([s.astype(np.float64) for s in sc], wl.seq_len, wl.blk_start, wl.blk_end, 0.25, w)
    assert np.array_equal(got, join_idx(ref))


# ------------------------------------------------------------------ refresh
@pytest.mark.parametrize("cfg,n", [("C0", None), ("C1", 2), ("C2", 2)])
def test_refresh_parity_configs(L, cfg, n):
    batch = synth.make_batch(synth.config(cfg, num_requests=n))
    p, out, scores = _run_refresh(L, batch)
    _check_refresh(batch, out, scores)


@pytest.mark.parametrize("name", sorted(EDGE))
def test_refresh_parity_edges(L, name):
    batch = synth.make_batch(EDGE[name])
    p, out, scores = _run_refresh(L, batch)
    _check_refresh(batch, out, scores)
    # without scores the outputs are identical
    p2, out2, _ = _run_refresh(L, batch, with_scores=False)
    assert np.array_equal(out, out2)


# ------------------------------------------------------------------ selection (ii): exact end to end
def _exact(wl):
    wl = synth.Workload(**{**wl.__dict__, "kind": "exact"})
    return wl


@pytest.mark.parametrize("cfg,n", [("C0", None), ("C1", 2), ("C2", 2), ("C3", 3)])
def test_selection_end_to_end_exact(L, cfg, n):
    batch = synth.make_batch(synth.config(cfg, num_requests=n, kind="exact"))
    p, out, scores = _run_refresh(L, batch)
    k, got = _run_select(L, p, scores)
    wl = batch.wl
    ref = [O.select_heads(f64(batch.q_req(b))[wl.blk_start[b]:wl.blk_end[b]], f64(batch.k_logical(b)),
                          wl.seq_len[b], wl.blk_start[b], wl.blk_end[b], wl.keep_ratio, wl.pool_window)
           for b in range(wl.num_requests)]
    assert np.array_equal(got, join_idx(ref))


@pytest.mark.parametrize("name", sorted(EDGE))
def test_selection_end_to_end_exact_edges(L, name):
    batch = synth.make_batch(_exact(EDGE[name]))
    p, out, scores = _run_refresh(L, batch)
    k, got = _run_select(L, p, scores)
    wl = batch.wl
    assert k == oracle_keep_counts(wl)
    ref = [O.select_heads(f64(batch.q_req(b))[wl.blk_start[b]:wl.blk_end[b]], f64(batch.k_logical(b)),
                          wl.seq_len[b], wl.blk_start[b], wl.blk_end[b], wl.keep_ratio, wl.pool_window)
           for b in range(wl.num_requests)]
    assert np.array_equal(got, join_idx(ref))


# ------------------------------------------------------------------ reuse
def _check_reuse(batch, got, idx_list, requests=None):
    wl = batch.wl
    for b in (range(wl.num_requests) if requests is None else requests):
        ref = O.attention_with_cache(f64(batch.q_blk_req(b)), f64(batch.k_logical(b)), f64(batch.v_logical(b)),
                                     wl.blk_start[b], wl.blk_end[b], idx_list[b])
        c0, c1 = batch.cu_blk[b], batch.cu_blk[b + 1]
        assert_close(got[c0:c1], ref, f"{wl.name} reuse req {b}")


# D = 16 / 32 / 64 run the tcgen05 kernels on their 64-dim layout (round 2): batches large
# enough for several rounds of the Reuse grid (512 units: 128 CTAs x 4, the balanced
# grid) and many Refresh units per CTA, every request checked against the oracle
@pytest.mark.parametrize("D,H,Hk", [(64, 32, 32), (32, 16, 4), (16, 8, 8)])
def test_narrow_head_dims_multiround(L, D, H, Hk):
    nreq = 512 // H
    Ls = [384 + 64 * (b % 5) for b in range(nreq)]
    bs = [Lb - 32 * (1 + b % 3) for b, Lb in enumerate(Ls)]
    wl = custom(f"e_d{D}_multi", Ls, bs, [x + 32 for x in bs], H=H, Hk=Hk, D=D, P=64)
    batch = synth.make_batch(wl)
    p, out, sc = _run_refresh(L, batch)
    _check_refresh(batch, out, sc, requests=range(0, nreq, 3))
    k = oracle_keep_counts(wl)
    idx = synth.indices(wl, k, mode="random")
    got = _run_reuse(L, batch, p, join_idx(idx))
    _check_reuse(batch, got, idx)


@pytest.mark.parametrize("mode", ["random", "shared"])
@pytest.mark.parametrize("cfg,n", [("C0", None), ("C1", 4), ("C2", 4), ("C3", 6)])
def test_reuse_parity_generated_indices(L, cfg, n, mode):
    batch = synth.make_batch(synth.config(cfg, num_requests=n))
    p = problem_of(batch)
    k = oracle_keep_counts(batch.wl)
    assert k == p.layout()[0]
    idx = synth.indices(batch.wl, k, mode=mode)
    got = _run_reuse(L, batch, p, join_idx(idx))
    _check_reuse(batch, got, idx)


@pytest.mark.parametrize("name", sorted(EDGE))
def test_reuse_parity_edges(L, name):
    batch = synth.make_batch(EDGE[name])
    p = problem_of(batch)
    k = oracle_keep_counts(batch.wl)
    idx = synth.indices(batch.wl, k)
    got = _run_reuse(L, batch, p, join_idx(idx))
    _check_reuse(batch, got, idx)


def test_reuse_r1_equals_refresh_rows(L):
    """keep ratio 1 + Q_blk = Q[bs:be]: Reuse rows == Refresh rows."""
    wl = custom("e_r1eq", [320, 200], [128, 40], [160, 72], H=4, Hk=2, D=128, r=1.0)
    batch = synth.make_batch(wl)
    batch.q_blk = torch.cat([batch.q_req(b)[wl.blk_start[b]:wl.blk_end[b]] for b in range(2)])
    p, out, scores = _run_refresh(L, batch)
    k, idx = _run_select(L, p, scores)
    got = _run_reuse(L, batch, p, idx)
    for b in range(2):
        ref = out[batch.cu_seqlens[b] + wl.blk_start[b]: batch.cu_seqlens[b] + wl.blk_end[b]]
        d = np.abs(got[batch.cu_blk[b]:batch.cu_blk[b + 1]] - ref)
        assert d.max() <= 1.6e-2 and d.mean() <= 1e-3


# ------------------------------------------------------------------ end to end (iii), determinism
def _selection_flips(batch, got_l, requests):
    """Tier (iii): on realistic inputs the GPU's selection must be a
    valid top-k of the oracle's fp64 pooled scores up to fp32 rounding.  With S the
    fp64 pooled scores, O the oracle's set, G the GPU's and s_k = min over O of S
    (the k-th largest), every GPU-only pick g must satisfy S[g] >= s_k - (eps_g +
    eps_k), and every oracle-only pick o (dropped by the GPU) S[o] <= s_k + eps_o +
    max(eps): nothing the GPU dropped beats what it kept beyond the rounding bound.
    eps_c = D 2^-22 max_{q in blk, m in win(c)} sum_d |Q[q,h,d] K[m,kv,d]| bounds the
    fp32 error of pooled score c (tensor-core accumulation; 2^-22 keeps a factor 2
    over the 2^-23 unit roundoff).  Returns (flips, picks checked)."""
    wl = batch.wl
    g = wl.num_heads // wl.num_kv_heads
    flips = picks = 0
    for b in requests:
        q, K = f64(batch.q_req(b)), f64(batch.k_logical(b))
        bs, be, Lb = wl.blk_start[b], wl.blk_end[b], wl.seq_len[b]
        C = O.candidates(Lb, bs, be)
        S = O.pool_scores(O.raw_scores(q[bs:be], K[C]), wl.pool_window)
        ref = O.select_heads(q[bs:be], K, Lb, bs, be, wl.keep_ratio, wl.pool_window)
        pos2c = np.full(Lb, -1)
        pos2c[C] = np.arange(len(C))
        for h in range(wl.num_heads):
            absdot = (np.abs(q[bs:be, h]) @ np.abs(K[C, h // g]).T).max(axis=0)
            eps = wl.head_dim * 2.0 ** -22 * O.pool_scores(absdot, wl.pool_window) + 1e-6
            gs, rs = set(got_l[b][h].tolist()), set(ref[h].tolist())
            assert len(gs) == len(rs) == len(got_l[b][h]), f"req {b} head {h}: duplicates / wrong k"
            oc = pos2c[ref[h]]
            kth = oc[np.argmin(S[h, oc])]
            for p in gs - rs:
                c = pos2c[p]
                assert c >= 0, f"req {b} head {h}: position {p} is not a candidate"
                assert S[h, c] >= S[h, kth] - (eps[c] + eps[kth]), \
                    f"req {b} head {h}: GPU kept {p} (S={S[h, c]:.6g}) below the k-th score {S[h, kth]:.6g}"
                flips += 1
            for p in rs - gs:
                c = pos2c[p]
                assert S[h, c] <= S[h, kth] + eps[c] + eps.max(), \
                    f"req {b} head {h}: GPU dropped {p} (S={S[h, c]:.6g}) above its kept scores"
            picks += len(gs)
    return flips, picks


@pytest.mark.parametrize("cfg,r,n,sample", [("C1", None, 2, [0, 1]), ("C2", None, 4, [0, 3]),
                                            ("C4", 0.05, 4, [0, 3]), ("C4", 0.25, 4, [1, 2])])
def test_end_to_end_realistic_selection_valid(L, cfg, r, n, sample):
    batch = synth.make_batch(synth.config(cfg, keep_ratio=r, num_requests=n))
    wl = batch.wl
    p, out, scores = _run_refresh(L, batch)
    k, got = _run_select(L, p, scores)
    got_l = split_idx(got, wl, k)
    flips, picks = _selection_flips(batch, got_l, sample)
    assert flips <= max(4, picks // 2000), f"{flips} rounding-level selection flips of {picks} picks"
    # Reuse with the selected lists (compared against the oracle on the GPU's own lists)
    gotr = _run_reuse(L, batch, p, got)
    _check_reuse(batch, gotr, got_l, requests=sample)


def test_realistic_full_c1_batch_every_row(L):
    """The whole C1 batch (16 requests, the bench's launch) on realistic inputs:
    every Refresh row and every Reuse row of every request against the oracle."""
    batch = synth.make_batch(synth.config("C1"))
    wl = batch.wl
    p = problem_of(batch)
    q, q_blk, kc, vc = to_dev(batch)
    buf = L.alloc_buffers(p)
    L.hot_path(p, q, q_blk, kc, vc, buf)
    torch.cuda.synchronize()
    k, total_idx, rows, blk_rows = p.layout()
    _check_refresh(batch, buf.out.float().cpu().numpy(), None)
    got_l = split_idx(buf.idx.cpu().numpy()[:total_idx], wl, k)
    _check_reuse(batch, buf.out_blk.float().cpu().numpy(), got_l)


def test_realistic_c3_subset_mixed_launch(L):
    """32 requests of the burst mix (C3 lengths 512..4096) in ONE mixed launch on
    realistic inputs: every Refresh row of the Refresh requests and every Reuse row
    of the others against the oracle."""
    from tests.test_gpu_mixed import _outputs, _split
    wl = synth.config("C3", num_requests=32)
    batch = synth.make_batch(wl)
    kc, vc = batch.k_cache.cuda(), batch.v_cache.cuda()
    ri = [i for i in range(32) if i % 8 == 0]
    ui = [i for i in range(32) if i % 8 != 0]
    sr, pr, su, pu, q, qb, idx, idx_list = _split(L, wl, batch, ri, ui)
    out, sc, ob = _outputs(wl, pr, pu, q)
    L.mixed_attn(pr, q, out, sc, pu, qb, idx, ob, kc, vc)
    torch.cuda.synchronize()
    out, ob = out.float().cpu().numpy(), ob.float().cpu().numpy()
    o = 0
    for b in ri:
        qq, K, V = f64(batch.q_req(b)), f64(batch.k_logical(b)), f64(batch.v_logical(b))
        assert_close(out[o:o + wl.seq_len[b]], O.attention_dense(qq, K, V), f"C3 refresh req {b}")
        o += wl.seq_len[b]
    o = 0
    for j, b in enumerate(ui):
        ref = O.attention_with_cache(f64(batch.q_blk_req(b)), f64(batch.k_logical(b)), f64(batch.v_logical(b)),
                                     wl.blk_start[b], wl.blk_end[b], idx_list[j])
        assert_close(ob[o:o + wl.blk[b]], ref, f"C3 reuse req {b}")
        o += wl.blk[b]


def test_determinism_and_page_permutation_invariance(L):
    wl = synth.config("C2", num_requests=2)
    b1 = synth.make_batch(wl)
    b2 = synth.make_batch(wl, page_seed=12345)
    assert not torch.equal(b1.block_table, b2.block_table)
    res = []
    for bb in (b1, b1, b2):
        p, out, scores = _run_refresh(L, bb)
        k, idx = _run_select(L, p, scores)
        ob = _run_reuse(L, bb, p, idx)
        res.append((out, scores, idx, ob))
    for other in res[1:]:
        for a, b in zip(res[0], other):
            assert np.array_equal(a.view(np.uint8), b.view(np.uint8))


def test_check_indices(L):
    batch = synth.make_batch(synth.config("C1", num_requests=3))
    p = problem_of(batch)
    k = p.layout()[0]
    idx = join_idx(synth.indices(batch.wl, k))
    viol = torch.zeros(1, dtype=torch.int32, device="cuda")
    L.check_indices(p, torch.from_numpy(idx).cuda(), viol)
    torch.cuda.synchronize()
    assert int(viol.item()) == 0
    bad = idx.copy()
    bad[5] = batch.wl.blk_start[0]          # inside the block
    bad[k[0] * 3 + 7] = 10 ** 6             # out of range (and breaks ascending order)
    L.check_indices(p, torch.from_numpy(bad).cuda(), viol)
    torch.cuda.synchronize()
    assert int(viol.item()) >= 2


# ------------------------------------------------------------------ full-size configs, sampled outputs
@pytest.mark.parametrize("cfg,sample,r,n", [("C1", [0, 9, 15], None, None), ("C2", [0, 31], None, None),
                                           ("C3", [0, 77, 255], None, None), ("C4", [0, 7], 0.05, 8),
                                           ("C4", [3], 1.0, 4)])
def test_full_config_hot_path_sampled(L, cfg, sample, r, n):
    """BASELINE sizes, the launch configuration bench.py times: whole batch on the
    GPU, oracle on sampled requests (exact-integer Q/K so the selection is bit-exact)."""
    wl = synth.config(cfg, kind="exact", keep_ratio=r, num_requests=n)
    batch = synth.make_batch(wl)
    p = problem_of(batch)
    q, q_blk, kc, vc = to_dev(batch)
    buf = L.alloc_buffers(p)
    L.hot_path(p, q, q_blk, kc, vc, buf)
    torch.cuda.synchronize()
    out = buf.out.float().cpu().numpy()
    k, total_idx, rows, blk_rows = p.layout()
    idx = split_idx(buf.idx.cpu().numpy()[:total_idx], wl, k)
    ob = buf.out_blk.float().cpu().numpy()
    for b in sample:
        qb, K, V = f64(batch.q_req(b)), f64(batch.k_logical(b)), f64(batch.v_logical(b))
        bs, be = wl.blk_start[b], wl.blk_end[b]
        c0, c1 = batch.cu_seqlens[b], batch.cu_seqlens[b + 1]
        # exact-integer logits are large; compare Refresh on a row sample with the stated tolerance
        rows_s = np.r_[0:4, bs:be, wl.seq_len[b] - 4:wl.seq_len[b]]
        ref = O.attention_dense(qb[rows_s], K, V)
        assert_close(out[c0:c1][rows_s], ref, f"{cfg} refresh req {b}")
        sel = O.select_heads(qb[bs:be], K, wl.seq_len[b], bs, be, wl.keep_ratio, wl.pool_window)
        assert np.array_equal(idx[b], sel), f"{cfg} selection req {b}"
        ref_u = O.attention_with_cache(f64(batch.q_blk_req(b)), K, V, bs, be, sel)
        assert_close(ob[batch.cu_blk[b]:batch.cu_blk[b + 1]], ref_u, f"{cfg} reuse req {b}")


# ------------------------------------------------------------------ N2: uniform (global) selection
@pytest.mark.parametrize("cfg,n", [("C0", None), ("C1", 4), ("C2", 4), ("C3", 8)])
def test_select_global_bitexact_integer_scores(L, cfg, n):
    """dllm_select_global vs the oracle's Eq. 5 selection on integer scores (head sums exact in fp32)."""
    wl = synth.config(cfg, num_requests=n)
    p = L.Problem(wl.seq_len, wl.blk_start, wl.blk_end, num_heads=wl.num_heads, num_kv_heads=wl.num_kv_heads,
                  head_dim=wl.head_dim, keep_ratio=wl.keep_ratio, pool_window=wl.pool_window, page_size=1024,
                  block_table=torch.zeros((wl.num_requests, 8), dtype=torch.int32).cuda())
    sc = synth.scores(wl, mode="ties")
    k, total_idx, _, _ = p.layout()
    idx = torch.full((max(total_idx, 1),), -7, dtype=torch.int32, device="cuda")
    L.select_global(p, torch.from_numpy(join_scores(sc)).cuda(), idx)
    torch.cuda.synchronize()
    got = split_idx(idx.cpu().numpy()[:total_idx], wl, k)
    ref = O.select_global_batch([s.astype(np.float64) for s in sc], wl.seq_len, wl.blk_start, wl.blk_end,
                                wl.keep_ratio, wl.pool_window)
    for b in range(wl.num_requests):
        assert all(np.array_equal(got[b][h], ref[b]) for h in range(wl.num_heads)), f"{cfg} req {b}"


def test_uniformity_trap_witness_on_gpu(L):
    """PAPER.md:143-145 / SPEC.md:270: per-head selection keeps every head's top key,
    the uniform set drops head 1's."""
    wl = custom("e_trap", [3], [2], [3], H=2, Hk=2, D=16, r=0.5, w=1, P=16)
    p = L.Problem(wl.seq_len, wl.blk_start, wl.blk_end, num_heads=2, num_kv_heads=2, head_dim=16, keep_ratio=0.5,
                  pool_window=1, page_size=16, block_table=torch.zeros((1, 1), dtype=torch.int32).cuda())
    raw = torch.tensor([9.0, 0.0, 5.0, 0.0, 9.0, 5.0], device="cuda")
    ph = torch.full((2,), -1, dtype=torch.int32, device="cuda")
    gl = torch.full((2,), -1, dtype=torch.int32, device="cuda")
    L.select_heads(p, raw, ph)
    L.select_global(p, raw, gl)
    torch.cuda.synchronize()
    assert ph.cpu().tolist() == [0, 1] and gl.cpu().tolist() == [0, 0]


def test_uniform_baseline_end_to_end(L):
    """select_global -> reuse equals the oracle's attention over the shared set (Eq. 4 with one I for all heads)."""
    batch = synth.make_batch(synth.config("C1", num_requests=2, kind="exact"))
    wl = batch.wl
    p, out, scores = _run_refresh(L, batch)
    k, total_idx, _, _ = p.layout()
    idx = torch.full((max(total_idx, 1),), -7, dtype=torch.int32, device="cuda")
    L.select_global(p, torch.from_numpy(np.ascontiguousarray(scores)).cuda(), idx)
    torch.cuda.synchronize()
    flat = idx.cpu().numpy()[:total_idx]
    got_sets = split_idx(flat, wl, k)
    for b in range(wl.num_requests):
        qb, K = f64(batch.q_req(b)), f64(batch.k_logical(b))
        ref = O.select_global(qb[wl.blk_start[b]:wl.blk_end[b]], K, wl.seq_len[b], wl.blk_start[b], wl.blk_end[b],
                              wl.keep_ratio, wl.pool_window)
        assert all(np.array_equal(got_sets[b][h], ref) for h in range(wl.num_heads))
    gotr = _run_reuse(L, batch, p, flat)
    _check_reuse(batch, gotr, got_sets)


# ------------------------------------------------------------------ N1: pack-at-Refresh layout
@pytest.mark.parametrize("cfg,n", [("C0", None), ("C1", 3), ("C2", 3)])
def test_pack_and_reuse_packed(L, cfg, n):
    """dllm_pack_kv copies exactly the selected rows (bit-identical gathering) and
    dllm_reuse_packed equals the gather-in-place Reuse bit for bit (same keys, same order)."""
    batch = synth.make_batch(synth.config(cfg, num_requests=n))
    wl = batch.wl
    p = problem_of(batch)
    k = oracle_keep_counts(wl)
    idx_list = synth.indices(wl, k)
    flat = join_idx(idx_list)
    q, q_blk, kc, vc = to_dev(batch)
    _, total_idx, _, blk_rows = p.layout()
    idx = torch.from_numpy(flat).cuda()
    kp = torch.full((total_idx, wl.head_dim), float("nan"), dtype=torch.bfloat16, device="cuda")
    vp = torch.full_like(kp, float("nan"))
    L.pack_kv(p, kc, vc, idx, kp, vp)
    out_p = torch.full((blk_rows, wl.num_heads, wl.head_dim), float("nan"), dtype=torch.bfloat16, device="cuda")
    L.reuse_packed(p, q_blk, kc, vc, kp, vp, out_p)
    torch.cuda.synchronize()
    kp_h, vp_h = kp.cpu(), vp.cpu()
    off = 0
    g = wl.num_heads // wl.num_kv_heads
    for b in range(wl.num_requests):
        Kl, Vl = batch.k_logical(b), batch.v_logical(b)
        for h in range(wl.num_heads):
            rows = torch.from_numpy(idx_list[b][h].astype(np.int64))
            assert torch.equal(kp_h[off:off + k[b]].view(torch.int16), Kl[rows, h // g].view(torch.int16))
            assert torch.equal(vp_h[off:off + k[b]].view(torch.int16), Vl[rows, h // g].view(torch.int16))
            off += k[b]
    # the packed path shares the persistent mma.sync kernel's arithmetic: bit-identical to
    # gathering in place with that kernel (the tcgen05 default rounds P.V differently)
    os.environ["DLLM_REUSE_IMPL"] = "ws"
    try:
        out_g = _run_reuse(L, batch, p, flat)
    finally:
        del os.environ["DLLM_REUSE_IMPL"]
    assert np.array_equal(out_p.float().cpu().numpy().view(np.uint32), out_g.view(np.uint32))
    _check_reuse(batch, out_p.float().cpu().numpy(), idx_list)


# ------------------------------------------------------------------ N2: per-KV-group selection (GQA)
@pytest.mark.parametrize("cfg,n", [("C1", 3), ("C2", 4), ("C3", 8)])
def test_select_groups_bitexact_integer_scores(L, cfg, n):
    """dllm_select_groups vs the oracle's per-KV-group selection on integer scores
    (group sums exact in fp32); with H_kv = H (C1, C3) it equals dllm_select_heads."""
    wl = synth.config(cfg, num_requests=n)
    p = L.Problem(wl.seq_len, wl.blk_start, wl.blk_end, num_heads=wl.num_heads, num_kv_heads=wl.num_kv_heads,
                  head_dim=wl.head_dim, keep_ratio=wl.keep_ratio, pool_window=wl.pool_window, page_size=1024,
                  block_table=torch.zeros((wl.num_requests, 8), dtype=torch.int32).cuda())
    sc = synth.scores(wl, mode="ties")
    k, total_idx, _, _ = p.layout()
    idx = torch.full((max(total_idx, 1),), -7, dtype=torch.int32, device="cuda")
    L.select_groups(p, torch.from_numpy(join_scores(sc)).cuda(), idx)
    torch.cuda.synchronize()
    got = split_idx(idx.cpu().numpy()[:total_idx], wl, k)
    ref = O.select_groups_batch([s.astype(np.float64) for s in sc], wl.seq_len, wl.blk_start, wl.blk_end,
                                wl.keep_ratio, wl.pool_window, wl.num_kv_heads)
    g = wl.num_heads // wl.num_kv_heads
    for b in range(wl.num_requests):
        assert all(np.array_equal(got[b][h], ref[b][h // g]) for h in range(wl.num_heads)), f"{cfg} req {b}"
    if wl.num_kv_heads == wl.num_heads:
        k2, per_head = _run_select(L, p, join_scores(sc))
        assert np.array_equal(per_head, idx.cpu().numpy()[:total_idx])


def test_select_groups_end_to_end_exact_gqa(L):
    """Refresh -> per-group select -> Reuse on the Dream GQA shape (exact-integer Q/K):
    the group sets equal the oracle's, every head of a group reads them, and the
    Reuse rows match the oracle's attention over the shared sets."""
    batch = synth.make_batch(synth.config("C2", num_requests=2, kind="exact"))
    wl = batch.wl
    p, out, scores = _run_refresh(L, batch)
    k, total_idx, _, _ = p.layout()
    idx = torch.full((max(total_idx, 1),), -7, dtype=torch.int32, device="cuda")
    L.select_groups(p, torch.from_numpy(np.ascontiguousarray(scores)).cuda(), idx)
    torch.cuda.synchronize()
    flat = idx.cpu().numpy()[:total_idx]
    got = split_idx(flat, wl, k)
    g = wl.num_heads // wl.num_kv_heads
    for b in range(wl.num_requests):
        qb, K = f64(batch.q_req(b)), f64(batch.k_logical(b))
        ref = O.select_groups(qb[wl.blk_start[b]:wl.blk_end[b]], K, wl.seq_len[b], wl.blk_start[b], wl.blk_end[b],
                              wl.keep_ratio, wl.pool_window, wl.num_kv_heads)
        assert all(np.array_equal(got[b][h], ref[h // g]) for h in range(wl.num_heads)), f"req {b}"
    gotr = _run_reuse(L, batch, p, flat)
    _check_reuse(batch, gotr, got)
