"""GPU parity of dllm_reuse_group_sets (next row N2, GQA; R21): Eq. 4
 over one key set per KV group, every head of the group
attending to the group's positions, vs the fp64 oracle's attention_with_cache on
the same sets.  The group kernel stacks up to 4 heads of a group in one work
unit: the cases cover full and partial sub-groups (G = 7 -> 4 + 3, G = 5 -> 4 + 1,
G = 8 -> 4 + 4, G = 2, 3), several 32-row groups, ragged tails, block tables
larger than the kernel's shared-memory cache, and the fallbacks (H = H_kv, D != 128)."""
import numpy as np
import pytest
import torch

import oracle as O
from paper_2512_17077_b200 import synth
from tests._util import assert_close, f64, join_idx, oracle_keep_counts, problem_of, to_dev

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def L():
    assert torch.cuda.is_available(), "GPU tests need a B200"
    from paper_2512_17077_b200 import lib
    return lib


def custom(name, L_, bs, be, H, Hk, D=128, r=0.25, P=64):
    return synth.Workload(name, H, Hk, D, list(L_), list(bs), list(be), r, 3, P, "realistic")


CASES = {
    "C2": synth.config("C2", num_requests=3),
    "C0": synth.config("C0"),
    "g5_ragged": custom("g_g5", [300, 1025, 77], [250, 993, 40], [282, 1025, 72], H=10, Hk=2),
    "g8_blk128": custom("g_g8", [700], [500], [628], H=8, Hk=1),
    "g3_mixed": custom("g_g3", [640, 129, 1025, 64], [608, 0, 993, 32], [640, 32, 1025, 64], H=6, Hk=2),
    "g2_p16": custom("g_g2", [300, 77], [250, 40], [282, 72], H=4, Hk=2, P=16),
    "g7_long_bt": custom("g_long", [40000], [39000], [39032], H=7, Hk=1, r=0.02, P=64),   # 625 pages > 512 cached
    "g4_blk1_r1": custom("g_r1", [200, 97], [100, 96], [101, 97], H=4, Hk=1, r=1.0),
    "mha_fallback": custom("g_mha", [300], [200], [232], H=4, Hk=4),
    "d64_fallback": custom("g_d64", [300], [200], [232], H=4, Hk=1, D=64),
}


def _run(L, batch, fn, idx_list):
    p = problem_of(batch)
    q, q_blk, kc, vc = to_dev(batch)
    _, _, _, blk_rows = p.layout()
    wl = batch.wl
    out = torch.full((blk_rows, wl.num_heads, wl.head_dim), float("nan"), dtype=torch.bfloat16, device="cuda")
    flat = join_idx(idx_list)
    idx = torch.from_numpy(flat).cuda() if flat.size else torch.zeros(1, dtype=torch.int32, device="cuda")
    fn(p, q_blk, kc, vc, idx, out)
    torch.cuda.synchronize()
    return out.float().cpu().numpy()


@pytest.mark.parametrize("name", sorted(CASES))
def test_reuse_group_sets_parity(L, name):
    batch = synth.make_batch(CASES[name])
    wl = batch.wl
    k = oracle_keep_counts(wl)
    idx = synth.indices(wl, k, mode="shared")   # one set per KV group, in every head's slot
    got = _run(L, batch, L.reuse_group_sets, idx)
    for b in range(wl.num_requests):
        ref = O.attention_with_cache(f64(batch.q_blk_req(b)), f64(batch.k_logical(b)), f64(batch.v_logical(b)),
                                     wl.blk_start[b], wl.blk_end[b], idx[b])
        c0, c1 = batch.cu_blk[b], batch.cu_blk[b + 1]
        assert_close(got[c0:c1], ref, f"{name} group reuse req {b}")


def test_reuse_group_sets_matches_per_head_kernel(L, monkeypatch):
    """Same sets through both Reuse kernels: equal within the fp32 rounding of two
    accumulation orders (both are checked against the oracle above)."""
    batch = synth.make_batch(synth.config("C2", num_requests=4))
    k = oracle_keep_counts(batch.wl)
    idx = synth.indices(batch.wl, k, mode="shared")
    a = _run(L, batch, L.reuse_group_sets, idx)
    monkeypatch.setenv("DLLM_REUSE_IMPL", "tc")
    b = _run(L, batch, L.reuse_sparse_attn, idx)
    assert np.isfinite(a).all()
    d = np.abs(a - b)
    assert d.max() <= 8e-3 and d.mean() <= 2e-4, (d.max(), d.mean())


def test_reuse_group_sets_after_select_groups(L):
    """Refresh -> dllm_select_groups -> dllm_reuse_group_sets on exact-integer Q/K
    at the Dream shape: the selected sets equal the oracle's per-group sets and the
    rows match the oracle's attention over them."""
    batch = synth.make_batch(synth.config("C2", num_requests=2, kind="exact"))
    wl = batch.wl
    p = problem_of(batch)
    q, q_blk, kc, vc = to_dev(batch)
    k, total_idx, rows, blk_rows = p.layout()
    out = torch.empty((rows, wl.num_heads, wl.head_dim), dtype=torch.bfloat16, device="cuda")
    sc = torch.empty((wl.num_heads * rows,), dtype=torch.float32, device="cuda")
    L.refresh_attn(p, q, kc, vc, out, sc)
    idx = torch.full((max(total_idx, 1),), -7, dtype=torch.int32, device="cuda")
    L.select_groups(p, sc, idx)
    ob = torch.full((blk_rows, wl.num_heads, wl.head_dim), float("nan"), dtype=torch.bfloat16, device="cuda")
    L.reuse_group_sets(p, q_blk, kc, vc, idx, ob)
    torch.cuda.synchronize()
    flat = idx.cpu().numpy()[:total_idx]
    got = ob.float().cpu().numpy()
    g = wl.num_heads // wl.num_kv_heads
    off = 0
    for b in range(wl.num_requests):
        sets = flat[off:off + wl.num_heads * k[b]].reshape(wl.num_heads, k[b])
        off += wl.num_heads * k[b]
        qb, K = f64(batch.q_req(b)), f64(batch.k_logical(b))
        ref_sets = O.select_groups(qb[wl.blk_start[b]:wl.blk_end[b]], K, wl.seq_len[b], wl.blk_start[b],
                                   wl.blk_end[b], wl.keep_ratio, wl.pool_window, wl.num_kv_heads)
        assert all(np.array_equal(sets[h], ref_sets[h // g]) for h in range(wl.num_heads)), f"req {b}"
        ref = O.attention_with_cache(f64(batch.q_blk_req(b)), K, f64(batch.v_logical(b)), wl.blk_start[b],
                                     wl.blk_end[b], sets)
        c0, c1 = batch.cu_blk[b], batch.cu_blk[b + 1]
        assert_close(got[c0:c1], ref, f"select_groups -> reuse_group_sets req {b}")


def test_reuse_group_sets_full_c2_sampled(L):
    """The full C2 batch (32 requests, the bench's launch): sampled requests vs the oracle."""
    batch = synth.make_batch(synth.config("C2"))
    wl = batch.wl
    k = oracle_keep_counts(wl)
    idx = synth.indices(wl, k, mode="shared")
    got = _run(L, batch, L.reuse_group_sets, idx)
    assert np.isfinite(got).all()
    for b in (0, 13, wl.num_requests - 1):
        ref = O.attention_with_cache(f64(batch.q_blk_req(b)), f64(batch.k_logical(b)), f64(batch.v_logical(b)),
                                     wl.blk_start[b], wl.blk_end[b], idx[b])
        c0, c1 = batch.cu_blk[b], batch.cu_blk[b + 1]
        assert_close(got[c0:c1], ref, f"C2 full group reuse req {b}")


def test_reuse_group_sets_empty_batch(L):
    p = L.Problem([], [], [], num_heads=28, num_kv_heads=4, head_dim=128, keep_ratio=0.2, pool_window=3,
                  page_size=64, block_table=torch.zeros((0, 1), dtype=torch.int32, device="cuda"))
    e = torch.empty(0, dtype=torch.bfloat16, device="cuda")
    L.reuse_group_sets(p, e, e, e, torch.zeros(1, dtype=torch.int32, device="cuda"), e)
    torch.cuda.synchronize()


# ------------------------------------------------------------------ union mode (per-head sets, GQA)
# DLLM_REUSE_IMPL=union: dllm_reuse_sparse_attn runs GQA batches (G >= 2, D = 128,
# L <= 8192) on the same kernel over the UNION of the sub-group's per-head sets,
# each head masked to its own keys; longer sequences fall back to the per-head kernel.
UNION_CASES = {
    "C2": synth.config("C2", num_requests=3),
    "g5_ragged": CASES["g5_ragged"],
    "g8_blk128": CASES["g8_blk128"],
    "g3_mixed": CASES["g3_mixed"],
    "g2_p16": CASES["g2_p16"],
    "g4_blk1_r1": CASES["g4_blk1_r1"],
    "g7_sparse": custom("u_sparse", [3000, 517], [2900, 480], [2932, 512], H=7, Hk=1, r=0.01),
    "g4_k0": custom("u_k0", [32, 64], [0, 0], [32, 64], H=4, Hk=1),   # no context keys at all
    "g7_long": custom("u_long", [8192, 300], [8100, 100], [8132, 132], H=7, Hk=1, r=0.05),
    "g7_over_union_len": custom("u_over", [9000], [8900], [8932], H=7, Hk=1, r=0.05),   # per-head fallback
}


@pytest.mark.parametrize("name", sorted(UNION_CASES))
@pytest.mark.parametrize("mode", ["random", "shared"])
def test_reuse_union_parity(L, name, mode, monkeypatch):
    monkeypatch.setenv("DLLM_REUSE_IMPL", "union")
    batch = synth.make_batch(UNION_CASES[name])
    wl = batch.wl
    k = oracle_keep_counts(wl)
    idx = synth.indices(wl, k, mode=mode)
    got = _run(L, batch, L.reuse_sparse_attn, idx)
    for b in range(wl.num_requests):
        ref = O.attention_with_cache(f64(batch.q_blk_req(b)), f64(batch.k_logical(b)), f64(batch.v_logical(b)),
                                     wl.blk_start[b], wl.blk_end[b], idx[b])
        c0, c1 = batch.cu_blk[b], batch.cu_blk[b + 1]
        assert_close(got[c0:c1], ref, f"{name}/{mode} union reuse req {b}")


def test_reuse_union_matches_per_head_kernel(L, monkeypatch):
    batch = synth.make_batch(synth.config("C2", num_requests=4))
    k = oracle_keep_counts(batch.wl)
    idx = synth.indices(batch.wl, k)
    monkeypatch.setenv("DLLM_REUSE_IMPL", "union")
    a = _run(L, batch, L.reuse_sparse_attn, idx)
    monkeypatch.setenv("DLLM_REUSE_IMPL", "tc")
    b = _run(L, batch, L.reuse_sparse_attn, idx)
    d = np.abs(a - b)
    assert np.isfinite(a).all() and d.max() <= 8e-3 and d.mean() <= 2e-4, (d.max(), d.mean())


def test_reuse_union_full_c2_sampled(L, monkeypatch):
    """The full C2 batch with per-head sets through the union kernel."""
    monkeypatch.setenv("DLLM_REUSE_IMPL", "union")
    batch = synth.make_batch(synth.config("C2"))
    wl = batch.wl
    k = oracle_keep_counts(wl)
    idx = synth.indices(wl, k)
    got = _run(L, batch, L.reuse_sparse_attn, idx)
    assert np.isfinite(got).all()
    for b in (0, 17, wl.num_requests - 1):
        ref = O.attention_with_cache(f64(batch.q_blk_req(b)), f64(batch.k_logical(b)), f64(batch.v_logical(b)),
                                     wl.blk_start[b], wl.blk_end[b], idx[b])
        c0, c1 = batch.cu_blk[b], batch.cu_blk[b + 1]
        assert_close(got[c0:c1], ref, f"C2 full union reuse req {b}")
