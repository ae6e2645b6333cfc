"""Pins for the fp64 oracle (``-m "not gpu"``).

Every oracle function is checked against something other than itself: the
SPEC/paper worked examples (tests/golden/spec_examples.json, each entry
citing its line), closed forms, library routines (torch SDPA / max_pool1d in
float64), invariants of the mathematics, and brute force on tiny inputs.
The checks are chosen so that a dropped term, a wrong sign or index, or a
transposed operand in the oracle fails at least one of them.
"""
import itertools
import json
import math
import os

import numpy as np
import pytest
import torch

import oracle as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def rnd(shape, seed):
    return np.random.default_rng(seed).standard_normal(shape)


# ---------------------------------------------------------------- keep_count
def test_keep_count_golden():
    for r, n, k in GOLD["keep_count"]["cases"]:
        assert O.keep_count(r, n) == k, (r, n)


def test_keep_count_bounds_and_errors():
    for n in range(0, 50):
        for r in (1e-9, 0.1, 0.33, 0.5, 0.999, 1.0):
            k = O.keep_count(r, n)
            assert (k == 0) if n == 0 else (1 <= k <= n)
            if n:
                assert k >= r * n - 1e-9 and k - 1 < r * n  # ceil
    for bad in (0.0, -0.1, 1.0001):
        with pytest.raises(ValueError):
            O.keep_count(bad, 10)


def test_candidates():
    assert O.candidates(8, 2, 5).tolist() == [0, 1, 5, 6, 7]
    assert O.candidates(4, 0, 4).tolist() == []
    assert O.candidates(4, 3, 4).tolist() == [0, 1, 2]
    with pytest.raises(ValueError):
        O.candidates(4, 2, 2)


# ---------------------------------------------------------------- Eq. 3
def test_attention_dense_golden_and_closed_forms():
    g = GOLD["attention_dense"]
    assert np.allclose(O.attention_dense(g["q"], g["k"], g["v"], 1.0), g["expect"])
    # closed form: two keys with logits 0 and ln 3 -> p = [1/4, 3/4]
    q = np.array([[[math.log(3.0)]]])
    k = np.array([[[0.0]], [[1.0]]])
    v = np.array([[[0.0]], [[4.0]]])
    assert abs(O.attention_dense(q, k, v, 1.0)[0, 0, 0] - 3.0) < 1e-14
    # default scale is 1/sqrt(D): D=4, q.k = 2*ln(3) -> logit ln 3
    q = np.array([[[math.log(3.0), math.log(3.0), 0, 0]]])
    k = np.array([[[0, 0, 0, 0.0]], [[1.0, 1.0, 0, 0]]])
    v = np.zeros((2, 1, 4)); v[1, 0, 2] = 4.0
    assert abs(O.attention_dense(q, k, v)[0, 0, 2] - 3.0) < 1e-14
    # n = 1 -> O = V
    V = rnd((1, 3, 5), 1)
    assert np.allclose(O.attention_dense(rnd((1, 3, 5), 2), rnd((1, 3, 5), 3), V), V, atol=0, rtol=0)
    # identical K rows -> uniform softmax -> O = column mean of V
    K = np.repeat(rnd((1, 2, 6), 4), 7, axis=0)
    V = rnd((7, 2, 6), 5)
    assert np.allclose(O.attention_dense(rnd((3, 2, 6), 6), K, V), V.mean(axis=0)[None], atol=1e-14)


def test_attention_dense_rows_sum_to_one_and_convexity():
    Q, K = rnd((9, 4, 8), 7) * 3, rnd((13, 2, 8), 8) * 3
    ones = np.ones((13, 2, 8))
    assert np.abs(O.attention_dense(Q, K, ones) - 1).max() < 1e-12
    V = rnd((13, 2, 8), 9)
    out = O.attention_dense(Q, K, V)
    for h in range(4):
        kh = h // 2
        assert (out[:, h] <= V[:, kh].max(axis=0) + 1e-12).all()
        assert (out[:, h] >= V[:, kh].min(axis=0) - 1e-12).all()


def test_attention_dense_vs_torch_sdpa_f64():
    Q, K, V = rnd((11, 6, 16), 10), rnd((17, 3, 16), 11), rnd((17, 3, 16), 12)
    ours = O.attention_dense(Q, K, V)
    tq = torch.from_numpy(Q).permute(1, 0, 2)
    tk = torch.from_numpy(np.repeat(K, 2, axis=1)).permute(1, 0, 2)
    tv = torch.from_numpy(np.repeat(V, 2, axis=1)).permute(1, 0, 2)
    ref = torch.nn.functional.scaled_dot_product_attention(tq, tk, tv).permute(1, 0, 2).numpy()
    assert np.abs(ours - ref).max() < 1e-12


def test_attention_dense_loops_equals_vectorised():
    Q, K, V = rnd((4, 2, 3), 13), rnd((5, 1, 3), 14), rnd((5, 1, 3), 15)
    assert np.abs(O.attention_dense_loops(Q, K, V) - O.attention_dense(Q, K, V)).max() < 1e-12


def test_gqa_equals_expanded_kv_and_key_permutation():
    Q, K, V = rnd((6, 8, 4), 16), rnd((9, 2, 4), 17), rnd((9, 2, 4), 18)
    a = O.attention_dense(Q, K, V)
    b = O.attention_dense(Q, np.repeat(K, 4, axis=1), np.repeat(V, 4, axis=1))
    assert np.abs(a - b).max() == 0.0
    perm = np.random.default_rng(0).permutation(9)
    assert np.abs(O.attention_dense(Q, K[perm], V[perm]) - a).max() < 1e-13
    # heads 0..3 read KV head 0, heads 4..7 read KV head 1 (not interleaved)
    K2 = K.copy(); K2[:, 1] = 0
    c = O.attention_dense(Q, K2, V)
    assert np.abs(c[:, :4] - a[:, :4]).max() == 0.0 and np.abs(c[:, 4:] - a[:, 4:]).max() > 1e-6
    with pytest.raises(ValueError):
        O.attention_dense(rnd((2, 3, 4), 1), rnd((2, 2, 4), 2), rnd((2, 2, 4), 3))


# ---------------------------------------------------------------- Eq. 6
def test_score_per_head_golden():
    g = GOLD["score_per_head"]
    raw = O.raw_scores(g["q_blk"], g["k"])
    assert raw.tolist() == g["raw"]
    assert O.pool_scores(raw, g["window"]).tolist() == g["pooled"]


def test_raw_scores_is_max_over_block_rows_unscaled():
    Qb, K = rnd((5, 4, 7), 20), rnd((11, 2, 7), 21)
    raw = O.raw_scores(Qb, K)
    assert np.abs(raw - O.raw_scores_loops(Qb, K)).max() < 1e-12
    # a single block row: the plain unscaled dot product; rows can only raise it
    r1 = O.raw_scores(Qb[:1], K)
    assert np.abs(r1[1] - Qb[0, 1] @ K[:, 0].T).max() < 1e-12
    assert (raw >= r1 - 1e-12).all()
    # scaling K by 2 scales the raw score by 2 (linearity, no softmax scale)
    assert np.abs(O.raw_scores(Qb, 2 * K) - 2 * raw).max() < 1e-12


def test_pool_identity_and_vs_torch_maxpool():
    raw = rnd((3, 17), 22)
    assert np.array_equal(O.pool_scores(raw, 1), raw)
    for w in (3, 5, 7):
        t = torch.nn.functional.max_pool1d(torch.from_numpy(raw)[None], w, stride=1, padding=w // 2)[0]
        assert np.array_equal(O.pool_scores(raw, w), t.numpy())
    # a single key: no neighbours
    assert O.pool_scores(np.array([[2.5]]), 3).tolist() == [[2.5]]
    with pytest.raises(ValueError):
        O.pool_scores(raw, 2)


def test_pool_is_on_compacted_candidate_axis():
    # block [2,4) in L=6: candidates [0,1,4,5]; pooling joins 1 and 4 across the block
    Qb = np.ones((2, 1, 1))
    K = np.array([0, 0, 50, 50, 9, 0], dtype=np.float64).reshape(6, 1, 1)
    idx = O.select_heads(Qb, K, 6, 2, 4, 0.5, 3)                            # k = 2
    # raw on C: [0, 0, 9, 0]; pooled: [0, 9, 9, 9]; top-2 lowest-index ties: c = 1, 2 -> pos 1, 4
    assert idx.tolist() == [[1, 4]]


# ---------------------------------------------------------------- TopK
def test_select_topk_golden():
    for case in GOLD["select_topk"]:
        assert O.select_topk(case["S"], case["k"]).tolist() == case["expect"], case["cite"]


def test_select_topk_brute_force_and_order():
    rng = np.random.default_rng(23)
    for trial in range(300):
        n = int(rng.integers(1, 9))
        S = rng.integers(-2, 3, size=n).astype(np.float64)       # heavy ties
        k = int(rng.integers(0, n + 1))
        got = O.select_topk(S, k).tolist()
        assert got == sorted(got) and len(set(got)) == k
        # brute force over all k-subsets: the selection is the unique subset that
        # (a) maximises the sum, then (b) is lexicographically smallest
        best = None
        for sub in itertools.combinations(range(n), k):
            key = (-sum(S[list(sub)]), list(sub))
            if best is None or key < best:
                best = key
        assert got == best[1], (S, k)
        # every kept beats every dropped under (score desc, index asc)
        dropped = [c for c in range(n) if c not in got]
        for c in got:
            for d in dropped:
                assert S[c] > S[d] or (S[c] == S[d] and c < d)


def test_signed_zero_is_a_tie():
    assert O.select_topk([-0.0, 0.0, -1.0], 1).tolist() == [0]
    assert O.select_topk([0.0, -0.0, -1.0], 1).tolist() == [0]


def test_uniformity_trap_witness():
    g = GOLD["select_global"]
    Spool = np.array(g["per_head_pooled"])
    assert O.select_topk(Spool.sum(axis=0), g["k"]).tolist() == g["expect"]
    assert O.select_topk(Spool, 1).tolist() == [[0], [1]]
    sg = GOLD["score_global"]
    assert np.array_equal(np.array(sg["per_head_pooled"]).sum(axis=0), sg["expect"])
    # constructive: per-head selection keeps each head's argmax key; global drops head 1's
    Qb = np.array([[[1.0, 0.0], [0.0, 1.0]]])                   # blk=1, H=2, D=2
    K = np.array([[[9.0, 0.0], [9.0, 0.0]], [[0.0, 9.0], [0.0, 9.0]]])     # L=2, H_kv=2
    K = np.concatenate([K, np.zeros((1, 2, 2))])                 # block row at position 2
    ph = O.select_heads(Qb, K, 3, 2, 3, 0.5, 1)                 # k = ceil(0.5*2) = 1
    gl = O.select_global(Qb, K, 3, 2, 3, 0.5, 1)
    assert ph.tolist() == [[0], [1]] and gl.tolist() == [0]
    assert np.array_equal(O.score_global(Qb, K[:2], 1), [9.0, 9.0])


# ---------------------------------------------------------------- Eq. 4
def _rand_request(seed, L=20, H=4, Hk=2, D=8, bs=7, be=11, r=0.3):
    Q = rnd((L, H, D), seed)
    K, V = rnd((L, Hk, D), seed + 1), rnd((L, Hk, D), seed + 2)
    Qb = rnd((be - bs, H, D), seed + 3)
    return Q, K, V, Qb


def test_reuse_gathered_equals_masked_dense():
    rng = np.random.default_rng(30)
    for t in range(200):                                         # SPEC.md:313 (200 instances)
        L = int(rng.integers(2, 40)); H_kv = int(rng.integers(1, 3)); H = H_kv * int(rng.integers(1, 3))
        D = int(rng.integers(1, 9)); bs = int(rng.integers(0, L)); be = int(rng.integers(bs + 1, L + 1))
        r = float(rng.choice([0.25, 0.5, 1.0]))
        K, V, Qb = rnd((L, H_kv, D), t), rnd((L, H_kv, D), t + 1000), rnd((be - bs, H, D), t + 2000)
        idx = O.select_heads(Qb, K, L, bs, be, r, 3)
        a = O.attention_with_cache(Qb, K, V, bs, be, idx)
        b = O.attention_masked_dense(Qb, K, V, bs, be, idx)
        assert np.abs(a - b).max() <= 1e-10 * max(1.0, np.abs(b).max())


def test_reuse_special_cases():
    Q, K, V, Qb = _rand_request(40)
    # empty context: block = whole sequence -> block-dense attention
    L = 20
    idx0 = O.select_heads(Qb, K, L, 7, 11, 0.3, 3)
    Qfull = rnd((L, 4, 8), 41)
    e = O.attention_with_cache(Qfull, K, V, 0, L, np.zeros((4, 0), np.int64))
    assert np.abs(e - O.attention_dense(Qfull, K, V)).max() < 1e-13
    # r = 1 with Q_blk = Q[bs:be] equals the Refresh rows [bs, be)
    idx1 = O.select_heads(Q[7:11], K, L, 7, 11, 1.0, 3)
    assert idx1.shape == (4, 16)
    full = O.attention_with_cache(Q[7:11], K, V, 7, 11, idx1)
    assert np.abs(full - O.attention_dense(Q, K, V)[7:11]).max() < 1e-13
    # selection excludes the block and is ascending
    for h in range(4):
        row = idx0[h].tolist()
        assert row == sorted(row) and not any(7 <= p < 11 for p in row)


def test_batch_drivers_match_per_request():
    wlL, bsL, beL = [12, 9], [3, 8], [6, 9]
    H, Hk, D = 4, 2, 4
    Q = rnd((21, H, D), 50)
    Ks = [rnd((12, Hk, D), 51), rnd((9, Hk, D), 52)]
    Vs = [rnd((12, Hk, D), 53), rnd((9, Hk, D), 54)]
    Ob, sc = O.refresh_batch(Q, Ks, Vs, wlL, bsL, beL)
    assert np.abs(Ob[12:] - O.attention_dense(Q[12:], Ks[1], Vs[1])).max() == 0
    sel = O.select_batch(sc, wlL, bsL, beL, 0.5, 3)
    assert np.array_equal(sel[0], O.select_heads(Q[3:6], Ks[0], 12, 3, 6, 0.5, 3))
    assert np.array_equal(sel[1], O.select_heads(Q[12 + 8:12 + 9], Ks[1], 9, 8, 9, 0.5, 3))
    Qb = np.concatenate([Q[3:6], Q[20:21]])
    Ou = O.reuse_batch(Qb, Ks, Vs, bsL, beL, sel)
    assert np.abs(Ou[3:] - O.attention_with_cache(Q[20:21], Ks[1], Vs[1], 8, 9, sel[1])).max() == 0


def test_select_global_batch_pins():
    # H = 1: the uniform sum degenerates to the per-head selection
    rng = np.random.default_rng(60)
    sc = [rng.integers(-3, 4, size=(1, 40)).astype(np.float64)]
    a = O.select_global_batch(sc, [40], [20], [24], 0.3, 3)[0]
    b = O.select_batch(sc, [40], [20], [24], 0.3, 3)[0][0]
    assert np.array_equal(a, b)
    # Uniformity-Trap witness through raw scores: per-head pooled
    # [[9,0],[0,9]] (w=1), k=1 -> heads keep {0} and {1}; the global sum ties -> {0}
    raw = [np.array([[9.0, 0.0, 5.0], [0.0, 9.0, 5.0]])]          # position 2 is the block
    assert O.select_batch(raw, [3], [2], [3], 0.5, 1)[0].tolist() == [[0], [1]]
    assert O.select_global_batch(raw, [3], [2], [3], 0.5, 1)[0].tolist() == [0]
    # permuting heads leaves the uniform selection unchanged (a sum), not the per-head one
    sc = [rng.standard_normal((4, 50))]
    g1 = O.select_global_batch(sc, [50], [10], [20], 0.4, 3)[0]
    g2 = O.select_global_batch([sc[0][::-1]], [50], [10], [20], 0.4, 3)[0]
    assert np.array_equal(g1, g2)


# ---------------------------------------------------------------- N2: per-KV-group selection
def test_select_groups_reduces_to_per_head_and_uniform():
    """score_groups sums Eq. 6's pooled scores over the heads sharing a KV head:
    with H_kv = H each group is one head (per-head Eq. 6 selection),
    with H_kv = 1 the group is every head (Eq. 5)."""
    rng = np.random.default_rng(7)
    L, bs, be, D = 37, 20, 25, 8
    Qb = rng.integers(-3, 4, size=(be - bs, 4, D)).astype(np.float64)
    K4 = rng.integers(-3, 4, size=(L, 4, D)).astype(np.float64)
    per_head = O.select_heads(Qb, K4, L, bs, be, 0.3, 3)
    assert np.array_equal(O.select_groups(Qb, K4, L, bs, be, 0.3, 3, 4), per_head)
    K1 = K4[:, :1]
    assert np.array_equal(O.select_groups(Qb, K1, L, bs, be, 0.3, 3, 1)[0],
                          O.select_global(Qb, K1, L, bs, be, 0.3, 3))


def test_select_groups_hand_worked():
    """H = 4 query heads over H_kv = 2 KV heads, w = 1, r = 0.5 on 4 candidates
    (k = 2), raw scores given: group 0 = heads {0, 1}: S = [4,0,0,1] + [0,3,2,1]
    = [4,3,2,2] -> {0, 1}; group 1 = heads {2, 3}: S = [0,0,5,0] + [1,1,0,4] =
    [1,1,5,4] -> {2, 3}.  (Per head the sets would be {0,3}, {1,2}, {0,2}, {0,3}.)"""
    raw = np.array([[4, 0, 0, 1, 9], [0, 3, 2, 1, 9], [0, 0, 5, 0, 9], [1, 1, 0, 4, 9]], dtype=np.float64)
    got = O.select_groups_batch([raw], [5], [4], [5], 0.5, 1, 2)[0]
    assert got.tolist() == [[0, 1], [2, 3]]
    per_head = O.select_batch([raw], [5], [4], [5], 0.5, 1)[0]
    assert per_head.tolist() == [[0, 3], [1, 2], [0, 2], [0, 3]]


def test_select_groups_batch_brute_force():
    """Against brute force over all k-subsets of each group's summed pooled scores
    (largest sum, ties to the lexicographically smallest subset)."""
    from itertools import combinations
    rng = np.random.default_rng(11)
    H, Hk, L, bs, be = 6, 2, 12, 3, 5
    raw = rng.integers(-2, 3, size=(H, L)).astype(np.float64)
    got = O.select_groups_batch([raw], [L], [bs], [be], 0.4, 3, Hk)[0]
    C = np.r_[0:bs, be:L]
    k = O.keep_count(0.4, len(C))
    for g in range(Hk):
        S = np.zeros(len(C))
        for h in range(g * H // Hk, (g + 1) * H // Hk):
            r = raw[h, C]
            S += [max(r[max(0, j - 1):j + 2]) for j in range(len(C))]
        best = min(combinations(range(len(C)), k), key=lambda s: (-sum(S[list(s)]), s))
        assert got[g].tolist() == C[list(best)].tolist()
