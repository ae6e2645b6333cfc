"""fp64 CPU oracle for dLLM-Serve's Head-Centric Sparse Attention (arXiv 2512.17077).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
module.  The product path (``paper_2512_17077_b200``) never imports it and has
no CPU fallback.  This file shares no code with the CUDA path: it is a plain,
slow, obviously-correct restatement of the paper's definitions in float64.

Citations are ``PAPER.md:<line>`` (the paper's LaTeX source) with the section /
equation, or ``SPEC.md:<line>`` for the CPU-program spec written from the
paper, or ``DESIGN.md R<n>`` for a reading we had to take where the paper is
silent or ambiguous (listed in DESIGN.md §3).

Notation (§2.3, §4.5): a request has L tokens, an active block
[bs, be), H query heads, H_kv KV heads (GQA, kv(h) = h // (H / H_kv), R10),
head_dim D, keep ratio r, pooling window w.

Tensors are numpy arrays.  Inputs may be any float dtype; everything is
widened to float64 on entry (bf16 -> f64 is exact).

Every function here is pinned by ``tests/test_oracle_pins.py`` against
something other than itself (closed forms, the paper/SPEC worked examples,
library routines, invariants, brute force).
"""
from __future__ import annotations

import math
from typing import Sequence

import numpy as np

__all__ = [
    "kv_head",
    "keep_count",
    "candidates",
    "attention_dense",
    "attention_dense_loops",
    "raw_scores",
    "raw_scores_loops",
    "pool_scores",
    "select_topk",
    "select_heads",
    "score_global",
    "select_global",
    "score_groups",
    "select_groups",
    "attention_with_cache",
    "attention_masked_dense",
    "refresh_batch",
    "select_batch",
    "select_global_batch",
    "select_groups_batch",
    "reuse_batch",
]


# ----------------------------------------------------------------------------
# small helpers
# ----------------------------------------------------------------------------

def _f64(x) -> np.ndarray:
    return np.asarray(x, dtype=np.float64)


def kv_head(h: int, num_heads: int, num_kv_heads: int) -> int:
    """GQA head sharing: query head h reads KV head floor(h / g), g = H / H_kv.

    DESIGN.md R10 (the paper assumes MHA for LLaDA; Dream-7B is GQA,
    PAPER.md:484).  H must be a multiple of H_kv.
    """
    if num_heads % num_kv_heads != 0:
        raise ValueError("num_heads must be a multiple of num_kv_heads")
    return h // (num_heads // num_kv_heads)


def keep_count(keep_ratio: float, n_ctx: int) -> int:
    """k = ceil(r * n_ctx), clamped to [1, n_ctx]; 0 when n_ctx == 0.

    PAPER.md:390 (§4.5) writes k = L*r; R5 takes n_ctx = L - blk
    (the candidate count) and ceil (SPEC.md:204 design decision),
    so r = 1 keeps every context token.  The product r*n_ctx is formed in IEEE
    double, as the paper's r is a real number.
    """
    if not (0.0 < keep_ratio <= 1.0):
        raise ValueError("keep_ratio must be in (0, 1]")
    if n_ctx < 0:
        raise ValueError("n_ctx must be >= 0")
    if n_ctx == 0:
        return 0
    k = math.ceil(float(keep_ratio) * float(n_ctx))
    return max(1, min(n_ctx, k))


def candidates(seq_len: int, blk_start: int, blk_end: int) -> np.ndarray:
    """Context positions C = [0, bs) ++ [be, L), ascending (R4).

    PAPER.md:115-117 (§2.3): Reuse treats "the context outside the active
    block" as cached; SPEC.md:323 includes the prompt among the candidates.
    """
    if not (0 <= blk_start < blk_end <= seq_len):
        raise ValueError("need 0 <= bs < be <= L")
    return np.concatenate([np.arange(0, blk_start), np.arange(blk_end, seq_len)]).astype(np.int64)


# ----------------------------------------------------------------------------
# Eq. 3 — Refresh dense attention
# ----------------------------------------------------------------------------

def attention_dense(Q, K, V, softmax_scale: float | None = None) -> np.ndarray:
    """O = Softmax(Q K^T / sqrt(d)) V per head — PAPER.md:106-113 (§2.3, Eq. 3).

    Q: [n_q, H, D]; K, V: [n_k, H_kv, D].  Bidirectional (no mask).  Softmax
    with max subtraction.  d = head_dim (R11) unless an
    explicit scale is given.  Vectorised per head with numpy matmul.
    """
    Q, K, V = _f64(Q), _f64(K), _f64(V)
    n_q, H, D = Q.shape
    n_k, H_kv, Dk = K.shape
    if Dk != D or V.shape != K.shape:
        raise ValueError("shape mismatch")
    tau = (1.0 / math.sqrt(D)) if not softmax_scale else float(softmax_scale)
    O = np.empty((n_q, H, D), dtype=np.float64)
    for h in range(H):
        kh = kv_head(h, H, H_kv)
        s = tau * (Q[:, h, :] @ K[:, kh, :].T)          # [n_q, n_k]
        m = s.max(axis=1, keepdims=True)
        p = np.exp(s - m)
        p /= p.sum(axis=1, keepdims=True)
        O[:, h, :] = p @ V[:, kh, :]
    return O


def attention_dense_loops(Q, K, V, softmax_scale: float | None = None) -> np.ndarray:
    """Nested-loop brute force of Eq. 3, tiny sizes only.

    Ascending-index summation, max subtraction.
    """
    Q, K, V = _f64(Q), _f64(K), _f64(V)
    n_q, H, D = Q.shape
    n_k, H_kv, _ = K.shape
    tau = (1.0 / math.sqrt(D)) if not softmax_scale else float(softmax_scale)
    O = np.zeros((n_q, H, D), dtype=np.float64)
    for h in range(H):
        kh = kv_head(h, H, H_kv)
        for i in range(n_q):
            s = []
            for j in range(n_k):
                acc = 0.0
                for d in range(D):
                    acc += Q[i, h, d] * K[j, kh, d]
                s.append(tau * acc)
            m = max(s)
            e = [math.exp(x - m) for x in s]
            z = 0.0
            for x in e:
                z += x
            for d in range(D):
                acc = 0.0
                for j in range(n_k):
                    acc += (e[j] / z) * V[j, kh, d]
                O[i, h, d] = acc
    return O


# ----------------------------------------------------------------------------
# Eq. 6 — per-head importance with local max pooling, and TopK
# ----------------------------------------------------------------------------

def raw_scores(Q_blk, K) -> np.ndarray:
    """raw[h, m] = max_{q in block} Q_blk[q, h] . K[m, kv(h)] for every key m.

    Inner term of Eq. 6, PAPER.md:385-389 (§4.5): the UNSCALED dot product
    (R8); the reduction over the block's query rows is max
    (R1).  Q_blk: [blk, H, D]; K: [n, H_kv, D].
    Returns [H, n].
    """
    Q_blk, K = _f64(Q_blk), _f64(K)
    blk, H, D = Q_blk.shape
    n, H_kv, _ = K.shape
    out = np.empty((H, n), dtype=np.float64)
    for h in range(H):
        kh = kv_head(h, H, H_kv)
        out[h] = (Q_blk[:, h, :] @ K[:, kh, :].T).max(axis=0)
    return out


def raw_scores_loops(Q_blk, K) -> np.ndarray:
    """Nested-loop brute force of raw_scores, tiny sizes only."""
    Q_blk, K = _f64(Q_blk), _f64(K)
    blk, H, D = Q_blk.shape
    n, H_kv, _ = K.shape
    out = np.empty((H, n), dtype=np.float64)
    for h in range(H):
        kh = kv_head(h, H, H_kv)
        for m in range(n):
            best = -math.inf
            for q in range(blk):
                acc = 0.0
                for d in range(D):
                    acc += Q_blk[q, h, d] * K[m, kh, d]
                best = max(best, acc)
            out[h, m] = best
    return out


def pool_scores(raw, window: int) -> np.ndarray:
    """S[h, j] = max_{m in [j - w//2, j + w//2] ∩ [0, n)} raw[h, m].

    Outer max of Eq. 6, PAPER.md:385-389 (§4.5), window w = "kernel size"
    (Table 3).  Half-width floor(w/2) (R2), window
    clipped at the edges (R3).  ``raw`` is on the
    compacted candidate axis (R4).  Works on [n] or [H, n].
    """
    raw = _f64(raw)
    if window < 1 or window % 2 == 0:
        raise ValueError("pool window must be odd and >= 1")
    half = window // 2
    n = raw.shape[-1]
    out = np.empty_like(raw)
    for j in range(n):
        lo, hi = max(0, j - half), min(n, j + half + 1)
        out[..., j] = raw[..., lo:hi].max(axis=-1)
    return out


def select_topk(S, k: int) -> np.ndarray:
    """I = TopK(S, k): the k largest scores, ties to the lower index, ascending.

    PAPER.md:390 (§4.5) "I^h = TopK(S_{h,:}, k)"; the tie rule and output
    order are DESIGN.md R6/R7.  S: [n] or [H, n]; returns int64
    indices into S's last axis, shape [k] or [H, k].
    """
    S = _f64(S)
    n = S.shape[-1]
    if not (0 <= k <= n):
        raise ValueError("k must be in [0, n]")
    if S.ndim == 1:
        order = sorted(range(n), key=lambda c: (-S[c], c))
        return np.array(sorted(order[:k]), dtype=np.int64)
    return np.stack([select_topk(S[h], k) for h in range(S.shape[0])]) if S.shape[0] else np.zeros((0, k), np.int64)


def select_heads(Q_blk, K, seq_len: int, blk_start: int, blk_end: int,
                 keep_ratio: float, window: int) -> np.ndarray:
    """Per-head selection for one request: positions I^h, [H, k], ascending.

    PAPER.md:383-390 (§4.5, Eq. 6 + TopK): raw scores of the candidates
    (R4), pooled on the compacted candidate axis, top-k per head with
    k = keep_count(r, n_ctx) (R5), mapped back to sequence positions.
    """
    C = candidates(seq_len, blk_start, blk_end)
    k = keep_count(keep_ratio, len(C))
    H = _f64(Q_blk).shape[1]
    if k == 0:
        return np.zeros((H, 0), dtype=np.int64)
    raw = raw_scores(Q_blk, _f64(K)[C])
    S = pool_scores(raw, window)
    return C[select_topk(S, k)]


def score_global(Q_blk, K, window: int) -> np.ndarray:
    """S_j = sum_h max_{m in win(j)} Q_{b,h} . K_{m,h} — PAPER.md:137-141 (§2.4, Eq. 5).

    The uniform (Sparse-dLLM) baseline: the per-head pooled scores summed
    across heads.  K here is the candidate rows.
    """
    return pool_scores(raw_scores(Q_blk, K), window).sum(axis=0)


def select_global(Q_blk, K, seq_len: int, blk_start: int, blk_end: int,
                  keep_ratio: float, window: int) -> np.ndarray:
    """One shared index set for all heads (§2.4): positions [k]."""
    C = candidates(seq_len, blk_start, blk_end)
    k = keep_count(keep_ratio, len(C))
    if k == 0:
        return np.zeros((0,), dtype=np.int64)
    return C[select_topk(score_global(Q_blk, _f64(K)[C], window), k)]


def score_groups(Q_blk, K, window: int, num_kv_heads: int) -> np.ndarray:
    """Per-KV-group scores S_g[j] = sum_{h in g} max_{m in win(j)} Q_{b,h} . K_{m,kv(h)}.

    Eq. 5 (§2.4) restricted to the query heads that share one
    KV head (GQA, R10, R21): the per-head pooled importance of Eq. 6
     summed over the group g = {h : kv(h) = g}.  Returns
    [H_kv, n] for the candidate rows K.  With H_kv = H it is the per-head Eq. 6
    score; with H_kv = 1 it is Eq. 5.
    """
    pooled = pool_scores(raw_scores(Q_blk, K), window)
    H = pooled.shape[0]
    return np.stack([pooled[[h for h in range(H) if kv_head(h, H, num_kv_heads) == g]].sum(axis=0)
                     for g in range(num_kv_heads)])


def select_groups(Q_blk, K, seq_len: int, blk_start: int, blk_end: int,
                  keep_ratio: float, window: int, num_kv_heads: int) -> np.ndarray:
    """One index set per KV group (next row N2): I_g = TopK(S_g, k) with the
    per-head rules (k = keep_count, R5; ties to the lower index, R6; ascending,
    R7), every head of group g reading I_g (§4.5: rL positions
    per head; here shared by the heads that share the KV rows).  [H_kv, k]."""
    C = candidates(seq_len, blk_start, blk_end)
    k = keep_count(keep_ratio, len(C))
    if k == 0:
        return np.zeros((num_kv_heads, 0), dtype=np.int64)
    S = score_groups(Q_blk, _f64(K)[C], window, num_kv_heads)
    return C[select_topk(S, k)]


# ----------------------------------------------------------------------------
# Eq. 4 — Reuse sparse attention
# ----------------------------------------------------------------------------

def attention_with_cache(Q_blk, K, V, blk_start: int, blk_end: int, idx,
                         softmax_scale: float | None = None) -> np.ndarray:
    """O_b = Softmax(Q_b [K_b; K_cache]^T / sqrt(d)) [V_b; V_cache], per head.

    PAPER.md:117-124 (§2.3, Eq. 4) with the per-head cache of §4.5
    (PAPER.md:390-395): for head h the key set is J^h = [bs, be) ++ I^h.
    K, V are the request's full logical K/V [L, H_kv, D] (the caller wrote the
    active block's rows); idx is [H, k] sequence positions.
    Gathered form: the keys are materialised and dense attention is applied.
    """
    Q_blk, K, V = _f64(Q_blk), _f64(K), _f64(V)
    blk, H, D = Q_blk.shape
    L, H_kv, _ = K.shape
    idx = np.asarray(idx, dtype=np.int64).reshape(H, -1)
    O = np.empty((blk, H, D), dtype=np.float64)
    for h in range(H):
        kh = kv_head(h, H, H_kv)
        J = np.concatenate([np.arange(blk_start, blk_end), idx[h]])
        O[:, h:h + 1, :] = attention_dense(Q_blk[:, h:h + 1, :], K[J, kh:kh + 1, :],
                                           V[J, kh:kh + 1, :], softmax_scale)
    return O


def attention_masked_dense(Q_blk, K, V, blk_start: int, blk_end: int, idx,
                           softmax_scale: float | None = None) -> np.ndarray:
    """Masked-dense form of Eq. 4: dense logits over all L keys, -inf on every
    context key not in I^h.  Independent of the gather."""
    Q_blk, K, V = _f64(Q_blk), _f64(K), _f64(V)
    blk, H, D = Q_blk.shape
    L, H_kv, _ = K.shape
    tau = (1.0 / math.sqrt(D)) if not softmax_scale else float(softmax_scale)
    idx = np.asarray(idx, dtype=np.int64).reshape(H, -1)
    O = np.empty((blk, H, D), dtype=np.float64)
    for h in range(H):
        kh = kv_head(h, H, H_kv)
        keep = np.zeros(L, dtype=bool)
        keep[blk_start:blk_end] = True
        keep[idx[h]] = True
        s = tau * (Q_blk[:, h, :] @ K[:, kh, :].T)
        s[:, ~keep] = -np.inf
        m = s.max(axis=1, keepdims=True)
        p = np.exp(s - m)
        p /= p.sum(axis=1, keepdims=True)
        O[:, h, :] = p @ V[:, kh, :]
    return O


# ----------------------------------------------------------------------------
# batch drivers (packed varlen layout of SURVEY §8(b)); same definitions,
# looped over requests.
# ----------------------------------------------------------------------------

def _offsets(lengths: Sequence[int]) -> np.ndarray:
    return np.concatenate([[0], np.cumsum(np.asarray(lengths, dtype=np.int64))])


def refresh_batch(Q, K_list, V_list, seq_len, blk_start, blk_end,
                  softmax_scale: float | None = None, requests=None):
    """Refresh for a packed batch.

    Q: [sum L, H, D]; K_list/V_list: per-request logical [L_b, H_kv, D].
    Returns (O [sum L, H, D] f64 -- rows of unselected requests are NaN,
    scores: list of [H, L_b] raw scores (Eq. 6 inner term, for every key,
    block rows included) or None for skipped requests).
    ``requests`` restricts the work to a subset (for bounded CPU samples).
    """
    Q = _f64(Q)
    cu = _offsets(seq_len)
    O = np.full(Q.shape, np.nan, dtype=np.float64)
    scores = [None] * len(seq_len)
    reqs = range(len(seq_len)) if requests is None else requests
    for b in reqs:
        q = Q[cu[b]:cu[b + 1]]
        O[cu[b]:cu[b + 1]] = attention_dense(q, K_list[b], V_list[b], softmax_scale)
        scores[b] = raw_scores(q[blk_start[b]:blk_end[b]], K_list[b])
    return O, scores


def select_batch(scores, seq_len, blk_start, blk_end, keep_ratio: float, window: int):
    """Per-head selection from precomputed raw scores [H, L_b] per request.

    PAPER.md:385-390 (Eq. 6 outer max + TopK).  Returns a list of [H, k_b]
    int64 position arrays (ascending per head).
    """
    out = []
    for b, sc in enumerate(scores):
        if sc is None:
            out.append(None)
            continue
        C = candidates(seq_len[b], blk_start[b], blk_end[b])
        k = keep_count(keep_ratio, len(C))
        sc = _f64(sc)
        if k == 0:
            out.append(np.zeros((sc.shape[0], 0), np.int64))
            continue
        out.append(C[select_topk(pool_scores(sc[:, C], window), k)])
    return out


def select_global_batch(scores, seq_len, blk_start, blk_end, keep_ratio: float, window: int):
    """Uniform (Sparse-dLLM) selection from precomputed raw scores [H, L_b]:
    S_j = sum_h pool(raw_h)[j] (§2.4, Eq. 5), one top-k per
    request with the same tie rule and order (R6, R7).  Returns a
    list of [k_b] int64 position arrays."""
    out = []
    for b, sc in enumerate(scores):
        C = candidates(seq_len[b], blk_start[b], blk_end[b])
        k = keep_count(keep_ratio, len(C))
        if k == 0:
            out.append(np.zeros((0,), np.int64))
            continue
        S = pool_scores(_f64(sc)[:, C], window).sum(axis=0)
        out.append(C[select_topk(S, k)])
    return out


def select_groups_batch(scores, seq_len, blk_start, blk_end, keep_ratio: float, window: int,
                        num_kv_heads: int):
    """Per-KV-group selection from precomputed raw scores [H, L_b] (score_groups
    on the candidate axis, one top-k per group).  Returns a list of [H_kv, k_b]
    int64 position arrays."""
    out = []
    for b, sc in enumerate(scores):
        C = candidates(seq_len[b], blk_start[b], blk_end[b])
        k = keep_count(keep_ratio, len(C))
        if k == 0:
            out.append(np.zeros((num_kv_heads, 0), np.int64))
            continue
        pooled = pool_scores(_f64(sc)[:, C], window)
        H = pooled.shape[0]
        S = np.stack([pooled[[h for h in range(H) if kv_head(h, H, num_kv_heads) == g]].sum(axis=0)
                      for g in range(num_kv_heads)])
        out.append(C[select_topk(S, k)])
    return out


def reuse_batch(Q_blk, K_list, V_list, blk_start, blk_end, idx_list,
                softmax_scale: float | None = None, requests=None):
    """Reuse for a packed batch: Q_blk [sum blk, H, D]; returns O_blk f64."""
    Q_blk = _f64(Q_blk)
    blks = [e - s for s, e in zip(blk_start, blk_end)]
    cu = _offsets(blks)
    O = np.full(Q_blk.shape, np.nan, dtype=np.float64)
    reqs = range(len(blks)) if requests is None else requests
    for b in reqs:
        O[cu[b]:cu[b + 1]] = attention_with_cache(Q_blk[cu[b]:cu[b + 1]], K_list[b], V_list[b],
                                                  blk_start[b], blk_end[b], idx_list[b],
                                                  softmax_scale)
    return O
