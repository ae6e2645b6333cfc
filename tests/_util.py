"""Shared test helpers: marshal a synth.Batch to the GPU, run the C-ABI, and
run the oracle on the same generated inputs.  The oracle side never sees a
value produced by the CUDA path."""
from __future__ import annotations

import numpy as np
import torch

import oracle as O
from paper_2512_17077_b200 import synth

# BASELINE.json north_star tolerances for attention outputs (bf16 in, fp32 acc)
MAX_ABS = 1e-2
MEAN_ABS = 1e-3


def problem_of(batch: synth.Batch, device="cuda"):
    from paper_2512_17077_b200 import lib
    wl = batch.wl
    bt = batch.block_table.to(device)
    return lib.Problem(wl.seq_len, wl.blk_start, wl.blk_end, num_heads=wl.num_heads,
                       num_kv_heads=wl.num_kv_heads, head_dim=wl.head_dim, keep_ratio=wl.keep_ratio,
                       pool_window=wl.pool_window, page_size=wl.page_size, block_table=bt)


def to_dev(batch: synth.Batch, device="cuda"):
    return (batch.q.to(device), batch.q_blk.to(device), batch.k_cache.to(device), batch.v_cache.to(device))


def f64(t: torch.Tensor) -> np.ndarray:
    return t.float().numpy().astype(np.float64)


def split_scores(flat: np.ndarray, wl) -> list:
    out, off = [], 0
    for L in wl.seq_len:
        out.append(flat[off:off + wl.num_heads * L].reshape(wl.num_heads, L))
        off += wl.num_heads * L
    return out


def join_scores(per_req) -> np.ndarray:
    return np.concatenate([np.asarray(s, dtype=np.float32).reshape(-1) for s in per_req])


def split_idx(flat: np.ndarray, wl, k) -> list:
    out, off = [], 0
    for kb in k:
        out.append(flat[off:off + wl.num_heads * kb].reshape(wl.num_heads, kb))
        off += wl.num_heads * kb
    return out


def join_idx(per_req) -> np.ndarray:
    return np.concatenate([np.asarray(x, dtype=np.int32).reshape(-1) for x in per_req]) if per_req else np.zeros(0, np.int32)


def assert_close(got: np.ndarray, ref: np.ndarray, what: str, max_abs=MAX_ABS, mean_abs=MEAN_ABS):
    assert got.shape == ref.shape, (what, got.shape, ref.shape)
    assert np.isfinite(got).all(), f"{what}: non-finite output"
    d = np.abs(got.astype(np.float64) - ref)
    assert d.max() <= max_abs, f"{what}: max-abs {d.max():.3e} > {max_abs}"
    assert d.mean() <= mean_abs, f"{what}: mean-abs {d.mean():.3e} > {mean_abs}"
    return float(d.max()), float(d.mean())


def oracle_keep_counts(wl) -> list:
    return [O.keep_count(wl.keep_ratio, L - (be - bs)) for L, bs, be in zip(wl.seq_len, wl.blk_start, wl.blk_end)]
