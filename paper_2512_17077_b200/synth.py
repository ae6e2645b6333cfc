"""Seeded synthetic inputs for the Head-Centric Sparse Attention path.

This module is shared by the tests (both the oracle side and the CUDA side),
``bench.py`` and ``__graft_entry__.smoke()``.  It holds NONE of the method's
arithmetic: it draws random tensors, places the active block, and lays the
logical K/V out in a paged cache.  Quantities the method derives (keep count
k, candidate scores, selections) are never computed here; where a generator
needs k (``indices``) the caller passes it in.

Recipe:
  * seed:   base seed S (env ``DLLM_SEED``, default 0); every tensor of every
            request gets its own sub-seed = hash(S, config, request, tensor),
            so one request can be regenerated alone (bounded oracle samples).
  * values: "realistic": Q, K ~ N(0, 1), V ~ U(-1, 1), rounded to bf16.
            "exact":     Q, K integers in [-3, 3] (every dot product is an
            integer <= 9*D, exact in fp32 under any summation order), V ~ U(-1, 1).
  * block:  generation region = the last min(256, L) tokens (gen length 256,
            PAPER.md:500); blk = 32 (Table 3 "KV Block Size", PAPER.md:502,
            read as the denoising block, R12); bs = L - G + 32*j with
            j uniform.  Configs may override.
  * pages:  page_size 64 (C0: 16); physical page ids are a random
            permutation; slots past L in a request's last page and all spare
            pages are filled with NaN (the kernels must never read them into a
            result).
"""
from __future__ import annotations

import hashlib
import os
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np
import torch

__all__ = ["Workload", "config", "CONFIG_NAMES", "request_tensors", "Batch", "make_batch",
           "indices", "scores", "replicate", "subset", "lm_head_inputs", "LM_HEAD_FULL"]


def _subseed(*parts) -> int:
    h = hashlib.sha256("/".join(str(p) for p in parts).encode()).digest()
    return int.from_bytes(h[:8], "little") & ((1 << 63) - 1)


def base_seed() -> int:
    return int(os.environ.get("DLLM_SEED", "0"))


@dataclass
class Workload:
    """One batch of requests in the paper's problem statement."""
    name: str
    num_heads: int
    num_kv_heads: int
    head_dim: int
    seq_len: List[int]
    blk_start: List[int]
    blk_end: List[int]
    keep_ratio: float
    pool_window: int = 3          # Table 3 "Kernel Size"
    page_size: int = 64
    kind: str = "realistic"       # or "exact"
    # for mixed batches (C3): which requests run Refresh (+select); the rest Reuse only
    refresh_mask: Optional[List[bool]] = None
    # global request ids (seeding) when this workload is a shard / replica of another
    req_ids: Optional[List[int]] = None

    @property
    def num_requests(self) -> int:
        return len(self.seq_len)

    @property
    def blk(self) -> List[int]:
        return [e - s for s, e in zip(self.blk_start, self.blk_end)]


def _place_blocks(seq_len: Sequence[int], blk: int, gen_len: int, rng: np.random.Generator):
    bs_list, be_list = [], []
    for L in seq_len:
        G = min(gen_len, L)
        nblk = max(1, G // blk)
        j = int(rng.integers(0, nblk))
        bs = max(0, L - G + blk * j)
        be = min(L, bs + blk)
        bs_list.append(bs)
        be_list.append(be)
    return bs_list, be_list


CONFIG_NAMES = ("C0", "C1", "C2", "C3", "C4")


def config(name: str, seed: Optional[int] = None, keep_ratio: Optional[float] = None,
           kind: str = "realistic", num_requests: Optional[int] = None) -> Workload:
    """The BASELINE.json configs.

    C0 tiny: 1 request, H=H_kv=2, D=16, L=64, block [32,40), r=0.25.
    C1 LLaDA-8B layer: B=16, H=H_kv=32, D=128, L=1024, block 32, r=0.25.
    C2 Dream-7B GQA: B=32, H=28, H_kv=4, D=128, L=2048, block 32, r=0.2.
    C3 burst: B=256, LLaDA heads, L ~ U{512..4096}, r=0.25, 8 Refresh + 248 Reuse.
    C4 sweep: B=128, LLaDA heads, L=4096, r in {0.05 .. 1.0} (default 0.25).
    ``num_requests`` truncates the batch (tests at reduced size).
    """
    seed = base_seed() if seed is None else seed
    rng = np.random.default_rng(_subseed(seed, name, "layout"))
    if name == "C0":
        wl = Workload("C0", 2, 2, 16, [64], [32], [40], 0.25, 3, 16, kind)
    elif name == "C1":
        L = [1024] * 16
        bs, be = _place_blocks(L, 32, 256, rng)
        wl = Workload("C1", 32, 32, 128, L, bs, be, 0.25, 3, 64, kind)
    elif name == "C2":
        L = [2048] * 32
        bs, be = _place_blocks(L, 32, 256, rng)
        wl = Workload("C2", 28, 4, 128, L, bs, be, 0.2, 3, 64, kind)
    elif name == "C3":
        L = [int(x) for x in rng.integers(512, 4097, size=256)]
        bs, be = _place_blocks(L, 32, 256, rng)
        mask = [False] * 256
        for i in rng.choice(256, size=8, replace=False):
            mask[int(i)] = True
        wl = Workload("C3", 32, 32, 128, L, bs, be, 0.25, 3, 64, kind, mask)
    elif name == "C4":
        L = [4096] * 128
        bs, be = _place_blocks(L, 32, 256, rng)
        wl = Workload("C4", 32, 32, 128, L, bs, be, 0.25, 3, 64, kind)
    else:
        raise KeyError(name)
    if keep_ratio is not None:
        wl.keep_ratio = keep_ratio
    if num_requests is not None:
        n = num_requests
        wl.seq_len, wl.blk_start, wl.blk_end = wl.seq_len[:n], wl.blk_start[:n], wl.blk_end[:n]
        if wl.refresh_mask is not None:
            wl.refresh_mask = wl.refresh_mask[:n]
    return wl


def replicate(wl: Workload, n: int) -> Workload:
    """n copies of a batch (weak scaling): replica 0 is bit-identical to ``wl``,
    replica r draws its own values (request ids offset by r * B)."""
    B = wl.num_requests
    ids = [r * B + b for r in range(n) for b in range(B)]
    mask = None if wl.refresh_mask is None else wl.refresh_mask * n
    return Workload(wl.name, wl.num_heads, wl.num_kv_heads, wl.head_dim, wl.seq_len * n, wl.blk_start * n,
                    wl.blk_end * n, wl.keep_ratio, wl.pool_window, wl.page_size, wl.kind, mask, ids)


def subset(wl: Workload, reqs: Sequence[int]) -> Workload:
    """The requests ``reqs`` of ``wl`` (a rank's shard); values are unchanged."""
    rid = wl.req_ids if wl.req_ids is not None else list(range(wl.num_requests))
    pick = lambda xs: [xs[i] for i in reqs]  # noqa: E731
    return Workload(wl.name, wl.num_heads, wl.num_kv_heads, wl.head_dim, pick(wl.seq_len), pick(wl.blk_start),
                    pick(wl.blk_end), wl.keep_ratio, wl.pool_window, wl.page_size, wl.kind,
                    None if wl.refresh_mask is None else pick(wl.refresh_mask), pick(rid))


def _bf16(x: torch.Tensor) -> torch.Tensor:
    return x.to(torch.bfloat16)


def _gen(seed: int) -> torch.Generator:
    g = torch.Generator(device="cpu")
    g.manual_seed(seed)
    return g


def request_tensors(wl: Workload, b: int, seed: Optional[int] = None):
    """Logical tensors of request b (bf16, CPU): Q [L,H,D], K, V [L,H_kv,D], Q_blk [blk,H,D].

    Q_blk is an independent input (the current block's queries at a Reuse
    step), drawn from the same distribution as Q.
    """
    seed = base_seed() if seed is None else seed
    L, H, Hk, D = wl.seq_len[b], wl.num_heads, wl.num_kv_heads, wl.head_dim
    blk = wl.blk_end[b] - wl.blk_start[b]
    rid = wl.req_ids[b] if wl.req_ids is not None else b
    tag = (seed, wl.name, wl.kind, rid, L, H, Hk, D)

    def qk(shape, t):
        g = _gen(_subseed(*tag, t))
        if wl.kind == "exact":
            return torch.randint(-3, 4, shape, generator=g).to(torch.bfloat16)
        return _bf16(torch.randn(shape, generator=g))

    q = qk((L, H, D), "Q")
    k = qk((L, Hk, D), "K")
    v = _bf16(torch.rand((L, Hk, D), generator=_gen(_subseed(*tag, "V"))) * 2 - 1)
    q_blk = qk((blk, H, D), "Qblk")
    return q, k, v, q_blk


@dataclass
class Batch:
    """Host-side (CPU) inputs of one batch in the library's layouts."""
    wl: Workload
    q: torch.Tensor            # [sum L, H, D] bf16
    q_blk: torch.Tensor        # [sum blk, H, D] bf16
    k_cache: torch.Tensor      # [num_pages, H_kv, P, D] bf16
    v_cache: torch.Tensor
    block_table: torch.Tensor  # [B, pages_per_req] int32 (-1 past the last page)
    seed: int = 0
    cu_seqlens: List[int] = field(default_factory=list)
    cu_blk: List[int] = field(default_factory=list)

    def k_logical(self, b: int) -> torch.Tensor:
        return _unpage(self.k_cache, self.block_table[b], self.wl.seq_len[b])

    def v_logical(self, b: int) -> torch.Tensor:
        return _unpage(self.v_cache, self.block_table[b], self.wl.seq_len[b])

    def q_req(self, b: int) -> torch.Tensor:
        return self.q[self.cu_seqlens[b]:self.cu_seqlens[b + 1]]

    def q_blk_req(self, b: int) -> torch.Tensor:
        return self.q_blk[self.cu_blk[b]:self.cu_blk[b + 1]]


def _unpage(cache: torch.Tensor, row: torch.Tensor, L: int) -> torch.Tensor:
    P = cache.shape[2]
    npg = (L + P - 1) // P
    pages = cache[row[:npg].long()]                       # [npg, H_kv, P, D]
    return pages.permute(0, 2, 1, 3).reshape(npg * P, cache.shape[1], cache.shape[3])[:L]


def make_batch(wl: Workload, seed: Optional[int] = None, spare_pages: int = 3,
               fill_nan: bool = True, page_seed: Optional[int] = None) -> Batch:
    """All requests' tensors, packed (Q, Q_blk) and paged (K, V).

    ``page_seed`` changes only the physical page permutation (same values)."""
    seed = base_seed() if seed is None else seed
    page_seed = seed if page_seed is None else page_seed
    B, H, Hk, D, P = wl.num_requests, wl.num_heads, wl.num_kv_heads, wl.head_dim, wl.page_size
    npg = [(L + P - 1) // P for L in wl.seq_len]
    pages_per_req = max(npg)
    total_pages = sum(npg) + spare_pages
    perm = torch.randperm(total_pages, generator=_gen(_subseed(page_seed, wl.name, "pages")))
    fill = float("nan") if fill_nan else 0.0
    k_cache = torch.full((total_pages, Hk, P, D), fill, dtype=torch.bfloat16)
    v_cache = torch.full((total_pages, Hk, P, D), fill, dtype=torch.bfloat16)
    block_table = torch.full((B, pages_per_req), -1, dtype=torch.int32)
    qs, qbs = [], []
    nxt = 0
    for b in range(B):
        q, k, v, q_blk = request_tensors(wl, b, seed)
        L = wl.seq_len[b]
        ids = perm[nxt:nxt + npg[b]]
        nxt += npg[b]
        block_table[b, :npg[b]] = ids.to(torch.int32)
        for i in range(npg[b]):
            lo, hi = i * P, min(L, (i + 1) * P)
            k_cache[ids[i], :, :hi - lo] = k[lo:hi].permute(1, 0, 2)
            v_cache[ids[i], :, :hi - lo] = v[lo:hi].permute(1, 0, 2)
        qs.append(q)
        qbs.append(q_blk)
    cu = [0]
    for L in wl.seq_len:
        cu.append(cu[-1] + L)
    cub = [0]
    for x in wl.blk:
        cub.append(cub[-1] + x)
    return Batch(wl, torch.cat(qs), torch.cat(qbs), k_cache, v_cache, block_table, seed, cu, cub)


def indices(wl: Workload, k_per_request: Sequence[int], seed: Optional[int] = None,
            mode: str = "random") -> List[np.ndarray]:
    """Valid per-head index lists (strictly ascending positions outside the
    active block), one [H, k_b] int32 array per request, for driving Reuse
    independently of selection.  k_b is supplied by the caller.

    mode "random": uniform subsets per head.  "shared": every head of a KV
    group gets the same set (maximal GQA overlap).
    """
    seed = base_seed() if seed is None else seed
    out = []
    for b, k in enumerate(k_per_request):
        L, bs, be = wl.seq_len[b], wl.blk_start[b], wl.blk_end[b]
        pool = np.concatenate([np.arange(0, bs), np.arange(be, L)])
        rid = b if wl.req_ids is None else wl.req_ids[b]
        rng = np.random.default_rng(_subseed(seed, wl.name, "idx", rid, mode))
        rows = []
        g = wl.num_heads // wl.num_kv_heads
        for h in range(wl.num_heads):
            if mode == "shared" and h % g:
                rows.append(rows[-1])
                continue
            rows.append(np.sort(rng.choice(pool, size=k, replace=False)))
        out.append(np.stack(rows).astype(np.int32) if rows else np.zeros((0, k), np.int32))
    return out


def scores(wl: Workload, seed: Optional[int] = None, mode: str = "ties") -> List[np.ndarray]:
    """fp32 raw-score tensors [H, L_b] per request, for driving selection
    independently of Refresh.  "ties": small integers (heavy ties, -0.0 mixed
    with +0.0);  "normal": N(0,1) fp32;  "wide": mixed magnitudes and signs."""
    seed = base_seed() if seed is None else seed
    out = []
    for b, L in enumerate(wl.seq_len):
        rng = np.random.default_rng(_subseed(seed, wl.name, "scores", b, mode))
        shape = (wl.num_heads, L)
        if mode == "ties":
            s = rng.integers(-4, 5, size=shape).astype(np.float32)
            zero = (s == 0) & (rng.random(shape) < 0.5)
            s[zero] = -0.0
        elif mode == "normal":
            s = rng.standard_normal(shape).astype(np.float32)
        elif mode == "wide":
            s = (rng.standard_normal(shape) * 10.0 ** rng.integers(-30, 30, size=shape)).astype(np.float32)
        else:
            raise KeyError(mode)
        out.append(s)
    return out


# ----------------------------------------------------------------------------- N4 inputs
# LM-head shapes (Table 3: at most 2,048 materialised logit rows;
# LLaDA-8B: d_model 4,096, vocabulary 126,464 -- the published model config).
LM_HEAD_FULL = {"n_tok": 2048, "d_model": 4096, "vocab": 126464, "max_num_logits": 2048}


def lm_head_inputs(n_tok: int, d_model: int, vocab: int, kind: str = "realistic", seed: Optional[int] = None):
    """(hidden [n_tok, d_model], weight [vocab, d_model]) bf16 CPU tensors.

    realistic: hidden ~ N(0, 1) (post-norm hidden states), weight ~ N(0, 0.02^2)
    (LM-head scale).  exact: integers in [-2, 2] for both, so every logit is an
    integer of magnitude <= 4 d_model, exact in fp32 under any summation order,
    with many exact ties (the lowest-index rule is exercised)."""
    seed = base_seed() if seed is None else seed
    gh = _gen(_subseed(seed, "lm_head", n_tok, d_model, vocab, kind, "hidden"))
    gw = _gen(_subseed(seed, "lm_head", n_tok, d_model, vocab, kind, "weight"))
    if kind == "exact":
        h = torch.randint(-2, 3, (n_tok, d_model), generator=gh).float()
        w = torch.randint(-2, 3, (vocab, d_model), generator=gw).float()
    elif kind == "realistic":
        h = torch.randn((n_tok, d_model), generator=gh)
        w = torch.randn((vocab, d_model), generator=gw) * 0.02
    else:
        raise ValueError(kind)
    return _bf16(h), _bf16(w)
