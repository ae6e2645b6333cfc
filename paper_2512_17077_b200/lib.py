"""Thin Python binding of libdllm's C-ABI (include/dllm.h).

Argument marshalling only: every step of the path runs in libdllm's CUDA
kernels.  Tensors are torch CUDA tensors (PyTorch supplies device memory and
streams); host arrays are plain Python/numpy int sequences.  There is no CPU
fallback: importing this module fails loudly if libdllm.so is missing, and a
compute call on tensors that are not on a CUDA device raises.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DLLM_LIB") or os.path.join(_HERE, "libdllm.so")   # DLLM_LIB: dev builds only

DLLM_OK = 0
DLLM_ERR_INVALID_ARG = -1
DLLM_ERR_UNSUPPORTED = -2
DLLM_ERR_SHAPE = -3
DLLM_ERR_K_RANGE = -4
DLLM_ERR_CUDA = -5

EXPORTED = ("dllm_workspace_bytes", "dllm_keep_count", "dllm_index_layout", "dllm_refresh_attn", "dllm_select_heads",
            "dllm_select_global", "dllm_select_groups",
            "dllm_refresh_select_attn", "dllm_mixed_select_attn",
            "dllm_reuse_sparse_attn", "dllm_reuse_group_sets", "dllm_pack_kv", "dllm_reuse_packed", "dllm_mixed_attn", "dllm_logit_chunks",
            "dllm_lm_head_workspace_bytes", "dllm_lm_head_argmax", "dllm_check_indices", "dllm_status_string",
            "dllm_last_error", "dllm_version")


class DllmError(RuntimeError):
    def __init__(self, status: int, where: str, detail: str):
        super().__init__(f"{where}: {detail or ''} [{status_string(status)}]")
        self.status = status


class _Problem(ctypes.Structure):
    _fields_ = [
        ("num_requests", ctypes.c_int32),
        ("num_heads", ctypes.c_int32),
        ("num_kv_heads", ctypes.c_int32),
        ("head_dim", ctypes.c_int32),
        ("seq_len", ctypes.POINTER(ctypes.c_int32)),
        ("blk_start", ctypes.POINTER(ctypes.c_int32)),
        ("blk_end", ctypes.POINTER(ctypes.c_int32)),
        ("keep_ratio", ctypes.c_double),
        ("pool_window", ctypes.c_int32),
        ("softmax_scale", ctypes.c_float),
        ("page_size", ctypes.c_int32),
        ("pages_per_req", ctypes.c_int32),
        ("block_table", ctypes.c_void_p),
        ("workspace", ctypes.c_void_p),
        ("workspace_bytes", ctypes.c_int64),
    ]


def _load() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libdllm.so not built ({LIB_PATH}); run `python -m paper_2512_17077_b200.build` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    P = ctypes.POINTER(_Problem)
    vp = ctypes.c_void_p
    if hasattr(lib, "dllm_workspace_bytes"):   # (absent in dev A/B builds of older sources)
        lib.dllm_workspace_bytes.argtypes = []
        lib.dllm_workspace_bytes.restype = ctypes.c_int64
    lib.dllm_keep_count.argtypes = [ctypes.c_double, ctypes.c_int32]
    lib.dllm_keep_count.restype = ctypes.c_int
    lib.dllm_index_layout.argtypes = [P, ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int64),
                                      ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64)]
    lib.dllm_index_layout.restype = ctypes.c_int
    lib.dllm_refresh_attn.argtypes = [P, vp, vp, vp, vp, vp, vp]
    lib.dllm_refresh_attn.restype = ctypes.c_int
    lib.dllm_select_heads.argtypes = [P, vp, vp, vp]
    lib.dllm_select_heads.restype = ctypes.c_int
    lib.dllm_select_global.argtypes = [P, vp, vp, vp]
    lib.dllm_select_global.restype = ctypes.c_int
    if hasattr(lib, "dllm_select_groups"):
        lib.dllm_select_groups.argtypes = [P, vp, vp, vp]
        lib.dllm_select_groups.restype = ctypes.c_int
    lib.dllm_reuse_sparse_attn.argtypes = [P, vp, vp, vp, vp, vp, vp]
    lib.dllm_reuse_sparse_attn.restype = ctypes.c_int
    lib.dllm_reuse_group_sets.argtypes = [P, vp, vp, vp, vp, vp, vp]
    lib.dllm_reuse_group_sets.restype = ctypes.c_int
    lib.dllm_pack_kv.argtypes = [P, vp, vp, vp, vp, vp, vp]
    lib.dllm_pack_kv.restype = ctypes.c_int
    lib.dllm_reuse_packed.argtypes = [P, vp, vp, vp, vp, vp, vp, vp]
    lib.dllm_reuse_packed.restype = ctypes.c_int
    lib.dllm_mixed_attn.argtypes = [P, vp, vp, vp, P, vp, vp, vp, vp, vp, vp]
    lib.dllm_mixed_attn.restype = ctypes.c_int
    lib.dllm_refresh_select_attn.argtypes = [P, vp, vp, vp, vp, vp, vp, vp]
    lib.dllm_refresh_select_attn.restype = ctypes.c_int
    lib.dllm_mixed_select_attn.argtypes = [P, vp, vp, vp, vp, P, vp, vp, vp, vp, vp, vp]
    lib.dllm_mixed_select_attn.restype = ctypes.c_int
    lib.dllm_logit_chunks.argtypes = [ctypes.c_int64, ctypes.c_int32, ctypes.POINTER(ctypes.c_int32), ctypes.c_int32]
    lib.dllm_logit_chunks.restype = ctypes.c_int
    lib.dllm_lm_head_workspace_bytes.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_int32]
    lib.dllm_lm_head_workspace_bytes.restype = ctypes.c_int64
    lib.dllm_lm_head_argmax.argtypes = [vp, vp, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, vp, vp,
                                        ctypes.c_int64, vp]
    lib.dllm_lm_head_argmax.restype = ctypes.c_int
    lib.dllm_check_indices.argtypes = [P, vp, vp, vp]
    lib.dllm_check_indices.restype = ctypes.c_int
    lib.dllm_status_string.argtypes = [ctypes.c_int]
    lib.dllm_status_string.restype = ctypes.c_char_p
    lib.dllm_last_error.argtypes = []
    lib.dllm_last_error.restype = ctypes.c_char_p
    lib.dllm_version.argtypes = []
    lib.dllm_version.restype = ctypes.c_char_p
    return lib


_lib = _load()


def lib() -> ctypes.CDLL:
    return _lib


def status_string(status: int) -> str:
    return _lib.dllm_status_string(status).decode()


def last_error() -> str:
    return _lib.dllm_last_error().decode()


def version() -> str:
    return _lib.dllm_version().decode()


def _check(status: int, where: str) -> None:
    if status != DLLM_OK:
        raise DllmError(status, where, last_error())


def keep_count(keep_ratio: float, n_ctx: int) -> int:
    k = _lib.dllm_keep_count(float(keep_ratio), int(n_ctx))
    _check(min(k, 0), "dllm_keep_count")
    return k


def _i32(xs) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(xs, dtype=np.int32))


def workspace_bytes() -> int:
    return int(_lib.dllm_workspace_bytes()) if hasattr(_lib, "dllm_workspace_bytes") else 16


def alloc_workspace(device="cuda") -> torch.Tensor:
    """A zeroed dllm_problem workspace (one per stream; it stays zeroed across launches)."""
    return torch.zeros(workspace_bytes(), dtype=torch.uint8, device=device)


class Problem:
    """Owns the host arrays, the device block table and the workspace behind a dllm_problem.

    workspace: "auto" (default) allocates a zeroed one on the block table's device,
    None runs without (Reuse keeps whole units, Refresh schedules statically), or a
    caller tensor of at least workspace_bytes() bytes."""

    def __init__(self, seq_len: Sequence[int], blk_start: Sequence[int], blk_end: Sequence[int], *,
                 num_heads: int, num_kv_heads: int, head_dim: int, keep_ratio: float, pool_window: int = 3,
                 softmax_scale: float = 0.0, page_size: int = 64, block_table: Optional[torch.Tensor] = None,
                 pages_per_req: Optional[int] = None, workspace="auto"):
        self.seq_len, self.blk_start, self.blk_end = _i32(seq_len), _i32(blk_start), _i32(blk_end)
        self.block_table = block_table
        if isinstance(workspace, str):
            assert workspace == "auto"
            workspace = (alloc_workspace(block_table.device) if block_table is not None and block_table.is_cuda
                         else None)
        self.workspace = workspace
        if pages_per_req is None:
            pages_per_req = int(block_table.shape[1]) if block_table is not None and block_table.dim() == 2 else 0
        self._s = _Problem()
        s = self._s
        s.num_requests = len(self.seq_len)
        s.num_heads, s.num_kv_heads, s.head_dim = num_heads, num_kv_heads, head_dim
        ptr = ctypes.POINTER(ctypes.c_int32)
        s.seq_len = self.seq_len.ctypes.data_as(ptr)
        s.blk_start = self.blk_start.ctypes.data_as(ptr)
        s.blk_end = self.blk_end.ctypes.data_as(ptr)
        s.keep_ratio = float(keep_ratio)
        s.pool_window = int(pool_window)
        s.softmax_scale = float(softmax_scale)
        s.page_size = int(page_size)
        s.pages_per_req = int(pages_per_req)
        if block_table is not None:
            assert block_table.dtype == torch.int32 and block_table.is_contiguous()
            s.block_table = block_table.data_ptr()
        else:
            s.block_table = None
        if workspace is not None:
            if not (workspace.is_cuda and workspace.is_contiguous()):
                raise ValueError("workspace must be a contiguous CUDA tensor")
            s.workspace = workspace.data_ptr()
            s.workspace_bytes = workspace.numel() * workspace.element_size()
        else:
            s.workspace, s.workspace_bytes = None, 0
        self._layout = None

    @property
    def ref(self):
        return ctypes.byref(self._s)

    @property
    def num_requests(self) -> int:
        return self._s.num_requests

    @property
    def num_heads(self) -> int:
        return self._s.num_heads

    @property
    def head_dim(self) -> int:
        return self._s.head_dim

    def layout(self):
        """(k per request, total idx elements, total rows, total block rows)."""
        if self._layout is None:
            self._layout = self._query_layout()
        return self._layout

    def _query_layout(self):
        B = self._s.num_requests
        k = (ctypes.c_int32 * max(B, 1))()
        ti, tr, tb = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        _check(_lib.dllm_index_layout(self.ref, k, ctypes.byref(ti), ctypes.byref(tr), ctypes.byref(tb)),
               "dllm_index_layout")
        return [k[i] for i in range(B)], ti.value, tr.value, tb.value


def _dev(t: Optional[torch.Tensor], name: str, dtype=None, need: int = 0) -> int:
    if t is None:
        return 0
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (libdllm has no CPU path)")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if dtype is not None and t.dtype != dtype:
        raise ValueError(f"{name} must be {dtype}, got {t.dtype}")
    if t.numel() < need:
        raise ValueError(f"{name} holds {t.numel()} elements, the problem's layout needs {need}")
    return t.data_ptr()


def _sizes(p: "Problem"):
    """Element counts the layout needs: (q/out rows*H*D, scores H*rows, idx, q_blk/out_blk)."""
    _, total_idx, rows, blk_rows = p.layout()
    HD = p.num_heads * p.head_dim
    return rows * HD, p.num_heads * rows, total_idx, blk_rows * HD


def _stream(stream) -> int:
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def refresh_attn(p: Problem, q, k_cache, v_cache, out, scores=None, stream=None) -> None:
    """dllm_refresh_attn (Eq. 3 + Eq. 6 raw importance)."""
    bf = torch.bfloat16
    nq, ns, _, _ = _sizes(p)
    _check(_lib.dllm_refresh_attn(p.ref, _dev(q, "q", bf, nq), _dev(k_cache, "k_cache", bf),
                                  _dev(v_cache, "v_cache", bf), _dev(out, "out", bf, nq),
                                  _dev(scores, "scores", torch.float32, ns), _stream(stream)), "dllm_refresh_attn")


def select_heads(p: Problem, scores, idx, stream=None) -> None:
    """dllm_select_heads (Eq. 6 pool + per-head TopK)."""
    _, ns, ni, _ = _sizes(p)
    _check(_lib.dllm_select_heads(p.ref, _dev(scores, "scores", torch.float32, ns), _dev(idx, "idx", torch.int32, ni),
                                  _stream(stream)), "dllm_select_heads")


def refresh_select_attn(p: Problem, q, k_cache, v_cache, out, scores, idx, stream=None) -> None:
    """dllm_refresh_select_attn: Refresh + Eq. 6 pool/TopK, the select fused into the Refresh kernel."""
    bf = torch.bfloat16
    nq, ns, ni, _ = _sizes(p)
    _check(_lib.dllm_refresh_select_attn(p.ref, _dev(q, "q", bf, nq), _dev(k_cache, "k_cache", bf),
                                         _dev(v_cache, "v_cache", bf), _dev(out, "out", bf, nq),
                                         _dev(scores, "scores", torch.float32, ns), _dev(idx, "idx", torch.int32, ni),
                                         _stream(stream)), "dllm_refresh_select_attn")


def select_global(p: Problem, scores, idx, stream=None) -> None:
    """dllm_select_global (Eq. 5 uniform baseline: one shared set per request)."""
    _, ns, ni, _ = _sizes(p)
    _check(_lib.dllm_select_global(p.ref, _dev(scores, "scores", torch.float32, ns),
                                   _dev(idx, "idx", torch.int32, ni), _stream(stream)), "dllm_select_global")


def select_groups(p: Problem, scores, idx, stream=None) -> None:
    """dllm_select_groups (N2, GQA: one shared set per KV group)."""
    _, ns, ni, _ = _sizes(p)
    _check(_lib.dllm_select_groups(p.ref, _dev(scores, "scores", torch.float32, ns),
                                   _dev(idx, "idx", torch.int32, ni), _stream(stream)), "dllm_select_groups")


def reuse_sparse_attn(p: Problem, q_blk, k_cache, v_cache, idx, out_blk, stream=None) -> None:
    """dllm_reuse_sparse_attn (Eq. 4 over per-head key subsets)."""
    bf = torch.bfloat16
    _, _, ni, nb = _sizes(p)
    _check(_lib.dllm_reuse_sparse_attn(p.ref, _dev(q_blk, "q_blk", bf, nb), _dev(k_cache, "k_cache", bf),
                                       _dev(v_cache, "v_cache", bf), _dev(idx, "idx", torch.int32, ni),
                                       _dev(out_blk, "out_blk", bf, nb), _stream(stream)), "dllm_reuse_sparse_attn")


def reuse_group_sets(p: Problem, q_blk, k_cache, v_cache, idx, out_blk, stream=None) -> None:
    """dllm_reuse_group_sets (Eq. 4 over one key set per KV group, as select_groups writes them)."""
    bf = torch.bfloat16
    _, _, ni, nb = _sizes(p)
    _check(_lib.dllm_reuse_group_sets(p.ref, _dev(q_blk, "q_blk", bf, nb), _dev(k_cache, "k_cache", bf),
                                      _dev(v_cache, "v_cache", bf), _dev(idx, "idx", torch.int32, ni),
                                      _dev(out_blk, "out_blk", bf, nb), _stream(stream)), "dllm_reuse_group_sets")


def pack_kv(p: Problem, k_cache, v_cache, idx, k_pack, v_pack, stream=None) -> None:
    """dllm_pack_kv (the paper's dense per-head layout)."""
    bf = torch.bfloat16
    _check(_lib.dllm_pack_kv(p.ref, _dev(k_cache, "k_cache", bf), _dev(v_cache, "v_cache", bf),
                             _dev(idx, "idx", torch.int32), _dev(k_pack, "k_pack", bf), _dev(v_pack, "v_pack", bf),
                             _stream(stream)), "dllm_pack_kv")


def reuse_packed(p: Problem, q_blk, k_cache, v_cache, k_pack, v_pack, out_blk, stream=None) -> None:
    """dllm_reuse_packed (Eq. 4 over the packed per-head context)."""
    bf = torch.bfloat16
    _check(_lib.dllm_reuse_packed(p.ref, _dev(q_blk, "q_blk", bf), _dev(k_cache, "k_cache", bf),
                                  _dev(v_cache, "v_cache", bf), _dev(k_pack, "k_pack", bf), _dev(v_pack, "v_pack", bf),
                                  _dev(out_blk, "out_blk", bf), _stream(stream)), "dllm_reuse_packed")


def mixed_attn(p_refresh: Problem, q, out, scores, p_reuse: Problem, q_blk, idx, out_blk, k_cache, v_cache,
               stream=None) -> None:
    """Refresh over p_refresh and Reuse over p_reuse in one launch (N3)."""
    bf = torch.bfloat16
    nq, ns, _, _ = _sizes(p_refresh)
    _, _, ni, nb = _sizes(p_reuse)
    _check(_lib.dllm_mixed_attn(p_refresh.ref, _dev(q, "q", bf, nq), _dev(out, "out", bf, nq),
                                _dev(scores, "scores", torch.float32, ns), p_reuse.ref, _dev(q_blk, "q_blk", bf, nb),
                                _dev(idx, "idx", torch.int32, ni), _dev(out_blk, "out_blk", bf, nb),
                                _dev(k_cache, "k_cache", bf), _dev(v_cache, "v_cache", bf), _stream(stream)),
           "dllm_mixed_attn")


def mixed_select_attn(p_refresh: Problem, q, out, scores, idx_refresh, p_reuse: Problem, q_blk, idx, out_blk, k_cache,
                      v_cache, stream=None) -> None:
    """dllm_mixed_select_attn: mixed_attn with the Refresh requests' selection fused in."""
    bf = torch.bfloat16
    nq, ns, nir, _ = _sizes(p_refresh)
    _, _, ni, nb = _sizes(p_reuse)
    _check(_lib.dllm_mixed_select_attn(p_refresh.ref, _dev(q, "q", bf, nq), _dev(out, "out", bf, nq),
                                       _dev(scores, "scores", torch.float32, ns),
                                       _dev(idx_refresh, "idx_refresh", torch.int32, nir),
                                       p_reuse.ref, _dev(q_blk, "q_blk", bf, nb), _dev(idx, "idx", torch.int32, ni),
                                       _dev(out_blk, "out_blk", bf, nb), _dev(k_cache, "k_cache", bf),
                                       _dev(v_cache, "v_cache", bf), _stream(stream)), "dllm_mixed_select_attn")


def logit_chunks(n_logit: int, max_num_logits: int) -> list:
    """SPEC.md:145-155 plan_logit_chunks through the C-ABI (host only)."""
    n = _lib.dllm_logit_chunks(int(n_logit), int(max_num_logits), None, 0)
    _check(min(n, 0), "dllm_logit_chunks")
    buf = (ctypes.c_int32 * max(n, 1))()
    n2 = _lib.dllm_logit_chunks(int(n_logit), int(max_num_logits), buf, n)
    _check(min(n2, 0), "dllm_logit_chunks")
    return [int(buf[i]) for i in range(n2)]


def lm_head_workspace_bytes(n_tok: int, vocab: int, max_num_logits: int) -> int:
    b = _lib.dllm_lm_head_workspace_bytes(int(n_tok), int(vocab), int(max_num_logits))
    _check(int(min(b, 0)), "dllm_lm_head_workspace_bytes")
    return int(b)


def lm_head_argmax(hidden, weight, ids, max_num_logits: int = 2048, workspace=None, stream=None) -> None:
    """ids[i] = lowest-index argmax_v hidden[i] . weight[v] (N4)."""
    n_tok, d_model = hidden.shape
    vocab = weight.shape[0]
    if weight.shape[1] != d_model:
        raise ValueError("weight must be [vocab, d_model]")
    if workspace is None:
        workspace = torch.empty(max(lm_head_workspace_bytes(n_tok, vocab, max_num_logits), 16), dtype=torch.uint8,
                                device=hidden.device)
    bf = torch.bfloat16
    _check(_lib.dllm_lm_head_argmax(_dev(hidden, "hidden", bf), _dev(weight, "weight", bf), int(n_tok), int(d_model),
                                    int(vocab), int(max_num_logits), _dev(ids, "ids", torch.int32),
                                    _dev(workspace, "workspace"), int(workspace.numel() * workspace.element_size()),
                                    _stream(stream)), "dllm_lm_head_argmax")


def check_indices(p: Problem, idx, violations, stream=None) -> None:
    _check(_lib.dllm_check_indices(p.ref, _dev(idx, "idx", torch.int32), _dev(violations, "violations", torch.int32),
                                   _stream(stream)), "dllm_check_indices")


@dataclass
class Buffers:
    """Caller-owned outputs sized from dllm_index_layout."""
    out: torch.Tensor
    scores: torch.Tensor
    idx: torch.Tensor
    out_blk: torch.Tensor
    k: list


def alloc_buffers(p: Problem, device="cuda") -> Buffers:
    k, total_idx, rows, blk_rows = p.layout()
    H, D = p.num_heads, p.head_dim
    return Buffers(
        out=torch.empty((rows, H, D), dtype=torch.bfloat16, device=device),
        scores=torch.empty((H * rows,), dtype=torch.float32, device=device),
        idx=torch.empty((max(total_idx, 1),), dtype=torch.int32, device=device),
        out_blk=torch.empty((blk_rows, H, D), dtype=torch.bfloat16, device=device),
        k=k,
    )


def hot_path(p: Problem, q, q_blk, k_cache, v_cache, buf: Buffers, stream=None) -> None:
    """One pass of the whole hot path: Refresh (+importance, select fused in) -> Reuse."""
    refresh_select_attn(p, q, k_cache, v_cache, buf.out, buf.scores, buf.idx, stream)
    reuse_sparse_attn(p, q_blk, k_cache, v_cache, buf.idx, buf.out_blk, stream)
