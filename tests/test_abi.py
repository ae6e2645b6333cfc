"""C-ABI checks that need no GPU: the library loads, exports every symbol
include/dllm.h declares, and its host-only logic (keep count, index layout,
all-or-nothing validation) behaves as documented.  No compute call is made."""
import ctypes
import json
import os
import re

import numpy as np
import pytest
import torch

import oracle as O
from paper_2512_17077_b200 import lib as L
from paper_2512_17077_b200 import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = open(os.path.join(ROOT, "include", "dllm.h")).read()
GOLD = json.load(open(os.path.join(ROOT, "tests", "golden", "spec_examples.json")))


def test_exports_every_declared_symbol():
    declared = re.findall(r"DLLM_API\s+[\w\s\*]+?\b(dllm_\w+)\s*\(", HEADER)
    assert len(declared) >= 9
    so = ctypes.CDLL(L.LIB_PATH)
    for name in declared:
        assert hasattr(so, name), name
    assert set(declared) == set(L.EXPORTED)


def test_status_strings_and_version():
    for code, name in [(0, "DLLM_OK"), (-1, "DLLM_ERR_INVALID_ARG"), (-2, "DLLM_ERR_UNSUPPORTED"),
                       (-3, "DLLM_ERR_SHAPE"), (-4, "DLLM_ERR_K_RANGE"), (-5, "DLLM_ERR_CUDA")]:
        assert L.status_string(code) == name
        assert re.search(rf"#define {name}\s+\(?{code}\)?", HEADER)
    assert "sm_100a" in L.version()


def test_keep_count_matches_golden_and_oracle():
    for r, n, k in GOLD["keep_count"]["cases"]:
        assert L.keep_count(r, n) == k
    rng = np.random.default_rng(0)
    for _ in range(2000):
        r = float(rng.choice([rng.random(), 0.05, 0.1, 0.2, 0.25, 0.5, 0.75, 1.0]))
        if r == 0.0:
            continue
        n = int(rng.integers(0, 70000))
        assert L.keep_count(r, n) == O.keep_count(r, n), (r, n)
    for bad in (0.0, -1.0, 1.5, float("nan")):
        with pytest.raises(L.DllmError) as e:
            L.keep_count(bad, 10)
        assert e.value.status == L.DLLM_ERR_INVALID_ARG


def _fake_bt(B, pages):
    # validation never dereferences the device block table; any non-NULL pointer will do
    return torch.zeros((B, pages), dtype=torch.int32)


def _prob(wl, **kw):
    args = dict(num_heads=wl.num_heads, num_kv_heads=wl.num_kv_heads, head_dim=wl.head_dim,
                keep_ratio=wl.keep_ratio, pool_window=wl.pool_window, page_size=wl.page_size,
                block_table=_fake_bt(wl.num_requests, 64))
    args.update(kw)
    return L.Problem(wl.seq_len, wl.blk_start, wl.blk_end, **args)


@pytest.mark.parametrize("cfg", ["C0", "C1", "C2", "C3", "C4"])
def test_index_layout_matches_oracle(cfg):
    wl = synth.config(cfg)
    k, total_idx, rows, blk_rows = _prob(wl).layout()
    ko = [O.keep_count(wl.keep_ratio, Lb - (be - bs)) for Lb, bs, be in zip(wl.seq_len, wl.blk_start, wl.blk_end)]
    assert k == ko
    assert total_idx == wl.num_heads * sum(ko)
    assert rows == sum(wl.seq_len) and blk_rows == sum(wl.blk)
    if cfg == "C1":
        assert set(k) == {248}
    if cfg == "C2":
        assert set(k) == {404}


def _status(fn):
    with pytest.raises(L.DllmError) as e:
        fn()
    return e.value.status


def test_validation_rejects_bad_problems():
    wl = synth.config("C1", num_requests=2)
    q = torch.zeros(8, dtype=torch.bfloat16)      # never touched: validation fails first
    dummy = (q, q, q, q)
    cases = {
        "even window": (dict(pool_window=2), L.DLLM_ERR_INVALID_ARG),
        "r=0": (dict(keep_ratio=0.0), L.DLLM_ERR_INVALID_ARG),
        "r>1": (dict(keep_ratio=1.01), L.DLLM_ERR_INVALID_ARG),
        "D=96": (dict(head_dim=96), L.DLLM_ERR_UNSUPPORTED),
        "H%Hkv": (dict(num_heads=32, num_kv_heads=5), L.DLLM_ERR_SHAPE),
        "page 48": (dict(page_size=48), L.DLLM_ERR_UNSUPPORTED),
        "pages_per_req": (dict(pages_per_req=3), L.DLLM_ERR_SHAPE),
        "neg scale": (dict(softmax_scale=-1.0), L.DLLM_ERR_INVALID_ARG),
        "no block table": (dict(block_table=None, pages_per_req=16), L.DLLM_ERR_INVALID_ARG),
    }
    for name, (kw, code) in cases.items():
        p = _prob(wl, **kw)
        assert _status(p.layout) == code, name
        # the compute entry points validate identically before touching the device
        assert L.lib().dllm_refresh_attn(p.ref, None, None, None, None, None, None) == code, name
        assert L.lib().dllm_reuse_sparse_attn(p.ref, None, None, None, None, None, None) == code, name
        assert L.lib().dllm_select_heads(p.ref, None, None, None) == code, name
        assert L.lib().dllm_refresh_select_attn(p.ref, None, None, None, None, None, None, None) == code, name
        assert L.last_error() != ""
    bad_blocks = [([10], [5], [5]), ([10], [-1], [3]), ([10], [2], [11]), ([0], [0], [1]), ([300], [0], [200])]
    for Ls, bs, be in bad_blocks:
        p = L.Problem(Ls, bs, be, num_heads=2, num_kv_heads=2, head_dim=64, keep_ratio=0.5,
                      block_table=_fake_bt(1, 32))
        assert _status(p.layout) in (L.DLLM_ERR_SHAPE, L.DLLM_ERR_UNSUPPORTED), (Ls, bs, be)
    # NULL tensors on a valid problem are rejected before any launch
    p = _prob(wl)
    assert L.lib().dllm_refresh_attn(p.ref, None, None, None, None, None, None) == L.DLLM_ERR_INVALID_ARG
    assert L.lib().dllm_select_heads(p.ref, None, None, None) == L.DLLM_ERR_INVALID_ARG
    # the one-call Refresh + select requires both scores and idx
    assert L.lib().dllm_refresh_select_attn(p.ref, None, None, None, None, None, None, None) == L.DLLM_ERR_INVALID_ARG
    assert L.lib().dllm_mixed_select_attn(p.ref, None, None, None, None, p.ref, None, None, None, None, None,
                                          None) == L.DLLM_ERR_INVALID_ARG
    # misaligned bf16 pointers
    base = q.data_ptr()
    assert L.lib().dllm_refresh_attn(p.ref, base + 2, base, base, base, None, None) == L.DLLM_ERR_SHAPE


def test_empty_batch_is_a_noop():
    p = L.Problem([], [], [], num_heads=4, num_kv_heads=4, head_dim=128, keep_ratio=0.5, block_table=None,
                  pages_per_req=0)
    assert p.layout() == ([], 0, 0, 0)
    for fn in (lambda: L.lib().dllm_refresh_attn(p.ref, None, None, None, None, None, None),
               lambda: L.lib().dllm_select_heads(p.ref, None, None, None),
               lambda: L.lib().dllm_reuse_sparse_attn(p.ref, None, None, None, None, None, None)):
        assert fn() == L.DLLM_OK


def test_binding_refuses_cpu_tensors():
    wl = synth.config("C0")
    p = _prob(wl)
    t = torch.zeros((64, 2, 16), dtype=torch.bfloat16)
    with pytest.raises(ValueError):
        L.refresh_attn(p, t, t, t, t)


def test_logit_chunks_abi_matches_oracle():
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "logit_examples.json")))
    for case in gold["chunk_plans"]:
        assert L.logit_chunks(case["n_logit"], case["max_num_logits"]) == case["plan"]
    rng = np.random.default_rng(5)
    for _ in range(100):
        n, m = int(rng.integers(0, 100000)), int(rng.integers(1, 5000))
        assert L.logit_chunks(n, m) == O.logit_chunks(n, m)
    assert L.lib().dllm_logit_chunks(-1, 5, None, 0) == -1
    assert L.lib().dllm_logit_chunks(10, 0, None, 0) == -1
    buf = (ctypes.c_int32 * 1)()
    assert L.lib().dllm_logit_chunks(10, 3, buf, 1) == -1      # 4 chunks do not fit


def test_lm_head_validation_without_gpu():
    so = L.lib()
    # workspace size: rows x ceil(V / 256) x 8
    assert L.lm_head_workspace_bytes(2048, 126464, 2048) == 2048 * 494 * 8
    assert L.lm_head_workspace_bytes(5000, 300, 2048) == 2048 * 2 * 8
    assert so.dllm_lm_head_workspace_bytes(-1, 10, 10) < 0
    fake = 1 << 20   # aligned non-null pointers: every call below must fail before any launch
    assert so.dllm_lm_head_argmax(fake, fake, 16, 100, 512, 16, fake, fake, 1 << 20, None) == -2   # d % 64
    assert so.dllm_lm_head_argmax(fake, fake, 16, 128, 0, 16, fake, fake, 1 << 20, None) == -1     # vocab
    assert so.dllm_lm_head_argmax(fake, fake, 16, 128, 512, 16, fake, fake, 8, None) == -1         # workspace
    assert so.dllm_lm_head_argmax(fake + 4, fake, 16, 128, 512, 16, fake, fake, 1 << 20, None) == -3  # alignment
    assert so.dllm_lm_head_argmax(None, fake, 16, 128, 512, 16, fake, fake, 1 << 20, None) == -1
    assert so.dllm_lm_head_argmax(None, None, 0, 128, 512, 16, None, None, 0, None) == 0            # empty: no-op
