"""GPU parity for the logit-decomposition row (N4): dllm_lm_head_argmax vs the
fp64 oracle (oracle/logits.py).

* exact-integer inputs: every logit is an exact fp32 integer, so the ids must
  equal the oracle's bit-exactly, ties included (lowest index);
* realistic inputs: the GPU id must be a valid ArgMax within the fp32
  accumulation error bound eps_row = d * 2^-23 * max_v sum_k |h_k w_vk|
  (fp32 vs fp64 decide the argmax differently only inside that band);
* the full LLaDA-8B shape (2,048 x 4,096 x 126,464) on sampled rows."""
import numpy as np
import pytest
import torch

import oracle as O
from paper_2512_17077_b200 import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def L():
    from paper_2512_17077_b200 import lib
    return lib


def _run(L, h, w, max_num_logits):
    ids = torch.full((h.shape[0],), -7, dtype=torch.int32, device="cuda")
    L.lm_head_argmax(h.cuda(), w.cuda(), ids, max_num_logits=max_num_logits)
    torch.cuda.synchronize()
    return ids.cpu().numpy()


@pytest.mark.parametrize("n_tok,d,vocab,mnl", [
    (1, 64, 1, 2048), (1, 64, 256, 2048), (77, 64, 255, 2048), (128, 128, 1000, 2048),
    (300, 256, 4099, 100), (300, 256, 4099, 64), (513, 64, 300, 512), (1000, 128, 7000, 333)])
def test_exact_inputs_bit_exact(L, n_tok, d, vocab, mnl):
    h, w = synth.lm_head_inputs(n_tok, d, vocab, "exact")
    got = _run(L, h, w, mnl)
    want = O.chunked_decode(h.float().numpy(), w.float().numpy(), mnl)
    assert np.array_equal(got, want)


def _check_valid(h, w, got, rows=None):
    hf, wf = h.double().numpy(), w.double().numpy()
    rows = np.arange(hf.shape[0]) if rows is None else np.asarray(rows)
    z = hf[rows] @ wf.T
    absz = np.abs(hf[rows]) @ np.abs(wf).T
    eps = hf.shape[1] * 2.0 ** -23 * absz.max(axis=1)
    best = z.max(axis=1)
    g = got[rows] if got.shape[0] != rows.shape[0] else got
    assert np.all((g >= 0) & (g < wf.shape[0]))
    zg = z[np.arange(rows.shape[0]), g]
    assert np.all(zg >= best - 2 * eps), (best - zg).max()
    return int(np.sum(g != O.argmax_lowest(z)))


@pytest.mark.parametrize("n_tok,d,vocab,mnl", [(300, 512, 5000, 2048), (257, 1024, 3001, 128)])
def test_realistic_inputs_valid_argmax(L, n_tok, d, vocab, mnl):
    h, w = synth.lm_head_inputs(n_tok, d, vocab, "realistic")
    got = _run(L, h, w, mnl)
    flips = _check_valid(h, w, got)
    assert flips <= max(1, n_tok // 100)   # near-ties inside the fp32 band only


def test_full_shape_sampled_rows(L):
    f = synth.LM_HEAD_FULL
    h, w = synth.lm_head_inputs(f["n_tok"], f["d_model"], f["vocab"], "realistic")
    got = _run(L, h, w, f["max_num_logits"])
    assert np.all((got >= 0) & (got < f["vocab"]))
    rows = [0, 1, 127, 128, 1000, 2047]
    flips = _check_valid(h, w, got[rows], rows)
    assert flips <= 1


def test_full_shape_exact_chunked(L):
    # exact arithmetic at the full vocabulary with chunking (3 chunks), sampled rows
    n, d, v = 1100, 4096, 126464
    h, w = synth.lm_head_inputs(n, d, v, "exact")
    got = _run(L, h, w, 512)
    rows = [0, 511, 512, 1023, 1024, 1099]
    want = O.argmax_rows(h.float().numpy(), w.float().numpy(), rows)
    assert np.array_equal(got[rows], want)


def test_deterministic(L):
    h, w = synth.lm_head_inputs(200, 256, 3000, "realistic")
    a, b = _run(L, h, w, 2048), _run(L, h, w, 64)
    assert np.array_equal(a, b)
