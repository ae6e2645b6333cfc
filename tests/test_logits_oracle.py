"""Pins for the logit-decomposition oracle (N4): SPEC worked examples, brute
force, and the chunked == monolithic invariant."""
import json
import os

import numpy as np
import pytest

import oracle as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "logit_examples.json")))


@pytest.mark.parametrize("case", GOLD["chunk_plans"], ids=lambda c: c["cite"][:14])
def test_chunk_plan_spec_examples(case):
    assert O.logit_chunks(case["n_logit"], case["max_num_logits"]) == case["plan"]


@pytest.mark.parametrize("case", GOLD["decodes"], ids=lambda c: c["cite"][:14])
def test_decode_spec_examples(case):
    z = np.asarray(case["logits"], dtype=np.float64)
    # logits given directly: hidden = the logit rows, weight = identity (V = d)
    ids = O.chunked_decode(z, np.eye(z.shape[1]), case["max_num_logits"])
    assert ids.tolist() == case["ids"]


def test_chunk_plan_properties():
    rng = np.random.default_rng(1)
    for _ in range(200):
        n, m = int(rng.integers(0, 10000)), int(rng.integers(1, 3000))
        plan = O.logit_chunks(n, m)
        assert sum(plan) == n and all(0 < c <= m for c in plan)
        assert all(c == m for c in plan[:-1])
    with pytest.raises(ValueError):
        O.logit_chunks(5, 0)


def test_argmax_lowest_brute_force():
    rng = np.random.default_rng(2)
    z = rng.integers(-3, 4, size=(200, 37)).astype(np.float64)   # many ties
    ids = O.argmax_lowest(z)
    for i in range(z.shape[0]):
        best = max(z[i])
        assert ids[i] == min(j for j in range(z.shape[1]) if z[i, j] == best)


def test_logits_brute_force():
    rng = np.random.default_rng(3)
    h, w = rng.normal(size=(5, 7)), rng.normal(size=(11, 7))
    z = O.logits(h, w)
    for i in range(5):
        for v in range(11):
            assert abs(z[i, v] - sum(h[i, k] * w[v, k] for k in range(7))) < 1e-12


def test_chunked_equals_monolithic():
    rng = np.random.default_rng(4)
    h = rng.integers(-2, 3, size=(301, 16)).astype(np.float64)
    w = rng.integers(-2, 3, size=(97, 16)).astype(np.float64)
    mono = O.argmax_lowest(O.logits(h, w))
    for m in (1, 7, 64, 300, 301, 5000):
        assert np.array_equal(O.chunked_decode(h, w, m), mono)
    assert np.array_equal(O.argmax_rows(h, w, [0, 5, 300]), mono[[0, 5, 300]])
