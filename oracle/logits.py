"""fp64 CPU oracle for dLLM-Serve's Logit Decomposition (next row N4).

TEST INFRASTRUCTURE ONLY (same rules as ``oracle/hcsa.py``): only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs may import it; it shares
no code with ``paper_2512_17077_b200``.

The paper (§4.3 "Logit Decomposition"; §5)
splits the LM-head projection along the token axis into chunks of at most
``max_num_logits`` tokens, "computes the logits, immediately applies the
decoding operator (e.g., ArgMax ...)" per chunk and frees the chunk's logits
before the next.  SPEC.md:145-165 states the two operations:
``plan_logit_chunks`` and ``chunked_decode`` (ArgMax, ties toward the lower
index, result identical to the monolithic ArgMax over the full [N, V] logits).
"""
from __future__ import annotations

from typing import List

import numpy as np


def logit_chunks(n_logit: int, max_num_logits: int) -> List[int]:
    """plan_logit_chunks ("If N_logit >
    max_num_logits, the runtime decomposes the output projection into serial
    sub-batches"): greedy full chunks of max_num_logits, then one remainder."""
    if n_logit < 0 or max_num_logits < 1:
        raise ValueError("n_logit >= 0 and max_num_logits >= 1 required")
    out, left = [], n_logit
    while left > 0:
        c = min(left, max_num_logits)
        out.append(c)
        left -= c
    return out


def logits(hidden, weight) -> np.ndarray:
    """Z = H W^T, the output projection (Z in R^{B x L x V}),
    in float64 from the given (bf16-representable) inputs.  hidden [N, d],
    weight [V, d] (the LM-head weight, one row per vocabulary entry)."""
    return np.asarray(hidden, dtype=np.float64) @ np.asarray(weight, dtype=np.float64).T


def argmax_lowest(z) -> np.ndarray:
    """ArgMax per row with ties toward the LOWER index.
    numpy's argmax returns the first occurrence of the maximum, which is that
    rule; kept as its own function so tests can pin it against brute force."""
    z = np.asarray(z)
    if z.shape[0] == 0:
        return np.zeros((0,), np.int64)
    return np.argmax(z, axis=1).astype(np.int64)


def chunked_decode(hidden, weight, max_num_logits: int) -> np.ndarray:
    """chunked_decode with ArgMax: for each
    planned chunk compute its logits, decode them, drop them, concatenate the
    ids in plan order.  Returns the ids and never holds more than one chunk of
    logits."""
    h = np.asarray(hidden, dtype=np.float64)
    ids, r0 = [], 0
    for c in logit_chunks(h.shape[0], max_num_logits):
        z = logits(h[r0:r0 + c], weight)
        ids.append(argmax_lowest(z))
        del z
        r0 += c
    return np.concatenate(ids) if ids else np.zeros((0,), np.int64)


def argmax_rows(hidden, weight, rows) -> np.ndarray:
    """Monolithic ArgMax of the selected rows only (sampled checks at full size)."""
    h = np.asarray(hidden, dtype=np.float64)[np.asarray(rows)]
    return argmax_lowest(logits(h, weight))
