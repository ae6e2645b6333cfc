"""fp64 CPU oracle for the Head-Centric Sparse Attention hot path.

TEST INFRASTRUCTURE ONLY: import it from ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s cpu_baseline / ``--impl reference`` legs, nowhere else.
It shares no code with ``paper_2512_17077_b200`` and never calls into it.
"""
from .hcsa import *  # noqa: F401,F403
from .logits import argmax_lowest, argmax_rows, chunked_decode, logit_chunks, logits  # noqa: F401
