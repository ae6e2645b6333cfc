"""Request-level data parallelism over 1/2/4/8 GPUs.

Requests are independent (Refresh, select and Reuse touch only their own
request's Q/K/V), so a batch is partitioned across ranks with no collective
on the data path.  The partition is LPT-greedy on an estimated per-request
cost (Refresh FLOPs at the tensor peak + Reuse bytes at HBM bandwidth).
NCCL is used only to all-gather the per-request outputs afterwards
(`allgather_outputs`), mirroring the north_star's "all-gather per-request
outputs"; the gather is timed separately from the compute.
"""
from __future__ import annotations

import heapq
import math
from typing import List, Sequence

import torch


def request_cost(L: int, blk: int, H: int, H_kv: int, D: int, k: int, refresh: bool = True, reuse: bool = True,
                 tflops: float = 1642.7, gbs: float = 6468.9) -> float:
    """Estimated seconds of one request on one GPU (roofline estimate): Refresh
    FLOPs at the tensor peak and/or Reuse bytes at HBM bandwidth."""
    t = 0.0
    if refresh:
        t += 4.0 * H * L * L * D / (tflops * 1e12)
    if reuse:
        t += (H * (blk + k) * 2 * D * 2 + 2 * H * blk * D * 2) / (gbs * 1e9)
    return t


def workload_costs(wl, k_per_request: Sequence[int]) -> List[float]:
    """Per-request cost estimates of one step of ``wl``: without a refresh_mask every
    request runs Refresh + select + Reuse; with one (a mixed burst batch, DESIGN.md
    R20) a Refresh request runs Refresh + select and a Reuse request Reuse only."""
    mask = wl.refresh_mask
    return [request_cost(L, e - s, wl.num_heads, wl.num_kv_heads, wl.head_dim, k,
                         refresh=True if mask is None else bool(mask[i]),
                         reuse=True if mask is None else not mask[i])
            for i, (L, s, e, k) in enumerate(zip(wl.seq_len, wl.blk_start, wl.blk_end, k_per_request))]


def lpt_partition(costs: Sequence[float], n: int) -> List[List[int]]:
    """Longest-processing-time-first greedy: each request (largest first) goes to
    the currently least-loaded rank.  Deterministic (ties: lower rank, lower id)."""
    order = sorted(range(len(costs)), key=lambda i: (-costs[i], i))
    heap = [(0.0, r) for r in range(n)]
    parts: List[List[int]] = [[] for _ in range(n)]
    for i in order:
        load, r = heapq.heappop(heap)
        parts[r].append(i)
        heapq.heappush(heap, (load + costs[i], r))
    return [sorted(p) for p in parts]


def makespan(costs: Sequence[float], parts: List[List[int]]) -> float:
    return max((sum(costs[i] for i in p) for p in parts), default=0.0)


def allgather_outputs(local: torch.Tensor, counts: Sequence[int], group=None) -> torch.Tensor:
    """All-gather variable-size per-rank outputs (rows along dim 0) to every rank.

    counts[r] = rows held by rank r.  Uses a padded all_gather_into_tensor (one
    NCCL collective) and strips the padding; returns [sum(counts), ...] in rank
    order."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    assert len(counts) == world
    rows = max(counts) if counts else 0
    pad = torch.zeros((rows,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[:local.shape[0]] = local
    gathered = torch.empty((world * rows,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(gathered, pad, group=group)
    return torch.cat([gathered[r * rows:r * rows + counts[r]] for r in range(world)])


def efficiency(costs: Sequence[float], n: int) -> float:
    parts = lpt_partition(costs, n)
    ms = makespan(costs, parts)
    return (sum(costs) / n) / ms if ms > 0 else 1.0


def reassemble(gathered: torch.Tensor, parts: List[List[int]], sizes: Sequence[int]) -> List[torch.Tensor]:
    """Per-request outputs in GLOBAL request order from an all-gathered tensor.

    Rank r contributed its requests ``parts[r]`` (ascending) back to back along dim
    0, request i taking ``sizes[i]`` rows (0 for requests without this output);
    ``gathered`` is the rank-order concatenation (``allgather_outputs``)."""
    out: List[torch.Tensor] = [None] * len(sizes)   # type: ignore[list-item]
    off = 0
    for p in parts:
        for i in p:
            out[i] = gathered[off:off + sizes[i]]
            off += sizes[i]
    assert off == gathered.shape[0], (off, gathered.shape)
    return out
