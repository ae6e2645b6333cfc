"""Request-level sharding: LPT partition and the output
all-gather layout, exercised with world-size-2 gloo on CPU."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2512_17077_b200 import shard, synth


def test_lpt_partition_properties():
    costs = [5.0, 3.0, 3.0, 2.0, 2.0, 2.0, 1.0]
    for n in (1, 2, 3, 4, 8):
        parts = shard.lpt_partition(costs, n)
        assert sorted(i for p in parts for i in p) == list(range(len(costs)))
        ms = shard.makespan(costs, parts)
        assert ms >= max(costs) and ms >= sum(costs) / n - 1e-12
        # LPT bound: makespan <= (4/3 - 1/(3n)) * OPT <= (4/3 - 1/(3n)) * max(lower bounds)...
        assert ms <= (4 / 3) * max(max(costs), sum(costs) / n) + 1e-9
    assert shard.lpt_partition(costs, 2) == shard.lpt_partition(costs, 2)   # deterministic


def test_lpt_on_burst_config_is_balanced():
    wl = synth.config("C3")
    costs = [shard.request_cost(L, e - s, 32, 32, 128, max(1, int(0.25 * (L - (e - s)))), refresh=bool(m))
             for L, s, e, m in zip(wl.seq_len, wl.blk_start, wl.blk_end, wl.refresh_mask)]
    # requests are indivisible: the bound is set by the largest Refresh request
    lb = max(max(costs), sum(costs) / 8)
    assert shard.makespan(costs, shard.lpt_partition(costs, 8)) <= (4 / 3) * lb
    assert shard.efficiency(costs, 2) >= 0.95


def test_weak_scaling_shards_replicate_c1():
    base = synth.config("C1")
    glob = synth.replicate(base, 4)
    costs = [1.0] * glob.num_requests
    parts = shard.lpt_partition(costs, 4)
    assert all(len(p) == base.num_requests for p in parts)
    sub = synth.subset(glob, list(range(base.num_requests)))
    a = synth.request_tensors(base, 5)[0]
    b = synth.request_tensors(sub, 5)[0]
    assert torch.equal(a, b)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, counts, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        local = torch.full((counts[rank], 3), float(rank + 1))
        local[:, 1] = torch.arange(counts[rank], dtype=torch.float32)
        got = shard.allgather_outputs(local, counts)
        q.put((rank, got))
    finally:
        dist.destroy_process_group()


def test_allgather_layout_gloo_world2():
    counts = [3, 5]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, counts, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    expect = torch.cat([torch.stack([torch.full((c,), float(r + 1)), torch.arange(c, dtype=torch.float32),
                                     torch.full((c,), float(r + 1))], 1) for r, c in enumerate(counts)])
    for r in range(2):
        assert torch.equal(res[r], expect)
