"""GPU: the dynamic unit scheduler of the tcgen05 Refresh kernel (device claim
counters in the caller's workspace, dllm_problem.workspace).
Which CTA computes which work unit must not change any result: repeated
launches (the counters self-reset), launches of two problems (two workspaces)
on two streams in flight at once, CUDA-graph replays and the static schedule
without a workspace are all bit-identical to one reference launch, and every
launch leaves the workspace zeroed."""
import pytest
import torch

from paper_2512_17077_b200 import synth
from tests._util import problem_of, to_dev

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def L():
    assert torch.cuda.is_available(), "GPU tests need a B200"
    from paper_2512_17077_b200 import lib
    return lib


def _setup(L, cfg, n):
    batch = synth.make_batch(synth.config(cfg, num_requests=n))
    p = problem_of(batch)
    q, q_blk, kc, vc = to_dev(batch)
    return p, q, q_blk, kc, vc


def _run(L, p, q, q_blk, kc, vc, stream=None):
    buf = L.alloc_buffers(p)
    L.refresh_attn(p, q, kc, vc, buf.out, buf.scores, stream)
    L.select_heads(p, buf.scores, buf.idx, stream)
    L.reuse_sparse_attn(p, q_blk, kc, vc, buf.idx, buf.out_blk, stream)
    return buf


def _same(a, b):
    assert torch.equal(a.out.view(torch.int16), b.out.view(torch.int16))
    assert torch.equal(a.scores.view(torch.int32), b.scores.view(torch.int32))
    assert torch.equal(a.idx, b.idx)
    assert torch.equal(a.out_blk.view(torch.int16), b.out_blk.view(torch.int16))


def test_repeated_launches_reset_the_counters(L):
    args = _setup(L, "C3", 12)
    ref = _run(L, *args)
    torch.cuda.synchronize()
    for _ in range(20):
        got = _run(L, *args)
    torch.cuda.synchronize()
    _same(ref, got)
    assert int(args[0].workspace.count_nonzero()) == 0, "the launches must leave the workspace zeroed"


def test_static_schedule_without_workspace(L):
    p, q, q_blk, kc, vc = _setup(L, "C2", 4)
    ref = _run(L, p, q, q_blk, kc, vc)
    wl = synth.config("C2", num_requests=4)
    p0 = L.Problem(wl.seq_len, wl.blk_start, wl.blk_end, num_heads=wl.num_heads, num_kv_heads=wl.num_kv_heads,
                   head_dim=wl.head_dim, keep_ratio=wl.keep_ratio, pool_window=wl.pool_window,
                   page_size=wl.page_size, block_table=p.block_table, workspace=None)
    got = _run(L, p0, q, q_blk, kc, vc)
    torch.cuda.synchronize()
    _same(ref, got)


def test_workspace_validation(L):
    p, q, q_blk, kc, vc = _setup(L, "C0", None)
    wl = synth.config("C0")
    small = torch.zeros(L.workspace_bytes() - 16, dtype=torch.uint8, device="cuda")
    with pytest.raises(L.DllmError):
        bad = L.Problem(wl.seq_len, wl.blk_start, wl.blk_end, num_heads=wl.num_heads, num_kv_heads=wl.num_kv_heads,
                        head_dim=wl.head_dim, keep_ratio=wl.keep_ratio, pool_window=wl.pool_window,
                        page_size=wl.page_size, block_table=p.block_table, workspace=small)
        _run(L, bad, q, q_blk, kc, vc)


def test_two_streams_in_flight(L):
    a1 = _setup(L, "C1", 6)
    a2 = _setup(L, "C2", 4)
    r1, r2 = _run(L, *a1), _run(L, *a2)
    torch.cuda.synchronize()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    outs = []
    for _ in range(4):
        outs.append((_run(L, *a1, stream=s1), _run(L, *a2, stream=s2)))
    torch.cuda.synchronize()
    for g1, g2 in outs:
        _same(r1, g1)
        _same(r2, g2)


def test_graph_replay(L):
    p, q, q_blk, kc, vc = _setup(L, "C1", 4)
    ref = _run(L, p, q, q_blk, kc, vc)
    buf = L.alloc_buffers(p)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        L.refresh_attn(p, q, kc, vc, buf.out, buf.scores, s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        L.refresh_attn(p, q, kc, vc, buf.out, buf.scores, s)
        L.select_heads(p, buf.scores, buf.idx, s)
        L.reuse_sparse_attn(p, q_blk, kc, vc, buf.idx, buf.out_blk, s)
    for _ in range(5):
        buf.out.zero_()
        buf.out_blk.zero_()
        g.replay()
        torch.cuda.synchronize()
        _same(ref, buf)
