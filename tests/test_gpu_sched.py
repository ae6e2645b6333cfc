"""GPU: the dynamic unit schedulers of the tcgen05 Refresh and Reuse kernels
(device claim counters in 64 self-resetting per-launch slots).
Which CTA computes which work unit must not change any result: repeated
launches (wrapping the slots), launches on two streams in flight at once and
CUDA-graph replays are all bit-identical to one reference launch."""
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


def test_repeated_launches_wrap_the_counter_slots(L):
    args = _setup(L, "C3", 12)
    ref = _run(L, *args)
    torch.cuda.synchronize()
    for _ in range(70):          # > 64 slots: every slot reused after its reset
        got = _run(L, *args)
    torch.cuda.synchronize()
    _same(ref, got)


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
