"""Dev: per-CTA / per-chunk timeline of the group-set Reuse kernel (reuse_grp.cu;
trace build: DLLM_TRACE_BUILD=1 python -c 'from paper_2512_17077_b200 import build; build.build()')."""
import ctypes, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["DLLM_LIB"] = os.environ.get("DLLM_LIB") or os.path.join(ROOT, "paper_2512_17077_b200", "libdllm_trace.so")
import torch
from paper_2512_17077_b200 import lib, synth
cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
n = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2] != "all" else None
wl = synth.config(cfg, num_requests=n)
b = synth.make_batch(wl)
p = lib.Problem(wl.seq_len, wl.blk_start, wl.blk_end, num_heads=wl.num_heads, num_kv_heads=wl.num_kv_heads,
                head_dim=wl.head_dim, keep_ratio=wl.keep_ratio, pool_window=wl.pool_window, page_size=wl.page_size,
                block_table=b.block_table.cuda())
q, qb, kc, vc = b.q.cuda(), b.q_blk.cuda(), b.k_cache.cuda(), b.v_cache.cuda()
buf = lib.alloc_buffers(p)
lib.refresh_attn(p, q, kc, vc, buf.out, buf.scores)
union = len(sys.argv) > 3 and sys.argv[3] == "union"   # per-head sets through the union kernel
(lib.select_heads if union else lib.select_groups)(p, buf.scores, buf.idx)
run = (lambda: lib.reuse_sparse_attn(p, qb, kc, vc, buf.idx, buf.out_blk)) if union else \
    (lambda: lib.reuse_group_sets(p, qb, kc, vc, buf.idx, buf.out_blk))
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for _ in range(3):
    flush.zero_()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    run()
    e.record()
    torch.cuda.synchronize()
print("event time us", s.elapsed_time(e) * 1e3)
tr = np.zeros((1024, 16), dtype=np.int64)
ch = np.zeros((16, 64), dtype=np.int64)
assert lib.lib().dllm_trace_rgs_read(tr.ctypes.data_as(ctypes.c_void_p), ch.ctypes.data_as(ctypes.c_void_p)) == 0
n = int((tr[:, 0] > 0).sum())
tr = tr[:n]
t0 = tr[:, 0].min()
rel = lambda x: (x - t0) / 1e3  # noqa: E731
print(f"CTAs {n}; start spread {rel(tr[:,0].max()):.2f} us; end min/med/max "
      f"{rel(tr[:,11].min()):.2f}/{np.median(rel(tr[:,11])):.2f}/{rel(tr[:,11].max()):.2f} us")
print(f"first offs published (median) {np.median(rel(tr[:,1]) - rel(tr[:,0])):.2f} us after CTA start; "
      f"first S issued {np.median(rel(tr[:,2]) - rel(tr[:,0])):.2f} us")
for u in range(8):
    col = tr[:, 3 + u]
    m = col > 0
    if not m.any():
        break
    prev = tr[:, 2] if u == 0 else tr[:, 2 + u]
    print(f"unit {u}: CTAs {m.sum()}, end median {np.median(rel(col[m])):.2f} us, "
          f"duration median {np.median((col[m] - prev[m]) / 1e3):.2f} us")
c0 = tr[0, 0]
print("CTA 0 chunks (us from CTA start): published, loader issued, S issued, softmax got S, head 0 done, "
      "P arrived, PV issued")
for t in range(min(24, int((ch[2] > 0).sum()))):
    print(f"  ch{t:3d} " + " ".join(f"{(ch[k, t] - c0) / 1e3:7.2f}" for k in (0, 1, 2, 3, 6, 4, 5)))
print("translator: union built (per unit), lookups done (per batch, first chunk index)")
print("  units " + " ".join(f"{(ch[12, u] - c0) / 1e3:7.2f}" for u in range(6) if ch[12, u] > 0))
print("  batches " + " ".join(f"{t}:{(ch[13, t] - c0) / 1e3:.2f}" for t in range(64) if ch[13, t] > 0))
print("unit: softmax row sums published, epilogue got O + sums, epilogue stored")
for u in range(6):
    if ch[9, u] > 0:
        print(f"{u:3d} " + " ".join(f"{(ch[k, u] - c0) / 1e3:7.2f}" for k in (9, 10, 11)))
