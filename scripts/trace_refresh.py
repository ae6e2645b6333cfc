"""Dev: timeline of CTA 0 of the tcgen05 refresh kernel (trace build)."""
import ctypes, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["DLLM_LIB"] = os.environ.get("DLLM_LIB") or os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                      "paper_2512_17077_b200", "libdllm_trace.so")
import torch
from paper_2512_17077_b200 import lib, synth
cfg = sys.argv[1] if len(sys.argv) > 1 else "C1"
wl = synth.config(cfg)
b = synth.make_batch(wl)
p = lib.Problem(wl.seq_len, wl.blk_start, wl.blk_end, num_heads=wl.num_heads, num_kv_heads=wl.num_kv_heads,
                head_dim=wl.head_dim, keep_ratio=wl.keep_ratio, pool_window=wl.pool_window, page_size=wl.page_size,
                block_table=b.block_table.cuda())
q, kc, vc = b.q.cuda(), b.k_cache.cuda(), b.v_cache.cuda()
buf = lib.alloc_buffers(p)
for _ in range(3):
    lib.refresh_attn(p, q, kc, vc, buf.out, buf.scores)
torch.cuda.synchronize()
tr = np.zeros((16, 512), dtype=np.int64)
lib.lib().dllm_trace_read(tr.ctypes.data_as(ctypes.c_void_p))
t0 = tr[0, 0]
names = ["sm0_wait", "sm1_wait", "sm0_gotS", "sm1_gotS", "sm0_P", "sm1_P", "mma_waitP0", "mma_gotP0",
         "mma_waitP1", "mma_gotP1", "mma_waitV", "mma_gotKV"]
print("iter " + " ".join(f"{n:>10s}" for n in names))
for i in range(40):
    print(f"{i:4d} " + " ".join(f"{(tr[k, i] - t0):10d}" for k in range(12)))
d = lambda a, c: np.diff(tr[a, :64])
print("softmax0 S->P (clk):", np.median(tr[4, :64] - tr[2, :64]), " wait for S:", np.median(tr[2, :64] - tr[0, :64]))
print("softmax1 S->P (clk):", np.median(tr[5, :64] - tr[3, :64]), " wait for S:", np.median(tr[3, :64] - tr[1, :64]))
print("mma wait P0:", np.median(tr[7, :64] - tr[6, :64]), " wait P1:", np.median(tr[9, :64] - tr[8, :64]),
      " wait V/K:", np.median(tr[11, :64] - tr[10, :64]))
print("period softmax0:", np.median(np.diff(tr[2, :64])))
print("softmax0 phases: ld", np.median(tr[12, :64] - tr[2, :64]), " turn-wait", np.median(tr[13, :64] - tr[12, :64]),
      " exp pass", np.median(tr[14, :64] - tr[13, :64]), " check+store+wait", np.median(tr[15, :64] - tr[14, :64]),
      " arrive", np.median(tr[4, :64] - tr[15, :64]))
