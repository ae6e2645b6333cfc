"""Dev: timeline of CTA 0 of the double-buffered tcgen05 refresh kernel (trace build)."""
import ctypes, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["DLLM_LIB"] = os.environ.get("DLLM_LIB") or os.path.join(ROOT, "paper_2512_17077_b200", "libdllm_trace.so")
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
lib.lib().dllm_trace2_read(tr.ctypes.data_as(ctypes.c_void_p))
t0 = tr[0, 0]
names = ["s0wait", "s1wait", "s0gotS", "s1gotS", "s0P", "s1P", "mWaitP0", "mGotP0", "mWaitP1", "mGotP1",
         "mWaitV", "mGotV", "mWaitK", "mGotK"]
print("iter " + " ".join(f"{n:>8s}" for n in names))
for i in list(range(0, 20)) + list(range(60, 72)):
    print(f"{i:4d} " + " ".join(f"{(tr[k, i] - t0):8d}" for k in range(14)))
N = 200
print("softmax0 S->P:", np.median(tr[4, :N] - tr[2, :N]), " wait S:", np.median(tr[2, :N] - tr[0, :N]))
print("softmax1 S->P:", np.median(tr[5, :N] - tr[3, :N]), " wait S:", np.median(tr[3, :N] - tr[1, :N]))
print("mma waitP0", np.median(tr[7, :N] - tr[6, :N]), "waitP1", np.median(tr[9, :N] - tr[8, :N]),
      "waitV", np.median(tr[11, :N] - tr[10, :N]), "waitK", np.median(tr[13, :N] - tr[12, :N]))
print("period (sm0 gotS):", np.median(np.diff(tr[2, :N])))
