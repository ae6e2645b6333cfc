"""Dev: phase timestamps of the select kernel (trace build), CTAs 0-7."""
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
lib.refresh_attn(p, q, kc, vc, buf.out, buf.scores)
for _ in range(3):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    lib.select_heads(p, buf.scores, buf.idx)
    e.record()
    torch.cuda.synchronize()
print("event us", s.elapsed_time(e) * 1e3)
tr = np.zeros((8, 10), dtype=np.int64)
lib.lib().dllm_trace_sel_read(tr.ctypes.data_as(ctypes.c_void_p))
names = ["wait", "find", "stage", "pool", "pass1", "pass2", "pass3", "pass4", "compact"]
for c in range(8):
    print(c, " ".join(f"{n}={int(tr[c, i + 1] - tr[c, i])}" for i, n in enumerate(names)), "total", int(tr[c, 9] - tr[c, 0]))
