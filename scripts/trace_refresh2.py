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
fused = len(sys.argv) > 2 and sys.argv[2] == "fused"
for _ in range(3):
    if fused:
        lib.refresh_select_attn(p, q, kc, vc, buf.out, buf.scores, buf.idx)
    else:
        lib.refresh_attn(p, q, kc, vc, buf.out, buf.scores)
torch.cuda.synchronize()
tr = np.zeros((34, 512), dtype=np.int64)
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
n_unit = (wl.seq_len[0] + 63) // 64
g = np.diff(tr[2, :N])
inner = [g[i] for i in range(len(g)) if (i + 1) % n_unit != 0]
bound = [g[i] for i in range(len(g)) if (i + 1) % n_unit == 0]
print(f"steps/unit {n_unit}: median inner period {np.median(inner):.0f}, median boundary gap {np.median(bound):.0f}, "
      f"boundary overhead per unit {np.median(bound) - np.median(inner):.0f} clk = "
      f"{(np.median(bound) - np.median(inner)) / (n_unit * np.median(inner)) * 100:.1f}% of a unit")
# unit boundary anatomy, relative to the last P of softmax WG0 in unit u-1 (clk)
for u_ in range(1, 7):
    e = u_ * n_unit - 1
    lastP = tr[4, e]
    r = lambda k, i: int(tr[k, i] - lastP)
    print(f"boundary {u_}: P1last {r(5, e)}; MMA gotP0 {r(7, e)} gotP1 {r(9, e)} unit-end {r(22, u_ - 1)} "
          f"decode {r(23, 2 * u_)}..{r(23, 2 * u_ + 1)} Qwait {r(16, u_)}..{r(17, u_)} K0 {r(18, u_)} K1 {r(19, u_)}; "
          f"Qprod QEMPTY wait {r(20, u_)}..{r(21, u_)}; sm0 waitS' {r(0, e + 1)} gotS' {r(2, e + 1)} P' {r(4, e + 1)} "
          f"gotS'1 {r(2, e + 2)}; sm1 gotS' {r(3, e + 1)}")
print("rows around the first boundary (absolute, minus t0):")
print("iter " + " ".join(f"{n:>8s}" for n in names))
for i in range(n_unit - 3, n_unit + 3):
    print(f"{i:4d} " + " ".join(f"{(tr[k, i] - t0):8d}" for k in range(14)))
print("MMA unit1 Qwait", tr[16, 1] - t0, tr[17, 1] - t0, "K0", tr[18, 1] - t0, "K1", tr[19, 1] - t0)
print("MMA end of unit0 (after last commit)", tr[22, 0] - t0, " unit1 decode start/end", tr[23, 2] - t0, tr[23, 3] - t0)

ct = np.zeros((1024, 4), dtype=np.int64)
lib.lib().dllm_trace2_cta(ct.ctypes.data_as(ctypes.c_void_p))
g = ct[:148]
start = g[:, 0] - g[:, 0].min(); dur = g[:, 1] - g[:, 0]
print(f"CTA start spread {start.max()/1e3:.1f} us; duration min/med/max {dur.min()/1e3:.1f}/{np.median(dur)/1e3:.1f}/{dur.max()/1e3:.1f} us; "
      f"kernel span {(g[:,1].max()-g[:,0].min())/1e3:.1f} us")
order = np.argsort(-dur)
print("slowest CTAs (cta, smid, us):", [(int(c), int(g[c, 3]), round(dur[c] / 1e3, 1)) for c in order[:12]])
print("fastest CTAs:", [(int(c), int(g[c, 3]), round(dur[c] / 1e3, 1)) for c in order[-6:]])
hist = np.histogram(dur / 1e3, bins=10)
print("hist", [int(x) for x in hist[0]], [round(float(x), 0) for x in hist[1]])

print("producer per step around the first two boundaries (abs - t0): K wait start, K got, V wait start, V got")
for i in list(range(n_unit - 5, n_unit + 3)) + list(range(2 * n_unit - 3, 2 * n_unit + 2)):
    print(f"{i:4d} " + " ".join(f"{(tr[k, i] - t0):8d}" for k in (24, 25, 26, 27)))
# softmax WG0 phase breakdown (clk): got S -> LDTM done -> max done -> exps done -> STTM waited -> P arrived
N = 200
ph = [tr[28, :N] - tr[2, :N], tr[29, :N] - tr[28, :N], tr[30, :N] - tr[29, :N], tr[31, :N] - tr[30, :N], tr[4, :N] - tr[31, :N]]
print("softmax0 phases median (ld, importance+mask+max, rescale-check+exp, st+wait, fence+arrive):",
      [float(np.median(x)) for x in ph])
nsel = int((tr[33] > 0).sum())
if nsel:
    print("fused selects in CTA 0:", nsel, "durations (clk):", [int(x) for x in (tr[33, :nsel] - tr[32, :nsel])],
          "start (clk from t0):", [int(x) for x in (tr[32, :nsel] - t0)])
