// Refresh dense attention on the 5th-generation tensor cores (sm_100a), with
// double-buffered score tiles: Eq. 3 (§2.3) + the raw
// per-head importance of Eq. 6 (inner term, §4.5).
//
// Why double buffering: when P_i(j) overwrites S_i(j) in TMEM (the P-aliases-S
// trick), Q_i K_{j+1}^T cannot start before P_i(j) has been consumed, so every
// softmax pass sits on the critical path of its own tile:
//   period = softmax + (P.V + Q.K^T) + latencies.
// Here K/V advance in 64-key steps and each 128-row Q tile owns TWO 64-column
// score buffers (TMEM: S_i[0], S_i[1], O_i; 2 tiles x 256 columns = 512), so
// Q_i K_{j+1}^T runs while the softmax works on S_i(j) and the softmax warps
// go from one step to the next without waiting for the tensor core.
//
// Persistent, warp-specialised, one CTA per SM (384 threads):
//   warp 8      TMA producer: Q tiles (3-D map over [sum L, H, D]) and 64-key
//               K/V tiles straight out of the paged cache (4-D map over
//               [pages, H_kv, P, D]) into 4-stage K and V rings (128-B swizzle).
//   warp 10     Q-tile producer (TMA);
//   warp 9      MMA issuer (one thread) + TMEM owner:
//               S_i(j) = Q_i K_j^T   (tcgen05.mma SS, M=128 N=64),
//               O_i   += P_i(j) V_j  (tcgen05.mma TS, P from TMEM, M=128 N=D).
//   warps 0-3   softmax warpgroup 0 (Q tile 0), one thread per query row;
//   warps 4-7   softmax warpgroup 1 (Q tile 1): tcgen05.ld of S, online
//               softmax in fp32 (log2 domain, lazy rescale: O is rescaled in
//               TMEM only when the running max grows by more than 2^8, after
//               waiting for the previous P.V), bf16 P back into the S buffer,
//               final O / l and store.
// Work unit = (request b, query head h, pair of 128-row Q tiles); the
// importance epilogue and the extra "score tile" for blocks that straddle a
// tile boundary are as in refresh_tc.cu.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdint.h>

#include <atomic>

#include "common.cuh"
#include "plan.h"
#include "tc_ptx.cuh"
#include "reuse_tc_body.cuh"
#include "workspace.h"

#ifdef DLLM_TRACE
__device__ long long g_trace2[34][512];
#define TRACE2(kind, it)                                                   \
  do {                                                                     \
    if (blockIdx.x == 0 && (it) < 512) g_trace2[kind][it] = clock64();     \
  } while (0)
__device__ long long g_cta2[1024][4];
extern "C" __attribute__((visibility("default"))) int dllm_trace2_read(long long *host) {
  return (int)cudaMemcpyFromSymbol(host, g_trace2, sizeof(g_trace2));
}
extern "C" __attribute__((visibility("default"))) int dllm_trace2_cta(long long *host) {
  return (int)cudaMemcpyFromSymbol(host, g_cta2, sizeof(g_cta2));
}
__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#else
#define TRACE2(kind, it)
#endif

namespace dllm {
namespace {

constexpr int TBM = 128;            // query rows per tile
constexpr int TBN = 64;             // keys per step
constexpr int NST = 4;              // K and V ring stages (3 measured 7% slower at C1, r01_ab_tc2_nst.log)
constexpr int THREADS = 512;
constexpr float kRescaleLog2 = 8.f; // lazy-rescale threshold (log2 units)
// of every kPolyPeriod exponential pairs of the softmax, kPolyPairs run as a
// degree-3 polynomial on the FMA pipe instead of MUFU ex2 (16/clk/SM, the same
// rate at which the tensor cores consume S elements at D = 128).  Swept in round 1
// (r01_ab_tc2_poly_sweep.log): 0 / 1 / 2 / 3 / 4 of 8 -> C1 972 / 1,002 / 973 /
// 987 / 935 TFLOP/s; 1 of 4 / 16, 3 of 16 and per-warpgroup shares all slower.
constexpr int kPolyPairs = 1;
constexpr int kPolyPeriod = 8;
// Dynamic unit scheduling: after its first (static) unit, a CTA claims the next
// work unit from a device counter (in the caller's workspace) when its K/V
// producer needs it and publishes the id to the other roles through a
// shared-memory ring, so CTAs that run faster (fewer importance-epilogue units,
// less contended SMs) take more units.
constexpr bool kDynSched = true;
// register split (setmaxnreg): 8 softmax warps, 4 epilogue warps, 4 others at 64;
// 2 * softmax + epilogue <= 448 for 64K registers per SM (136/176 vs 144/160 vs
// 152/144 measured neutral, r01_ab_tc2_regsplit.log)
#define DLLM_TC2_REG_SOFTMAX 136
#define DLLM_TC2_REG_EPI 176
static_assert(2 * DLLM_TC2_REG_SOFTMAX + DLLM_TC2_REG_EPI <= 448, "register budget");
// Measured in round 1 and removed: L2 prefetch of the next unit's K/V and Q
// (slower), next-unit decode mid-unit, one barrier pair per K/V stage, an MMA warp
// serving the two Q tiles in P-ready order (4-5% slower), a request cursor in
// decode_unit (0.5-1% slower), other warp-role placements (neutral).  Round 2: softmax
// warpgroup 1 held until warpgroup 0 finished each step's row max (to put the two
// exponential phases out of phase on the shared MUFU): C1 280 vs 272, C2 1,658 vs
// 1,584 us (profiles/r02_ab_tc2_skew.log).
#ifndef DLLM_TC2_FUSEDSEL
// 1: pool + TopK fused into the epilogue warpgroup (dllm_refresh_select_attn).  Off by
// default: measured ~13 us per (b, h) selection at C1 (~25k clk, issue-starved beside
// the softmax warps, and its unrolled code bloats the kernel ~2x), which made the
// fused call 16% slower than Refresh + the select launch at C1 (1% faster at C2).
#define DLLM_TC2_FUSEDSEL 0
#endif

template <int D>
struct Cfg {
  static constexpr int kChunks = D / 64;                 // 128-byte swizzle chunks per row
  static constexpr int kQBytes = TBM * D * 2;
  static constexpr int kKVBytes = TBN * D * 2;
  static constexpr int kOffQ = 0;                        // 2 Q tiles
  static constexpr int kOffK = 2 * kQBytes;              // NST K stages
  static constexpr int kOffV = kOffK + NST * kKVBytes;   // NST V stages
  static constexpr int kOffSc = kOffV + NST * kKVBytes;  // [2 wg][2 buf][4 warps][64] f32
  static constexpr int kOffBar = kOffSc + 2 * 2 * 4 * TBN * 4;
  static constexpr int kOffStage = kOffBar + 1024;       // [4 epilogue warps][32 rows][64 B] staging (SW64)
  static constexpr int kOffL = kOffStage + 4 * 32 * 64;  // [2 parity][2 tiles][128] f32 row sums
  static constexpr int kOffUnits = kOffL + 2 * 2 * 128 * 4;  // [kUnitRing][128 B] decoded units (K/V producer -> roles)
  static constexpr int kOffReq = kOffUnits + 4 * 128;
  // + nreq * sizeof(ReqInfo) + 1024 alignment slack, sized per launch
  static int bytes(int nreq) { return kOffReq + nreq * (int)sizeof(ReqInfo) + 1024; }
};

// barrier slots (8 bytes each)
enum : int {
  B_QFULL = 0, B_QEMPTY = 1,
  B_KFULL = 2, B_KEMPTY = B_KFULL + NST, B_VFULL = B_KEMPTY + NST, B_VEMPTY = B_VFULL + NST,
  B_VZ = B_VEMPTY + NST,
  B_SFULL = B_VZ + 1,          // [tile][buf]
  B_PFULL = B_SFULL + 4,       // [tile][buf]
  B_ODONE = B_PFULL + 4,       // [tile][buf]: P.V of that buffer completed
  B_OFULL = B_ODONE + 4,       // [tile]: last P.V of the unit completed
  B_OFREE = B_OFULL + 2,       // [tile]: epilogue has read O out of TMEM
  B_LFULL = B_OFREE + 2,       // [tile]: softmax row sums of the unit in smem
  B_TMEMSLOT = B_LFULL + 2,
  B_RFULL = B_TMEMSLOT + 1,    // [kRing]: unit id published by the K/V producer (dynamic scheduler)
  B_REMPTY = B_RFULL + 4       // [kRing]: read by every other role (kRingReaders arrivals)
};
constexpr int kRing = 4;
constexpr int kRingReaders = 1 /* Q producer */ + 1 /* MMA warp */ + 8 /* softmax warps */ + 4 /* epilogue warps */;
constexpr int kRingOff = 768;  // byte offset of the int ring[kRing] inside the barrier area
__host__ __device__ constexpr uint32_t tmem_s(int tile, int buf) { return (uint32_t)(tile * 128 + buf * 64); }
__host__ __device__ constexpr uint32_t tmem_o(int tile) { return tile ? 384u : 256u; }

__host__ __device__ __forceinline__ int regular_tiles(int L) { return (L + TBM - 1) / TBM; }
__host__ __device__ __forceinline__ bool straddles(int bs, int be) { return (bs / TBM) != ((be - 1) / TBM); }

struct Unit {
  int h, kvh;
  int L, bs, be;
  int q_off, bt_row;
  int64_t score_off;
  int n;          // 64-key steps
  int tile1;      // 1 if the second Q tile exists
  int origin0, origin1;
  int wend0, wend1;
  int sc0, sc1;   // importance epilogue on tile 0 / 1
  int k;          // k_b (fused select)
  int64_t idx_off;
};

// Work unit -> request (binary search over the request table in shared memory),
// head, Q-tile pair and importance-epilogue flags.  Called once per unit by the
// K/V producer only; the other roles receive the decoded Unit through shared memory.
__device__ __forceinline__ void decode_unit(const Plan &pl, const ReqInfo *rs, int unit, Unit &u) {
  // Unit order (the order in which the CTAs claim them).  With the importance
  // epilogue, the H * nreq pairs that carry it (the pair holding the active block's
  // tile, one per (request, head); their softmax warpgroup also reduces the block
  // rows' column maxima every step) come FIRST, the plain pairs after them: the
  // longest units are dealt first, so the last units of the launch -- which set
  // the tail of the dynamically scheduled grid -- are the short ones (LPT).
  int b, h, p;
  const ReqInfo *R;
  int nreg, ntiles, npairs;
  bool extra;
  auto shape = [&](const ReqInfo &r) {
    nreg = regular_tiles(r.L);
    extra = pl.with_scores && straddles(r.bs, r.be);
    ntiles = nreg + (extra ? 1 : 0);
    npairs = (ntiles + 1) >> 1;
  };
  if (pl.with_scores) {
    const int n_imp = pl.nreq * pl.H;
    if (unit < n_imp) {
      b = unit / pl.H;
      h = unit - b * pl.H;
      R = &rs[b];
      shape(*R);
      p = (extra ? nreg : R->bs / TBM) >> 1;
    } else {
      // plain pairs: request b owns [unit_off(b) - b H, unit_off(b + 1) - (b + 1) H)
      const int v = unit - n_imp;
      int lo = 0, hi = pl.nreq - 1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (rs[mid].unit_off - mid * pl.H <= v) lo = mid; else hi = mid - 1;
      }
      b = lo;
      R = &rs[b];
      shape(*R);
      const int np1 = npairs - 1;
      const int local = v - (R->unit_off - b * pl.H);
      h = local / np1;
      const int q = local - h * np1;
      const int p_imp = (extra ? nreg : R->bs / TBM) >> 1;
      p = q < p_imp ? q : q + 1;
    }
  } else {
    int lo = 0, hi = pl.nreq - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (rs[mid].unit_off <= unit) lo = mid; else hi = mid - 1;
    }
    b = lo;
    R = &rs[b];
    shape(*R);
    const int local = unit - R->unit_off;
    h = local / npairs;
    p = local - h * npairs;
  }
  u.L = R->L; u.bs = R->bs; u.be = R->be;
  u.q_off = R->q_off; u.bt_row = R->bt_row; u.score_off = R->score_off;
  u.k = R->k; u.idx_off = R->idx_off;
  u.h = h;
  u.kvh = h / (pl.H / pl.H_kv);
  u.n = (u.L + TBN - 1) / TBN;
  const int t0 = 2 * p, t1 = 2 * p + 1;
  u.tile1 = t1 < ntiles;
  u.origin0 = t0 < nreg ? t0 * TBM : u.bs;
  u.origin1 = t1 < nreg ? t1 * TBM : u.bs;
  u.wend0 = t0 < nreg ? u.L : 0;
  u.wend1 = t1 < nreg ? u.L : 0;
  u.sc0 = pl.with_scores && (t0 == nreg || (!extra && t0 == u.bs / TBM));
  u.sc1 = pl.with_scores && u.tile1 && (t1 == nreg || (!extra && t1 == u.bs / TBM));
}

// ---------------------------------------------------------------- fused select
// Pool + per-head TopK (Eq. 6 + TopK, §4.5) of ONE (request,
// head) by the 128 epilogue-warpgroup threads, right after the unit whose softmax
// warps wrote that head's raw scores (select fused into the
// Refresh epilogue).  The same definition and the same integer decisions as
// select_heads_kernel (select.cu; R2-R9): candidates C = [0,bs) ++
// [be,L), window of half-width w/2 clipped to the compacted axis, order-preserving
// 32-bit keys (-0 == +0), an exact 4-pass 8-bit MSB radix select of the k-th key,
// every key above it plus the lowest-index keys equal to it, written as ascending
// sequence positions.  Thread t owns the contiguous candidates [t P, t P + P),
// P = ceil(n/128) <= kFSelPer, held in registers, so the ascending output slots
// come from one block scan of per-thread counts.
constexpr int kFSelThreads = 128;
constexpr int kFSelPer = 32;                            // n_ctx <= 4096 (host-checked)
constexpr int kFSelMaxN = kFSelThreads * kFSelPer;
constexpr int kFSelBar = 5;                             // named barrier of the epilogue warpgroup
constexpr int kFSelHalfMax = 4;                         // windows w <= 9 pool from registers

__device__ __forceinline__ uint32_t fsel_key(float f) {
  const uint32_t u = __float_as_uint(f);
  if ((u & 0x7fffffffu) == 0u) return 0x80000000u;       // +-0 -> one key
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// raw: the head's L raw scores (written by this CTA in this kernel: plain loads,
// not the read-only path); scratch: >= 256 + 8 + 2 words of shared memory
__device__ __forceinline__ void fused_select(const float *raw, const int L, const int bs, const int be, const int half,
                                          const int k, int32_t *__restrict__ out, int *scratch, const int t) {
  int *hist = scratch;                                   // [256]
  int *wbuf = scratch + 256;                             // [4]
  int *sh = scratch + 264;                               // [2]: prefix, krem
  const int blk = be - bs, n = L - blk;
  const int P = (n + kFSelThreads - 1) / kFSelThreads;
  const int c0 = t * P;
  const int nv = max(0, min(P, n - c0));
  uint32_t key[kFSelPer];
  if (half <= kFSelHalfMax) {
    // the thread's P candidates and the half-windows around them: all loads in
    // flight together (one L2 round trip), -inf outside [0, n) == clipping
    float rv[kFSelPer + 2 * kFSelHalfMax];
#pragma unroll
    for (int i = 0; i < kFSelPer + 2 * kFSelHalfMax; ++i) {
      const int c = c0 - half + i;
      rv[i] = (i < P + 2 * half && c >= 0 && c < n) ? raw[c < bs ? c : c + blk] : -INFINITY;
    }
#pragma unroll
    for (int i = 0; i < kFSelPer; ++i) {
      float m = rv[i];
#pragma unroll
      for (int d = 1; d <= 2 * kFSelHalfMax; ++d)
        if (d <= 2 * half) m = fmaxf(m, rv[i + d]);
      key[i] = i < nv ? fsel_key(m) : 0u;
    }
  } else {
#pragma unroll
    for (int i = 0; i < kFSelPer; ++i) {
      uint32_t kk = 0u;
      if (i < nv) {
        const int c = c0 + i;
        const int lo = max(0, c - half), hi = min(n - 1, c + half);
        float m = -INFINITY;
        for (int j = lo; j <= hi; ++j) m = fmaxf(m, raw[j < bs ? j : j + blk]);
        kk = fsel_key(m);
      }
      key[i] = kk;
    }
  }
  uint32_t prefix = 0u, mask = 0u;
  int krem = k;
#pragma unroll 1
  for (int shift = 24; shift >= 0; shift -= 8) {
    for (int i = t; i < 256; i += kFSelThreads) hist[i] = 0;
    ptx::named_bar_sync(kFSelBar, kFSelThreads);
    // warp-aggregated: the keys crowd a few bins (similar exponents), so lanes with
    // equal bins are merged (match.any) into one shared atomic; P is CTA-uniform
#pragma unroll
    for (int i = 0; i < kFSelPer; ++i) {
      if (i >= P) break;
      const bool act = i < nv && (key[i] & mask) == prefix;
      const uint32_t bin = act ? ((key[i] >> shift) & 0xffu) : 0x100u;
      const uint32_t peers = __match_any_sync(0xffffffffu, bin);
      if (act && (t & 31) == __ffs(peers) - 1) atomicAdd(&hist[bin], __popc(peers));
    }
    ptx::named_bar_sync(kFSelBar, kFSelThreads);
    if (t < 32) {
      // lane l owns bins [8 (31 - l), 8 (31 - l) + 8): lane 0 the top bins
      const int base = 8 * (31 - t);
      int cnt[8], sum = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) { cnt[i] = hist[base + 7 - i]; sum += cnt[i]; }
      int incl = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (t >= o) incl += y;
      }
      const int above = incl - sum;
      if (above < krem && krem <= incl) {
        int acc = above;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          if (acc + cnt[i] >= krem) {
            sh[0] = (int)(prefix | ((uint32_t)(base + 7 - i) << shift));
            sh[1] = krem - acc;
            break;
          }
          acc += cnt[i];
        }
      }
    }
    ptx::named_bar_sync(kFSelBar, kFSelThreads);
    prefix = (uint32_t)sh[0];
    krem = sh[1];
    mask |= 0xffu << shift;
  }
  // compaction: slot of a selected candidate = #above before it + min(#equal before it, krem)
  int gt = 0, eq = 0;
#pragma unroll
  for (int i = 0; i < kFSelPer; ++i)
    if (i < nv) { gt += key[i] > prefix; eq += key[i] == prefix; }
  const int v = gt | (eq << 16);
  const int lane = t & 31, w = t >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wbuf[w] = x;
  ptx::named_bar_sync(kFSelBar, kFSelThreads);
  int basew = 0;
  for (int i = 0; i < w; ++i) basew += wbuf[i];
  const int pre = basew + x - v;
  int gt_pre = pre & 0xffff, eq_pre = pre >> 16;
#pragma unroll
  for (int i = 0; i < kFSelPer; ++i) {
    if (i < nv) {
      const int c = c0 + i;
      const int pos = c < bs ? c : c + blk;
      if (key[i] > prefix) {
        out[gt_pre + min(eq_pre, krem)] = pos;
        ++gt_pre;
      } else if (key[i] == prefix) {
        if (eq_pre < krem) out[gt_pre + eq_pre] = pos;
        ++eq_pre;
      }
    }
  }
  ptx::named_bar_sync(kFSelBar, kFSelThreads);        // scratch free again
}

// The kernel body, shared by refresh_tc2_kernel and the single-launch mixed
// Refresh/Reuse kernel below: CTA `cta` of `ncta` CTAs working on this plan.  The
// tensor maps are references to __grid_constant__ kernel parameters.
template <int D>
__device__ __forceinline__ void refresh_tc2_body(const Plan &plan, const CUtensorMap &tm_q, const CUtensorMap &tm_k,
                                                 const CUtensorMap &tm_v, const CUtensorMap &tm_o,
                                                 __nv_bfloat16 *__restrict__ out, float *__restrict__ scores,
                                                 int32_t *__restrict__ sel_idx, const int cta, const int ncta) {
  using C = Cfg<D>;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_u32 = smem_u32(smem_raw);
  const uint32_t sb = (raw_u32 + 1023u) & ~1023u;
  uint8_t *gb = smem_raw + (sb - raw_u32);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  auto bar = [&](int i) { return sb + C::kOffBar + 8u * (uint32_t)i; };
  // head dim of the tensors in global memory: D = 16 and 32 run on the 64-dim layout --
  // their tensor maps keep 64-column boxes over a Dg-column tensor, so the TMA fills
  // columns Dg..63 of every row with zeros (out-of-bounds fill) and Q.K^T, P.V are exact
  const int Dg = D == 128 ? 128 : plan.D;

#ifdef DLLM_TRACE
  if (threadIdx.x == 0 && blockIdx.x < 1024) { g_cta2[blockIdx.x][0] = gtimer(); g_cta2[blockIdx.x][2] = 0; }
#endif
  ReqInfo *rs = reinterpret_cast<ReqInfo *>(gb + C::kOffReq);
  for (int i = threadIdx.x; i < plan.nreq; i += blockDim.x) rs[i] = plan.r[i];
  if (threadIdx.x == 0) {
    ptx::mbar_init(bar(B_QFULL), 1);
    ptx::mbar_init(bar(B_QEMPTY), 1);
    for (int s = 0; s < NST; ++s) {
      ptx::mbar_init(bar(B_KFULL + s), 1);
      ptx::mbar_init(bar(B_KEMPTY + s), 1);
      ptx::mbar_init(bar(B_VFULL + s), 1);
      ptx::mbar_init(bar(B_VEMPTY + s), 1);
    }
    for (int i = 0; i < 4; ++i) {
      ptx::mbar_init(bar(B_SFULL + i), 1);
      ptx::mbar_init(bar(B_PFULL + i), 4);
      ptx::mbar_init(bar(B_ODONE + i), 1);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(bar(B_OFULL + i), 1);
      ptx::mbar_init(bar(B_OFREE + i), 4);
      ptx::mbar_init(bar(B_LFULL + i), 4);
    }
    for (int i = 0; i < kRing; ++i) {
      ptx::mbar_init(bar(B_RFULL + i), 1);
      ptx::mbar_init(bar(B_REMPTY + i), kRingReaders);
    }
    ptx::mbar_init(bar(B_VZ), 1);
    ptx::fence_mbar_init();
    ptx::tma_prefetch_desc(&tm_q);
    ptx::tma_prefetch_desc(&tm_k);
    ptx::tma_prefetch_desc(&tm_v);
  }
  // roles: warps 0-7 softmax (two aligned warpgroups, TMEM lane quarter = warp % 4),
  // warp 8 TMA producer, warp 9 MMA issuer.  The warp scheduler favours the highest
  // warp id among eligible warps of a sub-partition, so the producer and the MMA
  // issuer are placed above the softmax warps sharing their sub-partitions.
  constexpr int kProducerWarp = 8, kMmaWarp = 9, kQWarp = 10, kEpi0 = 12;
  if (warp == kMmaWarp) {
    ptx::tmem_alloc(bar(B_TMEMSLOT), 512);
    ptx::tmem_relinquish();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  // everything above (barriers, TMEM, tensor-map prefetch) is independent of the
  // preceding kernel's results: with programmatic dependent launch it overlaps that
  // kernel's tail; no role touches global memory (inputs, the scheduler counters)
  // before this wait
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t *>(gb + C::kOffBar + 8 * B_TMEMSLOT);
  // the device counter lives in the caller's workspace (dllm_problem.workspace):
  // without one the units go round-robin
  const bool dyn = kDynSched && plan.sched != nullptr;
  volatile int *ring = reinterpret_cast<volatile int *>(gb + C::kOffBar + kRingOff);
  Unit *uring = reinterpret_cast<Unit *>(gb + C::kOffUnits);
  // i-th unit of this CTA as seen by a reader role: the K/V producer claims it
  // (statically: cta + i * ncta; dynamically: from the device counter), decodes it
  // once and publishes id + decoded Unit through a kRing-slot shared-memory ring, so
  // the unit-boundary critical paths of the other roles carry no decode (measured
  // ~1,150 clk per decode_unit in every role, scripts/trace_refresh2.py).  A whole
  // warp reads the slot and lane 0 releases it after __syncwarp; a single-thread
  // role (the Q producer) reads and releases it alone.
  auto unit_at = [&](int i, bool whole_warp, Unit &u) -> int {
    const int slot = i % kRing;
    ptx::mbar_wait(bar(B_RFULL + slot), (i / kRing) & 1);
    const int un = ring[slot];
    if (un < plan.total_units) u = uring[slot];
    if (whole_warp) __syncwarp();
    if (!whole_warp || lane == 0) ptx::mbar_arrive(bar(B_REMPTY + slot));
    return un;
  };

  if (warp == kProducerWarp) {
    // ============================ TMA producer ============================
    asm volatile("setmaxnreg.dec.sync.aligned.u32 64;\n" ::: "memory");
    int it = 0, ucnt = 0;
    const int boxrows = plan.page_size < TBN ? plan.page_size : TBN;
    const int nsub = TBN / boxrows;
    const uint32_t boxbytes = (uint32_t)boxrows * 128u;
    auto claim = [&]() {
      const int c = ncta + atomicAdd(plan.sched, 1);
      return c < plan.total_units ? c : plan.total_units;
    };
    for (int i = 0;; ++i, ++ucnt) {
      // this role needs the next unit first: claim it, decode it, publish it
      int unit = 0;
      if (lane == 0) {
        unit = i == 0 ? cta : (dyn ? claim() : cta + i * ncta);
        unit = unit < plan.total_units ? unit : plan.total_units;
      }
      unit = __shfl_sync(0xffffffffu, unit, 0);
      Unit u;
      if (unit < plan.total_units) decode_unit(plan, rs, unit, u);
      if (lane == 0) {
        if (i > 0 && unit < plan.total_units) {
          // the unit's Q tiles go to L2 now, ~NST steps before the Q producer can load
          // them (after the current unit's last Q.K^T): the MMA warp's cross-unit
          // lookahead needs them ~1 step after that, and an HBM-cold 64 KB Q load took
          // ~2,900 clk there (trace)
          for (int t = 0; t < (u.tile1 ? 2 : 1); ++t)
            for (int c = 0; c < C::kChunks; ++c)
              ptx::tma_prefetch_3d(&tm_q, c * 64, u.h, u.q_off + (t ? u.origin1 : u.origin0));
        }
        const int slot = i % kRing;
        ptx::mbar_wait(bar(B_REMPTY + slot), ((i / kRing) & 1) ^ 1);
        ring[slot] = unit;
        if (unit < plan.total_units) uring[slot] = u;
        ptx::mbar_arrive(bar(B_RFULL + slot));
      }
      if (unit >= plan.total_units) break;
      const int32_t *bt = plan.block_table + (int64_t)u.bt_row * plan.pages_per_req;
      for (int j = 0; j < u.n; ++j, ++it) {
        const int s = it % NST;
        const uint32_t ph = (it / NST) & 1;
        const int key_end = min(TBN, u.L - j * TBN);      // valid keys in this step
        if (lane == 0) {
          int nvalid = 0;
          for (int sbx = 0; sbx < nsub; ++sbx) nvalid += (sbx * boxrows < key_end);
          const uint32_t bytes = (uint32_t)(nvalid * C::kChunks) * boxbytes;
          TRACE2(24, it);
          ptx::mbar_wait(bar(B_KEMPTY + s), ph ^ 1);
          TRACE2(25, it);
          ptx::mbar_arrive_expect_tx(bar(B_KFULL + s), bytes);
          for (int sbx = 0; sbx < nvalid; ++sbx) {
            const int key0 = j * TBN + sbx * boxrows;
            const int page = __ldg(bt + (key0 >> plan.page_shift));
            const int slot = key0 & (plan.page_size - 1);
            for (int c = 0; c < C::kChunks; ++c)
              ptx::tma_load_4d(sb + C::kOffK + s * C::kKVBytes + c * TBN * 128 + sbx * boxrows * 128, &tm_k,
                               bar(B_KFULL + s), c * 64, slot, u.kvh, page);
          }
          TRACE2(26, it);
          ptx::mbar_wait(bar(B_VEMPTY + s), ph ^ 1);
          TRACE2(27, it);
          ptx::mbar_arrive_expect_tx(bar(B_VFULL + s), bytes);
          for (int sbx = 0; sbx < nvalid; ++sbx) {
            const int key0 = j * TBN + sbx * boxrows;
            const int page = __ldg(bt + (key0 >> plan.page_shift));
            const int slot = key0 & (plan.page_size - 1);
            for (int c = 0; c < C::kChunks; ++c)
              ptx::tma_load_4d(sb + C::kOffV + s * C::kKVBytes + c * TBN * 128 + sbx * boxrows * 128, &tm_v,
                               bar(B_VFULL + s), c * 64, slot, u.kvh, page);
          }
        }
        __syncwarp();
        if (key_end < TBN) {
          // zero V rows >= key_end (P is 0 there, but 0 * NaN would poison O)
          ptx::mbar_wait(bar(B_VFULL + s), ph);
          uint8_t *vbase = gb + C::kOffV + s * C::kKVBytes;
          const int nrow = TBN - key_end;
          for (int e = lane; e < nrow * 8 * C::kChunks; e += 32) {
            const int c = e / (nrow * 8);
            const int rem = e - c * nrow * 8;
            const int r = key_end + rem / 8;
            *reinterpret_cast<uint4 *>(vbase + c * TBN * 128 + r * 128 + (rem & 7) * 16) = make_uint4(0, 0, 0, 0);
          }
          ptx::fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(bar(B_VZ));
        }
      }
    }
  } else if (warp == kQWarp) {
    // ============================ Q producer ============================
    asm volatile("setmaxnreg.dec.sync.aligned.u32 64;\n" ::: "memory");
    // (separate from the K/V producer so that the next unit's first K/V steps are
    // not queued behind the wait for the Q buffers to drain)
    if (lane == 0) {
      int ucnt = 0;
      for (int i = 0;; ++i, ++ucnt) {
        Unit u;
        const int unit = unit_at(i, false, u);
        if (unit >= plan.total_units) break;
        TRACE2(20, ucnt);
        ptx::mbar_wait(bar(B_QEMPTY), (ucnt & 1) ^ 1);
        TRACE2(21, ucnt);
        const int ntile = u.tile1 ? 2 : 1;
        ptx::mbar_arrive_expect_tx(bar(B_QFULL), (uint32_t)(ntile * C::kQBytes));
        for (int i = 0; i < ntile; ++i)
          for (int c = 0; c < C::kChunks; ++c)
            ptx::tma_load_3d(sb + C::kOffQ + i * C::kQBytes + c * TBM * 128, &tm_q, bar(B_QFULL), c * 64, u.h,
                             u.q_off + (i ? u.origin1 : u.origin0));
      }
    }
    __syncwarp();
  } else if (warp == kMmaWarp) {
    // ============================ MMA issuer ============================
    asm volatile("setmaxnreg.dec.sync.aligned.u32 64;\n" ::: "memory");
    // The whole warp runs this loop (warp-uniform control flow and descriptors,
    // kept in uniform registers); one elected lane issues each tcgen05 op.
    {
      constexpr uint32_t idesc_qk = ptx::idesc_bf16_f32(TBM, TBN, false, false);
      constexpr uint32_t idesc_pv = ptx::idesc_bf16_f32(TBM, D, false, true);
      const uint64_t dq = ptx::smem_desc_sw128(sb + C::kOffQ, 16, 1024);
      const uint64_t dk = ptx::smem_desc_sw128(sb + C::kOffK, 16, 1024);
      const uint64_t dv = ptx::smem_desc_sw128(sb + C::kOffV, TBN * 128, 1024);
      int it = 0, ucnt = 0, vzc = 0;
      int gs[2] = {0, 0};        // S tiles issued per Q tile (buffer = gs & 1)
      int gp[2] = {0, 0};        // P.V issued per Q tile
      int ou[2] = {0, 0};        // units per Q tile (O accumulator reuse)
      auto qk = [&](int i, int stage) {
        const int b = gs[i] & 1;
        const uint64_t a0 = dq + (uint64_t)((i * C::kQBytes) >> 4);
        const uint64_t b0 = dk + (uint64_t)((stage * C::kKVBytes) >> 4);
#pragma unroll
        for (int k = 0; k < D / 16; ++k) {
          const uint32_t ko = (uint32_t)(((k >> 2) * TBM * 128 + (k & 3) * 32) >> 4);
          const uint32_t kb = (uint32_t)(((k >> 2) * TBN * 128 + (k & 3) * 32) >> 4);
          ptx::mma_ss_elect(tmem + tmem_s(i, b), a0 + ko, b0 + kb, idesc_qk, k > 0);
        }
        ptx::mma_commit_elect(bar(B_SFULL + 2 * i + b));
        ++gs[i];
      };
      auto pv = [&](int i, int stage, bool acc, bool last) {
        const int b = gp[i] & 1;
        const uint64_t v0 = dv + (uint64_t)((stage * C::kKVBytes) >> 4);
#pragma unroll
        for (int k = 0; k < TBN / 16; ++k)
          ptx::mma_ts_elect(tmem + tmem_o(i), tmem + tmem_s(i, b) + (uint32_t)(k * 8), v0 + (uint64_t)((k * 16 * 128) >> 4),
                            idesc_pv, (acc || k > 0) ? 1u : 0u);
        ptx::mma_commit_elect(bar(B_ODONE + 2 * i + b));
        if (last) ptx::mma_commit_elect(bar(B_OFULL + i));
        ++gp[i];
      };
      // One continuous stream of 64-key steps over the CTA's units: at P.V step g the
      // MMA warp issues S(g + 2), also when step g + 2 belongs to the NEXT unit (its Q
      // tiles permitting: the Q buffer is refilled after the current unit's last Q.K^T,
      // checked without blocking).  Without this cross-unit lookahead every unit
      // boundary cost ~2,600-3,000 clk of softmax idle time (S'(0) issued only after the
      // last P.V of the previous unit): 8-11% of a C1 unit (scripts/trace_refresh2.py).
      Unit cu, nu;
      if (lane == 0) TRACE2(23, 0);
      int cur_id = unit_at(0, true, cu);
      int q_issued = 0;          // Q.K^T steps of cu already issued by the previous unit's lookahead
      bool q_ready = false;      // QFULL of cu acquired
      while (cur_id < plan.total_units) {
        const int nt = cu.tile1 ? 2 : 1;
        if (!q_ready) {
          if (lane == 0) TRACE2(16, ucnt);
          ptx::mbar_wait(bar(B_QFULL), ucnt & 1);
          if (lane == 0) TRACE2(17, ucnt);
        }
        ptx::tc_fence_after();
        // prologue: S(0) and S(1) of every tile, unless the lookahead issued them
        const int npro = cu.n < 2 ? cu.n : 2;
        for (int jj = q_issued; jj < npro; ++jj) {
          const int st = (it + jj) % NST;
          ptx::mbar_wait(bar(B_KFULL + st), ((it + jj) / NST) & 1);
          if (lane == 0) TRACE2(18 + jj, ucnt);
          ptx::tc_fence_after();
          for (int i = 0; i < nt; ++i) qk(i, st);
          ptx::mma_commit_elect(bar(B_KEMPTY + st));
          if (jj == cu.n - 1) ptx::mma_commit_elect(bar(B_QEMPTY));
        }
        int nxt_id = -1;         // next unit, read from the ring when the lookahead reaches it
        int nq = 0;              // Q.K^T steps of nu issued below
        bool nq_ready = false;
        for (int j = 0; j < cu.n; ++j) {
          const int sv = (it + j) % NST;
          if (lane == 0) TRACE2(10, it + j);
          ptx::mbar_wait(bar(B_VFULL + sv), ((it + j) / NST) & 1);
          if (lane == 0) TRACE2(11, it + j);
          if (j == cu.n - 1 && (cu.L % TBN) != 0) {
            ptx::mbar_wait(bar(B_VZ), vzc & 1);
            ++vzc;
          }
          // the lookahead Q.K^T of this step: global step it + j + 2
          int tg_nt = 0, tg_last = 0;
          bool tg_next = false;
          if (j + 2 < cu.n) {
            tg_nt = nt;
            tg_last = j + 2 == cu.n - 1;
          } else {
            if (nxt_id < 0) {
              if (lane == 0) TRACE2(23, 2 * ucnt + 1);
              nxt_id = unit_at(ucnt + 1, true, nu);
            }
            if (nxt_id < plan.total_units && nq < nu.n && nq <= j + 2 - cu.n) {
              if (!nq_ready) nq_ready = ptx::mbar_test_wait(bar(B_QFULL), (ucnt + 1) & 1);
              if (nq_ready) {
                tg_next = true;
                tg_nt = nu.tile1 ? 2 : 1;
                tg_last = nq == nu.n - 1;
              }
            }
          }
          const int gk = it + (tg_next ? cu.n + nq : j + 2);
          const int sk = gk % NST;
          for (int i = 0; i < 2; ++i) {
            if (i < nt) {
              const int b = gp[i] & 1;
              if (lane == 0) TRACE2(6 + 2 * i, gp[i]);
              ptx::mbar_wait(bar(B_PFULL + 2 * i + b), (gp[i] >> 1) & 1);
              if (lane == 0) TRACE2(7 + 2 * i, gp[i]);
              if (j == 0) {
                // the epilogue warpgroup must have read the previous unit's O_i
                ptx::mbar_wait(bar(B_OFREE + i), (ou[i] & 1) ^ 1);
                ++ou[i];
              }
              ptx::tc_fence_after();
              pv(i, sv, j > 0, j == cu.n - 1);
            }
            if (i < tg_nt) {
              if (i == 0) {
                if (lane == 0) TRACE2(12, it + j);
                ptx::mbar_wait(bar(B_KFULL + sk), (gk / NST) & 1);
                if (lane == 0) TRACE2(13, it + j);
                ptx::tc_fence_after();
              }
              qk(i, sk);
            }
          }
          if (tg_nt > 0) {
            ptx::mma_commit_elect(bar(B_KEMPTY + sk));
            if (tg_last) ptx::mma_commit_elect(bar(B_QEMPTY));
            if (tg_next) ++nq;
          }
          ptx::mma_commit_elect(bar(B_VEMPTY + sv));
          if (lane == 0 && j == cu.n - 1) TRACE2(22, ucnt);
        }
        it += cu.n;
        if (nxt_id < 0) nxt_id = unit_at(ucnt + 1, true, nu);
        cu = nu;
        cur_id = nxt_id;
        ++ucnt;
        q_issued = nq;
        q_ready = nq_ready;
      }
    }
    __syncwarp();
  } else if (warp < 8) {
    // ============================ softmax warpgroups ============================
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(DLLM_TC2_REG_SOFTMAX) : "memory");
    const int wg = warp >> 2;
    const int wq = warp & 3;                       // TMEM lane quarter
    const int row = wq * 32 + lane;                // row of the Q tile == TMEM lane
    const uint32_t lane_off = (uint32_t)(wq * 32) << 16;
    const uint32_t tO = tmem + lane_off + tmem_o(wg);
    float *sbuf = reinterpret_cast<float *>(gb + C::kOffSc) + wg * (2 * 4 * TBN);
    const float sl2 = plan.scale_log2;
    int sc = 0, oc = 0;
    for (int i = 0;; ++i) {
      Unit u;
      const int unit = unit_at(i, true, u);
      if (unit >= plan.total_units) break;
      if (wg == 1 && !u.tile1) continue;
      const int origin = wg ? u.origin1 : u.origin0;
      const bool sc_on = (wg ? u.sc1 : u.sc0) && scores != nullptr;
      const int rb0 = u.bs - origin, rb1 = u.be - origin;    // block rows within the tile
      const bool in_blk = sc_on && row >= rb0 && row < rb1;
      const bool warp_blk = sc_on && (wq * 32 < rb1) && (wq * 32 + 32 > rb0);
      float m_used = -INFINITY, lsum = 0.f;
      for (int j = 0; j < u.n; ++j, ++sc) {
        const int b = sc & 1;
        const uint32_t tS = tmem + lane_off + tmem_s(wg, b);
        if ((threadIdx.x & 127) == 0) TRACE2(0 + wg, sc);
        ptx::mbar_wait(bar(B_SFULL + 2 * wg + b), (sc >> 1) & 1);
        if ((threadIdx.x & 127) == 0) TRACE2(2 + wg, sc);
        ptx::tc_fence_after();
        uint32_t sr[64];
        DLLM_TMEM_LD32(tS + 0, (sr + 0));
        DLLM_TMEM_LD32(tS + 32, (sr + 32));
        ptx::tmem_wait_ld();
        if (threadIdx.x == 0) TRACE2(28, sc);
        float *s = reinterpret_cast<float *>(sr);
        if (sc_on) {
          // importance: column max of the UNSCALED S over the block rows
          float *buf = sbuf + (j & 1) * (4 * TBN);
          if (warp_blk) {
#pragma unroll
            for (int c = 0; c < 2; ++c) {
              float v[32];
#pragma unroll
              for (int i = 0; i < 32; ++i) v[i] = in_blk ? s[c * 32 + i] : -INFINITY;
#pragma unroll
              for (int o = 16; o >= 1; o >>= 1) {
                const bool up = (lane & o) != 0;
#pragma unroll
                for (int i = 0; i < o; ++i) {
                  const float send = up ? v[i] : v[i + o];
                  const float keep = up ? v[i + o] : v[i];
                  v[i] = fmaxf(keep, __shfl_xor_sync(0xffffffffu, send, o));
                }
              }
              buf[wq * TBN + c * 32 + lane] = v[0];
            }
          }
          ptx::named_bar_sync(1 + wg, 128);
          if (row < TBN) {
            float m = -INFINITY;
#pragma unroll
            for (int w2 = 0; w2 < 4; ++w2)
              if ((w2 * 32 < rb1) && (w2 * 32 + 32 > rb0)) m = fmaxf(m, buf[w2 * TBN + row]);
            const int key = j * TBN + row;
            if (key < u.L) scores[u.score_off + (int64_t)u.h * u.L + key] = m;
          }
        }
        if (j == u.n - 1) {
          const int key_end = u.L - j * TBN;
          if (key_end < TBN) {
#pragma unroll
            for (int c = 0; c < TBN; ++c)
              if (c >= key_end) s[c] = -INFINITY;
          }
        }
        float mx;
        {
          float t[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) t[i] = fmax3(s[i], s[8 + i], s[16 + i]);
#pragma unroll
          for (int i = 0; i < 8; ++i) t[i] = fmax3(t[i], s[24 + i], s[32 + i]);
#pragma unroll
          for (int i = 0; i < 8; ++i) t[i] = fmax3(t[i], s[40 + i], s[48 + i]);
#pragma unroll
          for (int i = 0; i < 8; ++i) t[i] = fmaxf(t[i], s[56 + i]);
          mx = fmax3(fmax3(t[0], t[1], t[2]), fmax3(t[3], t[4], t[5]), fmaxf(t[6], t[7])) * sl2;
        }
        if (threadIdx.x == 0) TRACE2(29, sc);
        if (j == 0) {
          m_used = mx;
        } else {
          // lazy rescale (warp-uniform: tcgen05.ld/st are warp-collective); O must
          // hold P(j-1).V first, so wait for that P.V to complete
          const bool need = mx > m_used + kRescaleLog2;
          if (__any_sync(0xffffffffu, need)) {
            const int pb = (sc - 1) & 1;
            ptx::mbar_wait(bar(B_ODONE + 2 * wg + pb), ((sc - 1) >> 1) & 1);
            ptx::tc_fence_after();
            const float alpha = need ? fast_exp2(m_used - mx) : 1.f;
            if (need) {
              lsum *= alpha;
              m_used = mx;
            }
#pragma unroll 1
            for (int c = 0; c < D; c += 32) {
              uint32_t o[32];
              DLLM_TMEM_LD32(tO + c, o);
              ptx::tmem_wait_ld();
#pragma unroll
              for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
              DLLM_TMEM_ST32(tO + c, o);
            }
          }
        }
        {
          const uint64_t sl2x2 = pack_f32x2(sl2, sl2);
          const uint64_t negm = pack_f32x2(-m_used, -m_used);
          uint64_t acc[4] = {0ull, 0ull, 0ull, 0ull};
          uint32_t pk[32];
#pragma unroll
          for (int c = 0; c < 32; ++c) {
            const uint64_t x = ffma2(pack_f32x2(s[2 * c], s[2 * c + 1]), sl2x2, negm);
            float p0, p1;
            if ((c & (kPolyPeriod - 1)) < kPolyPairs) {
              unpack_f32x2(exp2_poly2(x), p0, p1);          // FMA pipe
            } else {
              float x0, x1;
              unpack_f32x2(x, x0, x1);
              p0 = fast_exp2(x0);                           // MUFU
              p1 = fast_exp2(x1);
            }
            acc[c & 3] = fadd2(acc[c & 3], pack_f32x2(p0, p1));
            pk[c] = pack_bf16(p0, p1);
          }
          if (threadIdx.x == 0) TRACE2(30, sc);
          DLLM_TMEM_ST32(tS, pk);
          float a0, a1, a2, a3;
          unpack_f32x2(fadd2(acc[0], acc[1]), a0, a1);
          unpack_f32x2(fadd2(acc[2], acc[3]), a2, a3);
          lsum += (a0 + a1) + (a2 + a3);
        }
        ptx::tmem_wait_st();
        if (threadIdx.x == 0) TRACE2(31, sc);
        ptx::tc_fence_before();
        __syncwarp();
        if ((threadIdx.x & 127) == 0) TRACE2(4 + wg, sc);
        if (lane == 0) ptx::mbar_arrive(bar(B_PFULL + 2 * wg + b));
      }
      // ---- hand the row sums to the epilogue warpgroup (double-buffered by unit parity)
      float *lb = reinterpret_cast<float *>(gb + C::kOffL) + ((oc & 1) * 2 + wg) * 128;
      lb[row] = lsum;
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(bar(B_LFULL + wg));
      ++oc;
    }
  } else if (warp >= kEpi0 && warp < kEpi0 + 4) {
    // ============================ epilogue warpgroup ============================
    // Reads O_i out of TMEM as soon as the unit's last P.V completes, releases the
    // accumulator to the MMA warp, then normalises by the row sums and streams O to
    // global through the TMA store engine.  The softmax warps never wait for it.
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(DLLM_TC2_REG_EPI) : "memory");
    const int wq = warp & 3;
    const int row = wq * 32 + lane;
    const uint32_t lane_off = (uint32_t)(wq * 32) << 16;
    const int64_t HD = (int64_t)plan.H * Dg;
    uint8_t *stg = gb + C::kOffStage + wq * 32 * 64;
    const uint32_t stg_s = sb + C::kOffStage + wq * 32 * 64;
    int oc[2] = {0, 0};
    int selc = 0;
    (void)selc;
    for (int i = 0;; ++i) {
      Unit u;
      const int unit = unit_at(i, true, u);
      if (unit >= plan.total_units) break;
      for (int i = 0; i < (u.tile1 ? 2 : 1); ++i) {
        const uint32_t tO = tmem + lane_off + tmem_o(i);
        ptx::mbar_wait(bar(B_OFULL + i), oc[i] & 1);
        ptx::tc_fence_after();
        uint32_t o[D];
#pragma unroll
        for (int c = 0; c < D; c += 32) DLLM_TMEM_LD32(tO + c, (o + c));
        ptx::tmem_wait_ld();
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(bar(B_OFREE + i));
        ptx::mbar_wait(bar(B_LFULL + i), oc[i] & 1);
        const float lsum = reinterpret_cast<const float *>(gb + C::kOffL)[((oc[i] & 1) * 2 + i) * 128 + row];
        ++oc[i];
        const float inv = lsum > 0.f ? 1.f / lsum : 0.f;
        const int origin = i ? u.origin1 : u.origin0;
        const int wend = i ? u.wend1 : u.wend0;
        const int srow0 = origin + wq * 32;                // first tile row of this warp
        const bool full_warp = srow0 + 32 <= wend && Dg == D;   // (D < 64: direct stores)
#pragma unroll
        for (int c = 0; c < D; c += 32) {
          uint32_t pk[16];
#pragma unroll
          for (int e = 0; e < 16; ++e)
            pk[e] = pack_bf16(__uint_as_float(o[c + 2 * e]) * inv, __uint_as_float(o[c + 2 * e + 1]) * inv);
          if (full_warp) {
            if (lane == 0) ptx::bulk_wait_group_read0();   // previous chunk read out of staging
            __syncwarp();
#pragma unroll
            for (int q4 = 0; q4 < 4; ++q4) {
              const int chunk = q4 ^ ((lane >> 1) & 3);      // 64-byte swizzle
              *reinterpret_cast<uint4 *>(stg + lane * 64 + chunk * 16) =
                  make_uint4(pk[4 * q4], pk[4 * q4 + 1], pk[4 * q4 + 2], pk[4 * q4 + 3]);
            }
            ptx::fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              ptx::tma_store_3d(&tm_o, stg_s, c, u.h, u.q_off + srow0);
              ptx::bulk_commit_group();
            }
          } else if (srow0 + lane < wend && c < Dg) {
            uint4 *d4 = reinterpret_cast<uint4 *>(out + (int64_t)(u.q_off + srow0 + lane) * HD + (int64_t)u.h * Dg + c);
#pragma unroll
            for (int q4 = 0; q4 < 4; ++q4)
              if (c + 8 * q4 < Dg) d4[q4] = make_uint4(pk[4 * q4], pk[4 * q4 + 1], pk[4 * q4 + 2], pk[4 * q4 + 3]);
          }
        }
      }
      if (DLLM_TC2_FUSEDSEL && sel_idx != nullptr && scores != nullptr && (u.sc0 || u.sc1) && u.k > 0) {
        // this unit's softmax warps wrote the head's raw scores (every key, all steps)
        // before their row-sum arrivals, which the O loop above acquired
        if (lane == 0) ptx::bulk_wait_group_read0();   // staging tile becomes select scratch
        ptx::named_bar_sync(kFSelBar, kFSelThreads);
        if (warp == kEpi0 && lane == 0) TRACE2(32, selc);
        fused_select(scores + u.score_off + (int64_t)u.h * u.L, u.L, u.bs, u.be, plan.window >> 1, u.k,
                     sel_idx + u.idx_off + (int64_t)u.h * u.k, reinterpret_cast<int *>(gb + C::kOffStage),
                     (warp - kEpi0) * 32 + lane);
        if (warp == kEpi0 && lane == 0) TRACE2(33, selc);
        ++selc;
      }
    }
    if (lane == 0) ptx::bulk_wait_group0();
  } else {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 64;\n" ::: "memory");   // the idle warp of the producer group
  }

  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
#ifdef DLLM_TRACE
  if (threadIdx.x == 0 && cta < 1024) {
    g_cta2[blockIdx.x][1] = gtimer();
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    g_cta2[blockIdx.x][3] = smid;
  }
#endif
  if (warp == kMmaWarp) ptx::tmem_dealloc(tmem, 512);
  if (dyn && threadIdx.x == 0) {
    // the last CTA of the launch resets the counters for the next launch on this
    // workspace (every CTA's claims precede its increment: __syncthreads above + fence)
    __threadfence();
    if (atomicAdd(plan.sched + 1, 1) == ncta - 1) {
      atomicExch(plan.sched, 0);
      atomicExch(plan.sched + 1, 0);
    }
  }
}

template <int D>
__global__ void __launch_bounds__(THREADS, 1)
refresh_tc2_kernel(const __grid_constant__ Plan plan, const __grid_constant__ CUtensorMap tm_q,
                   const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
                   const __grid_constant__ CUtensorMap tm_o, __nv_bfloat16 *__restrict__ out,
                   float *__restrict__ scores, int32_t *__restrict__ sel_idx) {
  // (griddepcontrol.wait inside the body, after its input-independent prologue)
  refresh_tc2_body<D>(plan, tm_q, tm_k, tm_v, tm_o, out, scores, sel_idx, (int)blockIdx.x, (int)gridDim.x);
}

// Single-launch mixed-phase batch (the paper's single varlen
// dispatch over a packed batch of Refresh and Reuse requests, PAPER.md:366,
// 453-456): CTAs [0, n_ref) run the Refresh body over the Refresh requests'
// plan, CTAs [n_ref, grid) the Reuse body over the Reuse requests' plan, both
// persistent, in one launch with the same 512-thread block (the larger of the
// two shared-memory layouts; each body carves its own).  The tensor-bound and
// the HBM-bound phase finish together when n_ref follows their estimated times,
// and there is no kernel boundary between them.
__global__ void __launch_bounds__(THREADS, 1)
mixed_tc_kernel(const __grid_constant__ Plan rplan, const __grid_constant__ CUtensorMap tm_q,
                const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
                const __grid_constant__ CUtensorMap tm_o, __nv_bfloat16 *__restrict__ out, float *__restrict__ scores,
                const __grid_constant__ Plan uplan, const __nv_bfloat16 *__restrict__ q_blk,
                const __nv_bfloat16 *__restrict__ k_cache, const __nv_bfloat16 *__restrict__ v_cache,
                const int32_t *__restrict__ idx, __nv_bfloat16 *__restrict__ out_blk, const int n_ref,
                int32_t *__restrict__ sel_idx) {
  if ((int)blockIdx.x < n_ref) {
    // (griddepcontrol.wait inside both bodies, after their input-independent prologues)
    refresh_tc2_body<128>(rplan, tm_q, tm_k, tm_v, tm_o, out, scores, sel_idx, (int)blockIdx.x, n_ref);
  } else {
    // (griddepcontrol.wait inside the body, after its input-independent prologue)
    rtc::reuse_tc_body<128>(uplan, q_blk, k_cache, v_cache, idx, out_blk, (int)blockIdx.x - n_ref, (int)gridDim.x - n_ref);
  }
}
static_assert(THREADS == rtc::kTThreads, "mixed kernel: both bodies run 512-thread CTAs");

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void *p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

int num_sms() {
  int dev = 0, n = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

template <int D>
cudaError_t make_maps(const Plan &plan, const void *q, const void *k, const void *v, void *out, CUtensorMap &tq,
                      CUtensorMap &tk, CUtensorMap &tv, CUtensorMap &to) {
  auto enc = encode_fn();
  if (!enc) return cudaErrorNotSupported;
  // Dg <= D: D = 16 / 32 tensors on the 64-dim layout keep the 64-column boxes (the
  // TMA zero-fills the columns past Dg); their output goes out by direct stores
  const int Dg = plan.D;
  const cuuint32_t bq = 64, bo = 32;
  int64_t rows = 0;
  for (int b = 0; b < plan.nreq; ++b) rows = rows > plan.r[b].q_off + plan.r[b].L ? rows : plan.r[b].q_off + plan.r[b].L;
  {
    cuuint64_t dims[3] = {(cuuint64_t)Dg, (cuuint64_t)plan.H, (cuuint64_t)rows};
    cuuint64_t strides[2] = {(cuuint64_t)Dg * 2, (cuuint64_t)plan.H * Dg * 2};
    cuuint32_t box[3] = {bo, 1, 32};
    cuuint32_t es[3] = {1, 1, 1};
    if (enc(&to, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, out, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
        CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  {
    cuuint64_t dims[3] = {(cuuint64_t)Dg, (cuuint64_t)plan.H, (cuuint64_t)rows};
    cuuint64_t strides[2] = {(cuuint64_t)Dg * 2, (cuuint64_t)plan.H * Dg * 2};
    cuuint32_t box[3] = {bq, 1, TBM};
    cuuint32_t es[3] = {1, 1, 1};
    if (enc(&tq, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void *>(q), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  {
    const int P = plan.page_size;
    cuuint64_t dims[4] = {(cuuint64_t)Dg, (cuuint64_t)P, (cuuint64_t)plan.H_kv, (cuuint64_t)1 << 24};
    cuuint64_t strides[3] = {(cuuint64_t)Dg * 2, (cuuint64_t)P * Dg * 2, (cuuint64_t)plan.H_kv * P * Dg * 2};
    cuuint32_t box[4] = {bq, (cuuint32_t)(P < TBN ? P : TBN), 1, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    for (int w = 0; w < 2; ++w) {
      if (enc(w ? &tv : &tk, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void *>(w ? v : k), dims, strides, box,
              es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return cudaErrorInvalidValue;
    }
  }
  return cudaSuccess;
}

template <int D>
cudaError_t launch_d(const Plan &plan, const void *q, const void *k, const void *v, void *out, float *scores,
                     int32_t *sel_idx, void *workspace, cudaStream_t st) {
  CUtensorMap tq, tk, tv, to;
  cudaError_t me = make_maps<D>(plan, q, k, v, out, tq, tk, tv, to);
  if (me != cudaSuccess) return me;
  const int smem = Cfg<D>::bytes(plan.nreq);
  cudaError_t e = cudaFuncSetAttribute(refresh_tc2_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  const int grid = plan.total_units < num_sms() ? plan.total_units : num_sms();
  if (grid <= 0) return cudaSuccess;
  static thread_local Plan pl;   // + this launch's scheduler counters
  pl = plan;
  pl.sched = workspace_sched(workspace);
  return launch_pdl(refresh_tc2_kernel<D>, dim3(grid), dim3(THREADS), smem, st, pl, tq, tk, tv, to,
                    (__nv_bfloat16 *)out, scores, sel_idx);
}

}  // namespace

cudaError_t launch_mixed_tc(const Plan &rplan, const void *q, const void *k, const void *v, void *out, float *scores,
                            const Plan &uplan, const void *q_blk, const int32_t *idx, void *out_blk, int n_ref,
                            int grid, int32_t *sel_idx, void *workspace, cudaStream_t st) {
  if (rplan.D != 128 || uplan.D != 128) return cudaErrorInvalidValue;
  CUtensorMap tq, tk, tv, to;
  cudaError_t e = make_maps<128>(rplan, q, k, v, out, tq, tk, tv, to);
  if (e != cudaSuccess) return e;
  const int smem = Cfg<128>::bytes(rplan.nreq) > rtc::kTBytes ? Cfg<128>::bytes(rplan.nreq) : rtc::kTBytes;
  e = cudaFuncSetAttribute(mixed_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  if (grid <= 0) return cudaSuccess;
  static thread_local Plan rpl;
  rpl = rplan;
  rpl.sched = workspace_sched(workspace);
  (void)workspace;
  return launch_pdl(mixed_tc_kernel, dim3(grid), dim3(THREADS), smem, st, rpl, tq, tk, tv, to, (__nv_bfloat16 *)out,
                    scores, uplan, (const __nv_bfloat16 *)q_blk, (const __nv_bfloat16 *)k, (const __nv_bfloat16 *)v,
                    idx, (__nv_bfloat16 *)out_blk, n_ref, sel_idx);
}

int num_sms_mixed() { return num_sms(); }

// D = 64, 128 on their own layouts; D = 16, 32 on the 64-dim layout (zero-padded rows)
bool refresh_tc_supported(int D) { return D == 16 || D == 32 || D == 64 || D == 128; }

int fused_select_max_n() { return DLLM_TC2_FUSEDSEL ? kFSelMaxN : 0; }

int refresh_tc2_units(int L, int bs, int be, int H, bool with_scores) {
  const int nt = regular_tiles(L) + ((with_scores && straddles(bs, be)) ? 1 : 0);
  return H * ((nt + 1) / 2);
}

cudaError_t launch_refresh_tc2(const Plan &plan, const void *q, const void *k, const void *v, void *out,
                               float *scores, int32_t *sel_idx, void *workspace, cudaStream_t st) {
  switch (plan.D) {
    case 16:
    case 32:
    case 64: return launch_d<64>(plan, q, k, v, out, scores, sel_idx, workspace, st);
    case 128: return launch_d<128>(plan, q, k, v, out, scores, sel_idx, workspace, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace dllm
