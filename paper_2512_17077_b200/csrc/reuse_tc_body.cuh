#pragma once
// Reuse sparse attention on the 5th-generation tensor cores (tcgen05 + TMEM)
// (§2.3, Eq. 4; per-head key sets of §4.5).
//
// For request b, query head h and the active block's query rows q:
//   O_b[q,h] = softmax_j(tau Q_blk[q,h].K[j,kv(h)]) V[j,kv(h)],  j in [bs,be) ++ idx(b,h)
// with K/V gathered in place from the paged cache.
//
// Why transposed.  A work unit has only 32 query rows (one block of one head)
// but hundreds of keys, and tcgen05 needs M = 128 for the simple one-row-per-
// TMEM-lane accumulator layout.  So the unit is computed transposed, keys in
// the M dimension:
//   S^T[128 keys x 32 rows]  = K_chunk[128 x D] . Q^T           (A = K, K-major)
//   O^T[D=128 x 32 rows]    += V_chunk^T[D x 128] . P^T          (A = V, MN-major;
//                                                                 B = P^T, K-major)
// Each softmax thread owns one key of the chunk (its TMEM lane) and the 32
// query rows (columns); the per-row max / sum over keys are warp transpose-
// reductions plus a 4-warp exchange through shared memory.  The legacy
// mma.sync path peaks at ~2 kFLOP/clk/SM on sm_100a (profiles/
// r01_micro_tmem_mufu_hmma.log), which made the 64-key chunk of reuse_ws
// math-bound (~0.85 us per chunk, scripts/trace_reuse.py); here the math is
// a small fraction of the chunk's HBM time.
//
// Roles (16 warps = 512 threads, one CTA per SM, persistent over units; see the
// warp map below kTWarps):
//   warps 0-3, 6, 7  loaders: the unit's Q rows and 16-byte cp.async row gathers
//                    of K and V into an NS-stage ring laid out as the UMMA SW128
//                    operand tiles;
//   warp 4           translator: position -> physical cache row for every key of
//                    every chunk (block-table lookups, batched);
//   warp 5           MMA issuer (one elected lane issues; warp-uniform loop);
//   warps 8-11       softmax (thread = key = TMEM lane);
//   warps 12-15      epilogue (O^T / l -> bf16 rows -> bulk stores).
// P^T is written over the stage's K tile once S^T of that chunk is complete,
// so P needs no shared memory of its own.
// The data written by cp.async (generic proxy) is published to the tensor
// core (async proxy) by a proxy fence in the MMA warp after the full barrier.
#include <cuda_runtime.h>
#include <stdint.h>


#include "common.cuh"
#include "plan.h"
#include "tc_ptx.cuh"

namespace dllm {
namespace rtc {

constexpr int kTD = 128;            // head dim of the default layout (the mixed kernel's)
// The layout is built for a padded head dim DP in {64, 128}: D = 128 uses DP = 128;
// D = 16, 32, 64 use DP = 64 -- every row gathered into shared memory is zero-padded
// to DP dims (the 16-byte pieces past D are cp.async zero-fills), so S^T = K Q^T is
// unchanged, and O^T = V^T P^T keeps its M = 128 MMA: with DP = 64 its A operand's
// second 64-dim atom is read from the next 12 KB of shared memory (finite data) into
// TMEM lanes 64-127, which the epilogue never reads.
constexpr int kTRows = 32;          // query rows per unit (MMA N)
#ifndef DLLM_RTC_KEYS
#define DLLM_RTC_KEYS 96
#endif
// Keys per ring stage.  S^T is always an M = 128 MMA (the accumulator layout with
// one key per TMEM lane); with 96-key stages it reads 32 rows past the stage's K
// tile (the tile's second atom, then the stage's V tile: finite data) into TMEM
// lanes 96-127, which the softmax masks.  96-key stages fit 4 deep in the same
// 192 KB as 3 of 128 keys and waste less of the ring on a unit's partial last
// stage (C1: 280 keys = 3 x 96 (97% full) vs 2 x 128 + 24 (73%)).  Measured
// (profiles/r02_ab_reuse_keys96.log, two alternating runs on one box): C1 31.7 vs
// 33.8 us, C2 56.3 / 62.4 vs 56.3 / 56.3, C3 588 / 547 vs 542 / 555, C4 400 / 396 vs
// 401 / 410 us (96 vs 128).
constexpr int kTChunk = DLLM_RTC_KEYS;
constexpr int kTNS = kTChunk == 128 ? 3 : 4;     // K/V ring stages (2 x kTChunk x 256 B each)
static_assert(kTChunk % 32 == 0 && kTChunk <= 128, "reuse_tc: stage keys");
constexpr int kTNT = 4;             // translation ring depth (chunks)
constexpr int kTTG = 4;             // chunks translated per batch (2 vs 4: within box noise)
// Warp roles (16 warps; the warp schedulers favour the highest warp id among the
// eligible warps of a sub-partition, so the softmax and epilogue warps sit on top):
//   0-3, 6-7  loaders         4  translator       5  MMA issuer
//   8-11      softmax (TMEM lane quarter = warp % 4)
//   12-15     epilogue: O^T / l -> bf16 rows -> bulk (TMA) stores
constexpr int kTLoaders = 6, kTransWarp = 4, kMmaWarp = 5, kSoft0 = 8, kEpi0 = 12, kTWarps = 16;
__device__ __forceinline__ int loader_index(int w) { return w < 4 ? w : (w == 6 || w == 7 ? w - 2 : -1); }
constexpr int kTThreads = kTWarps * 32;

// shared memory (offsets from a 1024-byte aligned base)
constexpr int kBtMax = 1024;                          // block-table entries cached in shared memory
constexpr int kNumBars = 2 * kTNS + 2 * kTNT + 2 + 2 + 2 + 2 + 2 + 1 + 2 + 2 + 2 + 1;
template <int DP>
struct RL {
  static constexpr int kTileK = kTChunk * DP * 2;          // [DP/64 atoms][kTChunk rows][128 B]
  static constexpr int kStage = 2 * kTileK;                // K then V
  static constexpr int kQTile = kTRows * DP * 2;           // [DP/64 atoms][32 rows][128 B]
  static constexpr int kOffQ = kTNS * kStage;
  static constexpr int kOffOffs = kOffQ + 2 * kQTile;      // [kTNT][kTChunk] int32
  static constexpr int kOffRed = kOffOffs + kTNT * kTChunk * 4;   // [4 warps][32] chunk row maxima
  static constexpr int kOffL = kOffRed + 4 * 32 * 4;              // [2 O buffers][4 warps][32 rows] partial row sums
  static constexpr int kOffStage = kOffL + 2 * 4 * 32 * 4;        // output staging [32 rows][D] bf16
  static constexpr int kOffBt = kOffStage + kTRows * DP * 2;      // [kBtMax] int32
  static constexpr int kOffBar = kOffBt + kBtMax * 4;
  static constexpr int kBytes = kOffBar + 8 * kNumBars + 1024;    // + alignment slack
  static_assert(kBytes <= 227 * 1024, "reuse_tc shared memory");
  // the O^T MMA with DP = 64 reads a second 64-dim atom kTChunk * 128 bytes past each
  // stage's V tile: still inside the allocation (the next stage, or the Q tiles and
  // the offset ring after the last one).  Whatever it reads (NaN bit patterns
  // included) only reaches accumulator rows 64-127, which are never read.
  static_assert(DP == 128 || kTNS * kStage + kTChunk * 128 <= kOffBar, "reuse_tc DP = 64 overread");
};
constexpr int kTBytes = RL<kTD>::kBytes;

// TMEM columns: S^T double buffer (32 each), O^T double buffer (32 each)
constexpr uint32_t kTmemCols = 128;
__device__ __forceinline__ uint32_t tm_s(int b) { return (uint32_t)(b * 32); }
__device__ __forceinline__ uint32_t tm_o(int b) { return (uint32_t)(64 + b * 32); }

#ifdef DLLM_TRACE
// per-CTA timeline (globaltimer ns): [0] start, [1] translator: first offsets published,
// [2] MMA: first S issued, [3..10] softmax: end of unit i, [11] end, [12] SM id;
// CTA 0 per chunk: [0] published, [1] loader issued, [2] S issued, [3] softmax got S,
// [4] softmax P written, [5] P.V issued
static __device__ long long g_rtc[1024][16];
static __device__ long long g_rtc_chunk[16][64];
__device__ __forceinline__ long long rtc_timer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define RTC_CTA(slot)                                                          \
  do {                                                                         \
    if (lane == 0 && blockIdx.x < 1024) g_rtc[blockIdx.x][slot] = rtc_timer(); \
  } while (0)
#define RTC_CHUNK(kind, t)                                                              \
  do {                                                                                  \
    if (lane == 0 && blockIdx.x == 0 && (t) < 64) g_rtc_chunk[kind][t] = rtc_timer();   \
  } while (0)
#else
#define RTC_CTA(slot) \
  do {                \
  } while (0)
#define RTC_CHUNK(kind, t) \
  do {                     \
  } while (0)
#endif

struct TUnit {
  int b, h, kvh, rg, blk, bs, nk, k, blk_off, bt_row;
  int64_t idx_off;
};

__device__ __forceinline__ void tdecode(const Plan &pl, int unit, TUnit &u) {
  u.b = plan_find(pl, unit);
  const ReqInfo &R = pl.r[u.b];
  u.blk = R.be - R.bs;
  u.bs = R.bs;
  const int ngroups = (u.blk + kTRows - 1) / kTRows;
  const int local = unit - R.unit_off;
  u.h = local / ngroups;
  u.rg = local - u.h * ngroups;
  u.kvh = u.h / (pl.H / pl.H_kv);
  u.k = R.k;
  u.nk = u.blk + R.k;
  u.blk_off = R.blk_off;
  u.bt_row = R.bt_row;
  u.idx_off = R.idx_off + (int64_t)u.h * R.k;
}

__device__ __forceinline__ void cp_async_arrive_noinc(uint32_t bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(bar) : "memory");
}

// byte offset of 16-byte piece c (of a 2*D-byte row) of row r in a SW128 K-major
// operand tile with `rows` rows: [D/64 atoms][rows][128 B], piece index XOR (r & 7)
__device__ __forceinline__ uint32_t sw128_off(int rows, int r, int c) {
  return (uint32_t)((c >> 3) * rows * 128 + r * 128 + (((c & 7) ^ (r & 7)) << 4));
}

// Warp transpose-reduction of 32 per-lane values x[0..31] (x[n] = this lane's value
// for row n): returns, in lane j, op over the 32 lanes of x[j].  Destroys x.
template <bool MAX>
__device__ __forceinline__ float transpose_reduce32(float (&x)[32], int lane) {
#pragma unroll
  for (int w = 16; w >= 1; w >>= 1) {
    const bool up = (lane & w) != 0;
#pragma unroll
    for (int i = 0; i < w; ++i) {
      const float send = up ? x[i] : x[i + w];
      const float keep = up ? x[i + w] : x[i];
      const float r = __shfl_xor_sync(0xffffffffu, send, w);
      x[i] = MAX ? fmaxf(keep, r) : keep + r;
    }
  }
  return x[0];
}

// The kernel body, shared by reuse_tc_kernel (one launch per Reuse batch) and the
// single-launch mixed Refresh/Reuse kernel (refresh_tc2.cu): CTA `cta` of `ncta`
// CTAs working on this plan.  It executes griddepcontrol.wait itself, after its
// input-independent prologue: the caller must not read global memory before.
template <int DP>
__device__ __forceinline__ void reuse_tc_body(const Plan &plan, const __nv_bfloat16 *__restrict__ q_blk,
                                              const __nv_bfloat16 *__restrict__ k_cache,
                                              const __nv_bfloat16 *__restrict__ v_cache,
                                              const int32_t *__restrict__ idx, __nv_bfloat16 *__restrict__ out,
                                              const int cta, const int ncta) {
  using Lc = RL<DP>;
  constexpr int D = DP;        // padded head dim of the shared-memory layout and the MMAs
  const int Dg = DP == kTD ? kTD : plan.D;   // head dim of the tensors in global memory (<= DP)
  constexpr int CH = D / 8;    // 16-byte pieces per row
  constexpr int NS = kTNS;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t sb = (raw + 1023u) & ~1023u;
  uint8_t *gb = smem_raw + (sb - raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // barriers
  const uint32_t b_kvfull = sb + Lc::kOffBar;             // [NS] loaders (32*kTLoaders noinc)
  const uint32_t b_kvempty = b_kvfull + 8 * NS;       // [NS] MMA commit
  const uint32_t b_ofull_t = b_kvempty + 8 * NS;      // [kTNT] translator (1)
  const uint32_t b_oempty_t = b_ofull_t + 8 * kTNT;   // [kTNT] loaders (kTLoaders)
  const uint32_t b_qfull = b_oempty_t + 8 * kTNT;     // [2] loaders (32*kTLoaders noinc)
  const uint32_t b_qempty = b_qfull + 16;             // [2] MMA commit
  const uint32_t b_sfull = b_qempty + 16;             // [2] MMA commit
  const uint32_t b_sfree = b_sfull + 16;              // [2] softmax warps (4)
  const uint32_t b_pfull = b_sfree + 16;              // [2] softmax warps (4)
  const uint32_t b_pvdone = b_pfull + 16;             // [1] MMA commit after every P.V
  const uint32_t b_ofull = b_pvdone + 8;              // [2] MMA commit (unit's last P.V)
  const uint32_t b_ofree = b_ofull + 16;              // [2] epilogue warps (4): O^T and row sums consumed
  const uint32_t b_lfull = b_ofree + 16;              // [2] softmax warps (4): row sums written
  const uint32_t b_tslot = b_lfull + 16;              // TMEM base address slot
  // i-th unit of this CTA (static round-robin; a device-counter scheduler measured
  // 5-8% slower here, profiles/r01_ab_reuse_dynsched_qprefetch.log)
  auto unit_at = [&](int i) -> int { return cta + i * ncta; };
  int32_t *offs = reinterpret_cast<int32_t *>(gb + Lc::kOffOffs);

#ifdef DLLM_TRACE
  if (threadIdx.x == 0 && cta < 1024) {
    for (int i = 0; i < 16; ++i) g_rtc[blockIdx.x][i] = 0;
    g_rtc[blockIdx.x][0] = rtc_timer();
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    g_rtc[blockIdx.x][12] = smid;
  }
#endif
  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) {
      ptx::mbar_init(b_kvfull + 8 * i, 32 * kTLoaders);
      ptx::mbar_init(b_kvempty + 8 * i, 1);
    }
    for (int i = 0; i < kTNT; ++i) {
      ptx::mbar_init(b_ofull_t + 8 * i, 1);
      ptx::mbar_init(b_oempty_t + 8 * i, kTLoaders);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(b_qfull + 8 * i, 32 * kTLoaders);
      ptx::mbar_init(b_qempty + 8 * i, 1);
      ptx::mbar_init(b_sfull + 8 * i, 1);
      ptx::mbar_init(b_sfree + 8 * i, 4);
      ptx::mbar_init(b_pfull + 8 * i, 4);
      ptx::mbar_init(b_ofull + 8 * i, 1);
      ptx::mbar_init(b_ofree + 8 * i, 4);
      ptx::mbar_init(b_lfull + 8 * i, 4);
    }
    ptx::mbar_init(b_pvdone, 1);
    ptx::fence_mbar_init();
  }
  if (warp == kMmaWarp) {
    ptx::tmem_alloc(b_tslot, kTmemCols);
    ptx::tmem_relinquish();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  // everything above (barriers, TMEM) is independent of the preceding kernel's
  // results: with programmatic dependent launch it overlaps that kernel's tail
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t *>(gb + (b_tslot - sb));

  if (warp < kSoft0) asm volatile("setmaxnreg.dec.sync.aligned.u32 80;\n" ::: "memory");
  if (warp == kTransWarp) {
    // ============================ translator (+ Q rows) ============================
    int t = 0, bt_cached = -1;
    int *bts = reinterpret_cast<int *>(gb + Lc::kOffBt);
    int unit = cta;
    for (int i = 0;; ++i) {
      if (unit >= plan.total_units) break;
      const int cur = unit;
      unit += ncta;
      TUnit u;
      tdecode(plan, cur, u);
      // the next unit's index list and block-table row go to L2 while this one is
      // translated (warp-uniform lookup, one bulk prefetch each); for the CTA's first
      // unit only after its chunks are published (the lookup costs ~1k clk)
      auto prefetch_next = [&]() {
        TUnit v;
        tdecode(plan, unit, v);
        if (lane == 0 && v.k > 0) {
          const uintptr_t a0 = reinterpret_cast<uintptr_t>(idx + v.idx_off) & ~uintptr_t(15);
          const uintptr_t a1 = (reinterpret_cast<uintptr_t>(idx + v.idx_off + v.k) + 15) & ~uintptr_t(15);
          ptx::bulk_prefetch_l2(reinterpret_cast<const void *>(a0), (uint32_t)(a1 - a0));
        }
        if (lane == 1 && v.bt_row != u.bt_row) {
          const uintptr_t b0 = reinterpret_cast<uintptr_t>(plan.block_table + (int64_t)v.bt_row * plan.pages_per_req) &
                               ~uintptr_t(15);
          const uintptr_t b1 = (reinterpret_cast<uintptr_t>(plan.block_table + (int64_t)(v.bt_row + 1) * plan.pages_per_req) +
                                15) & ~uintptr_t(15);
          ptx::bulk_prefetch_l2(reinterpret_cast<const void *>(b0), (uint32_t)(b1 - b0));
        }
      };
      if (unit < plan.total_units && i > 0) prefetch_next();
      const int32_t *my_idx = idx + u.idx_off;
      const int32_t *bt = plan.block_table + (int64_t)u.bt_row * plan.pages_per_req;
      const int nchunks = (u.nk + kTChunk - 1) / kTChunk;
      const bool bt_smem = plan.pages_per_req <= kBtMax;
      for (int g0 = 0; g0 < nchunks; g0 += kTTG) {
        constexpr int Q = kTTG * kTChunk / 32;
        int pos[Q], off[Q];
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          const int j = g0 * kTChunk + q * 32 + lane;
          pos[q] = j < u.nk ? (j < u.blk ? u.bs + j : __ldg(my_idx + (j - u.blk))) : -1;
        }
        if (g0 == 0 && bt_smem && u.bt_row != bt_cached) {
          // the request's block-table row goes to shared memory while the index loads
          // above are in flight: a translation costs one memory round trip, not two
          __syncwarp();
          for (int i0 = 0; i0 < plan.pages_per_req; i0 += 8 * 32) {
            int v[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const int i = i0 + q * 32 + lane;
              v[q] = i < plan.pages_per_req ? __ldg(bt + i) : 0;
            }
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const int i = i0 + q * 32 + lane;
              if (i < plan.pages_per_req) bts[i] = v[q];
            }
          }
          bt_cached = u.bt_row;
        }
        __syncwarp();
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          const int pi = pos[q] >= 0 ? (pos[q] >> plan.page_shift) : 0;
          const int page = pos[q] >= 0 ? (bt_smem ? bts[pi] : __ldg(bt + pi)) : 0;
          off[q] = pos[q] >= 0 ? (page * plan.H_kv + u.kvh) * plan.page_size + (pos[q] & (plan.page_size - 1)) : -1;
        }
        const int ng = min(kTTG, nchunks - g0);
#pragma unroll
        for (int c = 0; c < kTTG; ++c) {
          if (c >= ng) break;
          const int slot = t % kTNT;
          ptx::mbar_wait(b_oempty_t + 8 * slot, ((t / kTNT) & 1) ^ 1);
#pragma unroll
          for (int rr = 0; rr < kTChunk / 32; ++rr) offs[slot * kTChunk + rr * 32 + lane] = off[c * (kTChunk / 32) + rr];
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(b_ofull_t + 8 * slot);
          if (t == 0) RTC_CTA(1);
          RTC_CHUNK(0, t);
          ++t;
        }
      }
      if (unit < plan.total_units && i == 0) prefetch_next();
    }
    cp_async_wait<0>();
  } else if (loader_index(warp) >= 0) {
    // ============================ loaders ============================
    const int li = loader_index(warp);
    const int64_t HD = (int64_t)plan.H * Dg;
    int t = 0, qc = 0;
    for (int i = 0;; ++i, ++qc) {
      const int unit = unit_at(i);
      if (unit >= plan.total_units) break;
      TUnit u;
      tdecode(plan, unit, u);
      const int nchunks = (u.nk + kTChunk - 1) / kTChunk;
      {
        // the unit's 32 query rows (zero rows past the block), SW128 K-major
        const int row0 = u.rg * kTRows;
        const int qb = qc & 1;
        ptx::mbar_wait(b_qempty + 8 * qb, ((qc >> 1) & 1) ^ 1);
        const uint32_t sq = sb + Lc::kOffQ + qb * Lc::kQTile;
        for (int i = li * 32 + lane; i < kTRows * CH; i += 32 * kTLoaders) {
          const int r = i / CH, c = i - r * CH;
          // rows past the block and (DP = 64) dims past D: zeros
          const bool ok = row0 + r < u.blk && (D == kTD || c * 8 < Dg);
          const __nv_bfloat16 *src = q_blk + (int64_t)(u.blk_off + (ok ? row0 + r : 0)) * HD + (int64_t)u.h * Dg + c * 8;
          cp_async16(sq + sw128_off(kTRows, r, c), src, ok ? 16 : 0);
        }
        cp_async_arrive_noinc(b_qfull + 8 * qb);
      }
      for (int c = 0; c < nchunks; ++c, ++t) {
        const int slot = t % kTNT, s = t % NS;
        ptx::mbar_wait(b_ofull_t + 8 * slot, (t / kTNT) & 1);
        ptx::mbar_wait(b_kvempty + 8 * s, ((t / NS) & 1) ^ 1);
        const uint32_t dk = sb + s * Lc::kStage, dv = dk + Lc::kTileK;
#pragma unroll 4
        for (int e = li * 32 + lane; e < kTChunk * CH; e += 32 * kTLoaders) {
          const int r = e / CH, cc = e - r * CH;
          const int off = offs[slot * kTChunk + r];
          const bool ok = off >= 0 && (D == Dg || cc * 8 < Dg);
          const int64_t goff = ok ? (int64_t)off * Dg + cc * 8 : 0;
          const int nb = ok ? 16 : 0;
          const uint32_t so = sw128_off(kTChunk, r, cc);
          cp_async16(dk + so, k_cache + goff, nb);
          cp_async16(dv + so, v_cache + goff, nb);
        }
        cp_async_arrive_noinc(b_kvfull + 8 * s);
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(b_oempty_t + 8 * slot);
        if (li == 0) RTC_CHUNK(1, t);
      }
    }
    cp_async_wait<0>();
  } else if (warp == kMmaWarp) {
    // ============================ MMA issuer ============================
    constexpr uint32_t idesc_s = ptx::idesc_bf16_f32(128, kTRows, false, false);
    constexpr uint32_t idesc_o = ptx::idesc_bf16_f32(128, kTRows, true, true);
    const uint64_t dk0 = ptx::smem_desc_sw128(sb, 16, 1024);                 // K tile (K-major) / P^T (K-major)
    const uint64_t dv0 = ptx::smem_desc_sw128(sb + Lc::kTileK, kTChunk * 128, 1024);   // V tile as MN-major A
    const uint64_t dq0 = ptx::smem_desc_sw128(sb + Lc::kOffQ, 16, 1024);
    // P^T MN-major SW64: one 32-row atom along N, 8-key groups 512 B apart along K
    const uint64_t dpm0 = ptx::smem_desc(sb, 64 * 8 * 2, 512, ptx::kSwizzle64B);
    int t = 0, uc = 0;
    int pv_t = -1, pv_s = 0, pv_ob = 0, pv_first = 0, pv_last = 0, pv_uc = 0;
    auto issue_pv = [&]() {
      ptx::mbar_wait(b_pfull + 8 * (pv_t & 1), (pv_t >> 1) & 1);
      if (pv_first) ptx::mbar_wait(b_ofree + 8 * pv_ob, ((pv_uc >> 1) & 1) ^ 1);
      ptx::tc_fence_after();
      const uint64_t a0 = dv0 + (uint64_t)((pv_s * Lc::kStage) >> 4);
      const uint64_t p0 = dpm0 + (uint64_t)((pv_s * Lc::kStage) >> 4);
#pragma unroll
      for (int k = 0; k < kTChunk / 16; ++k) {
        const uint32_t ao = (uint32_t)((k * 16 * 128) >> 4);
        const uint32_t bo = (uint32_t)((k * 16 * 64) >> 4);
        ptx::mma_ss_elect(tmem + tm_o(pv_ob), a0 + ao, p0 + bo, idesc_o, (!pv_first || k > 0) ? 1u : 0u);
      }
      ptx::mma_commit_elect(b_kvempty + 8 * pv_s);
      ptx::mma_commit_elect(b_pvdone);
      RTC_CHUNK(5, pv_t);
      if (pv_last) ptx::mma_commit_elect(b_ofull + 8 * pv_ob);
    };
    for (int i = 0;; ++i, ++uc) {
      const int unit = unit_at(i);
      if (unit >= plan.total_units) break;
      TUnit u;
      tdecode(plan, unit, u);
      const int nchunks = (u.nk + kTChunk - 1) / kTChunk;
      const int qb = uc & 1;
      ptx::mbar_wait(b_qfull + 8 * qb, (uc >> 1) & 1);
      for (int c = 0; c < nchunks; ++c, ++t) {
        const int s = t % NS, sbuf = t & 1;
        // P.V(t-1) goes out as soon as its P is ready, even when chunk t's K/V rows
        // are still in flight: its stage is released that much earlier
        while (!(ptx::mbar_test_wait(b_kvfull + 8 * s, (t / NS) & 1) &&
                 ptx::mbar_test_wait(b_sfree + 8 * sbuf, ((t >> 1) & 1) ^ 1))) {
          if (pv_t >= 0 && ptx::mbar_test_wait(b_pfull + 8 * (pv_t & 1), (pv_t >> 1) & 1) &&
              (!pv_first || ptx::mbar_test_wait(b_ofree + 8 * pv_ob, ((pv_uc >> 1) & 1) ^ 1))) {
            issue_pv();
            pv_t = -1;
          }
        }
        ptx::mbar_wait(b_kvfull + 8 * s, (t / NS) & 1);
        ptx::mbar_wait(b_sfree + 8 * sbuf, ((t >> 1) & 1) ^ 1);
        ptx::fence_proxy_async_smem();   // cp.async (generic proxy) data -> tensor core (async proxy)
        ptx::tc_fence_after();
        const uint64_t a0 = dk0 + (uint64_t)((s * Lc::kStage) >> 4);
        const uint64_t b0 = dq0 + (uint64_t)((qb * Lc::kQTile) >> 4);
#pragma unroll
        for (int k = 0; k < D / 16; ++k) {
          const uint32_t ao = (uint32_t)(((k >> 2) * kTChunk * 128 + (k & 3) * 32) >> 4);
          const uint32_t bo = (uint32_t)(((k >> 2) * kTRows * 128 + (k & 3) * 32) >> 4);
          ptx::mma_ss_elect(tmem + tm_s(sbuf), a0 + ao, b0 + bo, idesc_s, k > 0 ? 1u : 0u);
        }
        ptx::mma_commit_elect(b_sfull + 8 * sbuf);
        if (t == 0) RTC_CTA(2);
        RTC_CHUNK(2, t);
        if (c == nchunks - 1) ptx::mma_commit_elect(b_qempty + 8 * qb);
        if (pv_t >= 0) issue_pv();
        pv_t = t; pv_s = s; pv_ob = uc & 1; pv_first = c == 0; pv_last = c == nchunks - 1; pv_uc = uc;
      }
      // the unit's last P.V goes out now, not behind the next unit's first K chunk:
      // the epilogue waits for it
      if (pv_t >= 0) issue_pv();
      pv_t = -1;
    }
  } else if (warp < kEpi0) {
    // ============================ softmax (warps 8-11) ============================
    // Thread = one key of the chunk (TMEM lane), 32 query rows (columns).  Every
    // thread keeps the running row maxima m_run[0..31] (identical in all 128
    // threads).  Common case: no key of the chunk exceeds its row's running max
    // by more than 2^8 (lazy rescale), decided with one 128-thread barrier-OR,
    // and the chunk costs one exp2 per score plus four 16-byte P^T stores.
    // Otherwise the chunk's row maxima are exchanged (redux.sync + shared
    // memory) and l / O^T are rescaled.
    asm volatile("setmaxnreg.inc.sync.aligned.u32 200;\n" ::: "memory");
    const int sw = warp & 3;   // TMEM lane quarter
    const float sl2 = plan.scale_log2;
    float *red = reinterpret_cast<float *>(gb + Lc::kOffRed);   // [4 warps][32] chunk maxima
    float *lbuf = reinterpret_cast<float *>(gb + Lc::kOffL);
    const uint32_t lane_base = (uint32_t)(sw * 32) << 16;
    int t = 0, uc = 0;
    for (int i = 0;; ++i, ++uc) {
      const int unit = unit_at(i);
      if (unit >= plan.total_units) break;
      TUnit u;
      tdecode(plan, unit, u);
      const int nchunks = (u.nk + kTChunk - 1) / kTChunk;
      const int ob = uc & 1;
      float m_run[32], l_part[32];
#pragma unroll
      for (int n = 0; n < 32; ++n) { m_run[n] = -INFINITY; l_part[n] = 0.f; }
      for (int c = 0; c < nchunks; ++c, ++t) {
        const int sbuf = t & 1;
        ptx::mbar_wait(b_sfull + 8 * sbuf, (t >> 1) & 1);
        ptx::tc_fence_after();
        if (sw == 0) RTC_CHUNK(3, t);
        const int key = c * kTChunk + sw * 32 + lane;
        const bool valid = sw * 32 + lane < kTChunk && key < u.nk;   // lanes past the stage: masked
        float x[32];
        float dmax = -INFINITY;
        {
          uint32_t r[32];
          DLLM_TMEM_LD32(tmem + lane_base + tm_s(sbuf), r);
          ptx::tmem_wait_ld();
#pragma unroll
          for (int n = 0; n < 32; ++n) {
            x[n] = valid ? __uint_as_float(r[n]) * sl2 : -INFINITY;
            dmax = fmaxf(dmax, x[n] - m_run[n]);   // NaN (-inf - -inf) is ignored by fmaxf
          }
        }
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(b_sfree + 8 * sbuf);
        const bool rare = ptx::bar_red_or(1, 128, dmax > 8.f);
        if (sw == 0) RTC_CHUNK(6, t);
        if (rare) {
          // chunk row maxima: warp transpose-reduction (lane j <- max of row j over the
          // warp's 32 keys), the four warps through shared memory, broadcast by shuffles
          float wmx;
          {
            float tmp[32];
#pragma unroll
            for (int n = 0; n < 32; ++n) tmp[n] = x[n];
            wmx = transpose_reduce32<true>(tmp, lane);
          }
          red[sw * 32 + lane] = wmx;
          ptx::named_bar_sync(1, 128);
          // (the next write of `red` happens after the next barrier-OR, i.e. after every
          // warp has read it here)
          const float mc = fmaxf(fmaxf(red[lane], red[32 + lane]), fmaxf(red[64 + lane], red[96 + lane]));
          float alpha[32];
          if (c == 0) {
            // a unit's first chunk: nothing accumulated yet, no rescale factors
#pragma unroll
            for (int n = 0; n < 32; ++n) m_run[n] = __shfl_sync(0xffffffffu, mc, n);
          } else {
#pragma unroll
            for (int n = 0; n < 32; ++n) {
              const float mn = fmaxf(m_run[n], __shfl_sync(0xffffffffu, mc, n));
              alpha[n] = fast_exp2(m_run[n] - mn);
              m_run[n] = mn;
              l_part[n] *= alpha[n];
            }
          }
          if (c > 0) {
            // O^T of this unit holds chunks < c: wait for P.V(t-1), rescale its columns
            ptx::mbar_wait(b_pvdone, (t - 1) & 1);
            ptx::tc_fence_after();
#pragma unroll
            for (int n4 = 0; n4 < 8; ++n4) {
              uint32_t o4[4];
              DLLM_TMEM_LD4(tmem + lane_base + tm_o(ob) + 4 * n4, o4);
              ptx::tmem_wait_ld();
#pragma unroll
              for (int e = 0; e < 4; ++e) o4[e] = __float_as_uint(__uint_as_float(o4[e]) * alpha[4 * n4 + e]);
              DLLM_TMEM_ST4(tmem + lane_base + tm_o(ob) + 4 * n4, o4);
            }
            ptx::tmem_wait_st();
            ptx::tc_fence_before();
          }
        }
        if (sw == 0) RTC_CHUNK(7, t);
        // P^T over the stage's K tile, MN-major SW64 operand: key kc's 32 row values are
        // one 64-byte row (4 pieces of 16 B), piece j stored at j ^ ((kc >> 1) & 3)
        const int kc = sw * 32 + lane;
        uint8_t *prow = gb + (t % NS) * Lc::kStage + kc * 64;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          uint32_t w4[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int n = 8 * j + 2 * q;
            const uint32_t pp = pack_bf16(fast_exp2(x[n] - m_run[n]), fast_exp2(x[n + 1] - m_run[n + 1]));
            l_part[n] += __uint_as_float(pp << 16);
            l_part[n + 1] += __uint_as_float(pp & 0xffff0000u);
            w4[q] = pp;
          }
          *reinterpret_cast<uint4 *>(prow + ((j ^ ((kc >> 1) & 3)) << 4)) = make_uint4(w4[0], w4[1], w4[2], w4[3]);
        }
        if (sw == 0) RTC_CHUNK(8, t);
        ptx::fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(b_pfull + 8 * sbuf);
        if (sw == 0) RTC_CHUNK(4, t);
      }
      // ---- unit end: this warp's partial row sums -> shared memory for the epilogue
      const float wsum = transpose_reduce32<false>(l_part, lane);
      ptx::mbar_wait(b_ofree + 8 * ob, ((uc >> 1) & 1) ^ 1);   // unit uc-2's sums consumed
      lbuf[ob * 128 + sw * 32 + lane] = wsum;
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(b_lfull + 8 * ob);
      if (sw == 0) RTC_CHUNK(9, uc);
    }
  } else {
    // ============================ epilogue (warps 12-15) ============================
    // O^T (thread = head-dim lane d, 32 row columns) / l -> bf16 rows in a staging
    // tile -> one 256-byte bulk (TMA) store per row.  Plain global stores from the
    // warps on the critical path were measured to queue for microseconds behind
    // the gather traffic; here they are off the critical path and asynchronous.
    asm volatile("setmaxnreg.inc.sync.aligned.u32 152;\n" ::: "memory");
    const int ew = warp & 3;
    const uint32_t lane_base = (uint32_t)(ew * 32) << 16;
    const float *lbuf = reinterpret_cast<const float *>(gb + Lc::kOffL);
    int uc = 0;
    for (int i = 0;; ++i, ++uc) {
      const int unit = unit_at(i);
      if (unit >= plan.total_units) break;
      TUnit u;
      tdecode(plan, unit, u);
      const int ob = uc & 1;
      ptx::mbar_wait(b_lfull + 8 * ob, (uc >> 1) & 1);
      ptx::mbar_wait(b_ofull + 8 * ob, (uc >> 1) & 1);
      ptx::tc_fence_after();
      if (ew == 0) RTC_CHUNK(10, uc);
      const float lsum = lbuf[ob * 128 + lane] + lbuf[ob * 128 + 32 + lane] + lbuf[ob * 128 + 64 + lane] +
                         lbuf[ob * 128 + 96 + lane];
      const float inv = lsum > 0.f ? __frcp_rn(lsum) : 0.f;   // row `lane`
      uint32_t o[32];
      DLLM_TMEM_LD32(tmem + lane_base + tm_o(ob), o);
      ptx::tmem_wait_ld();
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(b_ofree + 8 * ob);
      if (ew == 0) ptx::bulk_wait_group_read0();   // previous unit's rows left the staging tile
      ptx::named_bar_sync(2, 128);
      // thread = head dim d (TMEM lane); rows of Dg dims in the staging tile
      const int d = ew * 32 + lane;
      uint8_t *stg = gb + Lc::kOffStage + d * 2;
#pragma unroll
      for (int n = 0; n < 32; ++n) {
        const float v = __uint_as_float(o[n]) * __shfl_sync(0xffffffffu, inv, n);
        if (D == kTD || d < Dg) *reinterpret_cast<__nv_bfloat16 *>(stg + n * (Dg * 2)) = __float2bfloat16_rn(v);
      }
      ptx::fence_proxy_async_smem();
      ptx::named_bar_sync(2, 128);
      const int row0 = u.rg * kTRows;
      const int nrows = min(kTRows, u.blk - row0);
      if (ew == 0 && lane < nrows) {
        ptx::bulk_s2g(out + ((int64_t)(u.blk_off + row0 + lane) * plan.H + u.h) * Dg,
                      sb + Lc::kOffStage + lane * (Dg * 2), Dg * 2);
        ptx::bulk_commit_group();
      }
      if (ew == 0) RTC_CHUNK(11, uc);
      if (ew == 0 && uc < 8) RTC_CTA(3 + uc);
    }
    if (ew == 0) ptx::bulk_wait_group0();
    if (ew == 0) RTC_CTA(11);
  }

  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (warp == kMmaWarp) ptx::tmem_dealloc(tmem, kTmemCols);
}

}  // namespace rtc
}  // namespace dllm
