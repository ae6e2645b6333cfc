// Reuse over per-KV-group key sets (next row N2, GQA; R21): Eq. 4
// for every query head h of request b,
//   O_b[q,h] = softmax_j(tau Q_blk[q,h].K[j,g]) V[j,g],  j in [bs,be) ++ idx(b,g),
// where every head h of KV group g = kv(h) attends to the SAME positions
// (dllm_select_groups writes one set per group into each head's idx slot).
//
// Why a kernel of its own.  With per-head sets (reuse_tc_body.cuh) a work unit is
// one head, and each of the G = H/H_kv heads of a group gathers the group's K/V
// rows again: at C2 (G = 7) the per-head kernel moves 7x the unique bytes.  Here
// a unit is (request, KV group, sub-group of up to kGH = 4 heads, 32-row block
// group): the unit's keys are gathered ONCE and the 4 x 32 query rows of the
// sub-group fill the M = 128 rows of the MMA, so nothing needs transposing (the
// per-head kernel puts keys on the TMEM lanes because one head has only 32 rows):
//   S[4*32 rows x 96 keys]  = [Q_h0; Q_h1; Q_h2; Q_h3] . K_chunk^T       (SS MMA)
//   O[4*32 rows x D]       += P . V_chunk                                (TS MMA: P in TMEM)
// which is the FlashAttention-4 layout of refresh_tc2.cu: thread = query row, row
// max / sum per thread, P written back over S in TMEM as bf16 pairs.
// TMEM: S double buffer 2 x 128 columns (96 used) + O double buffer 2 x 128 = 512.
//
// Roles as in reuse_tc_body.cuh (16 warps): loaders 0-3, 6, 7 (the stacked Q
// rows, 16-byte cp.async row gathers of K/V into a 3-stage ring of SW128 tiles);
// translator 4 (position -> physical row, block table cached in shared memory);
// MMA issuer 5; softmax 8-11 (warp j = head j of the sub-group); epilogue 12-15
// (O / l -> bf16, one contiguous 256-byte row per thread).  Static round-robin
// units over a persistent grid.
#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>

#include "reuse_tc_body.cuh"   // sw128_off, cp_async_arrive_noinc

namespace dllm {
namespace rgs {

using rtc::cp_async_arrive_noinc;
using rtc::sw128_off;

constexpr int kD = 128;
constexpr int kRows = 32;        // query rows per unit and head
constexpr int kGH = 4;           // heads per unit (stacked along N)
constexpr int kN = kGH * kRows;  // MMA M: the sub-group's stacked query rows
constexpr int kChunk = 96;       // keys per ring stage (MMA N of S, K of P.V)
constexpr int kNS = 3;           // ring stages
#ifndef DLLM_RGS_POLY
#define DLLM_RGS_POLY 3
#endif
// every kPolyEvery-th pair of exponentials runs on the FMA pipe (exp2_poly2), the
// rest on MUFU (16/clk/SM): per 96-key row 64 MUFU + 16 polynomial pairs
constexpr int kPolyEvery = DLLM_RGS_POLY;
constexpr int kNT = 4;           // translation ring depth (chunks)
constexpr int kTG = 4;           // chunks translated per batch
constexpr int kLoaders = 6, kTransWarp = 4, kMmaWarp = 5, kSoft0 = 8, kEpi0 = 12, kWarps = 16;
constexpr int kThreads = kWarps * 32;
__device__ __forceinline__ int loader_index(int w) { return w < 4 ? w : (w == 6 || w == 7 ? w - 2 : -1); }

constexpr int kTileK = kChunk * kD * 2;             // [2 atoms][kChunk rows][128 B]
constexpr int kStage = 2 * kTileK;                  // K then V
constexpr int kQTile = kN * kD * 2;                 // 32 KB: [2 atoms][128 rows = 4 heads x 32][128 B]
constexpr int kOffQ = kNS * kStage;
constexpr int kOffOffs = kOffQ + 2 * kQTile;        // [kNT][kChunk] int32
constexpr int kOffL = kOffOffs + kNT * kChunk * 4;  // [2 O buffers][128 rows] row sums
constexpr int kBtMax = 512;                         // block-table entries cached in shared memory
constexpr int kOffBt = kOffL + 2 * kN * 4;
// union mode (per-head sets): per-head position bitmaps of the unit, their union's
// word prefix counts, per-chunk head-membership masks and per-unit key counts
constexpr int kWMax = 256;                          // bitmap words: L <= 8192
constexpr int kMaxUnionLen = 32 * kWMax;
constexpr int kRing = 16;                           // > chunks the translator runs ahead of the softmax
constexpr int kOffBm = kOffBt + kBtMax * 4;         // [kGH][kWMax] u32
// union keys staged in ascending order (position | membership << 24): a batch of
// kTG chunks plus one 1024-position scan step (one bitmap word per lane)
constexpr int kStageKeys = 2048;
static_assert(kStageKeys >= kTG * kChunk + 1024 && (kStageKeys & (kStageKeys - 1)) == 0, "union staging ring");
constexpr int kOffStageK = kOffBm + kGH * kWMax * 4;   // [kStageKeys] int32
constexpr int kOffMask = kOffStageK + kStageKeys * 4;  // [kRing][kGH][kChunk / 32] u32
constexpr int kOffNk = kOffMask + kRing * kGH * (kChunk / 32) * 4;   // [kRing] int32
constexpr int kOffBar = kOffNk + kRing * 4;
constexpr int kNumBars = 2 * kNS + 2 * kNT + 2 * 7 + 1 + 1;
constexpr int kBytes = kOffBar + 8 * kNumBars + 1024;   // + alignment slack
static_assert(kBytes <= 227 * 1024, "reuse_grp shared memory");

constexpr uint32_t kTmemCols = 512;
static_assert(kChunk % 32 == 0 && kChunk <= 128, "S buffer columns");
__device__ __forceinline__ uint32_t tm_s(int b) { return (uint32_t)(b * kN); }
__device__ __forceinline__ uint32_t tm_o(int b) { return (uint32_t)(2 * kN + b * kN); }

#ifdef DLLM_TRACE
// per-CTA timeline (globaltimer ns): [0] start, [1] first offsets published, [2] first S
// issued, [3..10] epilogue: end of unit i, [11] end; CTA 0 per chunk t: [0] published,
// [1] loader issued, [2] S issued, [3] softmax got S, [6] head 0 done, [4] P arrived,
// [5] P.V issued; per unit: [9] row sums published, [10] epilogue got O, [11] stored
static __device__ long long g_rgs[1024][16];
static __device__ long long g_rgs_chunk[16][64];
__device__ __forceinline__ long long rgs_timer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define RGS_CTA(slot)                                                          \
  do {                                                                         \
    if (lane == 0 && blockIdx.x < 1024) g_rgs[blockIdx.x][slot] = rgs_timer(); \
  } while (0)
#define RGS_CHUNK(kind, t)                                                              \
  do {                                                                                  \
    if (lane == 0 && blockIdx.x == 0 && (t) < 64) g_rgs_chunk[kind][t] = rgs_timer();   \
  } while (0)
#else
#define RGS_CTA(slot) \
  do {                \
  } while (0)
#define RGS_CHUNK(kind, t) \
  do {                     \
  } while (0)
#endif

struct GUnit {
  int b, kvh, h0, nh, rg, blk, bs, nk, L, k, blk_off, bt_row;
  int64_t idx_off;
};

// unit -> (request, KV group, head sub-group, row group); the sub-groups of one
// (group, row group) are adjacent units, so they run in the same wave and the
// second gather of the group's rows is served by L2
__device__ __forceinline__ void gdecode(const Plan &pl, int unit, GUnit &u) {
  u.b = plan_find(pl, unit);
  const ReqInfo R = pl.r[u.b];
  const int G = pl.H / pl.H_kv;
  const int nsub = (G + kGH - 1) / kGH;
  u.blk = R.be - R.bs;
  u.bs = R.bs;
  const int ngroups = (u.blk + kRows - 1) / kRows;
  int local = unit - R.unit_off;
  const int sg = local % nsub;
  local /= nsub;
  u.rg = local % ngroups;
  u.kvh = local / ngroups;
  u.h0 = u.kvh * G + sg * kGH;
  u.nh = min(kGH, G - sg * kGH);
  u.nk = u.blk + R.k;   // group sets; union mode: blk + |union|, counted by the translator
  u.L = R.L;
  u.k = R.k;
  u.blk_off = R.blk_off;
  u.bt_row = R.bt_row;
  u.idx_off = R.idx_off + (int64_t)u.h0 * R.k;   // the group's set, read from the sub-group's first head
}

template <bool kUnion>
__global__ void __launch_bounds__(kThreads, 1)
reuse_grp_kernel(const __grid_constant__ Plan plan, const __nv_bfloat16 *__restrict__ q_blk,
                 const __nv_bfloat16 *__restrict__ k_cache, const __nv_bfloat16 *__restrict__ v_cache,
                 const int32_t *__restrict__ idx, __nv_bfloat16 *__restrict__ out) {
  constexpr int D = kD;
  constexpr int CH = D / 8;
  constexpr int NS = kNS;
  const int cta = blockIdx.x, ncta = gridDim.x;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t sb = (raw + 1023u) & ~1023u;
  uint8_t *gb = smem_raw + (sb - raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  const uint32_t b_kvfull = sb + kOffBar;             // [NS] loaders (32*kLoaders noinc)
  const uint32_t b_kvempty = b_kvfull + 8 * NS;       // [NS] MMA commit (P.V done)
  const uint32_t b_ofull_t = b_kvempty + 8 * NS;      // [kNT] translator
  const uint32_t b_oempty_t = b_ofull_t + 8 * kNT;    // [kNT] loaders (kLoaders)
  const uint32_t b_qfull = b_oempty_t + 8 * kNT;      // [2] loaders (32*kLoaders noinc)
  const uint32_t b_qempty = b_qfull + 16;             // [2] MMA commit
  const uint32_t b_sfull = b_qempty + 16;             // [2] MMA commit
  const uint32_t b_pfull = b_sfull + 16;              // [2] softmax warps (4)
  const uint32_t b_ofull = b_pfull + 16;              // [2] MMA commit (unit's last P.V)
  const uint32_t b_ofree = b_ofull + 16;              // [2] epilogue warps (4)
  const uint32_t b_lfull = b_ofree + 16;              // [2] softmax warps (4)
  const uint32_t b_pvdone = b_lfull + 16;             // [1] MMA commit after every P.V
  const uint32_t b_tslot = b_pvdone + 8;
  auto unit_at = [&](int i) -> int { return cta + i * ncta; };
  int32_t *offs = reinterpret_cast<int32_t *>(gb + kOffOffs);

#ifdef DLLM_TRACE
  if (threadIdx.x == 0 && cta < 1024) {
    for (int i = 0; i < 16; ++i) g_rgs[blockIdx.x][i] = 0;
    g_rgs[blockIdx.x][0] = rgs_timer();
  }
#endif
  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) {
      ptx::mbar_init(b_kvfull + 8 * i, 32 * kLoaders + 1);   // + loader 0's release of the translator's data
      ptx::mbar_init(b_kvempty + 8 * i, 1);
    }
    for (int i = 0; i < kNT; ++i) {
      ptx::mbar_init(b_ofull_t + 8 * i, 1);
      ptx::mbar_init(b_oempty_t + 8 * i, kLoaders);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(b_qfull + 8 * i, 32 * kLoaders);
      ptx::mbar_init(b_qempty + 8 * i, 1);
      ptx::mbar_init(b_sfull + 8 * i, 1);
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
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t *>(gb + (b_tslot - sb));

  // (setmaxnreg acts per warpgroup: every warp of a warpgroup requests the same count)
  if (warp < kSoft0) asm volatile("setmaxnreg.dec.sync.aligned.u32 80;\n" ::: "memory");
  if (warp == kTransWarp) {
    // ============================ translator ============================
    int t = 0, bt_cached = -1;
    int *bts = reinterpret_cast<int *>(gb + kOffBt);
    for (int i = 0;; ++i) {
      const int unit = unit_at(i);
      if (unit >= plan.total_units) break;
      GUnit u;
      gdecode(plan, unit, u);
      const int32_t *my_idx = idx + u.idx_off;
      const int32_t *bt = plan.block_table + (int64_t)u.bt_row * plan.pages_per_req;
      const int W = (u.L + 31) >> 5;
      const uint32_t *bm = reinterpret_cast<const uint32_t *>(gb + kOffBm);
      int *stage = reinterpret_cast<int *>(gb + kOffStageK);
      int staged = 0, scan_pos = 0, n_union = 0;
      if constexpr (kUnion) {
        // the sub-group's sets as position bitmaps (heads h0.. are consecutive in idx:
        // one contiguous list of nh * k entries), then the size of their union
        uint32_t *bmw = reinterpret_cast<uint32_t *>(gb + kOffBm);
        for (int j = 0; j < u.nh; ++j)
          for (int w = lane; w < W; w += 32) bmw[j * kWMax + w] = 0u;
        __syncwarp();
        const int total = u.nh * u.k;
        {
          // the next unit's lists go to L2 while this one is built and translated
          const int nu = unit_at(i + 1);
          if (nu < plan.total_units && lane == 0) {
            GUnit v;
            gdecode(plan, nu, v);
            if (v.k > 0) {
              const uintptr_t a0 = reinterpret_cast<uintptr_t>(idx + v.idx_off) & ~uintptr_t(15);
              const uintptr_t a1 =
                  (reinterpret_cast<uintptr_t>(idx + v.idx_off + (int64_t)v.nh * v.k) + 15) & ~uintptr_t(15);
              ptx::bulk_prefetch_l2(reinterpret_cast<const void *>(a0), (uint32_t)(a1 - a0));
            }
          }
        }
        for (int e0 = 0; e0 < total; e0 += 16 * 32) {
          int pv[16];
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            const int e = e0 + q * 32 + lane;
            pv[q] = e < total ? __ldg(my_idx + e) : -1;
          }
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            const int e = e0 + q * 32 + lane;
            const int j = (e >= u.k) + (e >= 2 * u.k) + (e >= 3 * u.k);
            if (pv[q] >= 0) atomicOr(bmw + j * kWMax + (pv[q] >> 5), 1u << (pv[q] & 31));
          }
        }
        __syncwarp();
        int cnt = 0;
        for (int w = lane; w < W; w += 32) {
          uint32_t uw = 0;
          for (int j = 0; j < u.nh; ++j) uw |= bm[j * kWMax + w];
          cnt += __popc(uw);
        }
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        n_union = cnt;
        u.nk = u.blk + n_union;
        if (lane == 0) reinterpret_cast<int *>(gb + kOffNk)[i % kRing] = u.nk;
        RGS_CHUNK(12, i);
        __syncwarp();
      }
      const int nchunks = (u.nk + kChunk - 1) / kChunk;
      const bool bt_smem = plan.pages_per_req <= kBtMax;
      for (int g0 = 0; g0 < nchunks; g0 += kTG) {
        constexpr int Q = kTG * kChunk / 32;
        int pos[Q], off[Q];
        uint32_t memb[Q];
        if constexpr (kUnion) {
          // stream the union in ascending position order into the staging ring until
          // it holds every union key of this batch: 128 positions per step, lane l
          // owning positions scan_pos + 4 l .. + 3 (membership nibbles from the
          // bitmaps, a warp prefix sum for the output slots)
          const int need = min((g0 + kTG) * kChunk - u.blk, n_union);
          while (staged < need) {
            // one bitmap word (32 positions) per lane; the lanes' output offsets are a
            // prefix sum of their counts, formed from ballots of the count bits (no
            // shuffle chain: the translator shares the MIO pipe with the gathers)
            const int w = scan_pos + lane;
            uint32_t bw[kGH], un = 0;
#pragma unroll
            for (int j = 0; j < kGH; ++j) {
              bw[j] = (j < u.nh && w < W) ? bm[j * kWMax + w] : 0u;
              un |= bw[j];
            }
            const int n = __popc(un);
            const uint32_t lt = (1u << lane) - 1u;
            int before = 0, tot = 0;
#pragma unroll
            for (int bit = 0; bit < 6; ++bit) {
              const uint32_t bal = __ballot_sync(0xffffffffu, (n >> bit) & 1);
              before += __popc(bal & lt) << bit;
              tot += __popc(bal) << bit;
            }
            int o = staged + before;
            while (un) {
              const int b = __ffs(un) - 1;
              un &= un - 1u;
              uint32_t m = 0;
#pragma unroll
              for (int j = 0; j < kGH; ++j) m |= ((bw[j] >> b) & 1u) << j;
              stage[o & (kStageKeys - 1)] = (w * 32 + b) | (int)(m << 24);
              ++o;
            }
            staged += tot;
            scan_pos += 32;
          }
          __syncwarp();
          RGS_CHUNK(13, t);
#pragma unroll
          for (int q = 0; q < Q; ++q) {
            const int j = g0 * kChunk + q * 32 + lane;
            if (j >= u.nk) {
              pos[q] = -1;
              memb[q] = 0u;
            } else if (j < u.blk) {   // block keys: every head
              pos[q] = u.bs + j;
              memb[q] = (1u << u.nh) - 1u;
            } else {
              const int v = stage[(j - u.blk) & (kStageKeys - 1)];
              pos[q] = v & 0xffffff;
              memb[q] = (uint32_t)v >> 24;
            }
          }
        } else {
#pragma unroll
          for (int q = 0; q < Q; ++q) {
            const int j = g0 * kChunk + q * 32 + lane;
            pos[q] = j < u.nk ? (j < u.blk ? u.bs + j : __ldg(my_idx + (j - u.blk))) : -1;
          }
        }
        if (g0 == 0 && bt_smem && u.bt_row != bt_cached) {
          __syncwarp();
          for (int i0 = 0; i0 < plan.pages_per_req; i0 += 8 * 32) {
            int v[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const int e = i0 + q * 32 + lane;
              v[q] = e < plan.pages_per_req ? __ldg(bt + e) : 0;
            }
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const int e = i0 + q * 32 + lane;
              if (e < plan.pages_per_req) bts[e] = v[q];
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
        const int ng = min(kTG, nchunks - g0);
#pragma unroll
        for (int c = 0; c < kTG; ++c) {
          if (c >= ng) break;
          const int slot = t % kNT;
          ptx::mbar_wait(b_oempty_t + 8 * slot, ((t / kNT) & 1) ^ 1);
#pragma unroll
          for (int rr = 0; rr < kChunk / 32; ++rr) offs[slot * kChunk + rr * 32 + lane] = off[c * (kChunk / 32) + rr];
          if constexpr (kUnion) {
            uint32_t *mk = reinterpret_cast<uint32_t *>(gb + kOffMask) + (t % kRing) * (kGH * (kChunk / 32));
#pragma unroll
            for (int rr = 0; rr < kChunk / 32; ++rr) {
#pragma unroll
              for (int j = 0; j < kGH; ++j) {
                const uint32_t bits = __ballot_sync(0xffffffffu, (memb[c * (kChunk / 32) + rr] >> j) & 1u);
                if (lane == 0) mk[j * (kChunk / 32) + rr] = bits;
              }
            }
          }
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(b_ofull_t + 8 * slot);
          if (t == 0) RGS_CTA(1);
          RGS_CHUNK(0, t);
          ++t;
        }
      }
    }
  } else if (loader_index(warp) >= 0) {
    // ============================ loaders ============================
    const int li = loader_index(warp);
    const int64_t HD = (int64_t)plan.H * D;
    int t = 0;
    for (int i = 0;; ++i) {
      const int unit = unit_at(i);
      if (unit >= plan.total_units) break;
      GUnit u;
      gdecode(plan, unit, u);
      int nchunks = kUnion ? 1 : (u.nk + kChunk - 1) / kChunk;   // union mode: known at the first chunk
      {
        // the sub-group's query rows, head j at tile rows 32j.. (zero rows past the
        // block; rows of absent heads are left as they are: their S^T / O^T columns
        // are never read)
        const int row0 = u.rg * kRows;
        const int qb = i & 1;
        ptx::mbar_wait(b_qempty + 8 * qb, ((i >> 1) & 1) ^ 1);
        const uint32_t sq = sb + kOffQ + qb * kQTile;
        const int n = u.nh * kRows * CH;
        for (int e = li * 32 + lane; e < n; e += 32 * kLoaders) {
          const int r = e / CH, c = e - r * CH;   // r = 32 j + row
          const int j = r >> 5, rr = r & 31;
          const bool ok = row0 + rr < u.blk;
          const __nv_bfloat16 *src =
              q_blk + (int64_t)(u.blk_off + (ok ? row0 + rr : 0)) * HD + (int64_t)(u.h0 + j) * D + c * 8;
          cp_async16(sq + sw128_off(kN, r, c), src, ok ? 16 : 0);
        }
        cp_async_arrive_noinc(b_qfull + 8 * qb);
      }
      for (int c = 0; c < nchunks; ++c, ++t) {
        const int slot = t % kNT, s = t % NS;
        ptx::mbar_wait(b_ofull_t + 8 * slot, (t / kNT) & 1);
        if (kUnion && c == 0) nchunks = (reinterpret_cast<const int *>(gb + kOffNk)[i % kRing] + kChunk - 1) / kChunk;
        ptx::mbar_wait(b_kvempty + 8 * s, ((t / NS) & 1) ^ 1);
        const uint32_t dk = sb + s * kStage, dv = dk + kTileK;
#pragma unroll 4
        for (int e = li * 32 + lane; e < kChunk * CH; e += 32 * kLoaders) {
          const int r = e / CH, cc = e - r * CH;
          const int off = offs[slot * kChunk + r];
          const int64_t goff = (int64_t)(off < 0 ? 0 : off) * D + cc * 8;
          const int nb = off < 0 ? 0 : 16;
          const uint32_t so = sw128_off(kChunk, r, cc);
          cp_async16(dk + so, k_cache + goff, nb);
          cp_async16(dv + so, v_cache + goff, nb);
        }
        cp_async_arrive_noinc(b_kvfull + 8 * s);
        // (a plain arrive: releases what this lane acquired from the translator -- the
        // unit's key count and the chunk's membership masks -- to the MMA and softmax warps)
        if (li == 0 && lane == 0) ptx::mbar_arrive(b_kvfull + 8 * s);
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(b_oempty_t + 8 * slot);
        if (li == 0) RGS_CHUNK(1, t);
      }
    }
    cp_async_wait<0>();
  } else if (warp == kMmaWarp) {
    // ============================ MMA issuer ============================
    // S(t) goes into S buffer t & 1, which held S(t-2) / P(t-2): P.V(t-2) was issued
    // before it, and tcgen05.mma ops from one thread execute in issue order, so the
    // buffer needs no release barrier of its own.
    constexpr uint32_t idesc_s = ptx::idesc_bf16_f32(kN, kChunk, false, false);   // M = 4 x 32 rows, N = keys
    constexpr uint32_t idesc_o = ptx::idesc_bf16_f32(kN, kD, false, true);        // A = P (TMEM), B = V MN-major
    const uint64_t dq0 = ptx::smem_desc_sw128(sb + kOffQ, 16, 1024);               // stacked Q, K-major A
    const uint64_t dk0 = ptx::smem_desc_sw128(sb, 16, 1024);                       // K tile, K-major B
    const uint64_t dv0 = ptx::smem_desc_sw128(sb + kTileK, kChunk * 128, 1024);    // V tile, MN-major B
    int t = 0;
    int pv_t = -1, pv_s = 0, pv_ob = 0, pv_first = 0, pv_last = 0, pv_uc = 0;
    auto issue_pv = [&]() {
      ptx::mbar_wait(b_pfull + 8 * (pv_t & 1), (pv_t >> 1) & 1);
      if (pv_first) ptx::mbar_wait(b_ofree + 8 * pv_ob, ((pv_uc >> 1) & 1) ^ 1);
      ptx::tc_fence_after();
      const uint64_t v0 = dv0 + (uint64_t)((pv_s * kStage) >> 4);
#pragma unroll
      for (int k = 0; k < kChunk / 16; ++k)
        ptx::mma_ts_elect(tmem + tm_o(pv_ob), tmem + tm_s(pv_t & 1) + (uint32_t)(k * 8),
                          v0 + (uint64_t)((k * 16 * 128) >> 4), idesc_o, (!pv_first || k > 0) ? 1u : 0u);
      ptx::mma_commit_elect(b_kvempty + 8 * pv_s);
      ptx::mma_commit_elect(b_pvdone);
      RGS_CHUNK(5, pv_t);
      if (pv_last) ptx::mma_commit_elect(b_ofull + 8 * pv_ob);
    };
    for (int i = 0;; ++i) {
      const int unit = unit_at(i);
      if (unit >= plan.total_units) break;
      GUnit u;
      gdecode(plan, unit, u);
      int nchunks = kUnion ? 1 : (u.nk + kChunk - 1) / kChunk;
      const int qb = i & 1;
      ptx::mbar_wait(b_qfull + 8 * qb, (i >> 1) & 1);
      for (int c = 0; c < nchunks; ++c, ++t) {
        const int s = t % NS;
        // P.V(t-1) goes out as soon as its P is ready, even when chunk t's rows are
        // still in flight
        while (!ptx::mbar_test_wait(b_kvfull + 8 * s, (t / NS) & 1)) {
          if (pv_t >= 0 && ptx::mbar_test_wait(b_pfull + 8 * (pv_t & 1), (pv_t >> 1) & 1) &&
              (!pv_first || ptx::mbar_test_wait(b_ofree + 8 * pv_ob, ((pv_uc >> 1) & 1) ^ 1))) {
            issue_pv();
            pv_t = -1;
          }
        }
        ptx::mbar_wait(b_kvfull + 8 * s, (t / NS) & 1);
        if (kUnion && c == 0) nchunks = (reinterpret_cast<const int *>(gb + kOffNk)[i % kRing] + kChunk - 1) / kChunk;
        ptx::fence_proxy_async_smem();   // cp.async (generic proxy) data -> tensor core (async proxy)
        ptx::tc_fence_after();
        const uint64_t a0 = dq0 + (uint64_t)((qb * kQTile) >> 4);
        const uint64_t b0 = dk0 + (uint64_t)((s * kStage) >> 4);
#pragma unroll
        for (int k = 0; k < D / 16; ++k) {
          const uint32_t ao = (uint32_t)(((k >> 2) * kN * 128 + (k & 3) * 32) >> 4);
          const uint32_t bo = (uint32_t)(((k >> 2) * kChunk * 128 + (k & 3) * 32) >> 4);
          ptx::mma_ss_elect(tmem + tm_s(t & 1), a0 + ao, b0 + bo, idesc_s, k > 0 ? 1u : 0u);
        }
        ptx::mma_commit_elect(b_sfull + 8 * (t & 1));
        if (t == 0) RGS_CTA(2);
        RGS_CHUNK(2, t);
        if (c == nchunks - 1) ptx::mma_commit_elect(b_qempty + 8 * qb);
        if (pv_t >= 0) issue_pv();
        pv_t = t; pv_s = s; pv_ob = i & 1; pv_first = c == 0; pv_last = c == nchunks - 1; pv_uc = i;
      }
      if (pv_t >= 0) issue_pv();
      pv_t = -1;
    }
  } else if (warp < kEpi0) {
    // ============================ softmax (warps 8-11) ============================
    // Thread = one query row of one head (TMEM lane 32 j + r: warp j = head j of the
    // sub-group), the chunk's keys along the columns: row max and row sum are
    // per-thread, the lazy rescale (2^8) is decided per warp (tcgen05.ld/st are
    // warp-collective).  P goes back into the S columns as packed bf16 pairs, the A
    // operand of the P.V MMA.  A warp whose head is absent (nh < 4) only arrives.
    asm volatile("setmaxnreg.inc.sync.aligned.u32 200;\n" ::: "memory");
    const int sw = warp & 3;
    const float sl2 = plan.scale_log2;
    float *lbuf = reinterpret_cast<float *>(gb + kOffL);
    const uint32_t lane_base = (uint32_t)(sw * 32) << 16;
    int t = 0;
    for (int i = 0;; ++i) {
      const int unit = unit_at(i);
      if (unit >= plan.total_units) break;
      GUnit u;
      gdecode(plan, unit, u);
      int nchunks = kUnion ? 1 : (u.nk + kChunk - 1) / kChunk;
      const int ob = i & 1;
      const bool active = sw < u.nh;
      const uint32_t tO = tmem + lane_base + tm_o(ob);
      float m_used = -INFINITY, lsum = 0.f;
      for (int c = 0; c < nchunks; ++c, ++t) {
        const int b = t & 1;
        const uint32_t tS = tmem + lane_base + tm_s(b);
        ptx::mbar_wait(b_sfull + 8 * b, (t >> 1) & 1);
        ptx::tc_fence_after();
        if (sw == 0) RGS_CHUNK(3, t);
        if constexpr (kUnion) {
          // (complete already -- S(t) was issued after it; acquires the translator's data)
          ptx::mbar_wait(b_kvfull + 8 * (t % NS), (t / NS) & 1);
          if (c == 0) {
            u.nk = reinterpret_cast<const int *>(gb + kOffNk)[i % kRing];
            nchunks = (u.nk + kChunk - 1) / kChunk;
          }
        }
        if (active) {
          uint32_t sr[kChunk];
          DLLM_TMEM_LD32(tS + 0, (sr + 0));
          DLLM_TMEM_LD32(tS + 32, (sr + 32));
          DLLM_TMEM_LD32(tS + 64, (sr + 64));
          ptx::tmem_wait_ld();
          float *x = reinterpret_cast<float *>(sr);
          if constexpr (kUnion) {
            // keys outside this head's own set (and padding): masked
            const uint32_t *mk = reinterpret_cast<const uint32_t *>(gb + kOffMask) +
                                 (t % kRing) * (kGH * (kChunk / 32)) + sw * (kChunk / 32);
#pragma unroll
            for (int rr = 0; rr < kChunk / 32; ++rr) {
              const uint32_t bits = mk[rr];
              if (bits != 0xffffffffu) {
#pragma unroll
                for (int e = 0; e < 32; ++e)
                  if (!((bits >> e) & 1u)) x[rr * 32 + e] = -INFINITY;
              }
            }
          } else {
            const int key_end = u.nk - c * kChunk;   // keys >= key_end of this chunk are padding
            if (key_end < kChunk) {
#pragma unroll
              for (int n = 0; n < kChunk; ++n)
                if (n >= key_end) x[n] = -INFINITY;
            }
          }
          float mx;
          {
            float m8[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) m8[e] = fmax3(x[e], x[8 + e], x[16 + e]);
#pragma unroll
            for (int g = 3; g < kChunk / 8; g += 2) {
#pragma unroll
              for (int e = 0; e < 8; ++e) m8[e] = g + 1 < kChunk / 8 ? fmax3(m8[e], x[8 * g + e], x[8 * g + 8 + e])
                                                                      : fmaxf(m8[e], x[8 * g + e]);
            }
            mx = fmax3(fmax3(m8[0], m8[1], m8[2]), fmax3(m8[3], m8[4], m8[5]), fmaxf(m8[6], m8[7])) * sl2;
          }
          if (c == 0) {
            m_used = mx;
          } else {
            const bool need = mx > m_used + 8.f;
            if (__any_sync(0xffffffffu, need)) {
              // O holds P(t-1).V: wait for that P.V, rescale this warp's rows
              ptx::mbar_wait(b_pvdone, (t - 1) & 1);
              ptx::tc_fence_after();
              const float alpha = need ? fast_exp2(m_used - mx) : 1.f;
              if (need) {
                lsum *= alpha;
                m_used = mx;
              }
#pragma unroll 1
              for (int cc = 0; cc < D; cc += 32) {
                uint32_t o[32];
                DLLM_TMEM_LD32(tO + cc, o);
                ptx::tmem_wait_ld();
#pragma unroll
                for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * alpha);
                DLLM_TMEM_ST32(tO + cc, o);
              }
            }
          }
          const uint64_t sl2x2 = pack_f32x2(sl2, sl2);
          const uint64_t negm = pack_f32x2(-m_used, -m_used);
          uint64_t acc[4] = {0ull, 0ull, 0ull, 0ull};
          uint32_t pk[kChunk / 2];
#pragma unroll
          for (int e = 0; e < kChunk / 2; ++e) {
            const uint64_t xx = ffma2(pack_f32x2(x[2 * e], x[2 * e + 1]), sl2x2, negm);
            float p0, p1;
            if (e % kPolyEvery == 0) {
              unpack_f32x2(exp2_poly2(xx), p0, p1);   // FMA pipe
            } else {
              unpack_f32x2(xx, p0, p1);
              p0 = fast_exp2(p0);                     // MUFU
              p1 = fast_exp2(p1);
            }
            acc[e & 3] = fadd2(acc[e & 3], pack_f32x2(p0, p1));
            pk[e] = pack_bf16(p0, p1);
          }
          DLLM_TMEM_ST32(tS, pk);
          DLLM_TMEM_ST16(tS + 32, (pk + 32));
          float a0, a1, a2, a3;
          unpack_f32x2(fadd2(acc[0], acc[1]), a0, a1);
          unpack_f32x2(fadd2(acc[2], acc[3]), a2, a3);
          lsum += (a0 + a1) + (a2 + a3);
          ptx::tmem_wait_st();
        }
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(b_pfull + 8 * b);
        if (sw == 0) RGS_CHUNK(4, t);
      }
      // unit end: the row sums -> shared memory for the epilogue
      ptx::mbar_wait(b_ofree + 8 * ob, ((i >> 1) & 1) ^ 1);
      lbuf[ob * kN + sw * 32 + lane] = lsum;
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(b_lfull + 8 * ob);
      if (sw == 0) RGS_CHUNK(9, i);
    }
  } else {
    // ============================ epilogue (warps 12-15) ============================
    // Thread = one output row (TMEM lane = 32 j + r: head h0 + j, block row row0 + r):
    // O / l -> bf16, one contiguous 256-byte row per thread (16-byte stores).
    asm volatile("setmaxnreg.inc.sync.aligned.u32 152;\n" ::: "memory");
    const int ew = warp & 3;
    const uint32_t lane_base = (uint32_t)(ew * 32) << 16;
    const float *lbuf = reinterpret_cast<const float *>(gb + kOffL);
    for (int i = 0;; ++i) {
      const int unit = unit_at(i);
      if (unit >= plan.total_units) break;
      GUnit u;
      gdecode(plan, unit, u);
      const int ob = i & 1;
      ptx::mbar_wait(b_lfull + 8 * ob, (i >> 1) & 1);
      ptx::mbar_wait(b_ofull + 8 * ob, (i >> 1) & 1);
      ptx::tc_fence_after();
      if (ew == 0) RGS_CHUNK(10, i);
      const int row = u.rg * kRows + lane;
      if (ew < u.nh) {
        const float l = lbuf[ob * kN + ew * 32 + lane];
        const float inv = l > 0.f ? __frcp_rn(l) : 0.f;
        uint4 *dst = reinterpret_cast<uint4 *>(out + ((int64_t)(u.blk_off + row) * plan.H + u.h0 + ew) * D);
#pragma unroll 1
        for (int cc = 0; cc < D; cc += 32) {
          uint32_t o[32];
          DLLM_TMEM_LD32(tmem + lane_base + tm_o(ob) + cc, o);
          ptx::tmem_wait_ld();
          if (row < u.blk) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              uint4 v;
              v.x = pack_bf16(__uint_as_float(o[8 * q + 0]) * inv, __uint_as_float(o[8 * q + 1]) * inv);
              v.y = pack_bf16(__uint_as_float(o[8 * q + 2]) * inv, __uint_as_float(o[8 * q + 3]) * inv);
              v.z = pack_bf16(__uint_as_float(o[8 * q + 4]) * inv, __uint_as_float(o[8 * q + 5]) * inv);
              v.w = pack_bf16(__uint_as_float(o[8 * q + 6]) * inv, __uint_as_float(o[8 * q + 7]) * inv);
              dst[cc / 8 + q] = v;
            }
          }
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(b_ofree + 8 * ob);
      if (ew == 0) RGS_CHUNK(11, i);
      if (ew == 0 && i < 8) RGS_CTA(3 + i);
    }
    if (ew == 0) RGS_CTA(11);
  }

  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (warp == kMmaWarp) ptx::tmem_dealloc(tmem, kTmemCols);
}

int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

}  // namespace rgs

#ifdef DLLM_TRACE
extern "C" __attribute__((visibility("default"))) int dllm_trace_rgs_read(long long *cta, long long *chunk) {
  cudaError_t e = cudaMemcpyFromSymbol(cta, rgs::g_rgs, sizeof(rgs::g_rgs));
  if (e == cudaSuccess) e = cudaMemcpyFromSymbol(chunk, rgs::g_rgs_chunk, sizeof(rgs::g_rgs_chunk));
  return (int)e;
}
#endif

// work units of request b: KV groups x head sub-groups x 32-row groups
int reuse_grp_units(int H, int H_kv, int blk) {
  const int G = H / H_kv;
  return H_kv * ((G + rgs::kGH - 1) / rgs::kGH) * ((blk + rgs::kRows - 1) / rgs::kRows);
}

bool reuse_grp_supported(int D) { return D == rgs::kD; }

// union mode keeps per-head position bitmaps of the whole sequence in shared memory
int reuse_union_max_len() { return rgs::kMaxUnionLen; }

cudaError_t launch_reuse_grp(const Plan &plan, const void *q_blk, const void *k_cache, const void *v_cache,
                             const int32_t *idx, void *out, bool union_sets, cudaStream_t st) {
  using namespace rgs;
  if (plan.D != kD) return cudaErrorInvalidValue;
  static std::once_flag once;
  static cudaError_t attr = cudaSuccess;
  std::call_once(once, [] {
    attr = cudaFuncSetAttribute(reuse_grp_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kBytes);
    if (attr == cudaSuccess)
      attr = cudaFuncSetAttribute(reuse_grp_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kBytes);
  });
  if (attr != cudaSuccess) return attr;
  // the fewest CTAs that keep the number of static rounds (as reuse_tc_grid)
  const int rounds = (plan.total_units + num_sms() - 1) / num_sms();
  const int tail = plan.total_units - (rounds - 1) * num_sms();
  const int grid = rounds <= 0 ? 0 : (rounds > 1 && 4 * tail < num_sms()) ? num_sms() : (plan.total_units + rounds - 1) / rounds;
  if (grid <= 0) return cudaSuccess;
  return launch_pdl(union_sets ? reuse_grp_kernel<true> : reuse_grp_kernel<false>, dim3(grid), dim3(kThreads),
                    (size_t)kBytes, st, plan, (const __nv_bfloat16 *)q_blk, (const __nv_bfloat16 *)k_cache,
                    (const __nv_bfloat16 *)v_cache, idx, (__nv_bfloat16 *)out);
}

}  // namespace dllm
