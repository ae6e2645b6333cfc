// Refresh dense attention on the 5th-generation tensor cores (sm_100a):
// Eq. 3 (§2.3) + the raw per-head importance of Eq. 6
// (inner term, §4.5) fused into the softmax pass.
//
// Persistent, warp-specialised, one CTA per SM (384 threads):
//   warp 0      TMA producer: Q tiles (3-D map over [sum L, H, D]) and K/V
//               tiles straight out of the paged cache (4-D map over
//               [pages, H_kv, P, D], one box per page slice) into a 2-stage
//               K ring and a 2-stage V ring, 128-byte swizzled.
//   warp 1      MMA issuer (one thread) + TMEM owner: S_i = Q_i K^T
//               (tcgen05.mma SS, M=128 N=128 K=16 steps, fp32 in TMEM) and
//               O_i += P_i V (tcgen05.mma TS: P read from TMEM, V from smem).
//   warps 4-7   softmax warpgroup 0 (Q tile 0), one thread per query row;
//   warps 8-11  softmax warpgroup 1 (Q tile 1).  Each reads its S tile from
//               TMEM (tcgen05.ld), does the online softmax in fp32 (log2
//               domain, lazy rescale: O is only rescaled when the running max
//               grows by more than 2^8), writes P as bf16 back into the S
//               columns (tcgen05.st) and finally normalises O and stores it.
// The two Q tiles of a unit ping-pong: while one warpgroup runs its softmax
// the tensor core runs the other tile's P.V and next Q.K^T.
//
// TMEM (512 columns): S0 [0,128), S1 [128,256), O0 [256,256+D), O1 [384,384+D).
// P_i aliases the first 64 columns of S_i (bf16 pairs).
//
// Work unit = (request b, query head h, pair of 128-row Q tiles).  A request
// has ceil(L/128) regular tiles; when its active block straddles a tile
// boundary one extra tile with origin bs is added whose O is discarded and
// which only serves the importance epilogue, so that exactly one tile per
// (b, h) holds all block rows.  Its softmax warps reduce the UNSCALED S over
// the block rows column-wise (warp transpose-reduce + shared memory) and
// write raw[b, h, m] for every key m (R1, R8).
// Keys past L in the last K/V tile are masked (-inf) and their V rows are
// zeroed in shared memory, so cache slots past L may hold anything (even NaN).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdint.h>

#include "common.cuh"
#include "plan.h"
#include "tc_ptx.cuh"

#ifdef DLLM_TRACE
__device__ long long g_trace[16][512];
#define TRACE(kind, it)                                                    \
  do {                                                                     \
    if (blockIdx.x == 0 && (it) < 512) g_trace[kind][it] = clock64();      \
  } while (0)
extern "C" __attribute__((visibility("default"))) int dllm_trace_read(long long *host) {
  return (int)cudaMemcpyFromSymbol(host, g_trace, sizeof(g_trace));
}
#else
#define TRACE(kind, it)
#endif

namespace dllm {
namespace {

constexpr int TBM = 128;            // query rows per tile
constexpr int TBN = 128;            // keys per K/V tile
constexpr int TC_THREADS = 384;
constexpr float kRescaleLog2 = 8.0f;
#ifndef DLLM_POLY_PAIRS
#define DLLM_POLY_PAIRS 0
#endif
constexpr int kPolyPairs = DLLM_POLY_PAIRS;
#ifndef DLLM_SPEC_MAX
#define DLLM_SPEC_MAX 0
#endif
#ifndef DLLM_PINGPONG
#define DLLM_PINGPONG 0
#endif
#ifndef DLLM_L2_PREFETCH
#define DLLM_L2_PREFETCH 0
#endif
constexpr bool kSpecMax = DLLM_SPEC_MAX;     // exponentials with the running max, check afterwards
constexpr bool kPingPong = DLLM_PINGPONG;    // strict MUFU turn-taking between the softmax warpgroups
constexpr bool kL2Prefetch = DLLM_L2_PREFETCH;   // of every 8 column pairs, this many use the FMA-pipe exp2
constexpr int kPrefetchLead = 4;     // K/V tiles before the end of a unit at which the next one is prefetched
constexpr int kPrefetchTiles = 2;    // K/V tiles of the next unit prefetched into L2

template <int D>
struct TcCfg {
  static constexpr int kChunks = D / 64;                 // 128-byte swizzle chunks per row
  static constexpr int kQBytes = TBM * D * 2;
  static constexpr int kKVBytes = TBN * D * 2;
  static constexpr int kOffQ = 0;                        // 2 Q tiles
  static constexpr int kOffK = 2 * kQBytes;              // 2 K stages
  static constexpr int kOffV = kOffK + 2 * kKVBytes;     // 2 V stages
  static constexpr int kOffSc = kOffV + 2 * kKVBytes;    // [2 wg][2 buf][4 warps][128] f32
  static constexpr int kOffBar = kOffSc + 2 * 2 * 4 * 128 * 4;
  static constexpr int kOffReq = kOffBar + 256;          // ReqInfo[nreq] copy of the plan
  static constexpr int kBytes = kOffReq + kMaxReqPerLaunch * (int)sizeof(ReqInfo) + 1024;  // + alignment slack
};

// barrier slots (8 bytes each)
enum : int {
  B_QFULL = 0, B_QEMPTY = 1, B_KFULL = 2, B_KEMPTY = 4, B_VFULL = 6, B_VEMPTY = 8, B_VZ = 10,
  B_SFULL = 11, B_PFULL = 13, B_OFULL = 15, B_TMEMSLOT = 17
};
__host__ __device__ constexpr uint32_t tmem_s(int i) { return i ? 128u : 0u; }
__host__ __device__ constexpr uint32_t tmem_o(int i) { return i ? 384u : 256u; }

__host__ __device__ __forceinline__ int tc_regular_tiles(int L) { return (L + TBM - 1) / TBM; }
__host__ __device__ __forceinline__ bool tc_straddles(int bs, int be) { return (bs / TBM) != ((be - 1) / TBM); }

struct Unit {
  int h, kvh;
  int L, bs, be;
  int q_off, bt_row;
  int64_t score_off;
  int n;          // K/V tiles
  int tile[2];    // tile ids (tile[1] = -1: single-tile unit)
  int origin[2];
  int write_end[2];
  bool scores_on[2];
};

// unit -> (request, head, tile pair); `rs` is the shared-memory copy of the plan's requests
__device__ __forceinline__ void decode_unit(const Plan &pl, const ReqInfo *rs, int unit, Unit &u) {
  int lo = 0, hi = pl.nreq - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (rs[mid].unit_off <= unit) lo = mid; else hi = mid - 1;
  }
  const ReqInfo &R = rs[lo];
  u.L = R.L; u.bs = R.bs; u.be = R.be;
  u.q_off = R.q_off; u.bt_row = R.bt_row; u.score_off = R.score_off;
  const int nreg = tc_regular_tiles(u.L);
  const bool extra = pl.with_scores && tc_straddles(u.bs, u.be);
  const int ntiles = nreg + (extra ? 1 : 0);
  const int npairs = (ntiles + 1) >> 1;
  const int local = unit - R.unit_off;
  u.h = local / npairs;
  const int p = (local - u.h * npairs + u.h) % npairs;   // rotate pairs by head (see refresh_tc2.cu)
  u.kvh = u.h / (pl.H / pl.H_kv);
  u.n = (u.L + TBN - 1) / TBN;
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int t = 2 * p + i;
    u.tile[i] = t < ntiles ? t : -1;
    u.origin[i] = t < nreg ? t * TBM : u.bs;
    u.write_end[i] = t < nreg ? u.L : 0;
    u.scores_on[i] = pl.with_scores && t < ntiles && (t == nreg || (!extra && t == u.bs / TBM));
  }
}

template <int D>
__global__ void __launch_bounds__(TC_THREADS, 1)
refresh_tc_kernel(const __grid_constant__ Plan plan, const __grid_constant__ CUtensorMap tm_q,
                  const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
                  __nv_bfloat16 *__restrict__ out, float *__restrict__ scores) {
  using C = TcCfg<D>;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_u32 = smem_u32(smem_raw);
  const uint32_t sb = (raw_u32 + 1023u) & ~1023u;
  uint8_t *gb = smem_raw + (sb - raw_u32);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  auto bar = [&](int i) { return sb + C::kOffBar + 8u * (uint32_t)i; };

  ReqInfo *rs = reinterpret_cast<ReqInfo *>(gb + C::kOffReq);
  for (int i = threadIdx.x; i < plan.nreq; i += blockDim.x) rs[i] = plan.r[i];
  if (threadIdx.x == 0) {
    ptx::mbar_init(bar(B_QFULL), 1);
    ptx::mbar_init(bar(B_QEMPTY), 1);
    for (int s = 0; s < 2; ++s) {
      ptx::mbar_init(bar(B_KFULL + s), 1);
      ptx::mbar_init(bar(B_KEMPTY + s), 1);
      ptx::mbar_init(bar(B_VFULL + s), 1);
      ptx::mbar_init(bar(B_VEMPTY + s), 1);
      ptx::mbar_init(bar(B_SFULL + s), 1);
      ptx::mbar_init(bar(B_PFULL + s), 4);
      ptx::mbar_init(bar(B_OFULL + s), 1);
    }
    ptx::mbar_init(bar(B_VZ), 1);
    ptx::fence_mbar_init();
    ptx::tma_prefetch_desc(&tm_q);
    ptx::tma_prefetch_desc(&tm_k);
    ptx::tma_prefetch_desc(&tm_v);
  }
  if (warp == 1) {
    ptx::tmem_alloc(bar(B_TMEMSLOT), 512);
    ptx::tmem_relinquish();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t *>(gb + C::kOffBar + 8 * B_TMEMSLOT);
  // register rebalancing (per role branch): the producer / MMA warpgroup needs
  // few registers, the softmax warpgroups hold a full 128-column S row per thread

  if (warp == 0) {
    // ============================ TMA producer ============================
    asm volatile("setmaxnreg.dec.sync.aligned.u32 104;\n" ::: "memory");
    int it = 0, ucnt = 0;
    const int boxrows = plan.page_size < TBN ? plan.page_size : TBN;
    const int nsub = TBN / boxrows;
    const uint32_t boxbytes = (uint32_t)boxrows * 128u;
    for (int unit = blockIdx.x; unit < plan.total_units; unit += gridDim.x, ++ucnt) {
      Unit u;
      decode_unit(plan, rs, unit, u);
      const int32_t *bt = plan.block_table + (int64_t)u.bt_row * plan.pages_per_req;
      if (lane == 0) {
        ptx::mbar_wait(bar(B_QEMPTY), (ucnt & 1) ^ 1);
        const int ntile = u.tile[1] >= 0 ? 2 : 1;
        ptx::mbar_arrive_expect_tx(bar(B_QFULL), (uint32_t)(ntile * C::kQBytes));
        for (int i = 0; i < ntile; ++i)
          for (int c = 0; c < C::kChunks; ++c)
            ptx::tma_load_3d(sb + C::kOffQ + i * C::kQBytes + c * TBM * 128, &tm_q, bar(B_QFULL), c * 64, u.h,
                             u.q_off + u.origin[i]);
      }
      for (int j = 0; j < u.n; ++j, ++it) {
        const int s = it & 1;
        const uint32_t ph = (it >> 1) & 1;
        const int key_end = min(TBN, u.L - j * TBN);      // valid keys in this tile
        if (kL2Prefetch && j == (u.n > kPrefetchLead ? u.n - kPrefetchLead : 0)) {
          // warm L2 with the next unit's Q tiles and first K/V tiles, so that the
          // unit boundary does not wait a full HBM round trip (all SMs cross unit
          // boundaries at about the same time)
          const int nu = unit + gridDim.x;
          if (nu < plan.total_units) {
            Unit v;
            decode_unit(plan, rs, nu, v);
            const int nt = v.tile[1] >= 0 ? 2 : 1;
            if (lane < nt * C::kChunks)
              ptx::tma_prefetch_3d(&tm_q, (lane % C::kChunks) * 64, v.h, v.q_off + v.origin[lane / C::kChunks]);
            const int32_t *btn = plan.block_table + (int64_t)v.bt_row * plan.pages_per_req;
            const int ntl = min(v.n, kPrefetchTiles);
            for (int e = lane; e < ntl * nsub; e += 32) {
              const int key0 = (e / nsub) * TBN + (e % nsub) * boxrows;
              if (key0 < v.L) {
                const int page = __ldg(btn + (key0 >> plan.page_shift));
                const int slot = key0 & (plan.page_size - 1);
                for (int c = 0; c < C::kChunks; ++c) {
                  ptx::tma_prefetch_4d(&tm_k, c * 64, slot, v.kvh, page);
                  ptx::tma_prefetch_4d(&tm_v, c * 64, slot, v.kvh, page);
                }
              }
            }
          }
          __syncwarp();
        }
        if (lane == 0) {
          int nvalid = 0;
          for (int sbx = 0; sbx < nsub; ++sbx) nvalid += (sbx * boxrows < key_end);
          const uint32_t bytes = (uint32_t)(nvalid * C::kChunks) * boxbytes;
          ptx::mbar_wait(bar(B_KEMPTY + s), ph ^ 1);
          ptx::mbar_arrive_expect_tx(bar(B_KFULL + s), bytes);
          for (int sbx = 0; sbx < nvalid; ++sbx) {
            const int key0 = j * TBN + sbx * boxrows;
            const int page = __ldg(bt + (key0 >> plan.page_shift));
            const int slot = key0 & (plan.page_size - 1);
            for (int c = 0; c < C::kChunks; ++c)
              ptx::tma_load_4d(sb + C::kOffK + s * C::kKVBytes + c * TBN * 128 + sbx * boxrows * 128, &tm_k,
                               bar(B_KFULL + s), c * 64, slot, u.kvh, page);
          }
          ptx::mbar_wait(bar(B_VEMPTY + s), ph ^ 1);
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
  } else if (warp == 1) {
    // ============================ MMA issuer ============================
    asm volatile("setmaxnreg.dec.sync.aligned.u32 104;\n" ::: "memory");
    {
      constexpr uint32_t idesc_qk = ptx::idesc_bf16_f32(TBM, TBN, false, false);
      constexpr uint32_t idesc_pv = ptx::idesc_bf16_f32(TBM, D, false, true);
      int it = 0, ucnt = 0, vzc = 0, pc[2] = {0, 0};
      for (int unit = blockIdx.x; unit < plan.total_units; unit += gridDim.x, ++ucnt) {
        Unit u;
        decode_unit(plan, rs, unit, u);
        const bool two = u.tile[1] >= 0;
        auto qk = [&](int i, int stage) {
#pragma unroll
          for (int k = 0; k < D / 16; ++k) {
            const uint32_t off = (uint32_t)((k >> 2) * TBM * 128 + (k & 3) * 32);
            const uint64_t a = ptx::smem_desc_sw128(sb + C::kOffQ + i * C::kQBytes + off, 16, 1024);
            const uint64_t b = ptx::smem_desc_sw128(sb + C::kOffK + stage * C::kKVBytes + off, 16, 1024);
            ptx::mma_ss_elect(tmem + tmem_s(i), a, b, idesc_qk, k > 0);
          }
        };
        auto pv = [&](int i, int stage, bool acc) {
#pragma unroll
          for (int k = 0; k < TBN / 16; ++k) {
            const uint64_t b = ptx::smem_desc_sw128(sb + C::kOffV + stage * C::kKVBytes + k * 16 * 128,
                                                    TBN * 128, 1024);
            ptx::mma_ts_elect(tmem + tmem_o(i), tmem + tmem_s(i) + (uint32_t)(k * 8), b, idesc_pv, (acc || k > 0) ? 1u : 0u);
          }
        };
        ptx::mbar_wait(bar(B_QFULL), ucnt & 1);
        ptx::tc_fence_after();
        {
          const int s0 = it & 1;
          ptx::mbar_wait(bar(B_KFULL + s0), (it >> 1) & 1);
          ptx::tc_fence_after();
          qk(0, s0);
          ptx::mma_commit_elect(bar(B_SFULL + 0));
          if (two) {
            qk(1, s0);
            ptx::mma_commit_elect(bar(B_SFULL + 1));
          }
          ptx::mma_commit_elect(bar(B_KEMPTY + s0));
          if (u.n == 1) ptx::mma_commit_elect(bar(B_QEMPTY));
        }
        for (int j = 0; j < u.n; ++j) {
          const int s = (it + j) & 1;
          const bool has_next = j + 1 < u.n;
          const int sn = (it + j + 1) & 1;
          if (lane == 0) TRACE(10, it + j);
          ptx::mbar_wait(bar(B_VFULL + s), ((it + j) >> 1) & 1);
          if (j == u.n - 1 && (u.L % TBN) != 0) {
            ptx::mbar_wait(bar(B_VZ), vzc & 1);
            ++vzc;
          }
          if (lane == 0) TRACE(11, it + j);
          ptx::tc_fence_after();
          if (lane == 0) TRACE(6, pc[0]);
          ptx::mbar_wait(bar(B_PFULL + 0), pc[0] & 1);
          if (lane == 0) TRACE(7, pc[0]);
          ++pc[0];
          ptx::tc_fence_after();
          pv(0, s, j > 0);
          if (!has_next) ptx::mma_commit_elect(bar(B_OFULL + 0));
          if (has_next) {
            ptx::mbar_wait(bar(B_KFULL + sn), ((it + j + 1) >> 1) & 1);
            ptx::tc_fence_after();
            qk(0, sn);
            ptx::mma_commit_elect(bar(B_SFULL + 0));
            if (!two && j + 1 == u.n - 1) ptx::mma_commit_elect(bar(B_QEMPTY));
          }
          if (two) {
            if (lane == 0) TRACE(8, pc[1]);
            ptx::mbar_wait(bar(B_PFULL + 1), pc[1] & 1);
            if (lane == 0) TRACE(9, pc[1]);
            ++pc[1];
            ptx::tc_fence_after();
            pv(1, s, j > 0);
            if (!has_next) ptx::mma_commit_elect(bar(B_OFULL + 1));
            if (has_next) {
              qk(1, sn);
              ptx::mma_commit_elect(bar(B_SFULL + 1));
              if (j + 1 == u.n - 1) ptx::mma_commit_elect(bar(B_QEMPTY));
            }
          }
          if (has_next) ptx::mma_commit_elect(bar(B_KEMPTY + sn));
          ptx::mma_commit_elect(bar(B_VEMPTY + s));
        }
        it += u.n;
      }
    }
    __syncwarp();
  } else if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 104;\n" ::: "memory");
  } else {
    // ============================ softmax warpgroups ============================
    asm volatile("setmaxnreg.inc.sync.aligned.u32 192;\n" ::: "memory");
    const int wg = (warp - 4) >> 2;
    const int wq = warp & 3;                       // TMEM lane quarter
    const int row = wq * 32 + lane;                // row of the Q tile == TMEM lane
    const uint32_t lane_off = (uint32_t)(wq * 32) << 16;
    const uint32_t tS = tmem + lane_off + tmem_s(wg);
    const uint32_t tO = tmem + lane_off + tmem_o(wg);
    float *sbuf = reinterpret_cast<float *>(gb + C::kOffSc) + wg * (2 * 4 * 128);
    const float sl2 = plan.scale_log2;
    const int64_t HD = (int64_t)plan.H * D;
    int sc = 0, oc = 0;
    for (int unit = blockIdx.x; unit < plan.total_units; unit += gridDim.x) {
      Unit u;
      decode_unit(plan, rs, unit, u);
      if ((wg ? u.tile[1] : u.tile[0]) < 0) continue;
      const int origin = (wg ? u.origin[1] : u.origin[0]);
      const bool sc_on = (wg ? u.scores_on[1] : u.scores_on[0]) && scores != nullptr;
      const int rb0 = u.bs - origin, rb1 = u.be - origin;    // block rows within the tile
      const bool in_blk = sc_on && row >= rb0 && row < rb1;
      float m_used = -INFINITY, lsum = 0.f;
      for (int j = 0; j < u.n; ++j) {
        if ((threadIdx.x & 127) == 0) TRACE(0 + wg, sc);
        ptx::mbar_wait(bar(B_SFULL + wg), sc & 1);
        if ((threadIdx.x & 127) == 0) TRACE(2 + wg, sc);
        ++sc;
        ptx::tc_fence_after();
        uint32_t sr[128];
        DLLM_TMEM_LD32(tS + 0, (sr + 0));
        DLLM_TMEM_LD32(tS + 32, (sr + 32));
        DLLM_TMEM_LD32(tS + 64, (sr + 64));
        DLLM_TMEM_LD32(tS + 96, (sr + 96));
        ptx::tmem_wait_ld();
        if (threadIdx.x == 128) TRACE(12, sc - 1);
        float *s = reinterpret_cast<float *>(sr);
        if (sc_on) {
          float *buf = sbuf + (j & 1) * (4 * 128);
          const bool warp_blk = (wq * 32 < rb1) && (wq * 32 + 32 > rb0);
          if (warp_blk) {
#pragma unroll
            for (int c = 0; c < 4; ++c) {
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
              buf[wq * 128 + c * 32 + lane] = v[0];
            }
          }
          ptx::named_bar_sync(1 + wg, 128);
          float m = -INFINITY;
#pragma unroll
          for (int w2 = 0; w2 < 4; ++w2)
            if ((w2 * 32 < rb1) && (w2 * 32 + 32 > rb0)) m = fmaxf(m, buf[w2 * 128 + row]);
          const int key = j * TBN + row;
          if (key < u.L) scores[u.score_off + (int64_t)u.h * u.L + key] = m;
        }
        if (j == u.n - 1) {
          const int key_end = u.L - j * TBN;
          if (key_end < TBN) {
#pragma unroll
            for (int c = 0; c < 128; ++c)
              if (c >= key_end) s[c] = -INFINITY;
          }
        }
        // Softmax with a speculative (stale) max: P = exp2(s*tau*log2e - m_used) is
        // computed with the running max of the previous tiles while the row max of
        // this tile is reduced alongside on the ALU pipe; only if it exceeds m_used
        // by more than 2^8 (rare after the first tile) is O rescaled and P redone
        // from S (still intact in TMEM).  The first tile of a unit takes its max first.
        auto rowmax = [&](const float *v) {
          float t[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) t[i] = fmax3(v[i], v[8 + i], v[16 + i]);
#pragma unroll
          for (int c = 24; c < 120; c += 16)
#pragma unroll
            for (int i = 0; i < 8; ++i) t[i] = fmax3(t[i], v[c + i], v[c + 8 + i]);
#pragma unroll
          for (int i = 0; i < 8; ++i) t[i] = fmaxf(t[i], v[120 + i]);
          return fmax3(fmax3(t[0], t[1], t[2]), fmax3(t[3], t[4], t[5]), fmaxf(t[6], t[7]));
        };
        // MUFU turn-taking: in a two-tile unit the warpgroups run their exponential
        // passes strictly alternately (WG0 j, WG1 j, WG0 j+1, ...) so that each pass
        // has the SM's 16 ex2/clk to itself while the tensor core works on the other tile
        const bool pingpong = kPingPong && u.tile[1] >= 0;
        if (pingpong) {
          if (wg == 0 && j > 0) ptx::named_bar_sync(3, 256);
          if (wg == 1) ptx::named_bar_sync(4, 256);
        }
        if (threadIdx.x == 128) TRACE(13, sc - 1);
        auto rescale_o = [&](float alpha) {
#pragma unroll 1
          for (int c = 0; c < D; c += 32) {
            uint32_t o[32];
            DLLM_TMEM_LD32(tO + c, o);
            ptx::tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
            DLLM_TMEM_ST32(tO + c, o);
          }
        };
        if (!kSpecMax) {
          // exact row max first, lazy rescale of O before the exponentials
          const float mx = rowmax(s) * sl2;
          if (j == 0) {
            m_used = mx;
          } else {
            const bool need = mx > m_used + kRescaleLog2;
            if (__any_sync(0xffffffffu, need)) {
              const float alpha = need ? fast_exp2(m_used - mx) : 1.f;
              if (need) {
                lsum *= alpha;
                m_used = mx;
              }
              rescale_o(alpha);
            }
          }
        } else if (j == 0) {
          m_used = rowmax(s) * sl2;
        }
        uint32_t pk[64];
        float lpart, mxr;
        auto exp_pass = [&](const float *v) {
          const uint64_t sl2x2 = pack_f32x2(sl2, sl2);
          const uint64_t negm = pack_f32x2(-m_used, -m_used);
          uint64_t acc[4] = {0ull, 0ull, 0ull, 0ull};
          float tm[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
          for (int c = 0; c < 64; ++c) {
            const int i = 2 * c;
            tm[c & 3] = fmax3(tm[c & 3], v[i], v[i + 1]);
            const uint64_t x = ffma2(pack_f32x2(v[i], v[i + 1]), sl2x2, negm);
            float p0, p1;
            if ((c & 7) < kPolyPairs) {
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
          float a0, a1, a2, a3;
          unpack_f32x2(fadd2(acc[0], acc[1]), a0, a1);
          unpack_f32x2(fadd2(acc[2], acc[3]), a2, a3);
          lpart = (a0 + a1) + (a2 + a3);
          mxr = fmaxf(fmaxf(tm[0], tm[1]), fmaxf(tm[2], tm[3]));
        };
        exp_pass(s);
        if (pingpong) {
          if (wg == 0) ptx::named_bar_arrive(4, 256);
          if (wg == 1 && j + 1 < u.n) ptx::named_bar_arrive(3, 256);
        }
        if (threadIdx.x == 128) TRACE(14, sc - 1);
        if (kSpecMax && j > 0) {
          const float mx = mxr * sl2;
          const bool need = mx > m_used + kRescaleLog2;
          // tcgen05.ld/st are warp-collective: the slow path is taken warp-uniformly
          if (__any_sync(0xffffffffu, need)) {
            const float alpha = need ? fast_exp2(m_used - mx) : 1.f;
            if (need) {
              lsum *= alpha;
              m_used = mx;
            }
            rescale_o(alpha);
            uint32_t sr2[128];
            DLLM_TMEM_LD32(tS + 0, (sr2 + 0));
            DLLM_TMEM_LD32(tS + 32, (sr2 + 32));
            DLLM_TMEM_LD32(tS + 64, (sr2 + 64));
            DLLM_TMEM_LD32(tS + 96, (sr2 + 96));
            ptx::tmem_wait_ld();
            float *s2 = reinterpret_cast<float *>(sr2);
            if (j == u.n - 1) {
              const int key_end = u.L - j * TBN;
#pragma unroll
              for (int c = 0; c < 128; ++c)
                if (c >= key_end) s2[c] = -INFINITY;
            }
            exp_pass(s2);
          }
        }
        lsum += lpart;
        DLLM_TMEM_ST32(tS + 0, (pk + 0));
        DLLM_TMEM_ST32(tS + 32, (pk + 32));
        ptx::tmem_wait_st();
        if (threadIdx.x == 128) TRACE(15, sc - 1);
        ptx::tc_fence_before();
        __syncwarp();
        if ((threadIdx.x & 127) == 0) TRACE(4 + wg, sc - 1);
        if (lane == 0) ptx::mbar_arrive(bar(B_PFULL + wg));
      }
      // ---- epilogue: O / l -> bf16 -> global
      ptx::mbar_wait(bar(B_OFULL + wg), oc & 1);
      ++oc;
      ptx::tc_fence_after();
      const float inv = lsum > 0.f ? 1.f / lsum : 0.f;
      const int grow = origin + row;
      const bool wr = grow < (wg ? u.write_end[1] : u.write_end[0]);
      __nv_bfloat16 *dst = out + (int64_t)(u.q_off + grow) * HD + (int64_t)u.h * D;
#pragma unroll 1
      for (int c = 0; c < D; c += 32) {
        uint32_t o[32];
        DLLM_TMEM_LD32(tO + c, o);
        ptx::tmem_wait_ld();
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 16; ++i)
          pk[i] = pack_bf16(__uint_as_float(o[2 * i]) * inv, __uint_as_float(o[2 * i + 1]) * inv);
        if (wr) {
          uint4 *d4 = reinterpret_cast<uint4 *>(dst + c);
#pragma unroll
          for (int i = 0; i < 4; ++i) d4[i] = make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
        }
      }
      ptx::tc_fence_before();
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (warp == 1) ptx::tmem_dealloc(tmem, 512);
}

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
cudaError_t launch_d(const Plan &plan, const void *q, const void *k, const void *v, void *out, float *scores,
                     cudaStream_t st) {
  auto enc = encode_fn();
  if (!enc) return cudaErrorNotSupported;
  int64_t rows = 0;
  for (int b = 0; b < plan.nreq; ++b) rows = rows > plan.r[b].q_off + plan.r[b].L ? rows : plan.r[b].q_off + plan.r[b].L;
  CUtensorMap tq, tk, tv;
  {
    cuuint64_t dims[3] = {(cuuint64_t)D, (cuuint64_t)plan.H, (cuuint64_t)rows};
    cuuint64_t strides[2] = {(cuuint64_t)D * 2, (cuuint64_t)plan.H * D * 2};
    cuuint32_t box[3] = {64, 1, TBM};
    cuuint32_t es[3] = {1, 1, 1};
    if (enc(&tq, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void *>(q), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  {
    const int P = plan.page_size;
    cuuint64_t dims[4] = {(cuuint64_t)D, (cuuint64_t)P, (cuuint64_t)plan.H_kv, (cuuint64_t)1 << 24};
    cuuint64_t strides[3] = {(cuuint64_t)D * 2, (cuuint64_t)P * D * 2, (cuuint64_t)plan.H_kv * P * D * 2};
    cuuint32_t box[4] = {64, (cuuint32_t)(P < TBN ? P : TBN), 1, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    for (int w = 0; w < 2; ++w) {
      if (enc(w ? &tv : &tk, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void *>(w ? v : k), dims, strides, box,
              es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return cudaErrorInvalidValue;
    }
  }
  const int smem = TcCfg<D>::kBytes;
  cudaError_t e = cudaFuncSetAttribute(refresh_tc_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  const int grid = plan.total_units < num_sms() ? plan.total_units : num_sms();
  if (grid <= 0) return cudaSuccess;
  refresh_tc_kernel<D><<<grid, TC_THREADS, smem, st>>>(plan, tq, tk, tv, (__nv_bfloat16 *)out, scores);
  return cudaGetLastError();
}

}  // namespace

bool refresh_tc_supported(int D) { return D == 64 || D == 128; }

int refresh_tc_units(int L, int bs, int be, int H, bool with_scores) {
  const int nt = tc_regular_tiles(L) + ((with_scores && tc_straddles(bs, be)) ? 1 : 0);
  return H * ((nt + 1) / 2);
}

cudaError_t launch_refresh_tc(const Plan &plan, const void *q, const void *k, const void *v, void *out,
                              float *scores, cudaStream_t st) {
  switch (plan.D) {
    case 64: return launch_d<64>(plan, q, k, v, out, scores, st);
    case 128: return launch_d<128>(plan, q, k, v, out, scores, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace dllm
