// Reuse sparse attention, persistent warp-specialised variant
// (§2.3, Eq. 4; per-head key sets of §4.5).
//
// For request b, query head h and the active block's query rows q:
//   O_b[q,h] = softmax_j(tau Q_blk[q,h].K[j,kv(h)]) V[j,kv(h)],  j in [bs,be) ++ idx(b,h)
// with K/V gathered in place from the paged cache (no pack, no assembly copy).
//
// Reuse is HBM-bound (~30 FLOP/B), and a work unit (b, h, 32 query rows) is
// short (C1: 280 keys = 143 KB), so a one-CTA-per-unit kernel spends most of
// its time filling and draining its pipeline.  Here one CTA per SM streams
// all of its units' 64-key chunks through ONE ring that never drains between
// units.  Roles (192 threads):
//   warp 4  translator: position -> physical cache row (block-table lookup)
//           for every key of every chunk, NT chunks ahead, into a smem ring;
//   warp 5  loader: Q rows of each unit + 16-byte cp.async row gathers of K
//           and V into an NS-stage ring, completion signalled with
//           cp.async.mbarrier.arrive.noinc;
//   warps 0-3 consumers: mma.sync m16n8k16 (bf16 -> fp32) S = Q K^T and
//           O += P V with a register online softmax; warp w owns rows
//           16*(w&1)..+16 and keys 32*(w>>1)..+32 of each chunk; the two key
//           halves are merged through shared memory at the end of a unit.
// Units of the heads of one KV group are adjacent in the unit order so their
// overlapping selections are served from L2.
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "plan.h"
#include "tc_ptx.cuh"

namespace dllm {
namespace {

constexpr int kWsConsumers = 4;
#ifndef DLLM_RWS_LOADERS
#define DLLM_RWS_LOADERS 4
#endif
#ifndef DLLM_RWS_NS
#define DLLM_RWS_NS 4
#endif
#ifndef DLLM_RWS_L2PF
#define DLLM_RWS_L2PF 1  // L2 prefetch of the CTA's index lists / block-table rows at start
#endif
#ifndef DLLM_RWS_DBG
#define DLLM_RWS_DBG 0   // dev only: 1 = consumers skip the math, 2 = loaders skip the gathers
#endif
constexpr int kLoaders = DLLM_RWS_LOADERS;   // cp.async issuing warps
constexpr int kWsThreads = (kWsConsumers + 1 + kLoaders) * 32;
constexpr int kRows = 32;          // query rows per unit
constexpr int kChunk = 64;         // keys per ring stage
constexpr int kNT = 8;             // translation ring depth (chunks)
constexpr int kTG = 8;             // chunks translated per batch

template <int D>
struct WsCfg {
  static constexpr int kNS = D >= 128 ? DLLM_RWS_NS : 6;  // data ring stages
  static constexpr int kRowB = D * 2 + 16;               // padded smem row (conflict-free ldmatrix)
  static constexpr int kKV = kChunk * kRowB;             // one K (or V) chunk
  static constexpr int kQ = kRows * D * 2;
  static constexpr int kXStride = D / 2 + 4;             // floats per lane record in the merge buffer
  static constexpr int kOffK = 0;
  static constexpr int kOffV = kOffK + kNS * kKV;
  static constexpr int kOffQ = kOffV + kNS * kKV;        // 2 buffers
  static constexpr int kOffOffs = kOffQ + 2 * kQ;        // [kNT][kChunk] int32
  static constexpr int kOffX = kOffOffs + kNT * kChunk * 4;   // [2 rh][32][kXStride] f32
  static constexpr int kOffBar = kOffX + 2 * 32 * kXStride * 4;
  static constexpr int kBytes = kOffBar + 8 * (2 * kNS + 2 * kNT + 4) + 128;
};

#ifdef DLLM_TRACE
// per-CTA timeline (globaltimer ns): [0] start, [1] translator: first offsets
// published, [2] consumer: first chunk ready, [3..10] consumer: end of unit i,
// [11] end, [12] SM id
__device__ long long g_rws[1024][16];
extern "C" __attribute__((visibility("default"))) int dllm_trace_rws_read(long long *host) {
  return (int)cudaMemcpyFromSymbol(host, g_rws, sizeof(g_rws));
}
__device__ __forceinline__ long long rws_timer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// CTA 0 per-chunk timeline: [0] translator published, [1] loader issued,
// [2] consumer: data ready, [3] consumer: chunk done, [4] consumer: wait start
__device__ long long g_rws_chunk[5][64];
extern "C" __attribute__((visibility("default"))) int dllm_trace_rws_chunk(long long *host) {
  return (int)cudaMemcpyFromSymbol(host, g_rws_chunk, sizeof(g_rws_chunk));
}
#define RWS_CHUNK(kind, t)                                                               \
  do {                                                                                   \
    if (lane == 0 && blockIdx.x == 0 && (t) < 64) g_rws_chunk[kind][t] = rws_timer();    \
  } while (0)
#define RWS_TRACE(slot)                                                                  \
  do {                                                                                   \
    if (lane == 0 && blockIdx.x < 1024) g_rws[blockIdx.x][slot] = rws_timer();           \
  } while (0)
#else
#define RWS_TRACE(slot) \
  do {                  \
  } while (0)
#define RWS_CHUNK(kind, t) \
  do {                     \
  } while (0)
#endif

struct RUnit {
  int b, h, kvh, rg, blk, bs, nk, k, blk_off, bt_row;
  int64_t idx_off;
};

__device__ __forceinline__ void decode(const Plan &pl, int unit, RUnit &u) {
  u.b = plan_find(pl, unit);
  const ReqInfo &R = pl.r[u.b];
  u.blk = R.be - R.bs;
  u.bs = R.bs;
  const int ngroups = (u.blk + kRows - 1) / kRows;
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

__device__ __forceinline__ void cp_async_mbar_arrive_noinc(uint32_t bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(bar) : "memory");
}

// PACKED: the context keys come from the paper's packed per-head buffers
// (k_pack / v_pack, row = the key's slot in the idx layout, written by
// dllm_pack_kv) instead of being gathered through the block table; the
// active block's rows still come from the paged cache.
template <int D, bool PACKED>
__global__ void __launch_bounds__(kWsThreads, 1)
reuse_ws_kernel(const __grid_constant__ Plan plan, const __nv_bfloat16 *__restrict__ q_blk,
                const __nv_bfloat16 *__restrict__ k_cache, const __nv_bfloat16 *__restrict__ v_cache,
                const int32_t *__restrict__ idx, __nv_bfloat16 *__restrict__ out,
                const __nv_bfloat16 *__restrict__ k_pack, const __nv_bfloat16 *__restrict__ v_pack) {
  using C = WsCfg<D>;
  constexpr int NS = C::kNS;
  constexpr int CH = D / 8;
  constexpr int KSTEPS = D / 16;
  extern __shared__ __align__(128) uint8_t smem[];
  const uint32_t sbase = smem_u32(smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // barriers
  const uint32_t b_full = sbase + C::kOffBar;                 // [NS] loader (32 noinc arrivals)
  const uint32_t b_empty = b_full + 8 * NS;                   // [NS] consumers (4)
  const uint32_t b_ofull = b_empty + 8 * NS;                  // [kNT] translator (1)
  const uint32_t b_oempty = b_ofull + 8 * kNT;                // [kNT] loader (1)
  const uint32_t b_qfull = b_oempty + 8 * kNT;                // [2] loader (32 noinc)
  const uint32_t b_qempty = b_qfull + 16;                     // [2] consumers (4)
  int32_t *offs = reinterpret_cast<int32_t *>(smem + C::kOffOffs);

#ifdef DLLM_TRACE
  if (threadIdx.x == 0 && blockIdx.x < 1024) {
    for (int i = 0; i < 16; ++i) g_rws[blockIdx.x][i] = 0;
    g_rws[blockIdx.x][0] = rws_timer();
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    g_rws[blockIdx.x][12] = smid;
  }
#endif
  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) {
      ptx::mbar_init(b_full + 8 * i, 32 * kLoaders);
      ptx::mbar_init(b_empty + 8 * i, kWsConsumers);
    }
    for (int i = 0; i < kNT; ++i) {
      ptx::mbar_init(b_ofull + 8 * i, 1);
      ptx::mbar_init(b_oempty + 8 * i, kLoaders);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(b_qfull + 8 * i, 32);
      ptx::mbar_init(b_qempty + 8 * i, kWsConsumers);
    }
    ptx::fence_mbar_init();
  }
  __syncthreads();

  if (warp == kWsConsumers) {
    // ============================ translator (+ Q rows) ============================
#if DLLM_RWS_L2PF
    // every index list and block-table row this CTA will translate, pulled into
    // L2 up front: the per-unit translation is two dependent memory round trips
    // (idx, then block table), and with few units per CTA they are the critical path
    for (int unit = blockIdx.x + lane * gridDim.x; unit < plan.total_units; unit += 32 * gridDim.x) {
      RUnit u;
      decode(plan, unit, u);
      if (!PACKED && u.k > 0) {
        const uintptr_t a0 = reinterpret_cast<uintptr_t>(idx + u.idx_off) & ~uintptr_t(15);
        const uintptr_t a1 = (reinterpret_cast<uintptr_t>(idx + u.idx_off + u.k) + 15) & ~uintptr_t(15);
        ptx::bulk_prefetch_l2(reinterpret_cast<const void *>(a0), (uint32_t)(a1 - a0));
      }
      const uintptr_t b0 = reinterpret_cast<uintptr_t>(plan.block_table + (int64_t)u.bt_row * plan.pages_per_req) &
                           ~uintptr_t(15);
      const uintptr_t b1 = (reinterpret_cast<uintptr_t>(plan.block_table + (int64_t)(u.bt_row + 1) * plan.pages_per_req) +
                            15) & ~uintptr_t(15);
      ptx::bulk_prefetch_l2(reinterpret_cast<const void *>(b0), (uint32_t)(b1 - b0));
    }
#endif
    int t = 0, qc = 0;
    for (int unit = blockIdx.x; unit < plan.total_units; unit += gridDim.x) {
      RUnit u;
      decode(plan, unit, u);
      const int32_t *my_idx = idx + u.idx_off;
      const int32_t *bt = plan.block_table + (int64_t)u.bt_row * plan.pages_per_req;
      const int nchunks = (u.nk + kChunk - 1) / kChunk;
      {
        // the unit's query rows (the translator runs ahead of the loaders, so Q of
        // the next unit is in flight long before the consumers need it)
        const int row0 = u.rg * kRows;
        const int qb = qc & 1;
        ptx::mbar_wait(b_qempty + 8 * qb, ((qc >> 1) & 1) ^ 1);
        uint8_t *sq = smem + C::kOffQ + qb * C::kQ;
        const int64_t HD = (int64_t)plan.H * D;
        for (int i = lane; i < kRows * CH; i += 32) {
          const int r = i / CH, c = i - r * CH;
          const bool ok = row0 + r < u.blk;
          const __nv_bfloat16 *src = q_blk + (int64_t)(u.blk_off + (ok ? row0 + r : 0)) * HD + (int64_t)u.h * D + c * 8;
          cp_async16(smem_u32(sq + swz<D>(r, c)), src, ok ? 16 : 0);
        }
        cp_async_mbar_arrive_noinc(b_qfull + 8 * qb);
        ++qc;
      }
      // batches of kTG chunks: all index loads of a batch are issued together, then
      // all block-table loads, so a batch costs two memory round trips, not 2 per chunk
      for (int g0 = 0; g0 < nchunks; g0 += kTG) {
        constexpr int Q = kTG * kChunk / 32;
        int pos[Q], off[Q];
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          const int j = g0 * kChunk + q * 32 + lane;
          if (PACKED)
            pos[q] = j < u.blk ? u.bs + j : -1;
          else
            pos[q] = j < u.nk ? (j < u.blk ? u.bs + j : __ldg(my_idx + (j - u.blk))) : -1;
        }
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          const int page = pos[q] >= 0 ? __ldg(bt + (pos[q] >> plan.page_shift)) : 0;
          off[q] = pos[q] >= 0 ? (page * plan.H_kv + u.kvh) * plan.page_size + (pos[q] & (plan.page_size - 1)) : -1;
          if (PACKED) {
            // packed context rows: slot of the key in the idx layout
            const int j = g0 * kChunk + q * 32 + lane;
            if (j >= u.blk && j < u.nk) off[q] = (int)(u.idx_off + (j - u.blk));
          }
        }
        const int ng = min(kTG, nchunks - g0);
#pragma unroll
        for (int c = 0; c < kTG; ++c) {
          if (c >= ng) break;
          const int slot = t % kNT;
          ptx::mbar_wait(b_oempty + 8 * slot, ((t / kNT) & 1) ^ 1);
#pragma unroll
          for (int rr = 0; rr < kChunk / 32; ++rr) offs[slot * kChunk + rr * 32 + lane] = off[c * (kChunk / 32) + rr];
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(b_ofull + 8 * slot);
          if (t == 0) RWS_TRACE(1);
          RWS_CHUNK(0, t);
          ++t;
        }
      }
    }
    cp_async_wait<0>();
  } else if (warp > kWsConsumers) {
    // ============================ loaders ============================
    const int li = warp - kWsConsumers - 1;
    int t = 0;
    for (int unit = blockIdx.x; unit < plan.total_units; unit += gridDim.x) {
      RUnit u;
      decode(plan, unit, u);
      const int nchunks = (u.nk + kChunk - 1) / kChunk;
      for (int c = 0; c < nchunks; ++c, ++t) {
        const int slot = t % kNT, s = t % NS;
        ptx::mbar_wait(b_ofull + 8 * slot, (t / kNT) & 1);
        ptx::mbar_wait(b_empty + 8 * s, ((t / NS) & 1) ^ 1);
        uint8_t *dk = smem + C::kOffK + s * C::kKV;
        uint8_t *dv = smem + C::kOffV + s * C::kKV;
        // 16-byte cp.async row gathers: consecutive lanes read consecutive 16-byte pieces
        // of the same 2D-byte row (coalesced per row); rows past the key list are
        // zero-filled (src-size 0); completion counted with cp.async.mbarrier.arrive.noinc
#pragma unroll 4
        for (int e = li * 32 + lane; e < (DLLM_RWS_DBG == 2 ? 0 : kChunk * CH); e += 32 * kLoaders) {
          const int r = e / CH, cc = e - r * CH;
          const int off = offs[slot * kChunk + r];
          const int64_t goff = (int64_t)(off < 0 ? 0 : off) * D + cc * 8;
          const int nb = off < 0 ? 0 : 16;
          const bool from_pack = PACKED && (c * kChunk + r) >= u.blk;
          cp_async16(smem_u32(dk + r * C::kRowB + cc * 16), (from_pack ? k_pack : k_cache) + goff, nb);
          cp_async16(smem_u32(dv + r * C::kRowB + cc * 16), (from_pack ? v_pack : v_cache) + goff, nb);
        }
        cp_async_mbar_arrive_noinc(b_full + 8 * s);
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(b_oempty + 8 * slot);
        if (li == 0) RWS_CHUNK(1, t);
      }
    }
    cp_async_wait<0>();
  } else {
    // ============================ consumers ============================
    const int rh = warp & 1, kh = warp >> 1;
    const float sl2 = plan.scale_log2;
    const int64_t HD = (int64_t)plan.H * D;
    float *xrec = reinterpret_cast<float *>(smem + C::kOffX) + (rh * 32 + lane) * C::kXStride;
    int t = 0, qc = 0;
    for (int unit = blockIdx.x; unit < plan.total_units; unit += gridDim.x, ++qc) {
      RUnit u;
      decode(plan, unit, u);
      const int nchunks = (u.nk + kChunk - 1) / kChunk;
      uint32_t qf[KSTEPS][4];
      {
        const int qb = qc & 1;
        ptx::mbar_wait(b_qfull + 8 * qb, (qc >> 1) & 1);
        const uint8_t *sq = smem + C::kOffQ + qb * C::kQ;
#pragma unroll
        for (int kk = 0; kk < KSTEPS; ++kk) {
          const int r = rh * 16 + (lane & 15);
          ldmatrix_x4(qf[kk][0], qf[kk][1], qf[kk][2], qf[kk][3], smem_u32(sq + swz<D>(r, kk * 2 + (lane >> 4))));
        }
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(b_qempty + 8 * qb);
      }
      float o[D / 8][4];
#pragma unroll
      for (int i = 0; i < D / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
      float m_r[2] = {-INFINITY, -INFINITY}, l_r[2] = {0.f, 0.f};

      for (int c = 0; c < nchunks; ++c, ++t) {
        const int s = t % NS;
        if (warp == 0) RWS_CHUNK(4, t);
        ptx::mbar_wait(b_full + 8 * s, (t / NS) & 1);
        if (t == 0 && warp == 0) RWS_TRACE(2);
        if (warp == 0) RWS_CHUNK(2, t);
        if (DLLM_RWS_DBG == 1) {
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(b_empty + 8 * s);
          continue;
        }
        const uint8_t *tk = smem + C::kOffK + s * C::kKV;
        const uint8_t *tv = smem + C::kOffV + s * C::kKV;
        float sc[4][4];
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) sc[nt][0] = sc[nt][1] = sc[nt][2] = sc[nt][3] = 0.f;
#pragma unroll
        for (int np = 0; np < 2; ++np) {
#pragma unroll
          for (int kk = 0; kk < KSTEPS; ++kk) {
            const int key = kh * 32 + np * 16 + (lane >> 4) * 8 + (lane & 7);
            const int cc = kk * 2 + ((lane >> 3) & 1);
            uint32_t b0, b1, b2, b3;
            ldmatrix_x4(b0, b1, b2, b3, smem_u32(tk + key * C::kRowB + cc * 16));
            mma_bf16_16816(sc[np * 2 + 0], qf[kk], b0, b1);
            mma_bf16_16816(sc[np * 2 + 1], qf[kk], b2, b3);
          }
        }
        const int kbase = c * kChunk + kh * 32 + (lane & 3) * 2;
        float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) {
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int j = kbase + nt * 8 + (e & 1);
            const float v = j < u.nk ? sc[nt][e] * sl2 : -INFINITY;
            sc[nt][e] = v;
            mx[e >> 1] = fmaxf(mx[e >> 1], v);
          }
        }
        float alpha[2], mbase[2];
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 1));
          mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 2));
          const float mnew = fmaxf(m_r[r], mx[r]);
          mbase[r] = mnew == -INFINITY ? 0.f : mnew;
          alpha[r] = fast_exp2(m_r[r] - mbase[r]);
          m_r[r] = mnew;
          l_r[r] *= alpha[r];
        }
#pragma unroll
        for (int i = 0; i < D / 8; ++i) {
          o[i][0] *= alpha[0]; o[i][1] *= alpha[0];
          o[i][2] *= alpha[1]; o[i][3] *= alpha[1];
        }
        uint32_t pa[2][4];
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) {
          const float p0 = fast_exp2(sc[nt][0] - mbase[0]);
          const float p1 = fast_exp2(sc[nt][1] - mbase[0]);
          const float p2 = fast_exp2(sc[nt][2] - mbase[1]);
          const float p3 = fast_exp2(sc[nt][3] - mbase[1]);
          const uint32_t lo = pack_bf16(p0, p1), hi = pack_bf16(p2, p3);
          const __nv_bfloat162 blo = *reinterpret_cast<const __nv_bfloat162 *>(&lo);
          const __nv_bfloat162 bhi = *reinterpret_cast<const __nv_bfloat162 *>(&hi);
          l_r[0] += __low2float(blo) + __high2float(blo);
          l_r[1] += __low2float(bhi) + __high2float(bhi);
          pa[nt >> 1][(nt & 1) * 2 + 0] = lo;
          pa[nt >> 1][(nt & 1) * 2 + 1] = hi;
        }
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
#pragma unroll
          for (int dp = 0; dp < D / 16; ++dp) {
            const int key = kh * 32 + ks * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
            const int cc = dp * 2 + (lane >> 4);
            uint32_t b0, b1, b2, b3;
            ldmatrix_x4_trans(b0, b1, b2, b3, smem_u32(tv + key * C::kRowB + cc * 16));
            mma_bf16_16816(o[dp * 2 + 0], pa[ks], b0, b1);
            mma_bf16_16816(o[dp * 2 + 1], pa[ks], b2, b3);
          }
        }
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(b_empty + 8 * s);
        if (warp == 0) RWS_CHUNK(3, t);
      }
      // ---- merge the two key halves and store
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        l_r[r] += __shfl_xor_sync(0xffffffffu, l_r[r], 1);
        l_r[r] += __shfl_xor_sync(0xffffffffu, l_r[r], 2);
      }
      if (kh == 1) {
#pragma unroll
        for (int i = 0; i < D / 8; ++i)
#pragma unroll
          for (int e = 0; e < 4; ++e) xrec[i * 4 + e] = o[i][e];
        xrec[D / 2 + 0] = m_r[0]; xrec[D / 2 + 1] = m_r[1];
        xrec[D / 2 + 2] = l_r[0]; xrec[D / 2 + 3] = l_r[1];
      }
      ptx::named_bar_sync(1, kWsConsumers * 32);
      if (kh == 0) {
        float sc_self[2], sc_other[2], inv[2];
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          const float m2 = xrec[D / 2 + r], l2 = xrec[D / 2 + 2 + r];
          const float m = fmaxf(m_r[r], m2);
          const float mb = m == -INFINITY ? 0.f : m;
          sc_self[r] = fast_exp2(m_r[r] - mb);
          sc_other[r] = fast_exp2(m2 - mb);
          const float l = l_r[r] * sc_self[r] + l2 * sc_other[r];
          inv[r] = l > 0.f ? 1.f / l : 0.f;
        }
        const int qr0 = u.rg * kRows + rh * 16 + (lane >> 2);
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          const int qrow = qr0 + r * 8;
          if (qrow >= u.blk) continue;
          __nv_bfloat16 *dst = out + (int64_t)(u.blk_off + qrow) * HD + (int64_t)u.h * D + (lane & 3) * 2;
#pragma unroll
          for (int i = 0; i < D / 8; ++i) {
            const float v0 = (o[i][r * 2 + 0] * sc_self[r] + xrec[i * 4 + r * 2 + 0] * sc_other[r]) * inv[r];
            const float v1 = (o[i][r * 2 + 1] * sc_self[r] + xrec[i * 4 + r * 2 + 1] * sc_other[r]) * inv[r];
            *reinterpret_cast<uint32_t *>(dst + i * 8) = pack_bf16(v0, v1);
          }
        }
      }
      ptx::named_bar_sync(1, kWsConsumers * 32);      // merge buffer free for the next unit
      if (warp == 0 && qc < 8) RWS_TRACE(3 + qc);
    }
    if (warp == 0) RWS_TRACE(11);
  }
}

int num_sms_ws() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

template <int D, bool PACKED>
cudaError_t launch_ws_d(const Plan &plan, const void *q_blk, const void *k_cache, const void *v_cache,
                        const int32_t *idx, void *out, const void *k_pack, const void *v_pack, cudaStream_t st) {
  const int smem = WsCfg<D>::kBytes;
  cudaError_t e = cudaFuncSetAttribute(reuse_ws_kernel<D, PACKED>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  const int grid = plan.total_units < num_sms_ws() ? plan.total_units : num_sms_ws();
  if (grid <= 0) return cudaSuccess;
  reuse_ws_kernel<D, PACKED><<<grid, kWsThreads, smem, st>>>(
      plan, (const __nv_bfloat16 *)q_blk, (const __nv_bfloat16 *)k_cache, (const __nv_bfloat16 *)v_cache, idx,
      (__nv_bfloat16 *)out, (const __nv_bfloat16 *)k_pack, (const __nv_bfloat16 *)v_pack);
  return cudaGetLastError();
}

// Pack (§4.5): the selected K/V rows of every (b, h) copied
// into dense per-head buffers, row order = the idx layout.  One CTA per (b, h);
// 16-byte loads through the block table, 16-byte stores.
template <int D>
__global__ void __launch_bounds__(256)
pack_kv_kernel(const __grid_constant__ Plan plan, const __nv_bfloat16 *__restrict__ k_cache,
               const __nv_bfloat16 *__restrict__ v_cache, const int32_t *__restrict__ idx,
               __nv_bfloat16 *__restrict__ k_pack, __nv_bfloat16 *__restrict__ v_pack) {
  constexpr int CH = D / 8;
  const int unit = blockIdx.x;
  const int b = plan_find(plan, unit);
  const ReqInfo &R = plan.r[b];
  const int h = unit - R.unit_off;
  const int kvh = h / (plan.H / plan.H_kv);
  const int64_t row0 = R.idx_off + (int64_t)h * R.k;
  const int32_t *bt = plan.block_table + (int64_t)R.bt_row * plan.pages_per_req;
#pragma unroll 4
  for (int e = threadIdx.x; e < R.k * CH; e += blockDim.x) {
    const int i = e / CH, cc = e - i * CH;
    const int pos = __ldg(idx + row0 + i);
    const int page = __ldg(bt + (pos >> plan.page_shift));
    const int64_t src = (((int64_t)page * plan.H_kv + kvh) * plan.page_size + (pos & (plan.page_size - 1))) * D + cc * 8;
    const int64_t dst = (row0 + i) * D + cc * 8;
    *reinterpret_cast<uint4 *>(k_pack + dst) = __ldg(reinterpret_cast<const uint4 *>(k_cache + src));
    *reinterpret_cast<uint4 *>(v_pack + dst) = __ldg(reinterpret_cast<const uint4 *>(v_cache + src));
  }
}

template <int D>
cudaError_t launch_pack_d(const Plan &plan, const void *k_cache, const void *v_cache, const int32_t *idx,
                          void *k_pack, void *v_pack, cudaStream_t st) {
  if (plan.total_units <= 0) return cudaSuccess;
  pack_kv_kernel<D><<<plan.total_units, 256, 0, st>>>(plan, (const __nv_bfloat16 *)k_cache,
                                                      (const __nv_bfloat16 *)v_cache, idx, (__nv_bfloat16 *)k_pack,
                                                      (__nv_bfloat16 *)v_pack);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_reuse_ws(const Plan &plan, const void *q_blk, const void *k_cache, const void *v_cache,
                            const int32_t *idx, void *out, cudaStream_t st) {
  switch (plan.D) {
    case 16: return launch_ws_d<16, false>(plan, q_blk, k_cache, v_cache, idx, out, nullptr, nullptr, st);
    case 32: return launch_ws_d<32, false>(plan, q_blk, k_cache, v_cache, idx, out, nullptr, nullptr, st);
    case 64: return launch_ws_d<64, false>(plan, q_blk, k_cache, v_cache, idx, out, nullptr, nullptr, st);
    case 128: return launch_ws_d<128, false>(plan, q_blk, k_cache, v_cache, idx, out, nullptr, nullptr, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_reuse_packed(const Plan &plan, const void *q_blk, const void *k_cache, const void *v_cache,
                                const void *k_pack, const void *v_pack, void *out, cudaStream_t st) {
  switch (plan.D) {
    case 16: return launch_ws_d<16, true>(plan, q_blk, k_cache, v_cache, nullptr, out, k_pack, v_pack, st);
    case 32: return launch_ws_d<32, true>(plan, q_blk, k_cache, v_cache, nullptr, out, k_pack, v_pack, st);
    case 64: return launch_ws_d<64, true>(plan, q_blk, k_cache, v_cache, nullptr, out, k_pack, v_pack, st);
    case 128: return launch_ws_d<128, true>(plan, q_blk, k_cache, v_cache, nullptr, out, k_pack, v_pack, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_pack_kv(const Plan &plan, const void *k_cache, const void *v_cache, const int32_t *idx,
                           void *k_pack, void *v_pack, cudaStream_t st) {
  switch (plan.D) {
    case 16: return launch_pack_d<16>(plan, k_cache, v_cache, idx, k_pack, v_pack, st);
    case 32: return launch_pack_d<32>(plan, k_cache, v_cache, idx, k_pack, v_pack, st);
    case 64: return launch_pack_d<64>(plan, k_cache, v_cache, idx, k_pack, v_pack, st);
    case 128: return launch_pack_d<128>(plan, k_cache, v_cache, idx, k_pack, v_pack, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace dllm
