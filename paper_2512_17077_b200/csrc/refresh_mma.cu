// Refresh dense attention, mma.sync variant (§2.3, Eq. 3)
// with the fused raw-importance epilogue (inner term of Eq. 6,
// PAPER.md:385-389, §4.5).
//
// This is the legacy-tensor-core (HMMA) reference kernel: the baseline the
// tcgen05/TMEM kernel (refresh_tc.cu) is measured against, and the path used
// for head_dim < 64.  Work unit = (b, h, 64-row Q tile); 4 warps x 16 rows;
// 64-key K/V chunks gathered from the paged cache with cp.async into a
// 3-stage ring; online softmax in registers.
//
// Importance: raw[b,h,m] = max_{q in [bs,be)} Q[q,h].K[m,kv(h)] (unscaled,
// DESIGN.md R1/R8) for every key m.  It is produced by exactly one CTA per
// (b, h): the regular tile that contains the whole block, or — when the block
// straddles a tile boundary — one extra "score-only" tile whose rows are the
// block rows (up to 128, in two 64-row passes), which computes S = Q K^T only.
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "plan.h"

namespace dllm {

constexpr int kRefThreads = 128;
constexpr int kRefRows = 64;
constexpr int kRefChunk = 64;
constexpr int kRefStages = 3;

template <int D>
struct RefSmem {
  static constexpr int kQ = kRefRows * D * 2;
  static constexpr int kKV = kRefChunk * D * 2;
  static constexpr int kScore = 4 * kRefChunk * 4;
  static constexpr int kBytes = kQ + kRefStages * 2 * kKV + kScore;
};

// Tiles of request b (shared with the host planner, dllm_api.cu).
__host__ __device__ __forceinline__ int ref_regular_tiles(int L) { return (L + kRefRows - 1) / kRefRows; }
__host__ __device__ __forceinline__ bool ref_block_straddles(int bs, int be) {
  return (bs / kRefRows) != ((be - 1) / kRefRows);
}

template <int D>
__global__ void __launch_bounds__(kRefThreads, 2)
refresh_mma_kernel(const __grid_constant__ Plan plan, const __nv_bfloat16 *__restrict__ q,
                   const __nv_bfloat16 *__restrict__ k_cache, const __nv_bfloat16 *__restrict__ v_cache,
                   __nv_bfloat16 *__restrict__ out, float *__restrict__ scores) {
  extern __shared__ __align__(128) uint8_t smem[];
  constexpr int CH = D / 8;
  constexpr int KSTEPS = D / 16;
  uint8_t *sQ = smem;
  uint8_t *sK = smem + RefSmem<D>::kQ;
  uint8_t *sV = sK + kRefStages * RefSmem<D>::kKV;
  float *sS = reinterpret_cast<float *>(sV + kRefStages * RefSmem<D>::kKV);   // [4 warps][64]

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int unit = blockIdx.x;
  const int b = plan_find(plan, unit);
  const ReqInfo &R = plan.r[b];
  const int L = R.L, bs = R.bs, be = R.be;
  const int nreg = ref_regular_tiles(L);
  const bool extra = plan.with_scores && ref_block_straddles(bs, be);
  const int ntiles = nreg + (extra ? 1 : 0);
  const int local = unit - R.unit_off;
  const int h = local / ntiles;
  const int t = local - h * ntiles;
  const int kvh = h / (plan.H / plan.H_kv);
  const bool score_only = t == nreg;
  const bool do_scores = plan.with_scores && (score_only || (!extra && t == bs / kRefRows));
  const int origin = score_only ? bs : t * kRefRows;
  const int npass = score_only ? (be - bs + kRefRows - 1) / kRefRows : 1;   // 1 or 2
  const int64_t HD = (int64_t)plan.H * D;
  const int32_t *bt = plan.block_table + (int64_t)R.bt_row * plan.pages_per_req;
  const int nchunks = (L + kRefChunk - 1) / kRefChunk;
  const int row_end = score_only ? be : L;      // rows >= row_end are zero-filled

  auto load_q = [&](int pass) {
    for (int i = tid; i < kRefRows * CH; i += kRefThreads) {
      const int r = i / CH, c = i - r * CH;
      const int row = origin + pass * kRefRows + r;
      const bool ok = row < row_end;
      const __nv_bfloat16 *src = q + (int64_t)(R.q_off + (ok ? row : 0)) * HD + (int64_t)h * D + c * 8;
      cp_async16(smem_u32(sQ + swz<D>(r, c)), src, ok ? 16 : 0);
    }
  };
  auto load_chunk = [&](int chunk, int stage) {
    uint8_t *dk = sK + stage * RefSmem<D>::kKV;
    uint8_t *dv = sV + stage * RefSmem<D>::kKV;
    constexpr int ROWS_PER_PASS = kRefThreads / CH;
    const int c = tid % CH;
#pragma unroll 4
    for (int r = tid / CH; r < kRefChunk; r += ROWS_PER_PASS) {
      const int pos = chunk * kRefChunk + r;
      const bool ok = pos < L;
      int64_t off = 0;
      if (ok) {
        const int page = __ldg(bt + (pos >> plan.page_shift));
        const int slot = pos & (plan.page_size - 1);
        off = (((int64_t)page * plan.H_kv + kvh) * plan.page_size + slot) * D + c * 8;
      }
      cp_async16(smem_u32(dk + swz<D>(r, c)), k_cache + off, ok ? 16 : 0);
      if (!score_only) cp_async16(smem_u32(dv + swz<D>(r, c)), v_cache + off, ok ? 16 : 0);
    }
  };

  // Q fragments (pass 0 always; pass 1 only for a >64-row score-only block)
  uint32_t qf[2][KSTEPS][4];
  load_q(0);
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
#pragma unroll
  for (int kk = 0; kk < KSTEPS; ++kk) {
    const int r = warp * 16 + (lane & 15);
    ldmatrix_x4(qf[0][kk][0], qf[0][kk][1], qf[0][kk][2], qf[0][kk][3], smem_u32(sQ + swz<D>(r, kk * 2 + (lane >> 4))));
  }
  if (npass > 1) {
    __syncthreads();
    load_q(1);
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < KSTEPS; ++kk) {
      const int r = warp * 16 + (lane & 15);
      ldmatrix_x4(qf[1][kk][0], qf[1][kk][1], qf[1][kk][2], qf[1][kk][3], smem_u32(sQ + swz<D>(r, kk * 2 + (lane >> 4))));
    }
  }

#pragma unroll
  for (int s = 0; s < kRefStages - 1; ++s) {
    if (s < nchunks) load_chunk(s, s);
    cp_async_commit();
  }

  float o[D / 8][4];
#pragma unroll
  for (int i = 0; i < D / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m_r[2] = {-INFINITY, -INFINITY}, l_r[2] = {0.f, 0.f};
  const float sl2 = plan.scale_log2;
  const float *dummy = nullptr; (void)dummy;
  float *score_row = scores ? scores + R.score_off + (int64_t)h * L : nullptr;

#pragma unroll 1
  for (int chunk = 0; chunk < nchunks; ++chunk) {
    cp_async_wait<kRefStages - 2>();
    __syncthreads();
    {
      const int nxt = chunk + kRefStages - 1;
      if (nxt < nchunks) load_chunk(nxt, nxt % kRefStages);
      cp_async_commit();
    }
    const int stage = chunk % kRefStages;
    const uint8_t *tk = sK + stage * RefSmem<D>::kKV;
    const uint8_t *tv = sV + stage * RefSmem<D>::kKV;

    float colmax[8][2];
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) colmax[nt][0] = colmax[nt][1] = -INFINITY;

    float s[8][4];
    auto compute_s = [&](const uint32_t (&qfr)[KSTEPS][4], int pass) {
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) s[nt][0] = s[nt][1] = s[nt][2] = s[nt][3] = 0.f;
#pragma unroll
      for (int np = 0; np < 4; ++np) {
#pragma unroll
        for (int kk = 0; kk < KSTEPS; ++kk) {
          const int key = np * 16 + (lane >> 4) * 8 + (lane & 7);
          const int c = kk * 2 + ((lane >> 3) & 1);
          uint32_t b0, b1, b2, b3;
          ldmatrix_x4(b0, b1, b2, b3, smem_u32(tk + swz<D>(key, c)));
          mma_bf16_16816(s[np * 2 + 0], qfr[kk], b0, b1);
          mma_bf16_16816(s[np * 2 + 1], qfr[kk], b2, b3);
        }
      }
      if (do_scores) {
        // column max over this thread's block rows of the UNSCALED S
        const int r0 = origin + pass * kRefRows + warp * 16 + (lane >> 2);
        const bool in0 = r0 >= bs && r0 < be, in1 = r0 + 8 >= bs && r0 + 8 < be;
#pragma unroll
        for (int nt = 0; nt < 8; ++nt) {
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            float v = -INFINITY;
            if (in0) v = s[nt][e];
            if (in1) v = fmaxf(v, s[nt][2 + e]);
            colmax[nt][e] = fmaxf(colmax[nt][e], v);
          }
        }
      }
    };
    compute_s(qf[0], 0);
    if (npass > 1) compute_s(qf[1], 1);
    if (do_scores) {
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          float v = colmax[nt][e];
          v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 4));
          v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 8));
          v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 16));
          colmax[nt][e] = v;
        }
      }
      if (lane < 4) {
#pragma unroll
        for (int nt = 0; nt < 8; ++nt) {
          sS[warp * kRefChunk + nt * 8 + lane * 2 + 0] = colmax[nt][0];
          sS[warp * kRefChunk + nt * 8 + lane * 2 + 1] = colmax[nt][1];
        }
      }
      __syncthreads();
      if (tid < kRefChunk) {
        const float v = fmaxf(fmaxf(sS[tid], sS[kRefChunk + tid]), fmaxf(sS[2 * kRefChunk + tid], sS[3 * kRefChunk + tid]));
        const int m = chunk * kRefChunk + tid;
        if (m < L) score_row[m] = v;
      }
    }
    if (score_only) continue;

    // online softmax (log2 domain); keys >= L masked
    float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int j = chunk * kRefChunk + nt * 8 + (lane & 3) * 2 + (e & 1);
        const float v = j < L ? s[nt][e] * sl2 : -INFINITY;
        s[nt][e] = v;
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
    uint32_t pa[4][4];
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      const float p0 = fast_exp2(s[nt][0] - mbase[0]);
      const float p1 = fast_exp2(s[nt][1] - mbase[0]);
      const float p2 = fast_exp2(s[nt][2] - mbase[1]);
      const float p3 = fast_exp2(s[nt][3] - mbase[1]);
      const uint32_t lo = pack_bf16(p0, p1), hi = pack_bf16(p2, p3);
      const __nv_bfloat162 blo = *reinterpret_cast<const __nv_bfloat162 *>(&lo);
      const __nv_bfloat162 bhi = *reinterpret_cast<const __nv_bfloat162 *>(&hi);
      l_r[0] += __low2float(blo) + __high2float(blo);
      l_r[1] += __low2float(bhi) + __high2float(bhi);
      pa[nt >> 1][(nt & 1) * 2 + 0] = lo;
      pa[nt >> 1][(nt & 1) * 2 + 1] = hi;
    }
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
#pragma unroll
      for (int dp = 0; dp < D / 16; ++dp) {
        const int key = ks * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
        const int c = dp * 2 + (lane >> 4);
        uint32_t b0, b1, b2, b3;
        ldmatrix_x4_trans(b0, b1, b2, b3, smem_u32(tv + swz<D>(key, c)));
        mma_bf16_16816(o[dp * 2 + 0], pa[ks], b0, b1);
        mma_bf16_16816(o[dp * 2 + 1], pa[ks], b2, b3);
      }
    }
  }
  cp_async_wait<0>();
  if (score_only) return;

#pragma unroll
  for (int r = 0; r < 2; ++r) {
    l_r[r] += __shfl_xor_sync(0xffffffffu, l_r[r], 1);
    l_r[r] += __shfl_xor_sync(0xffffffffu, l_r[r], 2);
  }
  const int qr0 = origin + warp * 16 + (lane >> 2);
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int row = qr0 + r * 8;
    if (row >= L) continue;
    const float inv = l_r[r] > 0.f ? 1.f / l_r[r] : 0.f;
    __nv_bfloat16 *dst = out + (int64_t)(R.q_off + row) * HD + (int64_t)h * D + (lane & 3) * 2;
#pragma unroll
    for (int i = 0; i < D / 8; ++i)
      *reinterpret_cast<uint32_t *>(dst + i * 8) = pack_bf16(o[i][r * 2] * inv, o[i][r * 2 + 1] * inv);
  }
}

template <int D>
static cudaError_t launch_refresh_mma_d(const Plan &plan, const void *q, const void *k, const void *v, void *out,
                                        float *scores, cudaStream_t st) {
  const int smem = RefSmem<D>::kBytes;
  cudaError_t e = cudaFuncSetAttribute(refresh_mma_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  refresh_mma_kernel<D><<<plan.total_units, kRefThreads, smem, st>>>(
      plan, (const __nv_bfloat16 *)q, (const __nv_bfloat16 *)k, (const __nv_bfloat16 *)v, (__nv_bfloat16 *)out,
      scores);
  return cudaGetLastError();
}

int refresh_mma_units(int L, int bs, int be, int H, bool with_scores) {
  return H * (ref_regular_tiles(L) + ((with_scores && ref_block_straddles(bs, be)) ? 1 : 0));
}

cudaError_t launch_refresh_mma(const Plan &plan, const void *q, const void *k, const void *v, void *out,
                               float *scores, cudaStream_t st) {
  switch (plan.D) {
    case 16: return launch_refresh_mma_d<16>(plan, q, k, v, out, scores, st);
    case 32: return launch_refresh_mma_d<32>(plan, q, k, v, out, scores, st);
    case 64: return launch_refresh_mma_d<64>(plan, q, k, v, out, scores, st);
    case 128: return launch_refresh_mma_d<128>(plan, q, k, v, out, scores, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace dllm
