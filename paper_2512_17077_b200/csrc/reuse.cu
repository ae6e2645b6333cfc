// Reuse sparse attention (§2.3, Eq. 4; per-head key sets
// of §4.5).
//
// For request b, query head h and the active block's query rows q:
//   O_b[q,h] = softmax_j(tau Q_blk[q,h].K[j,kv(h)]) V[j,kv(h)],
//   j in J^h = [bs, be) ++ idx(b,h)
// K/V are gathered IN PLACE from the paged cache through the block table:
// no pack, no assembly copy (the paper's assembly layer, is
// eliminated).
//
// Work unit = (b, h, 32-row group of the block); units of the heads of one
// KV group are adjacent so their overlapping selections hit L2.  128 threads
// = 4 warps: warp w owns query rows 16*(w&1) .. +16 and keys 32*(w>>1) .. +32
// of every 64-key chunk.  Chunks are gathered with 16-byte cp.async (one
// 256-byte K row and V row per key at D=128) into a 3-stage ring, then
// mma.sync m16n8k16 bf16 (fp32 accumulate) computes S = Q K^T and O += P V
// with a register-resident online softmax (exp2, quad shuffles).  The two
// key halves are merged through shared memory at the end.
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "plan.h"

namespace dllm {

constexpr int kReuseThreads = 128;
constexpr int kReuseRows = 32;     // query rows per unit
constexpr int kReuseChunk = 64;    // keys per pipeline stage
constexpr int kReuseStages = 3;

template <int D>
struct ReuseSmem {
  static constexpr int kQ = kReuseRows * D * 2;
  static constexpr int kKV = kReuseChunk * D * 2;
  static constexpr int kBytes = kQ + kReuseStages * 2 * kKV;
};

template <int D>
__global__ void __launch_bounds__(kReuseThreads, 2)
reuse_kernel(const __grid_constant__ Plan plan, const __nv_bfloat16 *__restrict__ q_blk,
             const __nv_bfloat16 *__restrict__ k_cache, const __nv_bfloat16 *__restrict__ v_cache,
             const int32_t *__restrict__ idx, __nv_bfloat16 *__restrict__ out) {
  extern __shared__ __align__(128) uint8_t smem[];
  constexpr int CH = D / 8;                              // 16-byte chunks per row
  constexpr int KSTEPS = D / 16;
  uint8_t *sQ = smem;
  uint8_t *sK = smem + ReuseSmem<D>::kQ;
  uint8_t *sV = sK + kReuseStages * ReuseSmem<D>::kKV;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int unit = blockIdx.x;
  const int b = plan_find(plan, unit);
  const ReqInfo &R = plan.r[b];
  const int blk = R.be - R.bs;
  const int ngroups = (blk + kReuseRows - 1) / kReuseRows;
  const int local = unit - R.unit_off;
  const int h = local / ngroups;
  const int rg = local - h * ngroups;
  const int kvh = h / (plan.H / plan.H_kv);
  const int nk = blk + R.k;
  const int nchunks = (nk + kReuseChunk - 1) / kReuseChunk;
  const int row0 = rg * kReuseRows;
  const int64_t HD = (int64_t)plan.H * D;
  const int32_t *my_idx = idx + R.idx_off + (int64_t)h * R.k;
  const int32_t *bt = plan.block_table + (int64_t)R.bt_row * plan.pages_per_req;

  // ---- Q rows of this unit (zero-filled past the block)
  for (int i = tid; i < kReuseRows * CH; i += kReuseThreads) {
    const int r = i / CH, c = i - r * CH;
    const bool ok = row0 + r < blk;
    const __nv_bfloat16 *src = q_blk + (int64_t)(R.blk_off + (ok ? row0 + r : 0)) * HD + (int64_t)h * D + c * 8;
    cp_async16(smem_u32(sQ + swz<D>(r, c)), src, ok ? 16 : 0);
  }

  auto load_chunk = [&](int chunk, int stage) {
    uint8_t *dk = sK + stage * ReuseSmem<D>::kKV;
    uint8_t *dv = sV + stage * ReuseSmem<D>::kKV;
    constexpr int ROWS_PER_PASS = kReuseThreads / CH;
    const int c = tid % CH;
#pragma unroll 4
    for (int r = tid / CH; r < kReuseChunk; r += ROWS_PER_PASS) {
      const int j = chunk * kReuseChunk + r;
      const bool ok = j < nk;
      int64_t off = 0;
      if (ok) {
        const int pos = j < blk ? R.bs + j : __ldg(my_idx + (j - blk));
        const int page = __ldg(bt + (pos >> plan.page_shift));
        const int slot = pos & (plan.page_size - 1);
        off = (((int64_t)page * plan.H_kv + kvh) * plan.page_size + slot) * D + c * 8;
      }
      cp_async16(smem_u32(dk + swz<D>(r, c)), k_cache + off, ok ? 16 : 0);
      cp_async16(smem_u32(dv + swz<D>(r, c)), v_cache + off, ok ? 16 : 0);
    }
  };

#pragma unroll
  for (int s = 0; s < kReuseStages - 1; ++s) {
    if (s < nchunks) load_chunk(s, s);
    cp_async_commit();
  }

  const int rh = warp & 1;          // row half: rows 16*rh .. +16
  const int kh = warp >> 1;         // key half: keys 32*kh .. +32 of a chunk
  uint32_t qf[KSTEPS][4];
  float o[D / 8][4];
#pragma unroll
  for (int i = 0; i < D / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m_r[2] = {-INFINITY, -INFINITY}, l_r[2] = {0.f, 0.f};
  const float sl2 = plan.scale_log2;

#pragma unroll 1
  for (int chunk = 0; chunk < nchunks; ++chunk) {
    cp_async_wait<kReuseStages - 2>();
    __syncthreads();
    {
      const int nxt = chunk + kReuseStages - 1;
      if (nxt < nchunks) load_chunk(nxt, nxt % kReuseStages);
      cp_async_commit();
    }
    if (chunk == 0) {
#pragma unroll
      for (int kk = 0; kk < KSTEPS; ++kk) {
        const int r = rh * 16 + (lane & 15);
        const int c = kk * 2 + (lane >> 4);
        ldmatrix_x4(qf[kk][0], qf[kk][1], qf[kk][2], qf[kk][3], smem_u32(sQ + swz<D>(r, c)));
      }
    }
    const int stage = chunk % kReuseStages;
    const uint8_t *tk = sK + stage * ReuseSmem<D>::kKV;
    const uint8_t *tv = sV + stage * ReuseSmem<D>::kKV;

    // S = Q K^T for this warp's 16 rows x 32 keys
    float s[4][4];
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) s[nt][0] = s[nt][1] = s[nt][2] = s[nt][3] = 0.f;
#pragma unroll
    for (int np = 0; np < 2; ++np) {
#pragma unroll
      for (int kk = 0; kk < KSTEPS; ++kk) {
        const int key = kh * 32 + np * 16 + (lane >> 4) * 8 + (lane & 7);
        const int c = kk * 2 + ((lane >> 3) & 1);
        uint32_t b0, b1, b2, b3;
        ldmatrix_x4(b0, b1, b2, b3, smem_u32(tk + swz<D>(key, c)));
        mma_bf16_16816(s[np * 2 + 0], qf[kk], b0, b1);
        mma_bf16_16816(s[np * 2 + 1], qf[kk], b2, b3);
      }
    }
    // mask keys past the end of the list; online softmax (log2 domain)
    const int kbase = chunk * kReuseChunk + kh * 32 + (lane & 3) * 2;
    float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int j = kbase + nt * 8 + (e & 1);
        float v = j < nk ? s[nt][e] * sl2 : -INFINITY;
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
    uint32_t pa[2][4];
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      const float p0 = fast_exp2(s[nt][0] - mbase[0]);
      const float p1 = fast_exp2(s[nt][1] - mbase[0]);
      const float p2 = fast_exp2(s[nt][2] - mbase[1]);
      const float p3 = fast_exp2(s[nt][3] - mbase[1]);
      // the row sum uses the bf16-rounded P that feeds P.V
      const uint32_t lo = pack_bf16(p0, p1), hi = pack_bf16(p2, p3);
      const __nv_bfloat162 blo = *reinterpret_cast<const __nv_bfloat162 *>(&lo);
      const __nv_bfloat162 bhi = *reinterpret_cast<const __nv_bfloat162 *>(&hi);
      l_r[0] += __low2float(blo) + __high2float(blo);
      l_r[1] += __low2float(bhi) + __high2float(bhi);
      pa[nt >> 1][(nt & 1) * 2 + 0] = lo;
      pa[nt >> 1][(nt & 1) * 2 + 1] = hi;
    }
    // O += P V  (k = this warp's 32 keys in two 16-key steps)
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
#pragma unroll
      for (int dp = 0; dp < D / 16; ++dp) {
        const int key = kh * 32 + ks * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
        const int c = dp * 2 + (lane >> 4);
        uint32_t b0, b1, b2, b3;
        ldmatrix_x4_trans(b0, b1, b2, b3, smem_u32(tv + swz<D>(key, c)));
        mma_bf16_16816(o[dp * 2 + 0], pa[ks], b0, b1);
        mma_bf16_16816(o[dp * 2 + 1], pa[ks], b2, b3);
      }
    }
  }
  cp_async_wait<0>();
  __syncthreads();

  // ---- merge the two key halves (warps w and w+2 share rows)
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    l_r[r] += __shfl_xor_sync(0xffffffffu, l_r[r], 1);
    l_r[r] += __shfl_xor_sync(0xffffffffu, l_r[r], 2);
  }
  constexpr int STRIDE = D / 2 + 4;                    // floats per lane record
  float *xbuf = reinterpret_cast<float *>(sK);         // [2 rh][32 lanes][STRIDE]
  float *rec = xbuf + (rh * 32 + lane) * STRIDE;
  if (kh == 1) {
#pragma unroll
    for (int i = 0; i < D / 8; ++i)
#pragma unroll
      for (int e = 0; e < 4; ++e) rec[i * 4 + e] = o[i][e];
    rec[D / 2 + 0] = m_r[0]; rec[D / 2 + 1] = m_r[1];
    rec[D / 2 + 2] = l_r[0]; rec[D / 2 + 3] = l_r[1];
  }
  __syncthreads();
  if (kh == 0) {
    float sc_self[2], sc_other[2], inv[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const float m2 = rec[D / 2 + r], l2 = rec[D / 2 + 2 + r];
      const float m = fmaxf(m_r[r], m2);
      const float mb = m == -INFINITY ? 0.f : m;
      sc_self[r] = fast_exp2(m_r[r] - mb);
      sc_other[r] = fast_exp2(m2 - mb);
      const float l = l_r[r] * sc_self[r] + l2 * sc_other[r];
      inv[r] = l > 0.f ? 1.f / l : 0.f;
    }
    const int qr0 = row0 + rh * 16 + (lane >> 2);
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int qrow = qr0 + r * 8;
      if (qrow >= blk) continue;
      __nv_bfloat16 *dst = out + (int64_t)(R.blk_off + qrow) * HD + (int64_t)h * D + (lane & 3) * 2;
#pragma unroll
      for (int i = 0; i < D / 8; ++i) {
        const float v0 = (o[i][r * 2 + 0] * sc_self[r] + rec[i * 4 + r * 2 + 0] * sc_other[r]) * inv[r];
        const float v1 = (o[i][r * 2 + 1] * sc_self[r] + rec[i * 4 + r * 2 + 1] * sc_other[r]) * inv[r];
        *reinterpret_cast<uint32_t *>(dst + i * 8) = pack_bf16(v0, v1);
      }
    }
  }
}

template <int D>
static cudaError_t launch_reuse_d(const Plan &plan, const void *q_blk, const void *k_cache,
                                  const void *v_cache, const int32_t *idx, void *out, cudaStream_t st) {
  const int smem = ReuseSmem<D>::kBytes;
  cudaError_t e = cudaFuncSetAttribute(reuse_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  reuse_kernel<D><<<plan.total_units, kReuseThreads, smem, st>>>(
      plan, (const __nv_bfloat16 *)q_blk, (const __nv_bfloat16 *)k_cache, (const __nv_bfloat16 *)v_cache,
      idx, (__nv_bfloat16 *)out);
  return cudaGetLastError();
}

cudaError_t launch_reuse(const Plan &plan, const void *q_blk, const void *k_cache, const void *v_cache,
                         const int32_t *idx, void *out, cudaStream_t st) {
  switch (plan.D) {
    case 16: return launch_reuse_d<16>(plan, q_blk, k_cache, v_cache, idx, out, st);
    case 32: return launch_reuse_d<32>(plan, q_blk, k_cache, v_cache, idx, out, st);
    case 64: return launch_reuse_d<64>(plan, q_blk, k_cache, v_cache, idx, out, st);
    case 128: return launch_reuse_d<128>(plan, q_blk, k_cache, v_cache, idx, out, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace dllm
