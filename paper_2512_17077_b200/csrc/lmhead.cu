// Logit decomposition: the LM-head projection with a fused
// lowest-index ArgMax (§4.3 "Logit Decomposition", 431-432
// §5; SPEC.md:145-165 plan_logit_chunks / chunked_decode).
//
//   ids[i] = argmax_v  sum_k hidden[i,k] * W[v,k]        (ties -> lowest v)
//
// The paper bounds the logit activation by running the LM head in token chunks
// of at most max_num_logits rows, decoding each chunk and freeing its
// [chunk, V] logit buffer before the next.  On B200 the logits never reach
// HBM at all: every 128 x 256 logit tile lives only in TMEM, its epilogue
// reduces each row to (max, lowest argmax) and writes one 8-byte partial per
// (row, vocab tile); a second kernel folds the partials of each row in
// vocabulary order.  The chunking by max_num_logits is kept (it now bounds the
// partials workspace, max_num_logits x ceil(V/256) x 8 B).
//
// GEMM: tcgen05.mma M=128 (tokens) x N=256 (vocab) x K=16, bf16 -> fp32 in
// TMEM (two 256-column accumulators, so the epilogue of one tile overlaps the
// mainloop of the next), operands by TMA (128-B swizzle) through a 4-stage
// ring of 64-wide K blocks.  Persistent CTAs walk tiles vocab-major so the
// CTAs in flight share a few W tiles and all of `hidden` in L2.
// Roles: warp 0 TMA producer, warp 1 MMA issuer, warps 4-7 epilogue.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdint.h>

#include "common.cuh"
#include "tc_ptx.cuh"

namespace dllm {
namespace {

constexpr int kLM = 128;           // token rows per tile (MMA M)
constexpr int kLN = 256;           // vocab columns per tile (MMA N)
constexpr int kLK = 64;            // K block per stage (one 128-B swizzle atom)
constexpr int kLStages = 4;
constexpr int kLThreads = 256;
constexpr int kATile = kLM * kLK * 2;        // 16 KB
constexpr int kBTile = kLN * kLK * 2;        // 32 KB
constexpr int kLStage = kATile + kBTile;
constexpr int kLOffBar = kLStages * kLStage;
constexpr int kLBytes = kLOffBar + 8 * (2 * kLStages + 4) + 16 + 1024;

struct LMArgs {
  int n_rows;       // rows of this chunk
  int row0;         // first row of the chunk in `hidden`
  int vocab;
  int d_model;
  int m_tiles, v_tiles;
  float2 *partial;  // [v_tiles][n_rows] (max, argmax as int bits)
};

__global__ void __launch_bounds__(kLThreads, 1)
lmhead_argmax_kernel(const __grid_constant__ CUtensorMap tm_h, const __grid_constant__ CUtensorMap tm_w,
                     const __grid_constant__ LMArgs a) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t sb = (raw + 1023u) & ~1023u;
  uint8_t *gb = smem_raw + (sb - raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t b_full = sb + kLOffBar;          // [kLStages] TMA tx
  const uint32_t b_empty = b_full + 8 * kLStages; // [kLStages] MMA commit
  const uint32_t b_afull = b_empty + 8 * kLStages;  // [2] MMA commit: accumulator ready
  const uint32_t b_aempty = b_afull + 16;           // [2] epilogue warps (4)
  const uint32_t b_tslot = b_aempty + 16;
  const int ntiles = a.m_tiles * a.v_tiles;
  const int kblocks = a.d_model / kLK;

  if (threadIdx.x == 0) {
    for (int i = 0; i < kLStages; ++i) {
      ptx::mbar_init(b_full + 8 * i, 1);
      ptx::mbar_init(b_empty + 8 * i, 1);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(b_afull + 8 * i, 1);
      ptx::mbar_init(b_aempty + 8 * i, 4);
    }
    ptx::fence_mbar_init();
    ptx::tma_prefetch_desc(&tm_h);
    ptx::tma_prefetch_desc(&tm_w);
  }
  if (warp == 1) {
    ptx::tmem_alloc(b_tslot, 512);
    ptx::tmem_relinquish();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t *>(gb + (b_tslot - sb));

  if (warp == 0) {
    // ============================ TMA producer ============================
    int it = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      const int vt = tile / a.m_tiles, mt = tile - vt * a.m_tiles;
      for (int kb = 0; kb < kblocks; ++kb, ++it) {
        const int s = it % kLStages;
        ptx::mbar_wait(b_empty + 8 * s, ((it / kLStages) & 1) ^ 1);
        if (lane == 0) {
          ptx::mbar_arrive_expect_tx(b_full + 8 * s, (uint32_t)kLStage);
          ptx::tma_load_2d(sb + s * kLStage, &tm_h, b_full + 8 * s, kb * kLK, a.row0 + mt * kLM);
          ptx::tma_load_2d(sb + s * kLStage + kATile, &tm_w, b_full + 8 * s, kb * kLK, vt * kLN);
        }
        __syncwarp();
      }
    }
  } else if (warp == 1) {
    // ============================ MMA issuer ============================
    constexpr uint32_t idesc = ptx::idesc_bf16_f32(kLM, kLN, false, false);
    const uint64_t da = ptx::smem_desc_sw128(sb, 16, 1024);
    const uint64_t db = ptx::smem_desc_sw128(sb + kATile, 16, 1024);
    int it = 0, tc = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++tc) {
      const int acc = tc & 1;
      ptx::mbar_wait(b_aempty + 8 * acc, ((tc >> 1) & 1) ^ 1);
      ptx::tc_fence_after();
      for (int kb = 0; kb < kblocks; ++kb, ++it) {
        const int s = it % kLStages;
        ptx::mbar_wait(b_full + 8 * s, (it / kLStages) & 1);
        ptx::tc_fence_after();
        const uint64_t off = (uint64_t)((s * kLStage) >> 4);
#pragma unroll
        for (int k = 0; k < kLK / 16; ++k)
          ptx::mma_ss_elect(tmem + (uint32_t)(acc * kLN), da + off + (uint64_t)(k * 2), db + off + (uint64_t)(k * 2),
                            idesc, (kb > 0 || k > 0) ? 1u : 0u);
        ptx::mma_commit_elect(b_empty + 8 * s);
      }
      ptx::mma_commit_elect(b_afull + 8 * acc);
    }
  } else if (warp >= 4) {
    // ============================ epilogue ============================
    // thread = token row (TMEM lane); strict '>' over ascending columns keeps the
    // lowest index among equal maxima
    const int ew = warp & 3;
    const uint32_t lane_base = (uint32_t)(ew * 32) << 16;
    int tc = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++tc) {
      const int vt = tile / a.m_tiles, mt = tile - vt * a.m_tiles;
      const int acc = tc & 1;
      ptx::mbar_wait(b_afull + 8 * acc, (tc >> 1) & 1);
      ptx::tc_fence_after();
      const int v0 = vt * kLN;
      const int ncols = min(kLN, a.vocab - v0);
      float best = -INFINITY;
      int bidx = v0;
#pragma unroll 1
      for (int cc = 0; cc < kLN / 32; ++cc) {
        uint32_t r[32];
        DLLM_TMEM_LD32(tmem + lane_base + (uint32_t)(acc * kLN + cc * 32), r);
        ptx::tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const float v = __uint_as_float(r[j]);
          const int col = cc * 32 + j;
          if (col < ncols && v > best) {
            best = v;
            bidx = v0 + col;
          }
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(b_aempty + 8 * acc);
      const int row = mt * kLM + ew * 32 + lane;
      if (row < a.n_rows) a.partial[(int64_t)vt * a.n_rows + row] = make_float2(best, __int_as_float(bidx));
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (warp == 1) ptx::tmem_dealloc(tmem, 512);
}

// per row: fold the vocab-tile partials in vocabulary order (strict '>' keeps
// the lowest index on ties, since tiles are visited in ascending order)
__global__ void lmhead_reduce_kernel(const float2 *__restrict__ partial, int n_rows, int v_tiles, int32_t *ids) {
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= n_rows) return;
  const float2 p0 = partial[row];
  float best = p0.x;
  int bidx = __float_as_int(p0.y);
  for (int vt = 1; vt < v_tiles; ++vt) {
    const float2 p = partial[(int64_t)vt * n_rows + row];
    if (p.x > best) {
      best = p.x;
      bidx = __float_as_int(p.y);
    }
  }
  ids[row] = bidx;
}

PFN_cuTensorMapEncodeTiled_v12000 lm_encode_fn() {
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

int lm_num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

}  // namespace

int64_t lmhead_vocab_tiles(int vocab) { return (vocab + kLN - 1) / kLN; }

// One chunk of rows [row0, row0 + n_rows): partials then ids[row0 ...].
cudaError_t launch_lmhead_chunk(const void *hidden, const void *weight, int n_tok, int d_model, int vocab, int row0,
                                int n_rows, int32_t *ids, void *workspace, cudaStream_t st) {
  if (n_rows <= 0) return cudaSuccess;
  auto enc = lm_encode_fn();
  if (!enc) return cudaErrorNotSupported;
  CUtensorMap th, tw;
  {
    cuuint64_t dims[2] = {(cuuint64_t)d_model, (cuuint64_t)n_tok};
    cuuint64_t strides[1] = {(cuuint64_t)d_model * 2};
    cuuint32_t box[2] = {(cuuint32_t)kLK, (cuuint32_t)kLM};
    cuuint32_t es[2] = {1, 1};
    if (enc(&th, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(hidden), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  {
    cuuint64_t dims[2] = {(cuuint64_t)d_model, (cuuint64_t)vocab};
    cuuint64_t strides[1] = {(cuuint64_t)d_model * 2};
    cuuint32_t box[2] = {(cuuint32_t)kLK, (cuuint32_t)kLN};
    cuuint32_t es[2] = {1, 1};
    if (enc(&tw, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(weight), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  LMArgs a;
  a.n_rows = n_rows;
  a.row0 = row0;
  a.vocab = vocab;
  a.d_model = d_model;
  a.m_tiles = (n_rows + kLM - 1) / kLM;
  a.v_tiles = (int)lmhead_vocab_tiles(vocab);
  a.partial = reinterpret_cast<float2 *>(workspace);
  cudaError_t e = cudaFuncSetAttribute(lmhead_argmax_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kLBytes);
  if (e != cudaSuccess) return e;
  const int ntiles = a.m_tiles * a.v_tiles;
  const int grid = ntiles < lm_num_sms() ? ntiles : lm_num_sms();
  lmhead_argmax_kernel<<<grid, kLThreads, kLBytes, st>>>(th, tw, a);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  lmhead_reduce_kernel<<<(n_rows + 255) / 256, 256, 0, st>>>(a.partial, n_rows, a.v_tiles, ids + row0);
  return cudaGetLastError();
}

}  // namespace dllm
