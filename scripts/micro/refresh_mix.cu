// dev microbench: the tensor-pipe time of one Refresh step's MMA mix, issued back to
// back with no data dependencies (one CTA per SM, all SMs):
//   per 64-key step and Q tile i: P.V  (TS, M128 N128, K = 64 keys: 4 x K16)
//                                 Q.K^T (SS, M128 N64,  K = D = 128: 8 x K16)
// against the same work with 128-key score tiles (QK^T SS N128, P.V K = 128) and
// with Q.K^T reading Q from TMEM (TS) -- what the softmax could at best overlap.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 refresh_mix.cu -o /tmp/mix
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2512_17077_b200/csrc/tc_ptx.cuh"
#include "../../paper_2512_17077_b200/csrc/common.cuh"
using namespace dllm;

// MODE 0: refresh_tc2 mix (2 tiles x (PV TS N128 K64 + QK SS N64 K128)) per 64-key step
// MODE 1: 128-key tiles: per 128-key step 2 tiles x (PV TS N128 K128 + QK SS N128 K128), reported per 64 keys
// MODE 2: as 0 but Q.K^T as TS (Q from TMEM, A operand), B = K from smem
// MODE 3: QK only (SS N64), MODE 4: PV only (TS N128 K64)
template <int MODE, int LDWARPS>
__global__ void mix_kernel(long long *out, int iters) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  __shared__ __align__(8) uint64_t bar2;
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t sb = (raw + 1023u) & ~1023u;
  uint8_t *gb = smem_raw + (sb - raw);
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  if (warp == 0) { ptx::tmem_alloc(smem_u32(&slot), 512); ptx::tmem_relinquish(); }
  if (threadIdx.x == 0) { ptx::mbar_init(smem_u32(&bar), 1); ptx::mbar_init(smem_u32(&bar2), 1 << 20); ptx::fence_mbar_init(); }
  for (int i = threadIdx.x; i < 128 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(gb)[i] = 0;
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before(); __syncthreads(); ptx::tc_fence_after();
  const uint32_t tmem = slot;
  long long t0 = 0, t1 = 0;
  // smem: Q 2 x 32 KB at 0, K 32 KB at 64 KB, V 32 KB at 96 KB (128-B swizzled K-major)
  const uint64_t dq = ptx::smem_desc_sw128(sb, 16, 1024);
  const uint64_t dk = ptx::smem_desc_sw128(sb + 65536, 16, 1024);
  const int TBN = MODE == 1 ? 128 : 64;
  const uint64_t dv = ptx::smem_desc_sw128(sb + 98304, TBN * 128, 1024);
  if (warp == 0) {
    constexpr uint32_t idesc_qk = ptx::idesc_bf16_f32(128, MODE == 1 ? 128 : 64, false, false);
    constexpr uint32_t idesc_pv = ptx::idesc_bf16_f32(128, 128, false, true);
    t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      for (int i = 0; i < 2; ++i) {
        const uint32_t ts = MODE == 1 ? (uint32_t)(i * 128) : (uint32_t)(i * 128 + (it & 1) * 64);
        const uint32_t to = i ? 384u : 256u;
        if (MODE != 3) {
#pragma unroll
          for (int k = 0; k < (MODE == 1 ? 8 : 4); ++k)
            ptx::mma_ts_elect(tmem + to, tmem + ts + (uint32_t)(k * 8), dv + (uint64_t)((k * 16 * 128) >> 4), idesc_pv, 1u);
          ptx::mma_commit_elect(smem_u32(&bar2));
        }
        if (MODE != 4) {
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const uint32_t ko = (uint32_t)(((k >> 2) * 128 * 128 + (k & 3) * 32) >> 4);
            const uint32_t kb = (uint32_t)(((k >> 2) * TBN * 128 + (k & 3) * 32) >> 4);
            if (MODE == 2)
              ptx::mma_ts_elect(tmem + ts, tmem + to + (uint32_t)(k * 8), dk + kb, idesc_qk, 1u);  // A from TMEM (timing only)
            else
              ptx::mma_ss_elect(tmem + ts, dq + (uint64_t)((i * 32768) >> 4) + ko, dk + kb, idesc_qk, 1u);
          }
          ptx::mma_commit_elect(smem_u32(&bar2));
        }
      }
    }
    ptx::mma_commit_elect(smem_u32(&bar));
    ptx::mbar_wait(smem_u32(&bar), 0);
    t1 = clock64();
  }
  if (LDWARPS && warp >= 4 && warp < 4 + LDWARPS) {
    // softmax-like TMEM traffic: 64 columns loaded + 32 stored per step per warp
    uint32_t acc = 0;
    const uint32_t t = tmem + (((warp & 3) * 32) << 16) + ((warp >> 2) & 1) * 128;
    for (int i = 0; i < iters; ++i) {
      uint32_t r[32], r2[32];
      DLLM_TMEM_LD32(t + (i & 1) * 64, r);
      DLLM_TMEM_LD32(t + (i & 1) * 64 + 32, r2);
      ptx::tmem_wait_ld();
#pragma unroll
      for (int k = 0; k < 32; ++k) r[k] ^= r2[k];
      DLLM_TMEM_ST32(t + (i & 1) * 64, r);
      ptx::tmem_wait_st();
      acc ^= r[lane];
    }
    if (acc == 0x1234567) out[1000] = acc;
  }
  __syncwarp();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  ptx::tc_fence_before(); __syncthreads(); ptx::tc_fence_after();
  if (warp == 0) ptx::tmem_dealloc(tmem, 512);
}

template <int MODE, int LW>
void run(long long *d, const char *name) {
  const int iters = 1024;
  const int smem = 128 * 1024 + 1024;
  cudaFuncSetAttribute(mix_kernel<MODE, LW>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  mix_kernel<MODE, LW><<<148, 384, smem>>>(d, iters);
  cudaDeviceSynchronize();
  mix_kernel<MODE, LW><<<148, 384, smem>>>(d, iters);
  cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, 8 * 148, cudaMemcpyDeviceToHost);
  double m = 0;
  for (int i = 0; i < 148; ++i) m += h[i];
  m /= 148;
  const double per = m / iters / (MODE == 1 ? 2 : 1);            // clk per 64 keys of both tiles
  const double nominal = MODE >= 3 ? 512.0 : 1024.0;             // 8192 FLOP/clk/SM
  printf("%-58s %7.1f clk per 64-key step (nominal %6.1f) -> %5.1f%% ; err=%s\n", name, per, nominal,
         100 * nominal / per, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  long long *d;
  cudaMalloc(&d, 8 * 2048);
  run<0, 0>(d, "tc2 mix: 2 x (PV TS N128 K64 + QK SS N64 K128)");
  run<0, 8>(d, "tc2 mix + 8 softmax-like TMEM warps");
  run<1, 0>(d, "128-key tiles: 2 x (PV TS N128 K128 + QK SS N128 K128)");
  run<1, 8>(d, "128-key tiles + 8 TMEM warps");
  run<2, 0>(d, "tc2 mix with QK as TS (Q in TMEM)");
  run<3, 0>(d, "QK only (SS N64 K128, 2 tiles)");
  run<4, 0>(d, "PV only (TS N128 K64, 2 tiles)");
}
