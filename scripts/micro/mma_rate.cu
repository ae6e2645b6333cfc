// dev microbench: tcgen05.mma issue/execute rate for the Refresh shapes (one CTA per SM)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2512_17077_b200/csrc/tc_ptx.cuh"
#include "../../paper_2512_17077_b200/csrc/common.cuh"
using namespace dllm;

template <int N, bool TS, int COMMIT_EVERY = 0, int LDWARPS = 0>
__global__ void mma_kernel(long long *out, int iters) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  __shared__ __align__(8) uint64_t bar2;
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  if (warp == 0) { ptx::tmem_alloc(smem_u32(&slot), 512); ptx::tmem_relinquish(); }
  if (threadIdx.x == 0) { ptx::mbar_init(smem_u32(&bar), 1); ptx::mbar_init(smem_u32(&bar2), 1 << 20); ptx::fence_mbar_init(); }
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(smem)[i] = 0;
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before(); __syncthreads(); ptx::tc_fence_after();
  const uint32_t tmem = slot;
  long long t0 = 0, t1 = 0;
  if (warp == 0 && lane == 0) {
    const uint32_t sa = smem_u32(smem), sbb = sa + 32768;
    constexpr uint32_t idesc = ptx::idesc_bf16_f32(128, N, false, TS);
    const uint64_t a0 = ptx::smem_desc_sw128(sa, 16, 1024);
    const uint64_t b0 = ptx::smem_desc_sw128(sbb, TS ? 8192 : 16, 1024);
    t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if (TS) ptx::mma_ts(tmem + 256, tmem + (uint32_t)(k * 8), b0 + (uint64_t)(k * 128), idesc, 1u);
        else ptx::mma_ss(tmem, a0 + (uint64_t)(k * 2), b0 + (uint64_t)(k * 2), idesc, 1u);
        if (COMMIT_EVERY && (k % COMMIT_EVERY) == COMMIT_EVERY - 1) ptx::mma_commit(smem_u32(&bar2));
      }
    }
    ptx::mma_commit(smem_u32(&bar));
    ptx::mbar_wait(smem_u32(&bar), 0);
    t1 = clock64();
  }
  if (LDWARPS && warp >= 1 && warp <= LDWARPS) {
    // concurrent TMEM readers (like the softmax warps): lanes of quarter warp%4, columns 128..191
    uint32_t acc = 0;
    const uint32_t t = tmem + (((warp & 3) * 32) << 16) + 128;
    for (int i = 0; i < iters * 2; ++i) {
      uint32_t r[32];
      DLLM_TMEM_LD32(t + (i & 1) * 32, r);
      ptx::tmem_wait_ld();
#pragma unroll
      for (int k = 0; k < 32; ++k) acc ^= r[k];
    }
    if (acc == 0x1234567) out[1000] = acc;
  }
  __syncwarp();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  ptx::tc_fence_before(); __syncthreads(); ptx::tc_fence_after();
  if (warp == 0) ptx::tmem_dealloc(tmem, 512);
}

template <int N, bool TS, int CE = 0, int LW = 0>
void run(long long *d, const char *name) {
  const int iters = 512;
  cudaFuncSetAttribute(mma_kernel<N, TS, CE, LW>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 1024);
  mma_kernel<N, TS, CE, LW><<<148, 384, 65536 + 1024>>>(d, iters);
  cudaDeviceSynchronize();
  long long h;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  const double per = (double)h / (iters * 8);
  const double ideal = 128.0 * N / 256.0;
  printf("%-28s %7.1f clk per MMA (ideal %5.1f) -> %5.1f%% ; err=%s\n", name, per, ideal, 100 * ideal / per,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  long long *d; cudaMalloc(&d, 8 * 256);
  run<64, false>(d, "SS M128 N64  K16 (QK tc2)");
  run<128, false>(d, "SS M128 N128 K16 (QK tc1)");
  run<256, false>(d, "SS M128 N256 K16");
  run<64, true>(d, "TS M128 N64  K16");
  run<128, true>(d, "TS M128 N128 K16 (PV)");
  run<128, false, 8>(d, "SS N128 + commit every 8");
  run<128, false, 4>(d, "SS N128 + commit every 4");
  run<128, false, 1>(d, "SS N128 + commit every 1");
  run<64, false, 8>(d, "SS N64 + commit every 8");
  run<128, false, 0, 4>(d, "SS N128 + 4 TMEM-ld warps");
  run<128, false, 0, 8>(d, "SS N128 + 8 TMEM-ld warps");
  run<64, false, 0, 8>(d, "SS N64 + 8 TMEM-ld warps");
  run<128, true, 0, 8>(d, "TS N128 + 8 TMEM-ld warps");
  run<128, true, 4>(d, "TS N128 + commit every 4");
}
