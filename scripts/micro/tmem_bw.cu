// Microbenchmarks (dev only): TMEM load bandwidth (32x32b.x32), MUFU ex2 rate,
// mma.sync m16n8k16 bf16 rate, per SM.  nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2512_17077_b200/csrc/tc_ptx.cuh"
#include "../../paper_2512_17077_b200/csrc/common.cuh"
using namespace dllm;

__global__ void tmem_ld_kernel(long long *out, int iters, int nwarps_active) {
  __shared__ uint32_t slot;
  int warp = threadIdx.x / 32;
  if (warp == 0) { ptx::tmem_alloc(smem_u32(&slot), 512); ptx::tmem_relinquish(); }
  ptx::tc_fence_before(); __syncthreads(); ptx::tc_fence_after();
  uint32_t t = slot + (((warp & 3) * 32) << 16);
  uint32_t acc = 0;
  long long t0 = clock64();
  if (warp < nwarps_active) {
    for (int i = 0; i < iters; ++i) {
      uint32_t r[32];
      DLLM_TMEM_LD32(t + (i & 3) * 32, r);
      ptx::tmem_wait_ld();
      #pragma unroll
      for (int k = 0; k < 32; ++k) acc ^= r[k];
    }
  }
  long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  if (acc == 12345) out[1000] = acc;
  ptx::tc_fence_before(); __syncthreads(); ptx::tc_fence_after();
  if (warp == 0) ptx::tmem_dealloc(slot, 512);
}

__global__ void mufu_kernel(long long *out, float *sink, int iters) {
  float x[8];
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3f + k;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    #pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = fast_exp2(x[k]) * -0.5f;
  }
  long long t1 = clock64();
  float s = 0; for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 1.2345f) sink[0] = s;
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}

__global__ void hmma_kernel(long long *out, float *sink, int iters) {
  uint32_t a[4] = {threadIdx.x, 1, 2, 3};
  float d[8][4] = {};
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    #pragma unroll
    for (int k = 0; k < 8; ++k) mma_bf16_16816(d[k], a, a[0] + k, a[1]);
  }
  long long t1 = clock64();
  float s = 0; for (int k = 0; k < 8; ++k) s += d[k][0];
  if (s == 1.2345f) sink[0] = s;
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}

int main() {
  long long *d; float *sink; cudaMalloc(&d, 8 * 2048); cudaMalloc(&sink, 64);
  long long h[148];
  int iters = 4096;
  for (int nw : {1, 4, 8}) {
    tmem_ld_kernel<<<148, 256>>>(d, iters, nw); cudaDeviceSynchronize();
    cudaMemcpy(h, d, 8 * 148, cudaMemcpyDeviceToHost);
    double bytes = (double)iters * nw * 32 * 32 * 4;
    printf("TMEM ld32x32b.x32: %d warps/SM: %.1f B/clk/SM (%.0f clk per warp-load)\n", nw, bytes / h[0], (double)h[0] / iters);
  }
  for (int nw : {4, 8, 16}) {
    mufu_kernel<<<148, nw * 32>>>(d, sink, iters); cudaDeviceSynchronize();
    cudaMemcpy(h, d, 8 * 148, cudaMemcpyDeviceToHost);
    printf("MUFU ex2: %d warps/SM: %.2f ex2/clk/SM\n", nw, (double)iters * 8 * nw * 32 / h[0]);
  }
  for (int nw : {4, 8, 16}) {
    hmma_kernel<<<148, nw * 32>>>(d, sink, iters); cudaDeviceSynchronize();
    cudaMemcpy(h, d, 8 * 148, cudaMemcpyDeviceToHost);
    printf("HMMA m16n8k16 bf16: %d warps/SM: %.0f FLOP/clk/SM\n", nw, (double)iters * 8 * nw * 4096.0 / h[0]);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
