// dev microbench: is F2FP.BF16.F32.PACK_AB on the MUFU (XU) pipe?
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2512_17077_b200/csrc/common.cuh"
using namespace dllm;
template <int MODE>
__global__ void k(long long *out, uint32_t *sink, int iters) {
  float x[16];
  for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-3f + i;
  uint32_t acc = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; i += 2) {
      if (MODE == 0) { acc ^= pack_bf16(x[i], x[i + 1]); x[i] += 1.f; }                       // F2FP only
      if (MODE == 1) { x[i] = fast_exp2(x[i]) * -0.5f; x[i + 1] = fast_exp2(x[i + 1]) * -0.5f; } // MUFU only
      if (MODE == 2) { float a = fast_exp2(x[i]), b = fast_exp2(x[i + 1]); acc ^= pack_bf16(a, b); x[i] = a * -0.5f; x[i+1] = b * -0.5f; }
      if (MODE == 3) { float a = fast_exp2(x[i]), b = fast_exp2(x[i + 1]);
                       uint32_t ua = __float_as_uint(a) + 0x8000u, ub = __float_as_uint(b) + 0x8000u;
                       acc ^= __byte_perm(ua, ub, 0x7632); x[i] = a * -0.5f; x[i+1] = b * -0.5f; }
    }
  }
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < 16; ++i) s += x[i];
  if (acc == 0x12345 || s == 1.234f) sink[0] = acc;
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}
int main() {
  long long *d; uint32_t *sink; cudaMalloc(&d, 8 * 2048); cudaMalloc(&sink, 64);
  long long h[4]; int iters = 2048;
  const char *names[] = {"F2FP pack only", "MUFU ex2 only", "MUFU + F2FP pack", "MUFU + IADD/PRMT pack"};
  for (int m = 0; m < 4; ++m) {
    for (int nw : {4, 8}) {
      if (m == 0) k<0><<<148, nw * 32>>>(d, sink, iters);
      if (m == 1) k<1><<<148, nw * 32>>>(d, sink, iters);
      if (m == 2) k<2><<<148, nw * 32>>>(d, sink, iters);
      if (m == 3) k<3><<<148, nw * 32>>>(d, sink, iters);
      cudaDeviceSynchronize();
      cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
      double pairs = (double)iters * 8 * nw * 32;
      printf("%-24s %d warps/SM: %.2f clk per warp-pair-op per SMSP (%.2f pairs/clk/SM)\n", names[m], nw,
             (double)h[0] / (iters * 8.0 * nw / 4), pairs / h[0]);
    }
  }
}
