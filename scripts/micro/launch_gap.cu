// dev micro: event-bracketed cost of ONE launch of an (almost) empty persistent
// kernel, as bench.py times a kernel: param size (16 B vs 12 KB __grid_constant__),
// dynamic smem (0 vs 200 KB: carveout switch after a preceding torch-like fill
// kernel), with and without a 512 MiB fill right before (the L2 flush).
#include <cstdio>
#include <cuda_runtime.h>
template <int N> struct P { int v[N]; };
template <int N> __global__ void __launch_bounds__(512) k(const __grid_constant__ P<N> p, int *out) {
  extern __shared__ int sm[];
  if (threadIdx.x == 0) { sm[0] = p.v[blockIdx.x % N]; if (sm[0] == 12345) out[0] = 1; }
}
__global__ void fill(uint4 *b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    b[i] = make_uint4(0, 0, 0, 0);
}
template <int N> float one(int *d, uint4 *fb, size_t fn, int smem, bool doflush) {
  P<N> p{};
  if (smem < 16) smem = 16;
  cudaFuncSetAttribute(k<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float tot = 0; int cnt = 0;
  for (int i = 0; i < 30; ++i) {
    if (doflush) fill<<<148 * 4, 512>>>(fb, fn);
    cudaEventRecord(a); k<N><<<148, 512, smem>>>(p, d); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); if (i >= 10) { tot += ms; ++cnt; }
  }
  return tot * 1e3f / cnt;
}
int main() {
  int *d; cudaMalloc(&d, 4);
  size_t fn = (512u << 20) / 16; uint4 *fb; cudaMalloc(&fb, fn * 16);
  for (int fl = 0; fl < 2; ++fl)
    for (int sm : {0, 200 * 1024}) {
      printf("flush=%d smem=%6d: 16B param %.2f us | 1KB %.2f us | 12KB %.2f us\n", fl, sm,
             one<4>(d, fb, fn, sm, fl), one<256>(d, fb, fn, sm, fl), one<3000>(d, fb, fn, sm, fl));
    }
  printf("last error: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
