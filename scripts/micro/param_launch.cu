// dev micro: launch cost of a kernel with a large __grid_constant__ parameter
// (the Plan is ~10 KB) vs a small one, 148 CTAs, back-to-back launches timed with events.
#include <cstdio>
#include <cuda_runtime.h>
template <int N> struct P { int v[N]; };
template <int N> __global__ void k(const __grid_constant__ P<N> p, int *out) {
  if (threadIdx.x == 0 && p.v[blockIdx.x % N] == 12345) out[0] = 1;
}
template <int N> float run(int *d, int iters) {
  P<N> p{}; cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int i = 0; i < 10; ++i) k<N><<<148, 288>>>(p, d);
  cudaEventRecord(a);
  for (int i = 0; i < iters; ++i) k<N><<<148, 288>>>(p, d);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b); return ms * 1e3f / iters;
}
template <int N> float run1(int *d) {  // single launch between events (what bench sees)
  P<N> p{}; cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float tot = 0;
  for (int i = 0; i < 20; ++i) {
    cudaEventRecord(a); k<N><<<148, 288>>>(p, d); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); if (i >= 5) tot += ms;
  }
  return tot * 1e3f / 15;
}
int main() {
  int *d; cudaMalloc(&d, 4);
  printf("16 B param : %.2f us/launch back-to-back, %.2f us single\n", run<4>(d, 200), run1<4>(d));
  printf("1 KB param : %.2f us/launch back-to-back, %.2f us single\n", run<256>(d, 200), run1<256>(d));
  printf("10 KB param: %.2f us/launch back-to-back, %.2f us single\n", run<2600>(d, 200), run1<2600>(d));
  printf("30 KB param: %.2f us/launch back-to-back, %.2f us single\n", run<7600>(d, 200), run1<7600>(d));
  return 0;
}
