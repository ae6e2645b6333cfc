// dev micro: does compute-sanitizer racecheck model mbarrier arrive (release) /
// try_wait (acquire) as synchronisation?  Warp 0 writes a shared buffer and arrives
// on an mbarrier; warp 1 waits on it and reads the buffer -- the textbook
// producer/consumer handoff the kernels use.  Any racecheck report here is a false
// positive of the tool, not of the pattern.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void k(int *out) {
  __shared__ int buf[32];
  __shared__ __align__(8) uint64_t bar;
  const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(b), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    buf[lane] = lane * 7;
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(b) : "memory");
  } else if (warp == 1) {
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
                   : "=r"(ok) : "r"(b), "r"(0) : "memory");
    out[lane] = buf[lane];
  }
}
int main() {
  int *d; cudaMalloc(&d, 128);
  k<<<1, 64>>>(d);
  int h[32]; cudaMemcpy(h, d, 128, cudaMemcpyDeviceToHost);
  printf("handoff %s\n", h[5] == 35 ? "ok" : "WRONG");
  return 0;
}
