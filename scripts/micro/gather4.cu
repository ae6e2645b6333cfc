// dev micro: semantics + throughput of TMA tile::gather4 (sm_100a) on a paged-cache-like
// 2D view [rows, D] bf16 with SWIZZLE_128B, box {64, BOXR}.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include <vector>
#include <cstdlib>

typedef CUresult (*EncodeFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                             const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void g4_kernel(const __grid_constant__ CUtensorMap tm, const int *rows, int nrows, uint16_t *out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar;
  const uint32_t b = su32(&bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    // nrows rows x 2 column halves (64 elems each): dst [2][nrows][128 B]
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(nrows * 256));
    for (int g = 0; g < nrows / 4; ++g)
      for (int h = 0; h < 2; ++h) {
        uint32_t dst = su32(sm + h * nrows * 128 + g * 512);
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
            ::"r"(dst), "l"(reinterpret_cast<uint64_t>(&tm)), "r"(h * 64), "r"(rows[4 * g]), "r"(rows[4 * g + 1]),
            "r"(rows[4 * g + 2]), "r"(rows[4 * g + 3]), "r"(b) : "memory");
      }
  }
  asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}" ::"r"(b));
  for (int i = threadIdx.x; i < nrows * 256 / 2; i += blockDim.x) out[i] = reinterpret_cast<uint16_t *>(sm)[i];
}

// throughput: every CTA gathers its own random rows, NST-stage ring of 128-row chunks
template <int NST>
__global__ void g4_bw(const __grid_constant__ CUtensorMap tm, const int *rows, int chunks_per_cta, int *sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bars[NST];
  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bars[s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const int lane = threadIdx.x;
  int acc = 0;
  for (int c = 0; c < chunks_per_cta + NST; ++c) {
    const int s = c % NST;
    if (c >= NST) {
      const int cc = c - NST;
      const uint32_t b = su32(&bars[s]);
      asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}" ::"r"(b),
                   "r"((cc / NST) & 1));
      acc += sm[s * 32768 + lane * 4];
      __syncwarp();
    }
    if (c < chunks_per_cta) {
      const int *r = rows + ((int64_t)blockIdx.x * chunks_per_cta + c) * 128 + lane * 4;
      const uint32_t b = su32(&bars[s]);
      if (lane == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(32768));
      __syncwarp();
      for (int h = 0; h < 2; ++h) {
        uint32_t dst = su32(sm + s * 32768 + h * 16384 + lane * 512);
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
            ::"r"(dst), "l"(reinterpret_cast<uint64_t>(&tm)), "r"(h * 64), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]),
            "r"(b) : "memory");
      }
    }
  }
  if (acc == 123456789) sink[0] = acc;
}

int main() {
  EncodeFn enc;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &q);
  const int D = 128;
  const int64_t R = 1 << 22;  // 4M rows x 256 B = 1 GiB
  uint16_t *cache;
  cudaMalloc(&cache, R * D * 2);
  std::vector<uint16_t> small(64 * 1024 * D);
  for (size_t i = 0; i < small.size(); ++i) small[i] = (uint16_t)(i * 2654435761u >> 7);
  cudaMemcpy(cache, small.data(), small.size() * 2, cudaMemcpyHostToDevice);
  for (int boxr : {1, 4}) {
    CUtensorMap tm;
    cuuint64_t dims[2] = {(cuuint64_t)D, (cuuint64_t)R};
    cuuint64_t strides[1] = {(cuuint64_t)D * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)boxr};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, cache, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("box {64,%d}: encode %d\n", boxr, (int)r);
    if (r) continue;
    const int n = 16;
    int hrows[n];
    for (int i = 0; i < n; ++i) hrows[i] = (i * 7919 + 13) % (64 * 1024);
    int *drows;
    uint16_t *dout;
    cudaMalloc(&drows, sizeof(hrows));
    cudaMalloc(&dout, n * 256);
    cudaMemcpy(drows, hrows, sizeof(hrows), cudaMemcpyHostToDevice);
    cudaMemset(dout, 0, n * 256);
    // rows pointer is read on device: copy to a device array first
    int *hr_dev = drows;
    cudaFuncSetAttribute(g4_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    // kernel reads rows[] from global
    g4_kernel<<<1, 128, 64 * 1024>>>(tm, hr_dev, n, dout);
    cudaError_t e = cudaDeviceSynchronize();
    printf("  run: %s\n", cudaGetErrorString(e));
    if (e) return 1;
    std::vector<uint16_t> o(n * 128);
    cudaMemcpy(o.data(), dout, n * 256, cudaMemcpyDeviceToHost);
    // expected: dst[h][i][chunk ^ (i%8)] holds row hrows[i], cols h*64 + chunk*8 ..
    int bad = 0, bad_noswz = 0;
    for (int h = 0; h < 2; ++h)
      for (int i = 0; i < n; ++i)
        for (int c = 0; c < 64; ++c) {
          const uint16_t want = small[(size_t)hrows[i] * D + h * 64 + c];
          const int chunk = c / 8, w = c % 8;
          const uint16_t got = o[h * n * 64 + i * 64 + ((chunk ^ (i % 8)) * 8) + w];
          const uint16_t got2 = o[h * n * 64 + i * 64 + c];
          bad += got != want;
          bad_noswz += got2 != want;
        }
    printf("  mismatches: swizzled-layout %d, plain-layout %d (of %d)\n", bad, bad_noswz, 2 * n * 64);
    // throughput
    const int ctas = 148, cpc = 64;
    std::vector<int> rr((size_t)ctas * cpc * 128);
    srand(1);
    for (auto &x : rr) x = (int)(((int64_t)rand() * 7 + rand()) % R);
    int *drr;
    cudaMalloc(&drr, rr.size() * 4);
    cudaMemcpy(drr, rr.data(), rr.size() * 4, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(g4_bw<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 32768);
    cudaFuncSetAttribute(g4_bw<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, 6 * 32768);
    for (int it = 0; it < 2; ++it) {
      cudaEvent_t a, bb;
      cudaEventCreate(&a);
      cudaEventCreate(&bb);
      cudaEventRecord(a);
      if (it == 0) g4_bw<4><<<ctas, 32, 4 * 32768>>>(tm, drr, cpc, (int *)dout);
      else g4_bw<6><<<ctas, 32, 6 * 32768>>>(tm, drr, cpc, (int *)dout);
      cudaEventRecord(bb);
      cudaEventSynchronize(bb);
      float ms;
      cudaEventElapsedTime(&ms, a, bb);
      printf("  gather4 bw (%d stages): %.1f GB/s (%s)\n", it ? 6 : 4, (double)ctas * cpc * 32768 / (ms * 1e-3) / 1e9,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
