// dev micro: where does tcgen05.mma (cta_group::1, kind::f16) with M=64 put the
// accumulator rows in TMEM?  A = 64 x 16 (K-major, no swizzle... we use SW128
// with K=64 elements), B = 32 x 64, D = A B^T; A row i = e_i pattern so that
// D[i][j] identifies i.  Reads all 128 lanes x 32 columns back.
#include <cstdio>
#ifndef LANE_OFF
#define LANE_OFF 0u
#endif
#include <cstdint>
#include <cuda_bf16.h>
#include "../../paper_2512_17077_b200/csrc/common.cuh"
#include "../../paper_2512_17077_b200/csrc/tc_ptx.cuh"
using namespace dllm;

__global__ void k(float *out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const uint32_t sb = (smem_u32(sm) + 1023u) & ~1023u;
  uint8_t *g = sm + (sb - smem_u32(sm));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // A: 64 rows x 64 K (bf16), SW128 K-major: row r, piece c at r*128 + ((c ^ (r&7))<<4)
  // A[r][kk] = (kk == 0) ? r : 0  -> D[r][j] = r * B[j][0]
  // B: 32 rows x 64 K: B[j][0] = 1, others 0   -> D[r][j] = r  (and add j via B[j][1] with A[r][1] = 1000)
  for (int e = threadIdx.x; e < 64 * 64; e += blockDim.x) {
    const int r = e / 64, kk = e % 64;
    float v = (kk == 0) ? (float)r : (kk == 1 ? 1000.f : 0.f);
    const int c = kk / 8, w = kk % 8;
    *reinterpret_cast<__nv_bfloat16 *>(g + r * 128 + ((c ^ (r & 7)) << 4) + w * 2) = __float2bfloat16(v);
  }
  for (int e = threadIdx.x; e < 32 * 64; e += blockDim.x) {
    const int r = e / 64, kk = e % 64;
    float v = (kk == 0) ? 1.f : (kk == 1 ? (float)r : 0.f);
    const int c = kk / 8, w = kk % 8;
    *reinterpret_cast<__nv_bfloat16 *>(g + 8192 + r * 128 + ((c ^ (r & 7)) << 4) + w * 2) = __float2bfloat16(v);
  }
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  if (threadIdx.x == 0) { ptx::mbar_init(smem_u32(&bar), 1); ptx::fence_mbar_init(); }
  ptx::fence_proxy_async_smem();
  if (warp == 0) { ptx::tmem_alloc(smem_u32(&tslot), 128); ptx::tmem_relinquish(); }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tslot;
  // zero the accumulator region first (write 0 via st) so unwritten lanes read 0
  {
    uint32_t z[32];
    for (int i = 0; i < 32; ++i) z[i] = 0xffffffffu;  // NaN marker
    DLLM_TMEM_ST32(tmem + ((uint32_t)(warp * 32) << 16), z);
    ptx::tmem_wait_st();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (warp == 0) {
    constexpr uint32_t idesc = ptx::idesc_bf16_f32(64, 32, false, false);
    const uint64_t da = ptx::smem_desc_sw128(sb, 16, 1024);
    const uint64_t db = ptx::smem_desc_sw128(sb + 8192, 16, 1024);
    for (int kk = 0; kk < 4; ++kk) ptx::mma_ss_elect(tmem + (LANE_OFF << 16), da + kk * 2, db + kk * 2, idesc, kk > 0);
    ptx::mma_commit_elect(smem_u32(&bar));
  }
  ptx::mbar_wait(smem_u32(&bar), 0);
  ptx::tc_fence_after();
  uint32_t r[32];
  DLLM_TMEM_LD32(tmem + ((uint32_t)(warp * 32) << 16), r);
  ptx::tmem_wait_ld();
  for (int j = 0; j < 32; ++j) out[(warp * 32 + lane) * 32 + j] = __uint_as_float(r[j]);
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) ptx::tmem_dealloc(tmem, 128);
}

int main() {
  float *d;
  cudaMalloc(&d, 128 * 32 * 4);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  k<<<1, 128, 64 * 1024>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  printf("run: %s\n", cudaGetErrorString(e));
  float h[128 * 32];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  // D[r][j] = r + 1000 * j (exact in fp32 and representable inputs)
  for (int lane = 0; lane < 128; ++lane) {
    printf("lane %3d:", lane);
    for (int j = 0; j < 4; ++j) printf(" %8.0f", h[lane * 32 + j]);
    printf(" ... col31 %8.0f\n", h[lane * 32 + 31]);
  }
  return 0;
}
