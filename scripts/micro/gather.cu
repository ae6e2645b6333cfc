// dev microbench: random 256-byte row gather bandwidth on B200 (the Reuse access pattern)
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>
#include "../../paper_2512_17077_b200/csrc/common.cuh"
using namespace dllm;

// (1) LDG.128 into registers, XOR-reduce (no smem)
template <int UNROLL>
__global__ void ldg_kernel(const uint4 *__restrict__ src, const int *__restrict__ rows, int nrows, uint4 *sink) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  uint4 acc = make_uint4(0, 0, 0, 0);
  // each warp handles 2 rows per step (lane>>4 selects the row, lane&15 the 16-B piece)
  for (int base = gw * 2 * UNROLL; base < nrows; base += nw * 2 * UNROLL) {
    uint4 v[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      const int r = base + u * 2 + (lane >> 4);
      v[u] = r < nrows ? __ldg(src + (size_t)rows[r] * 16 + (lane & 15)) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) { acc.x ^= v[u].x; acc.y ^= v[u].y; acc.z ^= v[u].z; acc.w ^= v[u].w; }
  }
  if (acc.x == 0x12345678) sink[0] = acc;
}

// (2) cp.async 16 B into a per-warp smem ring, wait_group
template <int STAGES>
__global__ void cpasync_kernel(const uint4 *__restrict__ src, const int *__restrict__ rows, int nrows, uint4 *sink) {
  extern __shared__ uint4 sm[];
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  uint4 *ring = sm + wl * STAGES * 32 * 4;     // per stage: 8 rows (4 x 512 B)
  uint32_t acc = 0;
  int s = 0;
  for (int base = gw * 8; base < nrows; base += nw * 8, s = (s + 1) % STAGES) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int r = base + u * 2 + (lane >> 4);
      const bool ok = r < nrows;
      cp_async16(smem_u32(ring + s * 128 + u * 32 + lane), src + (size_t)(ok ? rows[r] : 0) * 16 + (lane & 15), ok ? 16 : 0);
    }
    cp_async_commit();
    cp_async_wait<STAGES - 1>();
    acc ^= ring[((s + 1) % STAGES) * 128 + lane].x;
  }
  cp_async_wait<0>();
  if (acc == 0x12345678) sink[0] = make_uint4(acc, 0, 0, 0);
}

int main() {
  const size_t bytes = 268ull << 20;            // a C1-sized K+V cache
  const size_t nrow_total = bytes / 256;
  const int nrows = 82 * 1024 * 1024 / 256;     // ~82 MB gathered (C1 Reuse)
  std::mt19937 rng(1);
  std::vector<int> rows(nrows);
  // sorted groups of 16 rows within random 16 KB pages (the selection pattern)
  for (int i = 0; i < nrows; i += 16) {
    const int page = rng() % (nrow_total / 64);
    std::vector<int> pick(64); for (int j = 0; j < 64; ++j) pick[j] = j;
    std::shuffle(pick.begin(), pick.end(), rng); std::sort(pick.begin(), pick.begin() + 16);
    for (int j = 0; j < 16 && i + j < nrows; ++j) rows[i + j] = page * 64 + pick[j];
  }
  uint4 *src, *sink; int *drows;
  cudaMalloc(&src, bytes); cudaMemset(src, 1, bytes); cudaMalloc(&sink, 64);
  cudaMalloc(&drows, nrows * 4); cudaMemcpy(drows, rows.data(), nrows * 4, cudaMemcpyHostToDevice);
  void *flush; cudaMalloc(&flush, 512 << 20);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto timeit = [&](const char *name, auto launch) {
    float best = 1e9;
    for (int it = 0; it < 5; ++it) {
      cudaMemset(flush, it, 512 << 20);
      cudaEventRecord(a); launch(); cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); best = std::min(best, ms);
    }
    printf("%-40s %8.1f us  %7.1f GB/s  (%s)\n", name, best * 1e3, nrows * 256.0 / (best * 1e-3) / 1e9,
           cudaGetErrorString(cudaGetLastError()));
  };
  for (int tpb : {256, 512, 1024}) {
    char nm[64];
    snprintf(nm, 64, "LDG.128 unroll4  %4d thr x 148x2", tpb);
    timeit(nm, [&] { ldg_kernel<4><<<296, tpb>>>(src, drows, nrows, sink); });
    snprintf(nm, 64, "LDG.128 unroll8  %4d thr x 148x2", tpb);
    timeit(nm, [&] { ldg_kernel<8><<<296, tpb>>>(src, drows, nrows, sink); });
  }
  for (int tpb : {128, 256, 512}) {
    char nm[64];
    const int smem = (tpb / 32) * 4 * 128 * 16;
    cudaFuncSetAttribute(cpasync_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    snprintf(nm, 64, "cp.async 4 stages %4d thr x 148x2", tpb);
    timeit(nm, [&] { cpasync_kernel<4><<<296, tpb, smem>>>(src, drows, nrows, sink); });
  }
  // contiguous reference
  timeit("LDG.128 contiguous rows (identity)", [&] {
    static int *ident = nullptr;
    if (!ident) { std::vector<int> id(nrows); for (int i = 0; i < nrows; ++i) id[i] = i; cudaMalloc(&ident, nrows * 4); cudaMemcpy(ident, id.data(), nrows * 4, cudaMemcpyHostToDevice); }
    ldg_kernel<8><<<296, 1024>>>(src, ident, nrows, sink); });
}
