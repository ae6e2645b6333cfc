// Select: local max-pool + per-head TopK (§4.5, Eq. 6).
//
// One CTA per (request b, query head h).  The CTA
//   1. pools the raw scores of the n_ctx candidates C = [0,bs) ++ [be,L)
//      on the compacted candidate axis (window half-width w/2, clipped;
//      DESIGN.md R2-R4) straight from global memory (neighbour reads hit L1),
//      and stores order-preserving 32-bit keys in shared memory
//      (float -> uint, larger float -> larger key, -0 canonicalised to +0;
//      DESIGN.md R9);
//   2. finds the k-th largest key exactly with a 4-pass 8-bit MSB radix
//      select (shared-memory histograms);
//   3. compacts: every key above the threshold, plus the lowest-index
//      (k - #above) keys equal to it (R6), written as sequence
//      positions in ascending order (R7) with two ballot-based block scans.
// All decisions are integer comparisons of the fp32 inputs: bit-exact.
#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>

#include "common.cuh"
#include "plan.h"

namespace dllm {

#ifndef DLLM_SEL_THREADS
#define DLLM_SEL_THREADS 512
#endif
constexpr int kSelThreads = DLLM_SEL_THREADS;
constexpr int kSelWarps = kSelThreads / 32;
constexpr int kSelSmemStageMax = 24576;   // words of raw scores + keys staged in smem (96 KB)
constexpr int kSelSmemMaxWords = 32768;   // DLLM_MAX_SELECT_LEN keys (128 KB)
#ifdef DLLM_TRACE
// dev: phase timestamps (clock64) of a few CTAs: [cta][0 start, 1 after wait, 2 request found,
// 3 raw staged, 4 pooled, 5..8 radix passes, 9 compaction done]
__device__ long long g_sel_tr[8][10];
extern "C" __attribute__((visibility("default"))) int dllm_trace_sel_read(long long *h) {
  return (int)cudaMemcpyFromSymbol(h, g_sel_tr, sizeof(g_sel_tr));
}
#define SEL_TR(k) do { if (threadIdx.x == 0 && blockIdx.x < 8) g_sel_tr[blockIdx.x][k] = clock64(); } while (0)
#else
#define SEL_TR(k) do { } while (0)
#endif   // words of dynamic smem for staged raw scores + keys (96 KB)

__device__ __forceinline__ uint32_t order_key(float f) {
  uint32_t u = __float_as_uint(f);
  if ((u & 0x7fffffffu) == 0u) return 0x80000000u;     // +-0 -> the same key
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// Block-wide exclusive scan of one int per thread; returns the exclusive
// prefix and writes the block total to *total.
__device__ __forceinline__ int block_excl_scan(int v, int *warp_buf, int *total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_buf[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int w = lane < kSelWarps ? warp_buf[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < kSelWarps) warp_buf[lane] = w;        // inclusive warp prefix
  }
  __syncthreads();
  int base = warp ? warp_buf[warp - 1] : 0;
  *total = warp_buf[kSelWarps - 1];
  __syncthreads();
  return base + x - v;
}

__global__ void __launch_bounds__(kSelThreads)
select_heads_kernel(const __grid_constant__ Plan plan, const float *__restrict__ scores,
                    int32_t *__restrict__ idx, const int stage) {
  extern __shared__ uint32_t keys[];                  // [n_ctx]
  __shared__ int hist[2][256];      // double-buffered: the next pass's is cleared while this one fills
  __shared__ int warp_buf[32];
  __shared__ uint32_t s_prefix[2];
  __shared__ int s_krem[2];

  SEL_TR(0);
  pdl_wait_then_trigger();
  SEL_TR(1);
  const int unit = blockIdx.x;
  // every request owns exactly H units (one per head): no search over the plan
  // (a binary search in parameter memory cost ~1,200 clk of a ~14k clk CTA at C1)
  const int b = unit / plan.H;
  const ReqInfo &R = plan.r[b];
  const int h = unit - b * plan.H;
  const int L = R.L, bs = R.bs, blk = R.be - R.bs;
  const int n = L - blk;
  const int k = R.k;
  if (k <= 0) return;
  const float *raw = scores + R.score_off + (int64_t)h * L;
  int32_t *out = idx + R.idx_off + (int64_t)h * k;
  const int half = plan.window >> 1;
  SEL_TR(2);

  // 1. pool on the compacted axis, to order keys.  When every request's candidates
  // fit twice in shared memory (`stage`, decided for the whole launch by the host,
  // which sized the allocation accordingly), the raw scores are first staged there
  // with all loads of a thread in flight together (one memory round trip instead of
  // one per window element and candidate), then pooled from shared memory.
  if (stage) {
    float *rawc = reinterpret_cast<float *>(keys + n);
#pragma unroll 4
    for (int c = threadIdx.x; c < n; c += kSelThreads) rawc[c] = __ldg(raw + (c < bs ? c : c + blk));
    __syncthreads();
    SEL_TR(3);
    for (int c = threadIdx.x; c < n; c += kSelThreads) {
      const int lo = max(0, c - half), hi = min(n - 1, c + half);
      float m = -INFINITY;
      for (int j = lo; j <= hi; ++j) m = fmaxf(m, rawc[j]);
      keys[c] = order_key(m);
    }
  } else {
    for (int c = threadIdx.x; c < n; c += kSelThreads) {
      const int lo = max(0, c - half), hi = min(n - 1, c + half);
      float m = -INFINITY;
      for (int j = lo; j <= hi; ++j) {
        const int pos = j < bs ? j : j + blk;
        m = fmaxf(m, __ldg(raw + pos));
      }
      keys[c] = order_key(m);
    }
  }
  for (int i = threadIdx.x; i < 256; i += kSelThreads) hist[0][i] = 0;
  __syncthreads();
  SEL_TR(4);

  // 2. radix select of the k-th largest key (MSB first)
  uint32_t prefix = 0u, mask = 0u;
  int krem = k;
#pragma unroll 1
  for (int shift = 24; shift >= 0; shift -= 8) {
    // two block barriers per pass: hist[cur] fills while hist[cur ^ 1] (read by the
    // previous pass before its second barrier) is cleared for the next pass; the
    // digit goes through s_prefix[cur], next rewritten two passes later
    const int cur = ((24 - shift) >> 3) & 1;
    for (int i = threadIdx.x; i < 256; i += kSelThreads) hist[cur ^ 1][i] = 0;
    // warp-aggregated: the candidates' keys crowd a few bins (similar exponents), so
    // lanes with equal bins are merged (match.any) into one shared atomic
    for (int c0 = 0; c0 < n; c0 += kSelThreads) {
      const int c = c0 + threadIdx.x;
      const uint32_t key = c < n ? keys[c] : 0u;
      const bool act = c < n && (key & mask) == prefix;
      const uint32_t bin = act ? ((key >> shift) & 0xffu) : 0x100u;
      const uint32_t peers = __match_any_sync(0xffffffffu, bin);
      if (act && (threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&hist[cur][bin], __popc(peers));
    }
    __syncthreads();
    if (threadIdx.x < 32) {
      // lane l owns bins [8*(31-l), 8*(31-l)+8): lane 0 holds the top bins
      const int lane = threadIdx.x;
      const int base = 8 * (31 - lane);
      int cnt[8], sum = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) { cnt[i] = hist[cur][base + 7 - i]; sum += cnt[i]; }  // descending bins
      int incl = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      const int above = incl - sum;                   // keys in higher bins than this lane's
      const bool mine = above < krem && krem <= incl;
      if (mine) {
        int acc = above;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          if (acc + cnt[i] >= krem) {
            const uint32_t digit = (uint32_t)(base + 7 - i);
            s_prefix[cur] = prefix | (digit << shift);
            s_krem[cur] = krem - acc;
            break;
          }
          acc += cnt[i];
        }
      }
    }
    __syncthreads();
    prefix = s_prefix[cur];
    krem = s_krem[cur];
    mask |= 0xffu << shift;
    SEL_TR(5 + (24 - shift) / 8);
  }
  const uint32_t thr = prefix;   // exact key of the k-th largest
  const int need_eq = krem;      // how many keys equal to thr are taken (lowest index first)

  // 3. compaction in ascending candidate order
  // One block scan per 512 candidates of the packed pair (above, equal): a selected
  // candidate's output slot is (#above before it) + min(#equal before it, need_eq),
  // because exactly the first need_eq equal keys are taken.
  int eq_base = 0, gt_base = 0;
  for (int c0 = 0; c0 < n; c0 += kSelThreads) {
    const int c = c0 + threadIdx.x;
    uint32_t key = c < n ? keys[c] : 0u;
    const int gt = (c < n) && key > thr;
    const int eq = (c < n) && key == thr;
    int tot;
    const int pre = block_excl_scan(gt | (eq << 16), warp_buf, &tot);
    const int gt_pre = gt_base + (pre & 0xffff), eq_pre = eq_base + (pre >> 16);
    if (gt || (eq && eq_pre < need_eq)) out[gt_pre + min(eq_pre, need_eq)] = c < bs ? c : c + blk;
    gt_base += tot & 0xffff;
    eq_base += tot >> 16;
  }
  SEL_TR(9);
}

// Set selection over a group of heads (next row N2):
//  * uniform, the Sparse-dLLM baseline of PAPER.md:136-145 (§2.4, Eq. 5): the set
//    is every head of the request;
//  * per KV group (GQA): the set is the H / H_kv query heads sharing one KV head
//    (Eq. 5 restricted to the group, R21).
// S[c] = sum over the set's heads (ascending h, fp32) of the per-head pooled score,
// one top-k per (request, set) with the same radix select / tie rule, and the
// shared index set is written to every head's slot of the idx layout so that
// dllm_reuse_sparse_attn consumes it unchanged.  One CTA per (request, set).
__global__ void __launch_bounds__(kSelThreads)
select_global_kernel(const __grid_constant__ Plan plan, const float *__restrict__ scores,
                     int32_t *__restrict__ idx, const int heads_per_set) {
  extern __shared__ uint32_t keys[];                  // [n_ctx]
  __shared__ int hist[256];
  __shared__ int warp_buf[32];
  __shared__ uint32_t s_prefix;
  __shared__ int s_krem;
  // CTA = (request, head set): the set's heads are [h0, h0 + heads_per_set)
  const int sets = plan.H / heads_per_set;
  const ReqInfo &R = plan.r[blockIdx.x / sets];
  const int h0 = (blockIdx.x % sets) * heads_per_set;
  const int L = R.L, bs = R.bs, blk = R.be - R.bs;
  const int n = L - blk;
  const int k = R.k;
  if (k <= 0) return;
  const float *raw0 = scores + R.score_off;
  const int half = plan.window >> 1;
  for (int c = threadIdx.x; c < n; c += kSelThreads) {
    const int lo = max(0, c - half), hi = min(n - 1, c + half);
    float acc = 0.f;
    for (int h = h0; h < h0 + heads_per_set; ++h) {
      const float *raw = raw0 + (int64_t)h * L;
      float m = -INFINITY;
      for (int j = lo; j <= hi; ++j) m = fmaxf(m, __ldg(raw + (j < bs ? j : j + blk)));
      acc += m;
    }
    keys[c] = order_key(acc);
  }
  if (threadIdx.x == 0) { s_prefix = 0u; s_krem = k; }
  __syncthreads();
  uint32_t prefix = 0u, mask = 0u;
  int krem = k;
#pragma unroll 1
  for (int shift = 24; shift >= 0; shift -= 8) {
    for (int i = threadIdx.x; i < 256; i += kSelThreads) hist[i] = 0;
    __syncthreads();
    // warp-aggregated: the candidates' keys crowd a few bins (similar exponents), so
    // lanes with equal bins are merged (match.any) into one shared atomic
    for (int c0 = 0; c0 < n; c0 += kSelThreads) {
      const int c = c0 + threadIdx.x;
      const uint32_t key = c < n ? keys[c] : 0u;
      const bool act = c < n && (key & mask) == prefix;
      const uint32_t bin = act ? ((key >> shift) & 0xffu) : 0x100u;
      const uint32_t peers = __match_any_sync(0xffffffffu, bin);
      if (act && (threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&hist[bin], __popc(peers));
    }
    __syncthreads();
    if (threadIdx.x < 32) {
      const int lane = threadIdx.x;
      const int base = 8 * (31 - lane);
      int cnt[8], sum = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) { cnt[i] = hist[base + 7 - i]; sum += cnt[i]; }
      int incl = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      const int above = incl - sum;
      if (above < krem && krem <= incl) {
        int acc = above;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          if (acc + cnt[i] >= krem) {
            s_prefix = prefix | ((uint32_t)(base + 7 - i) << shift);
            s_krem = krem - acc;
            break;
          }
          acc += cnt[i];
        }
      }
    }
    __syncthreads();
    prefix = s_prefix;
    krem = s_krem;
    mask |= 0xffu << shift;
    __syncthreads();
  }
  int eq_base = 0, gt_base = 0;
  int32_t *out0 = idx + R.idx_off;
  for (int c0 = 0; c0 < n; c0 += kSelThreads) {
    const int c = c0 + threadIdx.x;
    const uint32_t key = c < n ? keys[c] : 0u;
    const int gt = (c < n) && key > prefix;
    const int eq = (c < n) && key == prefix;
    int tot;
    const int pre = block_excl_scan(gt | (eq << 16), warp_buf, &tot);
    const int gt_pre = gt_base + (pre & 0xffff), eq_pre = eq_base + (pre >> 16);
    if (gt || (eq && eq_pre < krem)) {
      const int pos = c < bs ? c : c + blk;
      const int pos_out = gt_pre + min(eq_pre, krem);
      for (int h = h0; h < h0 + heads_per_set; ++h) out0[(int64_t)h * k + pos_out] = pos;
    }
    gt_base += tot & 0xffff;
    eq_base += tot >> 16;
  }
}

// Debug checker: counts positions out of range, inside the block, or not
// strictly ascending.
__global__ void check_indices_kernel(const __grid_constant__ Plan plan, const int32_t *__restrict__ idx,
                                     int32_t *violations) {
  const int unit = blockIdx.x;
  const int b = plan_find(plan, unit);
  const ReqInfo &R = plan.r[b];
  const int h = unit - R.unit_off;
  const int32_t *row = idx + R.idx_off + (int64_t)h * R.k;
  int bad = 0;
  for (int i = threadIdx.x; i < R.k; i += blockDim.x) {
    const int p = row[i];
    if (p < 0 || p >= R.L || (p >= R.bs && p < R.be)) ++bad;
    if (i > 0 && row[i - 1] >= p) ++bad;
  }
  if (bad) atomicAdd(violations, bad);
}

cudaError_t launch_select(const Plan &plan, const float *scores, int32_t *idx, cudaStream_t st) {
  static std::once_flag once;
  static cudaError_t attr = cudaSuccess;
  std::call_once(once, [] {
    attr = cudaFuncSetAttribute(select_heads_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                kSelSmemMaxWords * (int)sizeof(uint32_t));
  });
  if (attr != cudaSuccess) return attr;
  int max_n = 0;
  for (int b = 0; b < plan.nreq; ++b) max_n = max(max_n, plan.r[b].L - (plan.r[b].be - plan.r[b].bs));
  // staging is decided for the whole launch: every CTA then has room for 2 n words
  const int stage = 2 * max_n <= kSelSmemStageMax ? 1 : 0;
  const size_t words = stage ? 2 * (size_t)max_n : (size_t)max_n;
  const size_t smem = (words > 0 ? words : 1) * sizeof(uint32_t);
  if (words > (size_t)kSelSmemMaxWords) return cudaErrorInvalidValue;
  return launch_pdl(select_heads_kernel, dim3(plan.total_units), dim3(kSelThreads), smem, st, plan, scores, idx,
                    stage);
}

cudaError_t launch_select_global(const Plan &plan, const float *scores, int32_t *idx, int heads_per_set,
                                 cudaStream_t st) {
  int max_n = 0;
  for (int b = 0; b < plan.nreq; ++b) max_n = max(max_n, plan.r[b].L - (plan.r[b].be - plan.r[b].bs));
  const size_t smem = (size_t)max(max_n, 1) * sizeof(uint32_t);
  static std::once_flag once;
  static cudaError_t attr = cudaSuccess;
  std::call_once(once, [] {
    attr = cudaFuncSetAttribute(select_global_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                kSelSmemMaxWords * (int)sizeof(uint32_t));
  });
  if (attr != cudaSuccess) return attr;
  if (smem > (size_t)kSelSmemMaxWords * sizeof(uint32_t)) return cudaErrorInvalidValue;
  select_global_kernel<<<plan.nreq * (plan.H / heads_per_set), kSelThreads, smem, st>>>(plan, scores, idx,
                                                                                        heads_per_set);
  return cudaGetLastError();
}

cudaError_t launch_check_indices(const Plan &plan, const int32_t *idx, int32_t *violations,
                                 cudaStream_t st) {
  check_indices_kernel<<<plan.total_units, 256, 0, st>>>(plan, idx, violations);
  return cudaGetLastError();
}

}  // namespace dllm
