// Select: local max-pool + per-head TopK (§4.5, Eq. 6).
//
// One CTA per (request b, query head h) (select_heads_kernel below).  The CTA
//   1. pools the raw scores of the n_ctx candidates C = [0,bs) ++ [be,L)
//      on the compacted candidate axis (window half-width w/2, clipped;
//      DESIGN.md R2-R4) and keeps order-preserving 32-bit keys in registers
//      (float -> uint, larger float -> larger key, -0 canonicalised to +0;
//      DESIGN.md R9);
//   2. finds the k-th largest key exactly with a 4-pass 8-bit MSB radix
//      select (shared-memory histograms);
//   3. compacts: every key above the threshold, plus the lowest-index
//      (k - #above) keys equal to it (R6), written as sequence
//      positions in ascending order (R7) after one block scan of the counts.
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
constexpr int kSelSmemMaxWords = 32772;
constexpr int kSelCollect = 32;   // threshold-bin size finished by one warp (select_heads_kernel)   // DLLM_MAX_SELECT_LEN raw scores (+ alignment slack)
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

// Block-wide exclusive scan for any multiple-of-32 block size.
__device__ __forceinline__ int block_excl_scan_any(int v, int *warp_buf, int *total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (nw == 1) {
    *total = __shfl_sync(0xffffffffu, x, 31);
    return x - v;
  }
  if (lane == 31) warp_buf[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int w = lane < nw ? warp_buf[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < nw) warp_buf[lane] = w;   // inclusive warp prefix
  }
  __syncthreads();
  const int base = warp ? warp_buf[warp - 1] : 0;
  *total = warp_buf[nw - 1];
  return base + x - v;
}

// One CTA of T = 32 * ceil(n_max / (32 E)) threads per (request, head); thread t
// keeps the keys of the E contiguous candidates c = t E + e in registers, so the
// radix passes touch shared memory only for the 256-bin histogram.
//   1. the raw scores are staged in shared memory (coalesced) and each thread pools
//      its candidates from a register window (16-byte loads + halo);
//   2. 4-pass 8-bit MSB radix select of the k-th largest key;
//   3. each thread counts its candidates above / equal to the threshold, one block
//      scan gives the output slots, and every thread writes its own positions --
//      ascending because thread order is candidate order.
template <int E>
__global__ void __launch_bounds__(1024)
select_heads_kernel(const __grid_constant__ Plan plan, const float *__restrict__ scores,
                    int32_t *__restrict__ idx) {
  extern __shared__ uint32_t sm[];   // raw scores [n]
  __shared__ int hist[256];
  __shared__ int warp_buf[32];
  __shared__ uint32_t s_prefix;
  __shared__ int s_krem;
  __shared__ int s_ncand, s_nbin;
  __shared__ uint32_t s_cand[kSelCollect];

  SEL_TR(0);
  // the request lookup reads only the launch plan: done before griddepcontrol.wait,
  // so with PDL it overlaps the producing kernel's tail (~450 clk of parameter loads)
  const int T = blockDim.x, tid = threadIdx.x;
  const int b = blockIdx.x / plan.H;
  const int h = blockIdx.x - b * plan.H;
  const ReqInfo &R = plan.r[b];
  const int L = R.L, bs = R.bs, blk = R.be - R.bs;
  const int n = L - blk;
  const int k = R.k;
  const float *raw = scores + R.score_off + (int64_t)h * L;
  int32_t *out = idx + R.idx_off + (int64_t)h * k;
  const int half = plan.window >> 1;
  if (tid == 0) s_ncand = 0;
  SEL_TR(1);
  pdl_wait_then_trigger();
  if (k <= 0) return;
  SEL_TR(2);

  // 1. stage the raw scores (coalesced), then every thread pools its own E
  // contiguous candidates c0 .. c0 + E - 1 from a register window (16-byte loads of
  // the E values plus the half-window halo on each side)
  float *rawc = reinterpret_cast<float *>(sm);
  for (int c = tid; c < n; c += T) rawc[c] = __ldg(raw + (c < bs ? c : c + blk));
  __syncthreads();
  SEL_TR(3);
  const int c0 = tid * E;
  uint32_t key[E];
  if (c0 + E <= n) {
    float x[E];
#pragma unroll
    for (int q = 0; q < E / 4; ++q) {
      const float4 v = reinterpret_cast<const float4 *>(rawc + c0)[q];
      x[4 * q] = v.x; x[4 * q + 1] = v.y; x[4 * q + 2] = v.z; x[4 * q + 3] = v.w;
    }
    if (half == 1) {
      const float left = c0 > 0 ? rawc[c0 - 1] : -INFINITY;
      const float right = c0 + E < n ? rawc[c0 + E] : -INFINITY;
#pragma unroll
      for (int e = 0; e < E; ++e)
        key[e] = order_key(fmaxf(fmaxf(e > 0 ? x[e - 1] : left, x[e]), e + 1 < E ? x[e + 1] : right));
    } else if (half == 0) {
#pragma unroll
      for (int e = 0; e < E; ++e) key[e] = order_key(x[e]);
    } else {
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int c = c0 + e;
        const int lo = max(0, c - half), hi = min(n - 1, c + half);
        float m = -INFINITY;
        for (int j = lo; j <= hi; ++j) m = fmaxf(m, rawc[j]);
        key[e] = order_key(m);
      }
    }
  } else {
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int c = c0 + e;
      float m = -INFINITY;
      if (c < n) {
        const int lo = max(0, c - half), hi = min(n - 1, c + half);
        for (int j = lo; j <= hi; ++j) m = fmaxf(m, rawc[j]);
      }
      key[e] = order_key(m);
    }
  }
  SEL_TR(4);

  // 2. radix select of the k-th largest key (MSB first).  (Measured alternatives,
  // slower: runs of equal bins per thread added with one atomic, and a double-
  // buffered histogram saving one barrier per pass: C1 13.3 -> 13.3 us, C4 138 -> 152.)
  uint32_t prefix = 0u, mask = 0u;
  int krem = k;
  int nbin = n;   // keys that share the current prefix
#pragma unroll 1
  for (int shift = 24; shift >= 0; shift -= 8) {
    if (shift < 24 && nbin <= kSelCollect) {
      // Few keys left in the threshold bin (on realistic scores the common case
      // after the second digit): collect them and finish with one warp instead of two more radix
      // passes (~1,300 clk each, mostly barriers).  Every key above the bin is
      // selected; among the bin's nbin keys the krem-th largest key is the threshold
      // -- the same threshold and the same tie rule as the full radix select.
#pragma unroll
      for (int e = 0; e < E; ++e)
        if (c0 + e < n && (key[e] & mask) == prefix) s_cand[atomicAdd(&s_ncand, 1)] = key[e];
      __syncthreads();
      if (tid < 32) {
        const uint32_t mine = tid < nbin ? s_cand[tid] : 0u;
        int gt = 0, ge = 0;
#pragma unroll
        for (int j = 0; j < kSelCollect; ++j) {
          const uint32_t o = __shfl_sync(0xffffffffu, mine, j);   // register rank, no smem chain
          gt += j < nbin && o > mine;
          ge += j < nbin && o >= mine;
        }
        // the lane whose key has fewer than krem keys above it and at least krem at
        // or above it holds the threshold (all such lanes hold the same key)
        const bool hit = tid < nbin && gt < krem && krem <= ge;
        const uint32_t who = __ballot_sync(0xffffffffu, hit);
        const int src = __ffs(who) - 1;
        const uint32_t thr_key = __shfl_sync(0xffffffffu, mine, src);
        const int gt_thr = __shfl_sync(0xffffffffu, gt, src);
        if (tid == 0) {
          s_prefix = thr_key;
          s_krem = krem - gt_thr;   // keys equal to the threshold still needed
        }
      }
      __syncthreads();
      prefix = s_prefix;
      krem = s_krem;
      SEL_TR(5 + (24 - shift) / 8);
      break;
    }
    for (int i = tid; i < 256; i += T) hist[i] = 0;
    __syncthreads();
    // (warp-aggregated atomics via match.any for the crowded first digit were
    // measured slower: C1 pass 2,500 vs 1,900 clk, C4 6,300-7,300 vs 3,000-4,400)
#pragma unroll
    for (int e = 0; e < E; ++e)
      if (c0 + e < n && (key[e] & mask) == prefix) atomicAdd(&hist[(key[e] >> shift) & 0xffu], 1);
    __syncthreads();
    if (tid < 32) {
      // lane l owns bins [8*(31-l), 8*(31-l)+8): lane 0 holds the top bins
      const int lane = tid;
      const int base = 8 * (31 - lane);
      int cnt[8], sum = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) { cnt[i] = hist[base + 7 - i]; sum += cnt[i]; }   // descending bins
      int incl = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
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
            s_nbin = cnt[i];      // keys in the chosen bin
            break;
          }
          acc += cnt[i];
        }
      }
    }
    __syncthreads();
    prefix = s_prefix;
    krem = s_krem;
    nbin = s_nbin;
    mask |= 0xffu << shift;
    SEL_TR(5 + (24 - shift) / 8);
  }
  const uint32_t thr = prefix;   // exact key of the k-th largest
  const int need_eq = krem;      // keys equal to thr taken, lowest index first

  // 3. compaction: slot = (#above before) + min(#equal before, need_eq)
  int ngt = 0, neq = 0;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const bool v = c0 + e < n;
    ngt += v && key[e] > thr;
    neq += v && key[e] == thr;
  }
  int tot;
  const int pre = block_excl_scan_any(ngt | (neq << 16), warp_buf, &tot);
  int gt_b = pre & 0xffff, eq_b = pre >> 16;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int c = c0 + e;
    if (c < n) {
      const bool gt = key[e] > thr, eq = key[e] == thr;
      if (gt || (eq && eq_b < need_eq)) out[gt_b + min(eq_b, need_eq)] = c < bs ? c : c + blk;
      gt_b += gt;
      eq_b += eq;
    }
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

// Keys per thread E: the smallest of 4, 8, 16, 32 that keeps the CTA at <= 256
// threads (C1, n = 992: E = 4, 256 threads; C4, n = 4,064: E = 16, 256 threads).
// Measured (profiles/r02_ab_select_v2.log): C1 13.3 us, C4 138 us, against 17.4 and
// 191-209 us for the round-1 kernel (512 threads, keys in shared memory).
template <int E>
cudaError_t launch_select_e(const Plan &plan, const float *scores, int32_t *idx, int max_n, cudaStream_t st) {
  static std::once_flag once;
  static cudaError_t attr = cudaSuccess;
  std::call_once(once, [] {
    attr = cudaFuncSetAttribute(select_heads_kernel<E>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                kSelSmemMaxWords * (int)sizeof(uint32_t));
  });
  if (attr != cudaSuccess) return attr;
  const int threads = 32 * max(1, (max_n + 32 * E - 1) / (32 * E));
  const size_t words = (size_t)max_n + 4;
  if (threads > 1024 || words > (size_t)kSelSmemMaxWords) return cudaErrorInvalidValue;
  return launch_pdl(select_heads_kernel<E>, dim3(plan.total_units), dim3(threads), words * sizeof(uint32_t), st,
                    plan, scores, idx);
}

cudaError_t launch_select(const Plan &plan, const float *scores, int32_t *idx, cudaStream_t st) {
  int max_n = 0;
  for (int b = 0; b < plan.nreq; ++b) max_n = max(max_n, plan.r[b].L - (plan.r[b].be - plan.r[b].bs));
#ifdef DLLM_SEL_E
  return launch_select_e<DLLM_SEL_E>(plan, scores, idx, max_n, st);
#else
  if (max_n <= 256 * 4) return launch_select_e<4>(plan, scores, idx, max_n, st);
  if (max_n <= 256 * 8) return launch_select_e<8>(plan, scores, idx, max_n, st);
  if (max_n <= 256 * 16) return launch_select_e<16>(plan, scores, idx, max_n, st);
  return launch_select_e<32>(plan, scores, idx, max_n, st);
#endif
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
