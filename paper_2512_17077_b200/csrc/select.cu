// Select: local max-pool + per-head TopK (§4.5, Eq. 6).
//
// One WARP per (request b, query head h), several rows per CTA and no block
// barrier (the rows are independent; a CTA-per-row kernel spent most of its
// time in block barriers and CTA dispatch):
//   1. the row's raw scores [0, L) go to the warp's smem region by one bulk (TMA)
//      copy (its unaligned head / tail, < 4 floats each, by plain loads);
//   2. pooling on the compacted candidate axis C = [0,bs) ++ [be,L) (window
//      half-width w/2, clipped; R2-R4) in 32-candidate chunks with a
//      register carry (previous / current / next chunk), written IN PLACE as
//      order-preserving 32-bit keys (float -> uint, larger float -> larger key,
//      -0 canonicalised to +0; R9): candidate c's raw score sits at region index
//      >= c and every value is in registers before its slot is overwritten; the
//      min and max key come out of the same pass;
//   3. the exact k-th largest key by MSB radix passes over a 256-bin histogram
//      (warp-aggregated smem atomics), the first digit right below the common
//      prefix of min and max so that every pass discriminates; the search ends
//      early when the threshold bin holds one key (recorded by the histogram) or
//      exactly the keys still needed;
//   4. ordered compaction: every key above the threshold plus the lowest-index
//      (k - #above) keys equal to it (R6), written as sequence positions in
//      ascending order (R7) from ballot prefix counts.
// All decisions are integer comparisons of the fp32 inputs: bit-exact.
#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>

#include "common.cuh"
#include "plan.h"
#include "tc_ptx.cuh"

namespace dllm {

constexpr int kSelThreads = 512;            // select_global / check kernels
constexpr int kSelWarps = kSelThreads / 32;
constexpr int kSelRowWarpsMax = 8;          // rows (warps) per CTA of select_heads_kernel
constexpr int kSelHist = 256;
constexpr int kSelSmemMax = 227 * 1024;

__device__ __forceinline__ uint32_t order_key(float f) {
  uint32_t u = __float_as_uint(f);
  if ((u & 0x7fffffffu) == 0u) return 0x80000000u;     // +-0 -> the same key
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// words of the per-warp smem region for rows of at most max_l scores: the raw row
// (+ up to 3 words of alignment offset), then the histogram and its key record
__host__ __device__ constexpr int sel_region_words(int max_l) { return ((max_l + 3 + 3) & ~3); }
__host__ __device__ constexpr int sel_warp_words(int max_l) { return sel_region_words(max_l) + 2 * kSelHist; }

__global__ void __launch_bounds__(kSelRowWarpsMax * 32)
select_heads_kernel(const __grid_constant__ Plan plan, const float *__restrict__ scores, int32_t *__restrict__ idx,
                    const int warp_words, const int nwarps) {
  extern __shared__ __align__(16) uint32_t sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t bar = smem_u32(sm) + 8u * warp;                      // [kSelRowWarpsMax] mbarriers
  uint32_t *reg = sm + 2 * kSelRowWarpsMax + warp * warp_words;       // 16-byte aligned
  const int region = warp_words - 2 * kSelHist;
  int *hist = reinterpret_cast<int *>(reg + region);
  uint32_t *hkey = reg + region + kSelHist;
  if (lane == 0) {
    ptx::mbar_init(bar, 1);
    ptx::fence_mbar_init();
  }
  __syncwarp();
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  const int row = blockIdx.x * nwarps + warp;
  if (row >= plan.total_units) return;
  // every request owns exactly H rows (one per head): no search over the plan
  const int b = row / plan.H;
  const ReqInfo &R = plan.r[b];
  const int h = row - b * plan.H;
  const int L = R.L, bs = R.bs, blk = R.be - R.bs;
  const int n = L - blk;
  const int k = R.k;
  if (k <= 0) return;
  int32_t *out = idx + R.idx_off + (int64_t)h * k;
  if (k >= n) {
    // every candidate is selected (r = 1): the positions in order
    for (int c = lane; c < n; c += 32) out[c] = c < bs ? c : c + blk;
    return;
  }

  // ---- 1. raw scores -> smem: region index of position p is p + off0
  const float *src = scores + R.score_off + (int64_t)h * L;
  const int off0 = (int)((reinterpret_cast<uintptr_t>(src) >> 2) & 3u);
  const int a1 = (4 - off0) & 3;                              // first position on a 16-byte boundary
  const int a2 = a1 + (((L - a1) > 0 ? (L - a1) : 0) & ~3);   // end of the 16-byte aligned interior
  float *regf = reinterpret_cast<float *>(reg);
  const bool bulk = a2 > a1;
  if (bulk && lane == 0) {
    const uint32_t bytes = (uint32_t)(a2 - a1) * 4u;
    ptx::mbar_arrive_expect_tx(bar, bytes);
    ptx::bulk_g2s(smem_u32(regf + off0 + a1), src + a1, bytes, bar);
  }
  for (int p = lane; p < L; p += 32)
    if (!bulk || p < a1 || p >= a2) regf[off0 + p] = __ldg(src + p);
  if (bulk) ptx::mbar_wait(bar, 0);
  __syncwarp();

  // ---- 2. pooling on the compacted axis, in place, as order keys
  const int half = plan.window >> 1;
  auto raw_at = [&](int c) -> float { return c < n ? regf[off0 + (c < bs ? c : c + blk)] : -INFINITY; };
  float prev = -INFINITY, cur = raw_at(lane);
  uint32_t lo = 0xffffffffu, hi = 0u;
  for (int c0 = 0; c0 < n; c0 += 32) {
    const float next = raw_at(c0 + 32 + lane);
    float m = cur;
    for (int o = 1; o <= half; ++o) {
      const float up = __shfl_up_sync(0xffffffffu, cur, o & 31);
      const float pv = __shfl_sync(0xffffffffu, prev, (lane - o) & 31);
      const float dn = __shfl_down_sync(0xffffffffu, cur, o & 31);
      const float nx = __shfl_sync(0xffffffffu, next, (lane + o) & 31);
      m = fmaxf(m, fmaxf(lane >= o ? up : pv, lane + o < 32 ? dn : nx));
    }
    const int c = c0 + lane;
    if (c < n) {
      const uint32_t key = order_key(m);
      reg[c] = key;
      lo = min(lo, key);
      hi = max(hi, key);
    }
    prev = cur;
    cur = next;
    __syncwarp();   // (w = 1 has no shuffle: keep the lanes in step over the in-place region)
  }
  lo = __reduce_min_sync(0xffffffffu, lo);
  hi = __reduce_max_sync(0xffffffffu, hi);
  __syncwarp();

  // ---- 3. radix select of the k-th largest key (MSB first, below the common prefix)
  uint32_t P = lo, pm = 0xffffffffu;   // keys with (key & pm) == P are still candidates
  int krem = k;
  bool ge_mode = false;                // the whole current bin is taken
  uint32_t thr = lo;
  if (lo != hi) {
    int top = 32 - __clz(lo ^ hi);     // low bits in which the keys differ
    pm = top == 32 ? 0u : ~((1u << top) - 1u);
    P = lo & pm;
    for (;;) {
      const int w = top < 8 ? top : 8, shift = top - w;
      const uint32_t dmask = (1u << w) - 1u;
      reinterpret_cast<int4 *>(hist)[lane] = make_int4(0, 0, 0, 0);
      reinterpret_cast<int4 *>(hist)[lane + 32] = make_int4(0, 0, 0, 0);
      __syncwarp();
      for (int c0 = 0; c0 < n; c0 += 32) {
        const int c = c0 + lane;
        const uint32_t key = c < n ? reg[c] : 0u;
        const bool act = c < n && (key & pm) == P;
        if (__ballot_sync(0xffffffffu, act) == 0u) continue;
        const uint32_t bin = act ? ((key >> shift) & dmask) : 0x100u;
        const uint32_t peers = __match_any_sync(0xffffffffu, bin);
        if (act && lane == __ffs(peers) - 1) {
          atomicAdd(&hist[bin], __popc(peers));
          hkey[bin] = key;
        }
      }
      __syncwarp();
      // lane l owns bins [8(31-l), 8(31-l)+8): lane 0 holds the top bins
      const int base = 8 * (31 - lane);
      int cnt[8], sum = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) { cnt[i] = hist[base + 7 - i]; sum += cnt[i]; }
      int incl = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      const int above = incl - sum;
      const bool mine = above < krem && krem <= incl;
      int dsel = 0, kin = 0, cb = 0;
      if (mine) {
        int acc = above;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          if (acc + cnt[i] >= krem) { dsel = base + 7 - i; kin = krem - acc; cb = cnt[i]; break; }
          acc += cnt[i];
        }
      }
      const int src_lane = __ffs(__ballot_sync(0xffffffffu, mine)) - 1;
      dsel = __shfl_sync(0xffffffffu, dsel, src_lane);
      kin = __shfl_sync(0xffffffffu, kin, src_lane);
      cb = __shfl_sync(0xffffffffu, cb, src_lane);
      P |= (uint32_t)dsel << shift;
      pm |= dmask << shift;
      krem = kin;
      top = shift;
      if (cb == krem) { ge_mode = true; break; }            // the whole bin is taken
      if (cb == 1) { thr = hkey[dsel]; break; }             // its only key is the k-th
      if (top == 0) { thr = P; break; }                      // exact key
      __syncwarp();                                          // hist / hkey reads before the next clear
    }
  } else {
    thr = lo;   // all keys equal: the k lowest indices
  }

  // ---- 4. ordered compaction
  int out_base = 0, eq_base = 0;
  for (int c0 = 0; c0 < n; c0 += 32) {
    const int c = c0 + lane;
    const uint32_t key = c < n ? reg[c] : 0u;
    bool sel;
    if (ge_mode) {
      sel = c < n && (key & pm) >= P;
    } else {
      const bool gt = c < n && key > thr, eq = c < n && key == thr;
      const uint32_t eqm = __ballot_sync(0xffffffffu, eq);
      sel = gt || (eq && eq_base + __popc(eqm & ((1u << lane) - 1u)) < krem);
      eq_base += __popc(eqm);
    }
    const uint32_t sm_ = __ballot_sync(0xffffffffu, sel);
    if (sel) out[out_base + __popc(sm_ & ((1u << lane) - 1u))] = c < bs ? c : c + blk;
    out_base += __popc(sm_);
  }
}

// Block-wide exclusive scan of one int per thread (select_global); returns the
// exclusive prefix and writes the block total to *total.
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

// Uniform (global) selection, the Sparse-dLLM baseline of PAPER.md:136-145
// (§2.4, Eq. 5): S[c] = sum over heads (ascending h, fp32) of the per-head pooled
// score, one top-k per request with the same radix select / tie rule, and the
// shared index set is written to EVERY head's slot of the idx layout so that
// dllm_reuse_sparse_attn consumes it unchanged.  One CTA per request.
__global__ void __launch_bounds__(kSelThreads)
select_global_kernel(const __grid_constant__ Plan plan, const float *__restrict__ scores,
                     int32_t *__restrict__ idx) {
  extern __shared__ uint32_t keys[];                  // [n_ctx]
  __shared__ int hist[256];
  __shared__ int warp_buf[32];
  __shared__ uint32_t s_prefix;
  __shared__ int s_krem;
  const ReqInfo &R = plan.r[blockIdx.x];
  const int L = R.L, bs = R.bs, blk = R.be - R.bs;
  const int n = L - blk;
  const int k = R.k;
  if (k <= 0) return;
  const int H = plan.H;
  const float *raw0 = scores + R.score_off;
  const int half = plan.window >> 1;
  for (int c = threadIdx.x; c < n; c += kSelThreads) {
    const int lo = max(0, c - half), hi = min(n - 1, c + half);
    float acc = 0.f;
    for (int h = 0; h < H; ++h) {
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
      for (int h = 0; h < H; ++h) out0[(int64_t)h * k + pos_out] = pos;
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

int num_sms_sel() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

cudaError_t launch_select(const Plan &plan, const float *scores, int32_t *idx, cudaStream_t st) {
  static std::once_flag once;
  static cudaError_t attr = cudaSuccess;
  std::call_once(once, [] {
    attr = cudaFuncSetAttribute(select_heads_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSelSmemMax);
  });
  if (attr != cudaSuccess) return attr;
  int max_l = 1;
  for (int b = 0; b < plan.nreq; ++b) max_l = max(max_l, plan.r[b].L);
  const int ww = sel_warp_words(max_l);
  const int rows = plan.total_units;
  // rows per CTA: enough CTAs to cover the SMs, at most what keeps 2 CTAs per SM
  // in shared memory (at least one row per CTA)
  int w = (rows + num_sms_sel() - 1) / num_sms_sel();
  w = w < 1 ? 1 : (w > kSelRowWarpsMax ? kSelRowWarpsMax : w);
  const int fixed = 2 * kSelRowWarpsMax * 4;
  while (w > 1 && fixed + (size_t)w * ww * 4 > (size_t)kSelSmemMax / 2) --w;
  const size_t smem = fixed + (size_t)w * ww * 4;
  if (smem > (size_t)kSelSmemMax) return cudaErrorInvalidValue;
  return launch_pdl(select_heads_kernel, dim3((rows + w - 1) / w), dim3(32 * w), smem, st, plan, scores, idx, ww, w);
}

cudaError_t launch_select_global(const Plan &plan, const float *scores, int32_t *idx, cudaStream_t st) {
  int max_n = 0;
  for (int b = 0; b < plan.nreq; ++b) max_n = max(max_n, plan.r[b].L - (plan.r[b].be - plan.r[b].bs));
  const size_t smem = (size_t)max(max_n, 1) * sizeof(uint32_t);
  static std::once_flag once;
  static cudaError_t attr = cudaSuccess;
  std::call_once(once, [] {
    attr = cudaFuncSetAttribute(select_global_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSelSmemMax);
  });
  if (attr != cudaSuccess) return attr;
  if (smem > (size_t)kSelSmemMax) return cudaErrorInvalidValue;
  select_global_kernel<<<plan.nreq, kSelThreads, smem, st>>>(plan, scores, idx);
  return cudaGetLastError();
}

cudaError_t launch_check_indices(const Plan &plan, const int32_t *idx, int32_t *violations,
                                 cudaStream_t st) {
  check_indices_kernel<<<plan.total_units, 256, 0, st>>>(plan, idx, violations);
  return cudaGetLastError();
}

}  // namespace dllm
