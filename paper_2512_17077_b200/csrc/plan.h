// Launch plan shared by the host library and the kernels.
//
// The host validates the problem and packs per-request metadata into a plan
// that travels BY VALUE as a __grid_constant__ kernel parameter (CUDA >= 12.1
// allows 32 KB of parameters), so there is no hidden host->device copy and
// the launches stay CUDA-graph capturable.  Batches larger than
// kMaxReqPerLaunch are split into several launches.
#pragma once
#include <stdint.h>

namespace dllm {

#ifndef DLLM_MAX_REQ
#define DLLM_MAX_REQ 256
#endif
constexpr int kMaxReqPerLaunch = DLLM_MAX_REQ;

struct ReqInfo {
  int32_t L;         // sequence length L_b
  int32_t bs, be;    // active block [bs, be)
  int32_t q_off;     // cu_L[b]: first row of the request in q / out
  int32_t blk_off;   // cu_blk[b]: first row in q_blk / out_blk
  int32_t k;         // k_b
  int64_t idx_off;   // H * cu_k[b]: first element of the request in idx
  int64_t score_off; // H * cu_L[b]: first element in scores
  int32_t unit_off;  // prefix of work units (kernel specific) before this request
  int32_t bt_row;    // row of the block table (request index in the caller's batch)
  int64_t cost_off;  // reuse: prefix of the work-unit costs (keys + kReuseUnitCost per unit) before this request
};

struct Plan {
  int32_t nreq;
  int32_t total_units;
  int32_t H, H_kv, D;
  int32_t page_size, page_shift, pages_per_req;
  int32_t window;
  int32_t with_scores;  // refresh: also emit the Eq. 6 raw importance
  int32_t units_per_req; // every request owns this many work units (0: they differ)
  int32_t req_cost;      // reuse: cost of every request when they are all equal (0: they differ)
  int64_t total_cost;    // reuse: sum of the unit costs of the plan
  float scale_log2;  // tau * log2(e)
  float scale;       // tau
  const int32_t *block_table;
  int32_t *sched;        // refresh_tc2: {claims, CTAs done} unit counters in the caller's workspace, or NULL
  ReqInfo r[kMaxReqPerLaunch];
};

// Reuse work balancing: a work unit (request, head, 32-row group) of nk = blk + k
// keys costs nk + kReuseUnitCost "key equivalents" (its Q rows, its output rows and
// the per-unit pipeline overheads); the launch's total cost is split evenly over
// the CTAs (reuse_tc_body.cuh).
constexpr int kReuseUnitCost = 32;

#if defined(__CUDACC__)
// Request owning work unit u: largest b with r[b].unit_off <= u.
__device__ __forceinline__ int plan_find(const Plan &p, int u) {
  if (p.units_per_req > 0) return u / p.units_per_req;   // uniform batch: no search
  int lo = 0, hi = p.nreq - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (p.r[mid].unit_off <= u) lo = mid; else hi = mid - 1;
  }
  return lo;
}
#endif

}  // namespace dllm
