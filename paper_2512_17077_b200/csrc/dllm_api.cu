// libdllm host side: the C-ABI of include/dllm.h.
//
// Validates the problem synchronously (all-or-nothing: nothing is enqueued
// on error), computes the per-request layout (k_b, offsets), packs it into
// by-value launch plans (plan.h) of at most kMaxReqPerLaunch requests, and
// enqueues the kernels on the caller's stream.  No device allocation, no
// host<->device copy, no synchronisation on any call path.
#include <cuda_runtime.h>
#include <math.h>
#include <stdarg.h>
#include <stdlib.h>
#include <stddef.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <string>
#include <vector>

#include "../../include/dllm.h"
#include "plan.h"
#include "workspace.h"

namespace dllm {
cudaError_t launch_select(const Plan &, const float *, int32_t *, cudaStream_t);
cudaError_t launch_check_indices(const Plan &, const int32_t *, int32_t *, cudaStream_t);
cudaError_t launch_select_global(const Plan &, const float *, int32_t *, int, cudaStream_t);
cudaError_t launch_reuse_packed(const Plan &, const void *, const void *, const void *, const void *, const void *,
                                void *, cudaStream_t);
cudaError_t launch_pack_kv(const Plan &, const void *, const void *, const int32_t *, void *, void *, cudaStream_t);
cudaError_t launch_refresh_mma(const Plan &, const void *, const void *, const void *, void *, float *,
                               cudaStream_t);
cudaError_t launch_reuse_ws(const Plan &, const void *, const void *, const void *, const int32_t *, void *,
                            cudaStream_t);
cudaError_t launch_mixed_tc(const Plan &rplan, const void *q, const void *k, const void *v, void *out, float *scores,
                            const Plan &uplan, const void *q_blk, const int32_t *idx, void *out_blk, int n_ref,
                            int grid, int32_t *sel_idx, void *workspace, cudaStream_t st);
int reuse_tc_grid(const Plan &plan, int max_ctas);
int num_sms_mixed();
int64_t lmhead_vocab_tiles(int vocab);
cudaError_t launch_lmhead_chunk(const void *hidden, const void *weight, int n_tok, int d_model, int vocab, int row0,
                                int n_rows, int32_t *ids, void *workspace, cudaStream_t st);
bool reuse_tc_supported(int D);
cudaError_t launch_reuse_tc(const Plan &, const void *, const void *, const void *, const int32_t *, void *,
                            void *, cudaStream_t);
int refresh_mma_units(int L, int bs, int be, int H, bool with_scores);
bool refresh_tc_supported(int D);
int refresh_tc2_units(int L, int bs, int be, int H, bool with_scores);
cudaError_t launch_refresh_tc2(const Plan &, const void *, const void *, const void *, void *, float *, int32_t *,
                               void *, cudaStream_t);
int fused_select_max_n();
int reuse_grp_units(int H, int H_kv, int blk);
bool reuse_grp_supported(int D);
cudaError_t launch_reuse_grp(const Plan &, const void *, const void *, const void *, const int32_t *, void *,
                             bool union_sets, cudaStream_t);
int reuse_union_max_len();
// union mode needs a KV group of at least 2 query heads
constexpr int kUnionMinGroup = 2;
}  // namespace dllm

using namespace dllm;

namespace {

thread_local std::string g_last_error;

int fail(int code, const char *fmt, ...) __attribute__((format(printf, 2, 3)));
int fail(int code, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

int ok() {
  g_last_error.clear();
  return DLLM_OK;
}

bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

int keep_count_impl(double r, int32_t n) {
  if (!(r > 0.0 && r <= 1.0) || n < 0) return DLLM_ERR_INVALID_ARG;
  if (n == 0) return 0;
  double k = ceil(r * (double)n);   // IEEE double product, then ceil (R5)
  if (k < 1.0) k = 1.0;
  if (k > (double)n) k = (double)n;
  return (int)k;
}

// Host-side validation of every field the calls read.  Fills k[] when given.
int validate(const dllm_problem *p, std::vector<int32_t> *k) {
  if (!p) return fail(DLLM_ERR_INVALID_ARG, "problem is NULL");
  const int B = p->num_requests;
  if (B < 0) return fail(DLLM_ERR_INVALID_ARG, "num_requests=%d < 0", B);
  if (p->num_heads < 1 || p->num_kv_heads < 1)
    return fail(DLLM_ERR_INVALID_ARG, "num_heads=%d num_kv_heads=%d must be >= 1", p->num_heads, p->num_kv_heads);
  if (p->num_heads % p->num_kv_heads)
    return fail(DLLM_ERR_SHAPE, "num_heads=%d is not a multiple of num_kv_heads=%d", p->num_heads,
                p->num_kv_heads);
  const int D = p->head_dim;
  if (D != 16 && D != 32 && D != 64 && D != 128)
    return fail(DLLM_ERR_UNSUPPORTED, "head_dim=%d not in {16,32,64,128}", D);
  if (!(p->keep_ratio > 0.0 && p->keep_ratio <= 1.0))
    return fail(DLLM_ERR_INVALID_ARG, "keep_ratio=%g not in (0,1]", p->keep_ratio);
  if (p->pool_window < 1 || (p->pool_window & 1) == 0)
    return fail(DLLM_ERR_INVALID_ARG, "pool_window=%d must be odd and >= 1", p->pool_window);
  if (p->pool_window > DLLM_MAX_POOL_WINDOW)
    return fail(DLLM_ERR_UNSUPPORTED, "pool_window=%d > %d", p->pool_window, DLLM_MAX_POOL_WINDOW);
  if (!(p->softmax_scale >= 0.f) || isinf(p->softmax_scale))
    return fail(DLLM_ERR_INVALID_ARG, "softmax_scale must be finite and >= 0 (0 = 1/sqrt(D))");
  const int P = p->page_size;
  if (P < 16 || P > 1024 || (P & (P - 1)))
    return fail(DLLM_ERR_UNSUPPORTED, "page_size=%d must be a power of two in [16,1024]", P);
  if (B == 0) {
    if (k) k->clear();
    return DLLM_OK;
  }
  if (!p->seq_len || !p->blk_start || !p->blk_end)
    return fail(DLLM_ERR_INVALID_ARG, "seq_len / blk_start / blk_end must be host arrays of length B");
  if (!p->block_table) return fail(DLLM_ERR_INVALID_ARG, "block_table is NULL");
  if (k) k->resize(B);
  int64_t rows = 0;
  for (int b = 0; b < B; ++b) {
    const int L = p->seq_len[b], bs = p->blk_start[b], be = p->blk_end[b];
    if (L < 1 || L > DLLM_MAX_SEQ_LEN)
      return fail(L < 1 ? DLLM_ERR_SHAPE : DLLM_ERR_UNSUPPORTED, "request %d: seq_len=%d outside [1,%d]", b, L,
                  DLLM_MAX_SEQ_LEN);
    if (!(0 <= bs && bs < be && be <= L))
      return fail(DLLM_ERR_SHAPE, "request %d: need 0 <= blk_start(%d) < blk_end(%d) <= seq_len(%d)", b, bs, be, L);
    if (be - bs > DLLM_MAX_BLOCK)
      return fail(DLLM_ERR_UNSUPPORTED, "request %d: block of %d rows > %d", b, be - bs, DLLM_MAX_BLOCK);
    if ((int64_t)(L + P - 1) / P > p->pages_per_req)
      return fail(DLLM_ERR_SHAPE, "request %d: seq_len=%d needs %d pages > pages_per_req=%d", b, L, (L + P - 1) / P,
                  p->pages_per_req);
    rows += L;
    if (k) (*k)[b] = keep_count_impl(p->keep_ratio, L - (be - bs));
  }
  if (rows * p->num_heads * D > ((int64_t)1 << 40)) return fail(DLLM_ERR_UNSUPPORTED, "batch too large");
  if (p->workspace && (((uintptr_t)p->workspace & 15u) || p->workspace_bytes < kWorkspaceBytes))
    return fail(DLLM_ERR_INVALID_ARG, "workspace must be 16-byte aligned and hold dllm_workspace_bytes() = %lld bytes",
                (long long)kWorkspaceBytes);
  return DLLM_OK;
}

float scale_of(const dllm_problem *p) {
  return p->softmax_scale > 0.f ? p->softmax_scale : (float)(1.0 / sqrt((double)p->head_dim));
}

// Packs requests [b0, b1) into a plan; units(b) gives each request's unit count.
template <class UnitsFn>
void fill_plan(Plan &pl, const dllm_problem *p, const std::vector<int32_t> &k, int b0, int b1,
               const std::vector<int64_t> &cu_L, const std::vector<int64_t> &cu_blk,
               const std::vector<int64_t> &cu_k, UnitsFn units) {
  memset(&pl, 0, offsetof(Plan, r));
  pl.nreq = b1 - b0;
  pl.H = p->num_heads;
  pl.H_kv = p->num_kv_heads;
  pl.D = p->head_dim;
  pl.page_size = p->page_size;
  int sh = 0;
  while ((1 << sh) < p->page_size) ++sh;
  pl.page_shift = sh;
  pl.pages_per_req = p->pages_per_req;
  pl.window = p->pool_window;
  pl.scale = scale_of(p);
  pl.scale_log2 = (float)((double)pl.scale * 1.4426950408889634);
  pl.block_table = p->block_table;
  int u = 0, upr = -1;
  int64_t cost = 0, rc = -1;
  for (int b = b0; b < b1; ++b) {
    ReqInfo &r = pl.r[b - b0];
    r.L = p->seq_len[b];
    r.bs = p->blk_start[b];
    r.be = p->blk_end[b];
    r.q_off = (int32_t)cu_L[b];
    r.blk_off = (int32_t)cu_blk[b];
    r.k = k[b];
    r.idx_off = (int64_t)p->num_heads * cu_k[b];
    r.score_off = (int64_t)p->num_heads * cu_L[b];
    r.unit_off = u;
    r.bt_row = b;
    const int ub = units(b);
    upr = upr < 0 ? ub : (upr == ub ? upr : 0);
    u += ub;
    // Reuse balancing (plan.h): a unit of request b costs blk_b + k_b + kReuseUnitCost
    r.cost_off = cost;
    const int64_t c = (int64_t)ub * (r.be - r.bs + r.k + kReuseUnitCost);
    rc = rc < 0 ? c : (rc == c ? rc : 0);
    cost += c;
  }
  pl.total_units = u;
  pl.units_per_req = upr > 0 ? upr : 0;
  pl.total_cost = cost;
  pl.req_cost = (rc > 0 && rc <= INT32_MAX && upr > 0) ? (int32_t)rc : 0;
}

struct Layout {
  std::vector<int32_t> k;
  std::vector<int64_t> cu_L, cu_blk, cu_k;
};

int make_layout(const dllm_problem *p, Layout &lay) {
  int st = validate(p, &lay.k);
  if (st) return st;
  const int B = p->num_requests;
  lay.cu_L.assign(B + 1, 0);
  lay.cu_blk.assign(B + 1, 0);
  lay.cu_k.assign(B + 1, 0);
  for (int b = 0; b < B; ++b) {
    lay.cu_L[b + 1] = lay.cu_L[b] + p->seq_len[b];
    lay.cu_blk[b + 1] = lay.cu_blk[b] + (p->blk_end[b] - p->blk_start[b]);
    lay.cu_k[b + 1] = lay.cu_k[b] + lay.k[b];
  }
  if (lay.cu_L[B] > INT32_MAX) return fail(DLLM_ERR_UNSUPPORTED, "sum of seq_len exceeds 2^31");
  return DLLM_OK;
}

int cuda_fail(cudaError_t e, const char *what) {
  return fail(DLLM_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

// Reuse kernel choice: 1 = persistent mma.sync (DLLM_REUSE_IMPL=ws), 2 = tcgen05 per
// head (=tc), 3 = tcgen05 over the union of up to 4 heads' sets of a KV group
// (=union, GQA, L <= 8192: one gather per sub-group, each head masked to its own
// keys; it pays only when the heads' sets overlap strongly -- on the synthetic C2
// selections 74.6 vs 56.3 us, profiles/r02_ab_reuse_union.log); default 0: per head
// (D = 128), else mma.sync.
int reuse_impl_env() {
  const char *s = getenv("DLLM_REUSE_IMPL");
  if (s && !strcmp(s, "ws")) return 1;
  if (s && !strcmp(s, "tc")) return 2;
  if (s && !strcmp(s, "union")) return 3;
  return 0;
}

int refresh_impl_env() {
  // DLLM_REFRESH_IMPL=mma selects the mma.sync kernel (A/B comparisons); default:
  // tcgen05 (D = 64, 128), else the mma.sync kernel.
  const char *s = getenv("DLLM_REFRESH_IMPL");
  if (s && !strcmp(s, "mma")) return 0;
  return 2;
}

}  // namespace

extern "C" {

int64_t dllm_workspace_bytes(void) { return kWorkspaceBytes; }

int dllm_keep_count(double keep_ratio, int32_t n_ctx) {
  const int k = keep_count_impl(keep_ratio, n_ctx);
  if (k < 0) return fail(k, "keep_count: keep_ratio=%g n_ctx=%d", keep_ratio, n_ctx);
  return k;
}

int dllm_index_layout(const dllm_problem *p, int32_t *k_out, int64_t *total_idx, int64_t *total_rows,
                      int64_t *total_blk_rows) {
  Layout lay;
  int st = make_layout(p, lay);
  if (st) return st;
  const int B = p->num_requests;
  if (k_out)
    for (int b = 0; b < B; ++b) k_out[b] = lay.k[b];
  if (total_idx) *total_idx = (int64_t)p->num_heads * (B ? lay.cu_k[B] : 0);
  if (total_rows) *total_rows = B ? lay.cu_L[B] : 0;
  if (total_blk_rows) *total_blk_rows = B ? lay.cu_blk[B] : 0;
  return ok();
}

}  // extern "C"

namespace {
// Refresh (+ optionally the fused select): sel_idx != NULL asks the tcgen05 kernel
// to run pool + TopK in its epilogue warpgroup (caller checked fused_ok()).
int refresh_impl(const dllm_problem *p, const void *q, const void *k_cache, const void *v_cache, void *out,
                 float *scores, int32_t *sel_idx, void *stream) {
  Layout lay;
  int st = make_layout(p, lay);
  if (st) return st;
  const int B = p->num_requests;
  if (B == 0) return ok();
  if (!q || !k_cache || !v_cache || !out) return fail(DLLM_ERR_INVALID_ARG, "refresh: NULL tensor pointer");
  if (!aligned16(q) || !aligned16(k_cache) || !aligned16(v_cache) || !aligned16(out))
    return fail(DLLM_ERR_SHAPE, "refresh: bf16 tensors must be 16-byte aligned");
  if (scores && ((uintptr_t)scores & 3u)) return fail(DLLM_ERR_SHAPE, "refresh: scores must be 4-byte aligned");
  const bool with_scores = scores != nullptr;
  const int impl = refresh_tc_supported(p->head_dim) ? refresh_impl_env() : 0;
  cudaStream_t s = (cudaStream_t)stream;
  static thread_local Plan pl;
  for (int b0 = 0; b0 < B; b0 += kMaxReqPerLaunch) {
    const int b1 = b0 + kMaxReqPerLaunch < B ? b0 + kMaxReqPerLaunch : B;
    fill_plan(pl, p, lay.k, b0, b1, lay.cu_L, lay.cu_blk, lay.cu_k, [&](int b) {
      const int L = p->seq_len[b], bs = p->blk_start[b], be = p->blk_end[b], H = p->num_heads;
      return impl == 2 ? refresh_tc2_units(L, bs, be, H, with_scores) : refresh_mma_units(L, bs, be, H, with_scores);
    });
    pl.with_scores = with_scores;
    cudaError_t e = impl == 2 ? launch_refresh_tc2(pl, q, k_cache, v_cache, out, scores, sel_idx, p->workspace, s)
                              : launch_refresh_mma(pl, q, k_cache, v_cache, out, scores, s);
    if (e != cudaSuccess) return cuda_fail(e, "refresh launch");
  }
  return ok();
}

// the select can run inside the Refresh kernel: tcgen05 path, every candidate set
// small enough for the epilogue warpgroup's registers
bool fused_ok(const dllm_problem *p, const float *scores, const int32_t *idx) {
  if (!scores || !idx || !refresh_tc_supported(p->head_dim) || refresh_impl_env() != 2) return false;
  if (const char *e = getenv("DLLM_FUSED_SELECT"))
    if (e[0] == '0') return false;
  for (int b = 0; b < p->num_requests; ++b)
    if (p->seq_len[b] - (p->blk_end[b] - p->blk_start[b]) > fused_select_max_n()) return false;
  return true;
}
}  // namespace

extern "C" {

int dllm_refresh_attn(const dllm_problem *p, const void *q, const void *k_cache, const void *v_cache, void *out,
                      float *scores, void *stream) {
  return refresh_impl(p, q, k_cache, v_cache, out, scores, nullptr, stream);
}

int dllm_refresh_select_attn(const dllm_problem *p, const void *q, const void *k_cache, const void *v_cache,
                             void *out, float *scores, int32_t *idx, void *stream) {
  Layout lay;
  int st = make_layout(p, lay);
  if (st) return st;
  if (p->num_requests == 0) return ok();
  if (!scores || !idx) return fail(DLLM_ERR_INVALID_ARG, "refresh_select: NULL scores / idx");
  for (int b = 0; b < p->num_requests; ++b)
    if (p->seq_len[b] > DLLM_MAX_SELECT_LEN)
      return fail(DLLM_ERR_UNSUPPORTED, "select: request %d seq_len=%d > %d", b, p->seq_len[b], DLLM_MAX_SELECT_LEN);
  if (fused_ok(p, scores, idx)) return refresh_impl(p, q, k_cache, v_cache, out, scores, idx, stream);
  st = refresh_impl(p, q, k_cache, v_cache, out, scores, nullptr, stream);
  if (st) return st;
  return dllm_select_heads(p, scores, idx, stream);
}

int dllm_select_heads(const dllm_problem *p, const float *scores, int32_t *idx, void *stream) {
  Layout lay;
  int st = make_layout(p, lay);
  if (st) return st;
  const int B = p->num_requests;
  if (B == 0) return ok();
  if (!scores || !idx) return fail(DLLM_ERR_INVALID_ARG, "select: NULL pointer");
  for (int b = 0; b < B; ++b)
    if (p->seq_len[b] > DLLM_MAX_SELECT_LEN)
      return fail(DLLM_ERR_UNSUPPORTED, "select: request %d seq_len=%d > %d", b, p->seq_len[b], DLLM_MAX_SELECT_LEN);
  static thread_local Plan pl;
  for (int b0 = 0; b0 < B; b0 += kMaxReqPerLaunch) {
    const int b1 = b0 + kMaxReqPerLaunch < B ? b0 + kMaxReqPerLaunch : B;
    fill_plan(pl, p, lay.k, b0, b1, lay.cu_L, lay.cu_blk, lay.cu_k, [&](int) { return p->num_heads; });
    if (pl.total_units == 0) continue;
    cudaError_t e = launch_select(pl, scores, idx, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "select launch");
  }
  return ok();
}

}  // extern "C"

namespace {
int select_sets(const dllm_problem *p, const float *scores, int32_t *idx, void *stream, int heads_per_set,
                const char *who) {
  Layout lay;
  int st = make_layout(p, lay);
  if (st) return st;
  const int B = p->num_requests;
  if (B == 0) return ok();
  if (!scores || !idx) return fail(DLLM_ERR_INVALID_ARG, "%s: NULL pointer", who);
  for (int b = 0; b < B; ++b)
    if (p->seq_len[b] > DLLM_MAX_SELECT_LEN)
      return fail(DLLM_ERR_UNSUPPORTED, "%s: request %d seq_len=%d > %d", who, b, p->seq_len[b], DLLM_MAX_SELECT_LEN);
  static thread_local Plan pl;
  for (int b0 = 0; b0 < B; b0 += kMaxReqPerLaunch) {
    const int b1 = b0 + kMaxReqPerLaunch < B ? b0 + kMaxReqPerLaunch : B;
    fill_plan(pl, p, lay.k, b0, b1, lay.cu_L, lay.cu_blk, lay.cu_k, [&](int) { return 1; });
    cudaError_t e = launch_select_global(pl, scores, idx, heads_per_set, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "select_global launch");
  }
  return ok();
}
}  // namespace

extern "C" {

int dllm_select_global(const dllm_problem *p, const float *scores, int32_t *idx, void *stream) {
  return select_sets(p, scores, idx, stream, p ? p->num_heads : 1, "select_global");
}

int dllm_select_groups(const dllm_problem *p, const float *scores, int32_t *idx, void *stream) {
  return select_sets(p, scores, idx, stream, p && p->num_kv_heads > 0 ? p->num_heads / p->num_kv_heads : 1,
                     "select_groups");
}

int dllm_reuse_sparse_attn(const dllm_problem *p, const void *q_blk, const void *k_cache, const void *v_cache,
                           const int32_t *idx, void *out_blk, void *stream) {
  Layout lay;
  int st = make_layout(p, lay);
  if (st) return st;
  const int B = p->num_requests;
  if (B == 0) return ok();
  if (!q_blk || !k_cache || !v_cache || !out_blk) return fail(DLLM_ERR_INVALID_ARG, "reuse: NULL tensor pointer");
  if (!idx && lay.cu_k[B] > 0) return fail(DLLM_ERR_INVALID_ARG, "reuse: idx is NULL");
  if (!aligned16(q_blk) || !aligned16(k_cache) || !aligned16(v_cache) || !aligned16(out_blk))
    return fail(DLLM_ERR_SHAPE, "reuse: bf16 tensors must be 16-byte aligned");
  static thread_local Plan pl;
  const int impl = reuse_impl_env();
  for (int b0 = 0; b0 < B; b0 += kMaxReqPerLaunch) {
    const int b1 = b0 + kMaxReqPerLaunch < B ? b0 + kMaxReqPerLaunch : B;
    int max_len = 0;
    for (int b = b0; b < b1; ++b) max_len = p->seq_len[b] > max_len ? p->seq_len[b] : max_len;
    const bool use_union = impl == 3 && p->num_heads / p->num_kv_heads >= kUnionMinGroup &&
                           reuse_grp_supported(p->head_dim) && max_len <= reuse_union_max_len();
    fill_plan(pl, p, lay.k, b0, b1, lay.cu_L, lay.cu_blk, lay.cu_k, [&](int b) {
      const int blk = p->blk_end[b] - p->blk_start[b];
      return use_union ? reuse_grp_units(p->num_heads, p->num_kv_heads, blk) : p->num_heads * ((blk + 31) / 32);
    });
    cudaError_t e = use_union
        ? launch_reuse_grp(pl, q_blk, k_cache, v_cache, idx, out_blk, true, (cudaStream_t)stream)
        : impl != 1 && reuse_tc_supported(p->head_dim)
              ? launch_reuse_tc(pl, q_blk, k_cache, v_cache, idx, out_blk, p->workspace, (cudaStream_t)stream)
              : launch_reuse_ws(pl, q_blk, k_cache, v_cache, idx, out_blk, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "reuse launch");
  }
  return ok();
}

int dllm_reuse_group_sets(const dllm_problem *p, const void *q_blk, const void *k_cache, const void *v_cache,
                          const int32_t *idx, void *out_blk, void *stream) {
  Layout lay;
  int st = make_layout(p, lay);
  if (st) return st;
  const int B = p->num_requests;
  if (B == 0) return ok();
  // one set per KV group is a special case of per-head sets: the per-head kernel
  // computes the same attention (head dims the group kernel does not cover,
  // MHA where a group is one head, and the A/B switch DLLM_REUSE_IMPL=ws)
  if (!reuse_grp_supported(p->head_dim) || p->num_heads == p->num_kv_heads || reuse_impl_env() == 1)
    return dllm_reuse_sparse_attn(p, q_blk, k_cache, v_cache, idx, out_blk, stream);
  if (!q_blk || !k_cache || !v_cache || !out_blk) return fail(DLLM_ERR_INVALID_ARG, "reuse_group_sets: NULL tensor pointer");
  if (!idx && lay.cu_k[B] > 0) return fail(DLLM_ERR_INVALID_ARG, "reuse_group_sets: idx is NULL");
  if (!aligned16(q_blk) || !aligned16(k_cache) || !aligned16(v_cache) || !aligned16(out_blk))
    return fail(DLLM_ERR_SHAPE, "reuse_group_sets: bf16 tensors must be 16-byte aligned");
  static thread_local Plan pl;
  for (int b0 = 0; b0 < B; b0 += kMaxReqPerLaunch) {
    const int b1 = b0 + kMaxReqPerLaunch < B ? b0 + kMaxReqPerLaunch : B;
    fill_plan(pl, p, lay.k, b0, b1, lay.cu_L, lay.cu_blk, lay.cu_k, [&](int b) {
      return reuse_grp_units(p->num_heads, p->num_kv_heads, p->blk_end[b] - p->blk_start[b]);
    });
    cudaError_t e = launch_reuse_grp(pl, q_blk, k_cache, v_cache, idx, out_blk, false, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "reuse_group_sets launch");
  }
  return ok();
}

int dllm_pack_kv(const dllm_problem *p, const void *k_cache, const void *v_cache, const int32_t *idx, void *k_pack,
                 void *v_pack, void *stream) {
  Layout lay;
  int st = make_layout(p, lay);
  if (st) return st;
  const int B = p->num_requests;
  if (B == 0 || lay.cu_k[B] == 0) return ok();
  if (!k_cache || !v_cache || !idx || !k_pack || !v_pack) return fail(DLLM_ERR_INVALID_ARG, "pack_kv: NULL pointer");
  if (!aligned16(k_cache) || !aligned16(v_cache) || !aligned16(k_pack) || !aligned16(v_pack))
    return fail(DLLM_ERR_SHAPE, "pack_kv: bf16 tensors must be 16-byte aligned");
  static thread_local Plan pl;
  for (int b0 = 0; b0 < B; b0 += kMaxReqPerLaunch) {
    const int b1 = b0 + kMaxReqPerLaunch < B ? b0 + kMaxReqPerLaunch : B;
    fill_plan(pl, p, lay.k, b0, b1, lay.cu_L, lay.cu_blk, lay.cu_k, [&](int) { return p->num_heads; });
    cudaError_t e = launch_pack_kv(pl, k_cache, v_cache, idx, k_pack, v_pack, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "pack_kv launch");
  }
  return ok();
}

int dllm_reuse_packed(const dllm_problem *p, const void *q_blk, const void *k_cache, const void *v_cache,
                      const void *k_pack, const void *v_pack, void *out_blk, void *stream) {
  Layout lay;
  int st = make_layout(p, lay);
  if (st) return st;
  const int B = p->num_requests;
  if (B == 0) return ok();
  if (!q_blk || !k_cache || !v_cache || !out_blk) return fail(DLLM_ERR_INVALID_ARG, "reuse_packed: NULL tensor pointer");
  if ((!k_pack || !v_pack) && lay.cu_k[B] > 0) return fail(DLLM_ERR_INVALID_ARG, "reuse_packed: NULL packed buffer");
  if (lay.cu_k[B] * (int64_t)p->num_heads > INT32_MAX)
    return fail(DLLM_ERR_UNSUPPORTED, "reuse_packed: more than 2^31 packed rows");
  if (!aligned16(q_blk) || !aligned16(k_cache) || !aligned16(v_cache) || !aligned16(out_blk) ||
      !aligned16(k_pack) || !aligned16(v_pack))
    return fail(DLLM_ERR_SHAPE, "reuse_packed: bf16 tensors must be 16-byte aligned");
  static thread_local Plan pl;
  for (int b0 = 0; b0 < B; b0 += kMaxReqPerLaunch) {
    const int b1 = b0 + kMaxReqPerLaunch < B ? b0 + kMaxReqPerLaunch : B;
    fill_plan(pl, p, lay.k, b0, b1, lay.cu_L, lay.cu_blk, lay.cu_k, [&](int b) {
      const int blk = p->blk_end[b] - p->blk_start[b];
      return p->num_heads * ((blk + 31) / 32);
    });
    cudaError_t e = launch_reuse_packed(pl, q_blk, k_cache, v_cache, k_pack, v_pack, out_blk, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "reuse_packed launch");
  }
  return ok();
}

int dllm_check_indices(const dllm_problem *p, const int32_t *idx, int32_t *d_violations, void *stream) {
  Layout lay;
  int st = make_layout(p, lay);
  if (st) return st;
  if (!d_violations) return fail(DLLM_ERR_INVALID_ARG, "check_indices: d_violations is NULL");
  const int B = p->num_requests;
  cudaError_t e = cudaMemsetAsync(d_violations, 0, sizeof(int32_t), (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "check_indices memset");
  if (B == 0) return ok();
  if (!idx && lay.cu_k[B] > 0) return fail(DLLM_ERR_INVALID_ARG, "check_indices: idx is NULL");
  static thread_local Plan pl;
  for (int b0 = 0; b0 < B; b0 += kMaxReqPerLaunch) {
    const int b1 = b0 + kMaxReqPerLaunch < B ? b0 + kMaxReqPerLaunch : B;
    fill_plan(pl, p, lay.k, b0, b1, lay.cu_L, lay.cu_blk, lay.cu_k, [&](int) { return p->num_heads; });
    e = launch_check_indices(pl, idx, d_violations, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "check_indices launch");
  }
  return ok();
}

}  // extern "C"

namespace {
int mixed_impl(const dllm_problem *p_refresh, const void *q, void *out, float *scores, int32_t *sel_idx,
               const dllm_problem *p_reuse, const void *q_blk, const int32_t *idx, void *out_blk,
               const void *k_cache, const void *v_cache, void *stream) {
  if (!p_refresh || !p_reuse) return fail(DLLM_ERR_INVALID_ARG, "mixed: NULL problem");
  Layout lr, lu;
  int st = make_layout(p_refresh, lr);
  if (st) return st;
  st = make_layout(p_reuse, lu);
  if (st) return st;
  const int Br = p_refresh->num_requests, Bu = p_reuse->num_requests;
  if (Br > 0 && Bu > 0 &&
      (p_refresh->num_heads != p_reuse->num_heads || p_refresh->num_kv_heads != p_reuse->num_kv_heads ||
       p_refresh->head_dim != p_reuse->head_dim || p_refresh->page_size != p_reuse->page_size))
    return fail(DLLM_ERR_SHAPE, "mixed: the two problems address one paged cache and must agree on H, H_kv, D, page");
  const bool single = Br > 0 && Bu > 0 && Br <= kMaxReqPerLaunch && Bu <= kMaxReqPerLaunch &&
                      p_refresh->head_dim == 128 && refresh_impl_env() == 2 && reuse_impl_env() != 1;
  if (!single) {
    // not expressible as one launch (a phase is empty, > kMaxReqPerLaunch requests, or
    // a head dim / A-B override outside the two tcgen05 kernels): the same work as
    // separate launches, same results
    st = sel_idx ? dllm_refresh_select_attn(p_refresh, q, k_cache, v_cache, out, scores, sel_idx, stream)
                 : dllm_refresh_attn(p_refresh, q, k_cache, v_cache, out, scores, stream);
    if (st) return st;
    return dllm_reuse_sparse_attn(p_reuse, q_blk, k_cache, v_cache, idx, out_blk, stream);
  }
  if (!q || !out || !q_blk || !out_blk || !k_cache || !v_cache)
    return fail(DLLM_ERR_INVALID_ARG, "mixed: NULL tensor pointer");
  if (!idx && lu.cu_k[Bu] > 0) return fail(DLLM_ERR_INVALID_ARG, "mixed: idx is NULL");
  if (!aligned16(q) || !aligned16(out) || !aligned16(q_blk) || !aligned16(out_blk) || !aligned16(k_cache) ||
      !aligned16(v_cache))
    return fail(DLLM_ERR_SHAPE, "mixed: bf16 tensors must be 16-byte aligned");
  if (scores && ((uintptr_t)scores & 3u)) return fail(DLLM_ERR_SHAPE, "mixed: scores must be 4-byte aligned");
  const bool with_scores = scores != nullptr;
  static thread_local Plan rp, up;
  fill_plan(rp, p_refresh, lr.k, 0, Br, lr.cu_L, lr.cu_blk, lr.cu_k, [&](int b) {
    return refresh_tc2_units(p_refresh->seq_len[b], p_refresh->blk_start[b], p_refresh->blk_end[b],
                             p_refresh->num_heads, with_scores);
  });
  rp.with_scores = with_scores;
  fill_plan(up, p_reuse, lu.k, 0, Bu, lu.cu_L, lu.cu_blk, lu.cu_k, [&](int b) {
    return p_reuse->num_heads * ((p_reuse->blk_end[b] - p_reuse->blk_start[b] + 31) / 32);
  });
  // split the SMs between the phases in proportion to their estimated times
  // (Refresh: 4 H L^2 D FLOP at ~1 PFLOP/s; Reuse: H (blk + k) rows of K and V at ~5 TB/s)
  double t_ref = 0, t_reu = 0;
  const double H = p_refresh->num_heads, D = p_refresh->head_dim;
  for (int b = 0; b < Br; ++b) t_ref += 4.0 * H * (double)p_refresh->seq_len[b] * p_refresh->seq_len[b] * D / 1.0e15;
  for (int b = 0; b < Bu; ++b)
    t_reu += H * (double)(p_reuse->blk_end[b] - p_reuse->blk_start[b] + lu.k[b]) * 4.0 * D / 5.0e12;
  const int nsm = num_sms_mixed();
  if (const char *e = getenv("DLLM_MIXED_REFRESH_WEIGHT")) t_ref *= atof(e);   // dev: A/B of the SM split
  int n_ref = (int)(nsm * t_ref / (t_ref + t_reu) + 0.5);
  n_ref = n_ref < 1 ? 1 : (n_ref > nsm - 1 ? nsm - 1 : n_ref);
  if (n_ref > rp.total_units) n_ref = rp.total_units;
  const int n_reu = reuse_tc_grid(up, nsm - n_ref);
  cudaError_t e = launch_mixed_tc(rp, q, k_cache, v_cache, out, scores, up, q_blk, idx, out_blk, n_ref, n_ref + n_reu,
                                  sel_idx, p_refresh->workspace, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "mixed launch");
  return ok();
}
}  // namespace

extern "C" {

int dllm_mixed_attn(const dllm_problem *p_refresh, const void *q, void *out, float *scores,
                    const dllm_problem *p_reuse, const void *q_blk, const int32_t *idx, void *out_blk,
                    const void *k_cache, const void *v_cache, void *stream) {
  return mixed_impl(p_refresh, q, out, scores, nullptr, p_reuse, q_blk, idx, out_blk, k_cache, v_cache, stream);
}

int dllm_mixed_select_attn(const dllm_problem *p_refresh, const void *q, void *out, float *scores, int32_t *idx_refresh,
                           const dllm_problem *p_reuse, const void *q_blk, const int32_t *idx, void *out_blk,
                           const void *k_cache, const void *v_cache, void *stream) {
  if (!p_refresh) return fail(DLLM_ERR_INVALID_ARG, "mixed: NULL problem");
  if (!scores || !idx_refresh) return fail(DLLM_ERR_INVALID_ARG, "mixed_select: NULL scores / idx_refresh");
  for (int b = 0; b < p_refresh->num_requests; ++b)
    if (p_refresh->seq_len[b] > DLLM_MAX_SELECT_LEN)
      return fail(DLLM_ERR_UNSUPPORTED, "select: request %d seq_len=%d > %d", b, p_refresh->seq_len[b],
                  DLLM_MAX_SELECT_LEN);
  if (fused_ok(p_refresh, scores, idx_refresh))
    return mixed_impl(p_refresh, q, out, scores, idx_refresh, p_reuse, q_blk, idx, out_blk, k_cache, v_cache, stream);
  int st = mixed_impl(p_refresh, q, out, scores, nullptr, p_reuse, q_blk, idx, out_blk, k_cache, v_cache, stream);
  if (st) return st;
  return dllm_select_heads(p_refresh, scores, idx_refresh, stream);
}

int dllm_logit_chunks(int64_t n_logit, int32_t max_num_logits, int32_t *chunk_sizes, int32_t capacity) {
  if (n_logit < 0 || max_num_logits < 1 || capacity < 0)
    return fail(DLLM_ERR_INVALID_ARG, "logit_chunks: n_logit %lld, max_num_logits %d, capacity %d",
                (long long)n_logit, max_num_logits, capacity);
  const int64_t n = (n_logit + max_num_logits - 1) / max_num_logits;
  if (n > capacity && (capacity > 0 || chunk_sizes))
    return fail(DLLM_ERR_INVALID_ARG, "logit_chunks: %lld chunks do not fit capacity %d", (long long)n, capacity);
  if (n > 0x7fffffff) return fail(DLLM_ERR_INVALID_ARG, "logit_chunks: too many chunks");
  for (int64_t i = 0; chunk_sizes && i < n; ++i) {
    const int64_t left = n_logit - i * max_num_logits;
    chunk_sizes[i] = (int32_t)(left < max_num_logits ? left : max_num_logits);
  }
  ok();
  return (int)n;
}

int64_t dllm_lm_head_workspace_bytes(int32_t n_tok, int32_t vocab, int32_t max_num_logits) {
  if (n_tok < 0 || vocab < 1 || max_num_logits < 1)
    return fail(DLLM_ERR_INVALID_ARG, "lm_head_workspace_bytes: n_tok %d, vocab %d, max_num_logits %d", n_tok, vocab,
                max_num_logits);
  const int64_t rows = n_tok < max_num_logits ? n_tok : max_num_logits;
  return rows * lmhead_vocab_tiles(vocab) * 8;
}

int dllm_lm_head_argmax(const void *hidden, const void *weight, int32_t n_tok, int32_t d_model, int32_t vocab,
                        int32_t max_num_logits, int32_t *ids, void *workspace, int64_t workspace_bytes,
                        void *stream) {
  if (n_tok < 0 || vocab < 1 || max_num_logits < 1 || d_model < 64 || d_model % 64)
    return fail(d_model > 0 && d_model % 64 ? DLLM_ERR_UNSUPPORTED : DLLM_ERR_INVALID_ARG,
                "lm_head_argmax: n_tok %d, d_model %d (multiple of 64), vocab %d, max_num_logits %d", n_tok, d_model,
                vocab, max_num_logits);
  if (n_tok == 0) return ok();
  if (!hidden || !weight || !ids || !workspace)
    return fail(DLLM_ERR_INVALID_ARG, "lm_head_argmax: NULL buffer");
  if (((uintptr_t)hidden | (uintptr_t)weight | (uintptr_t)workspace) & 15)
    return fail(DLLM_ERR_SHAPE, "lm_head_argmax: hidden / weight / workspace not 16-byte aligned");
  const int64_t need = dllm_lm_head_workspace_bytes(n_tok, vocab, max_num_logits);
  if (workspace_bytes < need)
    return fail(DLLM_ERR_INVALID_ARG, "lm_head_argmax: workspace %lld bytes < %lld", (long long)workspace_bytes,
                (long long)need);
  for (int64_t r0 = 0; r0 < n_tok; r0 += max_num_logits) {
    const int rows = (int)(n_tok - r0 < max_num_logits ? n_tok - r0 : max_num_logits);
    cudaError_t e = launch_lmhead_chunk(hidden, weight, n_tok, d_model, vocab, (int)r0, rows, ids, workspace,
                                        (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "lm_head_argmax launch");
  }
  return ok();
}

const char *dllm_status_string(int status) {
  switch (status) {
    case DLLM_OK: return "DLLM_OK";
    case DLLM_ERR_INVALID_ARG: return "DLLM_ERR_INVALID_ARG";
    case DLLM_ERR_UNSUPPORTED: return "DLLM_ERR_UNSUPPORTED";
    case DLLM_ERR_SHAPE: return "DLLM_ERR_SHAPE";
    case DLLM_ERR_K_RANGE: return "DLLM_ERR_K_RANGE";
    case DLLM_ERR_CUDA: return "DLLM_ERR_CUDA";
  }
  return "DLLM_ERR_UNKNOWN";
}

const char *dllm_last_error(void) { return g_last_error.c_str(); }

const char *dllm_version(void) {
  static const std::string v = std::string(
      "libdllm sm_100a: refresh=tcgen05/TMEM+TMA (D=16..128), select=radix-topk, "
      "reuse=paged cp.async gather + tcgen05 (D=16..128), mixed=one-launch Refresh+Reuse, "
      "lm_head=tcgen05 GEMM + fused argmax, select_in_refresh=") + (fused_select_max_n() > 0 ? "on" : "off");
  return v.c_str();
}

}  // extern "C"
