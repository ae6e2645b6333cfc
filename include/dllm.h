/*
 * dllm.h — C-ABI of libdllm: dLLM-Serve's Head-Centric Sparse Attention hot
 * path (arXiv 2512.17077) on NVIDIA B200 (sm_100a).
 *
 * Three calls make up one pass of the path:
 *   dllm_refresh_attn       Refresh, Eq. 3 (§2.3) + the raw
 *                           per-head importance of Eq. 6 (§4.5)
 *   dllm_select_heads       local max-pool + per-head TopK (§4.5)
 *   dllm_refresh_select_attn  the two above in one call (select fused into the
 *                           Refresh kernel's epilogue when eligible)
 *   dllm_reuse_sparse_attn  Reuse, Eq. 4 (§2.3) over the
 *                           per-head key subsets of §4.5
 *
 * Plain C: no torch or CUDA types in the signatures.  Device buffers are
 * plain device pointers owned by the caller; host arrays are read during the
 * call only.  The library never allocates device memory on a call path and
 * never writes the K/V cache.
 *
 * Execution: compute calls enqueue kernels on `stream` (a cudaStream_t cast
 * to void*, NULL = legacy default stream) and return without synchronising.
 * They are CUDA-graph capturable.  Validation is all-or-nothing: on any
 * error nothing is enqueued.  Faults inside a kernel surface at the caller's
 * next synchronisation.  Device state of a launch (the Refresh unit
 * counters) lives only in the caller's optional workspace
 * (dllm_problem.workspace); launches sharing one workspace must be
 * stream-ordered.
 *
 * Layouts (all bf16 tensors 16-byte aligned, row-major, innermost last):
 *   q, out         [sum_b L_b, H, D]   packed varlen, request b at rows
 *                                      cu_L[b] = sum_{b'<b} L_b'
 *   q_blk, out_blk [sum_b blk_b, H, D] the active blocks, request order,
 *                                      blk_b = be_b - bs_b
 *   k_cache,       [num_pages, H_kv, P, D]  paged, head-major inside a page:
 *   v_cache                            position p of request b is page
 *                                      block_table[b*pages_per_req + p/P],
 *                                      slot p%P.  Keys are post-RoPE
 *                                      (R13).
 *   scores (fp32)  scores[H*cu_L[b] + h*L_b + m], m in [0, L_b): the raw,
 *                  UNSCALED max_{q in [bs,be)} Q[q,h].K[m,kv(h)] (DESIGN.md
 *                  R1, R8); block positions are written but not used.
 *   idx (int32)    idx[H*cu_k[b] + h*k_b + i], i in [0, k_b): selected
 *                  sequence positions, strictly ascending per (b, h), outside
 *                  [bs, be); cu_k[b] = sum_{b'<b} k_b'; k_b = dllm_keep_count
 *                  (keep_ratio, L_b - blk_b).
 * GQA: query head h reads KV head h / (H / H_kv) (R10).
 */
#ifndef DLLM_H_
#define DLLM_H_

#include <stdint.h>

#if defined(__GNUC__)
#define DLLM_API __attribute__((visibility("default")))
#else
#define DLLM_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (0 = success) ---------------------------------------- */
#define DLLM_OK                0
#define DLLM_ERR_INVALID_ARG  (-1)  /* NULL pointer, r not in (0,1], w even, ... */
#define DLLM_ERR_UNSUPPORTED  (-2)  /* head_dim / page_size / length outside the built kernels */
#define DLLM_ERR_SHAPE        (-3)  /* H % H_kv != 0, bs/be outside [0, L], misaligned buffers */
#define DLLM_ERR_K_RANGE      (-4)  /* k > n_ctx (only reachable through dllm_check_indices) */
#define DLLM_ERR_CUDA         (-5)  /* a CUDA launch / attribute call failed */

#define DLLM_MAX_SEQ_LEN   65536   /* L_b upper bound for refresh / reuse            */
#define DLLM_MAX_SELECT_LEN 32768  /* L_b upper bound for dllm_select_heads (smem)   */
#define DLLM_MAX_BLOCK     128     /* blk_b = be_b - bs_b upper bound                */
#define DLLM_MAX_POOL_WINDOW 65    /* pool_window upper bound (Table 3 uses 3)       */

/* The problem statement of one batch (a packed batch
 * of requests with per-request sequence length and active-block position;
 * heads / KV heads / head_dim; keep ratio r; pooling
 * window w). */
typedef struct dllm_problem {
  int32_t num_requests;        /* B >= 0                                          */
  int32_t num_heads;           /* H >= 1                                          */
  int32_t num_kv_heads;        /* H_kv >= 1, H % H_kv == 0                        */
  int32_t head_dim;            /* D in {16, 32, 64, 128}                          */
  const int32_t *seq_len;      /* HOST [B]: 1 <= L_b <= DLLM_MAX_SEQ_LEN          */
  const int32_t *blk_start;    /* HOST [B]: 0 <= bs_b                             */
  const int32_t *blk_end;      /* HOST [B]: bs_b < be_b <= L_b, be-bs <= 128      */
  double keep_ratio;           /* r in (0, 1]                                     */
  int32_t pool_window;         /* w odd in [1, 65] (Table 3 "Kernel Size" = 3)    */
  float softmax_scale;         /* tau; 0 -> 1/sqrt(D) (Eq. 3/4 "sqrt(d)")         */
  int32_t page_size;           /* P: power of two in [16, 1024]                   */
  int32_t pages_per_req;       /* row stride of block_table, >= ceil(L_b / P)     */
  const int32_t *block_table;  /* DEVICE [B * pages_per_req] physical page ids    */
  void *workspace;             /* DEVICE, optional (NULL ok): dllm_workspace_bytes()
                                  bytes, 16-byte aligned, ZERO-initialised once by
                                  the caller; every launch leaves it zeroed again.
                                  It holds the Refresh kernel's dynamic work-unit
                                  counters, so launches using one workspace must be
                                  stream-ordered: one workspace per stream (a
                                  captured graph must not be replayed concurrently
                                  with another launch on the same workspace).
                                  NULL: Refresh schedules its units statically
                                  (round-robin; same results, slower tails).      */
  int64_t workspace_bytes;     /* size of `workspace` (>= dllm_workspace_bytes())  */
} dllm_problem;

/* Bytes of the optional DEVICE workspace of dllm_problem (a constant of the
 * build, 4 KB).  Host only. */
DLLM_API int64_t dllm_workspace_bytes(void);

/* k = ceil(r * n_ctx) in IEEE double, clamped to [1, n_ctx]; 0 if n_ctx == 0
 * ("k = L*r", R5).  Returns a negative status for
 * r not in (0, 1] or n_ctx < 0.  Host only. */
DLLM_API int dllm_keep_count(double keep_ratio, int32_t n_ctx);

/* Validates `p` (host fields only; no CUDA call) and reports the index
 * layout: k_out (HOST [B], may be NULL) receives k_b, *total_idx (may be
 * NULL) receives H * sum_b k_b, the int32 count `idx` must hold.  Also the
 * size helpers: *total_rows = sum L_b, *total_blk_rows = sum blk_b (NULL ok). */
DLLM_API int dllm_index_layout(const dllm_problem *p, int32_t *k_out, int64_t *total_idx,
                      int64_t *total_rows, int64_t *total_blk_rows);

/* Refresh (Eq. 3): out[q, h] = softmax_j(tau * Q[q,h].K[j,kv(h)]) . V[j,kv(h)]
 * over all j in [0, L_b) (bidirectional, no mask), for every row of every
 * request; bf16 in, fp32 accumulation and softmax statistics, P rounded to
 * bf16 before P.V, bf16 out (R14).  If `scores` is not NULL it also
 * writes the raw importance (see layout above).  q, k_cache, v_cache, out,
 * scores: DEVICE. */
DLLM_API int dllm_refresh_attn(const dllm_problem *p, const void *q, const void *k_cache,
                      const void *v_cache, void *out, float *scores, void *stream);

/* Selection (Eq. 6 + TopK): per (b, h), over the candidates
 * C = [0, bs) ++ [be, L) (R4): S[c] = max of scores[C[c']] for
 * |c' - c| <= w/2, c' in [0, n_ctx) (pooling on the compacted candidate axis,
 * R2-R4); I^h = the k_b candidates with the largest S, ties to the lower c
 * (R6), written as positions C[c] ascending (R7).  Bit-exact.  -0 == +0.
 * Scores must be finite.  scores, idx: DEVICE. */
DLLM_API int dllm_select_heads(const dllm_problem *p, const float *scores, int32_t *idx, void *stream);

/* Refresh + selection in one call (next row N1, second half: the select fused
 * into the Refresh epilogue; the paper selects at Refresh time
 * §4.5).  Exactly dllm_refresh_attn(p, q, k_cache, v_cache, out, scores) followed
 * by dllm_select_heads(p, scores, idx): out, scores and idx are bit-identical to
 * the two calls.  In a library built with DLLM_TC2_FUSEDSEL=1, with D = 128 / 64
 * and every n_ctx = L_b - blk_b <= 4096, the pool + TopK of each (b, h) runs
 * inside the tcgen05 Refresh kernel (its epilogue warpgroup, right after the work
 * unit that wrote that head's raw scores) and no select launch follows; the
 * default build (measured faster) and every other case (or
 * DLLM_FUSED_SELECT=0 in the environment) launch the two kernels.  scores and idx are required (not NULL); sizes from
 * dllm_index_layout.  All tensors DEVICE. */
DLLM_API int dllm_refresh_select_attn(const dllm_problem *p, const void *q, const void *k_cache,
                                      const void *v_cache, void *out, float *scores, int32_t *idx, void *stream);

/* Uniform selection, the Sparse-dLLM baseline (§2.4, Eq. 5):
 * S[c] = sum_h (pooled scores of head h)[c], summed in fp32 in ascending head
 * order; ONE top-k set per request (same pooling, tie rule and order as
 * dllm_select_heads), written to every head's slot of the idx layout so that
 * dllm_reuse_sparse_attn runs the uniform baseline unchanged.  Bit-exact when
 * the head sums are exact in fp32.  scores, idx: DEVICE. */
DLLM_API int dllm_select_global(const dllm_problem *p, const float *scores, int32_t *idx, void *stream);

/* Per-KV-group selection (next row N2, GQA): for every request and KV head g,
 * S_g[c] = sum over the query heads h with kv(h) = g (ascending h, fp32) of the
 * per-head pooled score (Eq. 6's pooling), i.e. Eq. 5
 * restricted to the heads sharing one KV head (DESIGN.md
 * R21); ONE top-k set per (request, KV head) with the per-head rules (k_b, ties
 * to the lower candidate, ascending positions), written to the idx slot of every
 * head of the group, so dllm_reuse_sparse_attn reads each group's K/V rows once
 * per head from the same positions.  H_kv = H gives dllm_select_heads, H_kv = 1
 * dllm_select_global.  Bit-exact when the head sums are exact in fp32.  scores,
 * idx: DEVICE. */
DLLM_API int dllm_select_groups(const dllm_problem *p, const float *scores, int32_t *idx, void *stream);

/* Reuse (Eq. 4): out_blk[q, h] = softmax_j(tau * Qb[q,h].K[j,kv(h)]) . V[j,kv(h)]
 * over J^h = [bs, be) ++ idx(b, h), K/V read in place through the block table
 * (no pack, no copy).  The caller has written the active block's K/V rows
 * into the cache.  idx must satisfy the layout precondition above (checked
 * only by dllm_check_indices).  q_blk, k_cache, v_cache, idx, out_blk: DEVICE. */
DLLM_API int dllm_reuse_sparse_attn(const dllm_problem *p, const void *q_blk, const void *k_cache,
                           const void *v_cache, const int32_t *idx, void *out_blk,
                           void *stream);

/* Reuse over per-KV-group sets (next row N2, GQA; R21): the same
 * result as dllm_reuse_sparse_attn (Eq. 4) when every head of
 * a KV group holds the same index list, as dllm_select_groups writes them.
 * Precondition (not checked): for every request b and KV head g, idx(b, h) is
 * equal for all h with kv(h) = g; only the list of the group's first head of
 * each run of up to 4 heads is read.  The group's K/V rows are gathered once
 * for up to 4 of its heads instead of once per head.  Same layouts, pointers
 * and errors as dllm_reuse_sparse_attn, to which it falls back when H = H_kv
 * or D != 128.  All DEVICE. */
DLLM_API int dllm_reuse_group_sets(const dllm_problem *p, const void *q_blk, const void *k_cache,
                                   const void *v_cache, const int32_t *idx, void *out_blk, void *stream);

/* Pack (the paper's physical layout, §4.5: "pack the sparse
 * tokens into a physically dense KV layout", [N_heads, rL, D_head]): for every
 * (b, h, i), k_pack[(H*cu_k[b] + h*k_b + i) * D + d] = K[idx(b,h,i), kv(h), d]
 * and likewise V; row order = the idx layout.  k_pack, v_pack: DEVICE bf16
 * [H * sum_b k_b, D], caller-owned.  idx must satisfy the layout precondition. */
DLLM_API int dllm_pack_kv(const dllm_problem *p, const void *k_cache, const void *v_cache, const int32_t *idx,
                          void *k_pack, void *v_pack, void *stream);

/* Reuse over the packed context (Eq. 4 with K_cache = the packed per-head rows,
 * read contiguously with no index indirection): keys
 * [bs, be) from the paged cache ++ the k_b packed rows of (b, h).  Same output
 * as dllm_reuse_sparse_attn on the idx the buffers were packed from. */
DLLM_API int dllm_reuse_packed(const dllm_problem *p, const void *q_blk, const void *k_cache, const void *v_cache,
                               const void *k_pack, const void *v_pack, void *out_blk, void *stream);

/* Single-launch mixed-phase batch (next row N3; the paper's single varlen
 * dispatch over a packed batch of Refresh and Reuse requests, PAPER.md:366,
 * 453-456): dllm_refresh_attn over p_refresh (q, out, scores as there) and
 * dllm_reuse_sparse_attn over p_reuse (q_blk, idx, out_blk as there), both
 * reading one paged cache (k_cache, v_cache) through their own block tables,
 * computed by ONE persistent launch whose CTAs are split between the two phases
 * in proportion to their estimated times.  Results are bit-identical to the two
 * separate calls.  The problems must agree on H, H_kv, D and page size.  When
 * one phase is empty, a phase has more than 256 requests, or D != 128, the same
 * work runs as the two separate launches.  The Reuse requests' idx come from an
 * earlier selection; dllm_select_heads(p_refresh, scores, ...) may follow on the
 * same stream.  All pointers DEVICE; returns DLLM_OK or a negative status. */
DLLM_API int dllm_mixed_attn(const dllm_problem *p_refresh, const void *q, void *out, float *scores,
                             const dllm_problem *p_reuse, const void *q_blk, const int32_t *idx, void *out_blk,
                             const void *k_cache, const void *v_cache, void *stream);

/* dllm_mixed_attn with the Refresh requests' selection fused in (as in
 * dllm_refresh_select_attn): also writes idx_refresh = dllm_select_heads(
 * p_refresh, scores, .) from inside the same launch when eligible, else by a
 * select launch after it.  scores and idx_refresh required.  All DEVICE. */
DLLM_API int dllm_mixed_select_attn(const dllm_problem *p_refresh, const void *q, void *out, float *scores,
                                    int32_t *idx_refresh, const dllm_problem *p_reuse, const void *q_blk,
                                    const int32_t *idx, void *out_blk, const void *k_cache, const void *v_cache,
                                    void *stream);

/* ---- Logit decomposition (next row N4; §4.3 "Logit
 * Decomposition", §5; SPEC.md:145-165 plan_logit_chunks /
 * chunked_decode).  The LM head in token chunks of at most max_num_logits rows,
 * each chunk decoded by ArgMax before the next. ---- */

/* plan_logit_chunks: greedy full chunks of max_num_logits
 * followed by one remainder chunk, covering [0, n_logit) in order.  Writes up to
 * `capacity` sizes into chunk_sizes (HOST, may be NULL when capacity is 0) and
 * returns the number of chunks (>= 0), or DLLM_ERR_INVALID_ARG if n_logit < 0,
 * max_num_logits < 1 or the chunks do not fit in `capacity`. */
DLLM_API int dllm_logit_chunks(int64_t n_logit, int32_t max_num_logits, int32_t *chunk_sizes, int32_t capacity);

/* Bytes of DEVICE workspace dllm_lm_head_argmax needs: one 8-byte (max, index)
 * partial per (row of a chunk, 256-wide vocabulary tile), i.e.
 * min(n_tok, max_num_logits) * ceil(vocab / 256) * 8.  Negative on bad args. */
DLLM_API int64_t dllm_lm_head_workspace_bytes(int32_t n_tok, int32_t vocab, int32_t max_num_logits);

/* chunked_decode with ArgMax: for every token row i,
 *   ids[i] = argmax_v sum_k hidden[i,k] * weight[v,k]     (fp32 accumulation
 *   of the bf16 products; ties -> the LOWEST v),
 * processing the rows in the chunks of dllm_logit_chunks(n_tok,
 * max_num_logits).  The [chunk, vocab] logits are never written to memory:
 * every 128 x 256 logit tile is reduced in the tensor-core accumulator and only
 * per-tile (max, index) partials reach the workspace.
 *   hidden:  DEVICE bf16 [n_tok, d_model] row-major (token-major), 16-B aligned
 *   weight:  DEVICE bf16 [vocab, d_model] row-major (nn.Linear layout)
 *   ids:     DEVICE int32 [n_tok], written
 *   workspace: DEVICE, >= dllm_lm_head_workspace_bytes(...) bytes, caller-owned
 * d_model must be a positive multiple of 64; vocab >= 1; n_tok >= 0 (0 is a
 * no-op).  Returns DLLM_OK or a negative status; nothing is enqueued on error. */
DLLM_API int dllm_lm_head_argmax(const void *hidden, const void *weight, int32_t n_tok, int32_t d_model,
                                 int32_t vocab, int32_t max_num_logits, int32_t *ids, void *workspace,
                                 int64_t workspace_bytes, void *stream);

/* Debug: counts index-layout violations (out of [0, L), inside the block,
 * not strictly ascending) into *d_violations (DEVICE int32, zeroed by the
 * call).  idx, d_violations: DEVICE. */
DLLM_API int dllm_check_indices(const dllm_problem *p, const int32_t *idx, int32_t *d_violations,
                       void *stream);

/* Static description of a status code. */
DLLM_API const char *dllm_status_string(int status);

/* Thread-local detail of the last failing call on this thread ("" if none). */
DLLM_API const char *dllm_last_error(void);

/* Library build / kernel identification string (architecture, kernels). */
DLLM_API const char *dllm_version(void);

#ifdef __cplusplus
}
#endif

#endif /* DLLM_H_ */
