#pragma once
// Reuse sparse attention on the 5th-generation tensor cores (tcgen05 + TMEM)
// (§2.3, Eq. 4; per-head key sets of §4.5).
//
// For request b, query head h and the active block's query rows q:
//   O_b[q,h] = softmax_j(tau Q_blk[q,h].K[j,kv(h)]) V[j,kv(h)],  j in [bs,be) ++ idx(b,h)
// with K/V gathered in place from the paged cache.
//
// Work units and balancing.  A unit is (request b, head h, 32-row group of the
// block) with nk = blk + k keys; it costs nk + kReuseUnitCost (plan.h).  The
// launch's total cost is cut into ncta EQUAL contiguous ranges of the unit
// sequence, one per CTA, so every CTA streams the same number of keys (no wave
// tail: C1's 512 units over 148 SMs would otherwise leave 68 CTAs a 4th unit).
// A unit cut by a range boundary is computed in pieces ("segments") by
// consecutive CTAs: the CTA holding the unit's first key (the owner) processes
// its piece LAST in its range, every other CTA holding a piece processes it
// FIRST and writes (O^T, row max m, row sum l) unnormalised to its slot of the
// caller's workspace; the owner merges them (flash-decoding style rescale) when
// it finishes, so it never waits in practice.  Without a workspace the ranges
// are rounded to whole units (no merge).
//
// Dense key stream.  A CTA's keys form one stream over its segments, cut into
// 128-key chunks that may span a segment boundary (at most two "parts": the end
// of one segment and the start of the next), so every ring stage but the last
// is full: with one unit per stage group (C1: 280 keys = 2.2 stages) a third of
// the ring slots carried a nearly empty chunk and the stream reached ~77% of
// HBM in its steady state (profiles/r02_trace_reuse_C1.log).
//
// Why transposed.  A unit has only 32 query rows and tcgen05 needs M = 128 for
// the one-row-per-TMEM-lane accumulator layout, so keys sit on the M axis:
//   S^T[128 keys x 32 rows]  = K_chunk[128 x D] . Q^T           (A = K, K-major)
//   O^T[D=128 x 32 rows]    += V_chunk^T[D x 128] . P^T          (A = V, MN-major;
//                                                                 B = P^T)
// A chunk with two parts runs two S^T MMAs (one per segment's Q) into two TMEM
// buffers and two P.V MMAs into the two segments' O^T accumulators; each part's
// P^T has zeros for the other part's keys.
//
// Roles (16 warps, one CTA per SM, persistent):
//   warp 4           translator: the index lists kLA chunks ahead (4-byte cp.async
//                    into a position ring, so an index load never sits behind the
//                    gathers it feeds), then position -> physical cache row for
//                    every key of a chunk (page ids from the block-table rows of the
//                    CTA's requests, staged once in smem) into a row-offset ring;
//   warps 0-3, 6, 7  loaders: the segments' Q rows and 16-byte cp.async row
//                    gathers of K and V into the NS-stage ring laid out as UMMA
//                    SW128 operand tiles (a lean loop: one offset read per row);
//   warp 5           MMA issuer (one elected lane issues; warp-uniform loop);
//   warps 8-11       softmax (thread = key = TMEM lane, 32 query rows in
//                    registers; lazy rescale, barrier-OR decides the rare case);
//   warps 12-15      epilogue: O^T / l -> bf16 rows -> bulk (TMA) stores; the
//                    partial write / merge of split units.
// P^T is written over the stage's K tile once its S^T MMAs completed (part A at
// +0, part B at +8 KB).  cp.async data (generic proxy) is published to the
// tensor core (async proxy) by a proxy fence in the MMA warp after the full
// barrier.  The ring is zeroed once: rows a chunk leaves empty keep finite data
// (masked to p = 0 by the softmax), so they need no load.
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "plan.h"
#include "tc_ptx.cuh"

namespace dllm {
namespace rtc {

constexpr int kTD = 128;            // head dim supported by this kernel
constexpr int kTRows = 32;          // query rows per unit (MMA N)
constexpr int kTChunk = 128;        // keys per ring stage (MMA M of S^T)
constexpr int kTNS = 3;             // K/V ring stages (64 KB each)
constexpr int kNP = 6;              // position ring slots (one chunk each)
constexpr int kLA = kNP - 1;        // index lookahead in chunks
constexpr int kTNT = 4;             // row-offset ring slots (translator -> loaders)
#ifndef DLLM_RTC_IDXLDG
#define DLLM_RTC_IDXLDG 0           // dev A/B: translator reads the index lists with __ldg (no lookahead staging)
#endif
constexpr int kBtCap = 512;         // block-table entries staged in smem
constexpr int kMaxCtas = 256;       // workspace partial slots (>= SMs per launch)
constexpr int kPartFloats = kTD * kTRows + 2 * kTRows;   // O^T [D][32] + m[32] + l[32]

// Warp roles (the warp schedulers favour the highest warp id among the eligible
// warps of a sub-partition, so the softmax and epilogue warps sit on top)
constexpr int kTLoaders = 6, kTransWarp = 4, kMmaWarp = 5, kSoft0 = 8, kEpi0 = 12, kTWarps = 16;
__device__ __forceinline__ int loader_index(int w) { return w < 4 ? w : (w == 6 || w == 7 ? w - 2 : -1); }
constexpr int kTThreads = kTWarps * 32;
constexpr int kLThreads = 32 * kTLoaders;

// shared memory (offsets from a 1024-byte aligned base)
constexpr int kTileK = kTChunk * kTD * 2;       // 32 KB: [2 atoms][128 rows][128 B]
constexpr int kStage = 2 * kTileK;              // K then V
constexpr int kQTile = kTRows * kTD * 2;        // 8 KB: [2 atoms][32 rows][128 B]
constexpr int kOffQ = kTNS * kStage;
constexpr int kOffPos = kOffQ + 2 * kQTile;               // [kNP][kTChunk] int32 positions
constexpr int kOffOffs = kOffPos + kNP * kTChunk * 4;    // [kTNT][kTChunk] int32 cache row offsets (-1: none)
constexpr int kOffBt = kOffOffs + kTNT * kTChunk * 4;     // [kBtCap] int32
constexpr int kOffRed = kOffBt + kBtCap * 4;              // [4 warps][32] chunk row maxima
constexpr int kOffL = kOffRed + 4 * 32 * 4;               // [2 O buffers][4 warps][32 rows] partial row sums
constexpr int kOffM = kOffL + 2 * 4 * 32 * 4;             // [2 O buffers][32 rows] running maxima (log2 domain)
constexpr int kOffStage = kOffM + 2 * 32 * 4;             // output staging [32 rows][D] bf16
constexpr int kOffReq = kOffStage + kTRows * kTD * 2;     // [kReqCache] ReqInfo of the CTA's requests
constexpr int kOffBar = kOffReq + 16 * (int)sizeof(ReqInfo);
constexpr int kNumBars = 2 * kTNS + 2 * kTNT + 2 * 2 + 2 * 3 + 1 + 2 * 3 + 1;
constexpr int kTBytes = kOffBar + 8 * kNumBars + 1024;    // + alignment slack
static_assert(kTBytes <= 227 * 1024, "reuse_tc shared memory");

// TMEM columns: S^T [2 chunk buffers][2 parts] (32 each), O^T [2 segment buffers]
constexpr uint32_t kTmemCols = 256;
__device__ __forceinline__ uint32_t tm_s(int b, int part) { return (uint32_t)(b * 64 + part * 32); }
__device__ __forceinline__ uint32_t tm_o(int b) { return (uint32_t)(128 + b * 32); }

#ifdef DLLM_TRACE
// per-CTA timeline (globaltimer ns): [0] start, [1] first gathers issued, [2] first
// S issued, [3..10] epilogue: end of segment i, [11] end, [12] SM id, [13] chunks;
// CTA 0 per chunk: [0] idx issued, [1] gathers issued, [2] S issued, [3] softmax
// got S, [4] P written, [5] P.V issued
static __device__ long long g_rtc[1024][16];
static __device__ long long g_rtc_chunk[16][64];
__device__ __forceinline__ long long rtc_timer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define RTC_CTA(slot, v)                                            \
  do {                                                              \
    if (lane == 0 && cta < 1024) g_rtc[cta][slot] = (v);            \
  } while (0)
#define RTC_CHUNK(kind, t)                                                          \
  do {                                                                              \
    if (lane == 0 && cta == 0 && (t) < 64) g_rtc_chunk[kind][t] = rtc_timer();      \
  } while (0)
#else
#define RTC_CTA(slot, v) \
  do {                   \
  } while (0)
#define RTC_CHUNK(kind, t) \
  do {                     \
  } while (0)
#endif

struct TUnit {
  int b, h, kvh, rg, blk, bs, nk, k, blk_off, bt_row;
  int64_t idx_off;     // first index of (b, h)
  int64_t cost0;       // cost position of the unit's first key
};

// The CTA's requests' metadata, staged in shared memory by the prologue: the plan
// lives in kernel-parameter (constant) space, whose reads miss the small constant
// cache (hundreds of clk each) and would sit on every role's per-chunk path.
// Requests outside [b0, b0 + n) (a range spanning more than kReqCache requests)
// fall back to the parameter copy.
constexpr int kReqCache = 16;
struct ReqCache {
  const ReqInfo *rq;   // smem [n]
  int b0, n;
  // by value, each source read with its own instructions (LDS / LDC): a reference
  // would merge the two into generic loads, slow on the parameter window
  __device__ __forceinline__ ReqInfo get(const Plan &pl, int b) const {
    ReqInfo R;
    if ((unsigned)(b - b0) < (unsigned)n) {
      R = rq[b - b0];
    } else {
      R = pl.r[b];
    }
    return R;
  }
  // request owning unit u
  __device__ __forceinline__ int find(const Plan &pl, int u) const {
    if (pl.units_per_req > 0) return u / pl.units_per_req;
    if (n > 0 && u >= rq[0].unit_off) {
      int b = 0;
      while (b + 1 < n && rq[b + 1].unit_off <= u) ++b;
      if (b + 1 < n || b0 + n == pl.nreq) return b0 + b;
    }
    return plan_find(pl, u);
  }
};

__device__ __forceinline__ void tdecode(const Plan &pl, const ReqCache &rc, int unit, TUnit &u) {
  u.b = rc.find(pl, unit);
  const ReqInfo R = rc.get(pl, u.b);
  u.blk = R.be - R.bs;
  u.bs = R.bs;
  const int ngroups = (u.blk + kTRows - 1) / kTRows;
  const int local = unit - R.unit_off;
  u.h = local / ngroups;
  u.rg = local - u.h * ngroups;
  u.kvh = u.h / (pl.H / pl.H_kv);
  u.k = R.k;
  u.nk = u.blk + R.k;
  u.blk_off = R.blk_off;
  u.bt_row = R.bt_row;
  u.idx_off = R.idx_off + (int64_t)u.h * R.k;
  u.cost0 = R.cost_off + (int64_t)local * (u.nk + kReuseUnitCost);
}

// (unit, key) at cost position x; a position in a unit's virtual cost tail maps to
// the next unit's first key
__device__ __forceinline__ void locate(const Plan &pl, int64_t x, int &u, int &j) {
  if (x >= pl.total_cost) {
    u = pl.total_units;
    j = 0;
    return;
  }
  int b;
  if (pl.req_cost > 0) {
    b = (int)(x / pl.req_cost);
    b = b < pl.nreq ? b : pl.nreq - 1;
  } else {
    int lo = 0, hi = pl.nreq - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (pl.r[mid].cost_off <= x) lo = mid; else hi = mid - 1;
    }
    b = lo;
  }
  const ReqInfo &R = pl.r[b];
  const int nk = R.be - R.bs + R.k, uc = nk + kReuseUnitCost;
  const int64_t rel = x - R.cost_off;
  const int ul = (int)(rel / uc);
  u = R.unit_off + ul;
  j = (int)(rel - (int64_t)ul * uc);
  if (j >= nk) {
    ++u;
    j = 0;
  }
}

__device__ __forceinline__ int64_t range_start(const Plan &pl, int c, int ncta) {
  return (int64_t)c * pl.total_cost / ncta;
}

// CTA whose range holds cost position x (largest c with range_start(c) <= x)
__device__ __forceinline__ int cta_of(const Plan &pl, int64_t x, int ncta) {
  int c = (int)(x * ncta / pl.total_cost);
  while (c + 1 < ncta && range_start(pl, c + 1, ncta) <= x) ++c;
  while (c > 0 && range_start(pl, c, ncta) > x) --c;
  return c;
}

// A CTA's key stream: from key j0 of unit u0 up to (excluding) key j1 of unit u1
// (j1 == 0: up to the end of unit u1 - 1).
struct Range {
  int u0, j0, u1, j1;
  __device__ __forceinline__ bool empty() const { return u0 > u1 || (u0 == u1 && j0 >= j1); }
  __device__ __forceinline__ int last_unit() const { return j1 > 0 ? u1 : u1 - 1; }
};

__device__ __forceinline__ Range cta_range(const Plan &pl, int cta, int ncta, bool split) {
  Range r;
  locate(pl, range_start(pl, cta, ncta), r.u0, r.j0);
  locate(pl, range_start(pl, cta + 1, ncta), r.u1, r.j1);
  if (!split) {
    // whole units only: a unit belongs to the CTA whose range holds its first key
    if (r.j0 > 0) { ++r.u0; r.j0 = 0; }
    if (r.j1 > 0) { ++r.u1; r.j1 = 0; }
  }
  return r;
}

// One part of a chunk: keys [j0, j0 + len) of unit u at chunk rows [row0, row0 + len)
struct Part {
  int u, j0, len, row0;
  bool first, last;   // first / last part of this CTA's segment of unit u
};

__device__ __forceinline__ int unit_nk(const Plan &pl, const ReqCache &rc, int u) {
  const ReqInfo R = rc.get(pl, rc.find(pl, u));
  return R.be - R.bs + R.k;
}

// Walks a CTA's key stream in chunks of at most kTChunk keys and two parts.  Every
// role runs its own copy over the same range, so all agree on the chunk sequence.
struct Gen {
  Range rg;
  int u, j;
  int cu, cnk;   // key count of unit cu (cache)
  __device__ __forceinline__ explicit Gen(const Range &r) : rg(r), u(r.u0), j(r.j0), cu(-1), cnk(0) {}
  __device__ __forceinline__ bool done() const { return u > rg.u1 || (u == rg.u1 && j >= rg.j1); }
  __device__ __forceinline__ int endk(const Plan &pl, const ReqCache &rc, int uu) {
    if (uu == rg.u1) return rg.j1;
    if (uu != cu) {
      cu = uu;
      cnk = unit_nk(pl, rc, uu);
    }
    return cnk;
  }
  __device__ __forceinline__ bool next(const Plan &pl, const ReqCache &rc, Part &a, Part &b, bool &hb) {
    hb = false;
    if (done()) return false;
    int e = endk(pl, rc, u);
    a.u = u; a.j0 = j; a.row0 = 0;
    a.len = min(kTChunk, e - j);
    a.first = j == (u == rg.u0 ? rg.j0 : 0);
    a.last = j + a.len == e;
    j += a.len;
    if (a.last) {
      ++u;
      j = 0;
      if (a.len < kTChunk && !done()) {
        e = endk(pl, rc, u);
        b.u = u; b.j0 = 0; b.row0 = a.len;
        b.len = min(kTChunk - a.len, e);
        b.first = true;
        b.last = b.len == e;
        j = b.len;
        hb = true;
        if (b.last) { ++u; j = 0; }
      }
    }
    return true;
  }
};

__device__ __forceinline__ void cp_async_arrive_noinc(uint32_t bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void cp_async4(uint32_t dst, const void *src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(dst), "l"(src));
}
__device__ __forceinline__ int ld_acquire(const int32_t *p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int32_t *p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}

// byte offset of 16-byte piece c (of a 2*D-byte row) of row r in a SW128 K-major
// operand tile with `rows` rows: [D/64 atoms][rows][128 B], piece index XOR (r & 7)
__device__ __forceinline__ uint32_t sw128_off(int rows, int r, int c) {
  return (uint32_t)((c >> 3) * rows * 128 + r * 128 + (((c & 7) ^ (r & 7)) << 4));
}

// Warp transpose-reduction of 32 per-lane values x[0..31] (x[n] = this lane's value
// for row n): returns, in lane j, op over the 32 lanes of x[j].  Destroys x.
template <bool MAX>
__device__ __forceinline__ float transpose_reduce32(float (&x)[32], int lane) {
#pragma unroll
  for (int w = 16; w >= 1; w >>= 1) {
    const bool up = (lane & w) != 0;
#pragma unroll
    for (int i = 0; i < w; ++i) {
      const float send = up ? x[i] : x[i + w];
      const float keep = up ? x[i + w] : x[i];
      const float r = __shfl_xor_sync(0xffffffffu, send, w);
      x[i] = MAX ? fmaxf(keep, r) : keep + r;
    }
  }
  return x[0];
}

// The kernel body, shared by reuse_tc_kernel (one launch per Reuse batch) and the
// single-launch mixed Refresh/Reuse kernel (refresh_tc2.cu): CTA `cta` of `ncta`
// CTAs working on this plan.  ws_part / ws_flags: the caller's workspace (NULL: no
// unit is split).  Must be entered by every thread of the CTA before any of them
// reads global memory written by a preceding kernel (it executes griddepcontrol.wait).
__device__ __forceinline__ void reuse_tc_body(const Plan &plan, const __nv_bfloat16 *__restrict__ q_blk,
                                              const __nv_bfloat16 *__restrict__ k_cache,
                                              const __nv_bfloat16 *__restrict__ v_cache,
                                              const int32_t *__restrict__ idx, __nv_bfloat16 *__restrict__ out,
                                              float *__restrict__ ws_part, int32_t *__restrict__ ws_flags,
                                              const int cta, const int ncta) {
  constexpr int D = kTD;
  constexpr int CH = D / 8;    // 16-byte pieces per row
  constexpr int NS = kTNS;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t sb = (raw + 1023u) & ~1023u;
  uint8_t *gb = smem_raw + (sb - raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // barriers
  const uint32_t b_kvfull = sb + kOffBar;             // [NS] loaders (kLThreads noinc)
  const uint32_t b_kvempty = b_kvfull + 8 * NS;       // [NS] MMA commit
  const uint32_t b_ofull_t = b_kvempty + 8 * NS;      // [kTNT] translator (1)
  const uint32_t b_oempty_t = b_ofull_t + 8 * kTNT;   // [kTNT] loaders (kTLoaders)
  const uint32_t b_qfull = b_oempty_t + 8 * kTNT;     // [2] loaders (kLThreads noinc)
  const uint32_t b_qempty = b_qfull + 16;             // [2] MMA commit
  const uint32_t b_sfull = b_qempty + 16;             // [2] MMA commit
  const uint32_t b_sfree = b_sfull + 16;              // [2] softmax warps (4)
  const uint32_t b_pfull = b_sfree + 16;              // [2] softmax warps (4)
  const uint32_t b_pvdone = b_pfull + 16;             // [1] MMA commit after every chunk's P.V
  const uint32_t b_ofull = b_pvdone + 8;              // [2] MMA commit (segment's last P.V)
  const uint32_t b_ofree = b_ofull + 16;              // [2] epilogue warps (4): O^T and row sums consumed
  const uint32_t b_lfull = b_ofree + 16;              // [2] softmax warps (4): row sums / maxima written
  const uint32_t b_tslot = b_lfull + 16;              // TMEM base address slot

#ifdef DLLM_TRACE
  const long long t_start = rtc_timer();
#endif
  const bool split = ws_part != nullptr && ws_flags != nullptr;
  const Range rg = cta_range(plan, cta, ncta, split);
  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) {
      ptx::mbar_init(b_kvfull + 8 * i, kLThreads);
      ptx::mbar_init(b_kvempty + 8 * i, 1);
    }
    for (int i = 0; i < kTNT; ++i) {
      ptx::mbar_init(b_ofull_t + 8 * i, 1);
      ptx::mbar_init(b_oempty_t + 8 * i, kTLoaders);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(b_qfull + 8 * i, kLThreads);
      ptx::mbar_init(b_qempty + 8 * i, 1);
      ptx::mbar_init(b_sfull + 8 * i, 1);
      ptx::mbar_init(b_sfree + 8 * i, 4);
      ptx::mbar_init(b_pfull + 8 * i, 4);
      ptx::mbar_init(b_ofull + 8 * i, 1);
      ptx::mbar_init(b_ofree + 8 * i, 4);
      ptx::mbar_init(b_lfull + 8 * i, 4);
    }
    ptx::mbar_init(b_pvdone, 1);
    ptx::fence_mbar_init();
  }
  if (warp == kMmaWarp) {
    ptx::tmem_alloc(b_tslot, kTmemCols);
    ptx::tmem_relinquish();
  }
  {
    // zero the K/V ring once: rows a chunk does not fill keep finite data
    const uint4 z = make_uint4(0u, 0u, 0u, 0u);
    for (int i = threadIdx.x; i < NS * kStage / 16; i += kTThreads) reinterpret_cast<uint4 *>(gb)[i] = z;
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  // everything above is independent of the preceding kernel's results
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  asm volatile("griddepcontrol.wait;\n" ::: "memory");

  const int li = loader_index(warp);
  int32_t *pos_ring = reinterpret_cast<int32_t *>(gb + kOffPos);
  int32_t *bts = reinterpret_cast<int32_t *>(gb + kOffBt);
  const int ppr = plan.pages_per_req;
  int b_first = 0, b_last = -1;
  if (!rg.empty()) {
    b_first = plan_find(plan, rg.u0);
    b_last = plan_find(plan, rg.last_unit());
  }
  const int nbt = (b_last - b_first + 1) * ppr;
  const bool bt_smem = nbt <= kBtCap;
  ReqInfo *rq = reinterpret_cast<ReqInfo *>(gb + kOffReq);
  const int nrq = min(b_last - b_first + 1, kReqCache);
  {
    // this CTA's requests' metadata -> smem (4-byte words, all threads)
    constexpr int W = (int)(sizeof(ReqInfo) / 4);
    const int32_t *src = reinterpret_cast<const int32_t *>(&plan.r[b_first]);
    int32_t *dst = reinterpret_cast<int32_t *>(rq);
    for (int i = threadIdx.x; i < nrq * W; i += kTThreads) dst[i] = src[i];
  }

  // translator: the index lists of the first kLA chunks go out before anything else
  // (one memory round trip in parallel with the block-table rows below); one
  // cp.async group per chunk (empty past the end), so that cp.async.wait_group<kLA>
  // means "chunk t's positions have landed"
  // (before the barrier below the request cache is not yet visible: the prologue's
  // lookahead reads the parameter copy, n = 0)
  ReqCache RCs{rq, b_first, 0};
  Gen ga(rg);
  auto issue_idx = [&](int tt) {
    Part a, b;
    bool hb;
    if (!DLLM_RTC_IDXLDG && ga.next(plan, RCs, a, b, hb)) {
      const uint32_t dst = smem_u32(pos_ring + (tt % kNP) * kTChunk);
#pragma unroll
      for (int rr = 0; rr < kTChunk / 32; ++rr) {
        const int r = rr * 32 + lane;
        const bool inA = r < a.len, inB = !inA && hb && r < a.len + b.len;
        if (inA || inB) {
          const int uu = inA ? a.u : b.u;
          const ReqInfo R = RCs.get(plan, RCs.find(plan, uu));
          const int blk = R.be - R.bs;
          const int h = (uu - R.unit_off) / ((blk + kTRows - 1) / kTRows);
          const int j = inA ? a.j0 + r : r - a.len;
          if (j >= blk) cp_async4(dst + 4 * r, idx + R.idx_off + (int64_t)h * R.k + (j - blk));
        }
      }
      RTC_CHUNK(0, tt);
    }
    cp_async_commit();
  };
  if (warp == kTransWarp)
    for (int tt = 0; tt < kLA; ++tt) issue_idx(tt);
  // block-table rows of this CTA's requests (consecutive rows of the caller's table)
  if (bt_smem && nbt > 0) {
    const int32_t *bt0 = plan.block_table + (int64_t)plan.r[b_first].bt_row * ppr;
    for (int i = threadIdx.x; i < nbt; i += kTThreads) bts[i] = __ldg(bt0 + i);
  }
  __syncthreads();
  RCs.n = nrq;
  const ReqCache &rc = RCs;
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t *>(gb + (b_tslot - sb));

  // register split (64K per SM): loaders + MMA 80, softmax 200, epilogue 152
  if (warp < kSoft0) asm volatile("setmaxnreg.dec.sync.aligned.u32 80;\n" ::: "memory");
  if (warp == kTransWarp) {
    // ============================ translator ============================
    // position -> physical cache row for every key of every chunk: the index list
    // entry (staged kLA chunks ahead) or bs + j for block keys, the page id from the
    // staged block-table rows; -1 for rows past the chunk's keys
    const int P = plan.page_size, pshift = plan.page_shift, hkv = plan.H_kv;
    Gen gt(rg);
    TUnit ua, ub;
    int uau = -1, ubu = -1;
    for (int t = 0;; ++t) {
      Part a, b;
      bool hb;
      if (!gt.next(plan, rc, a, b, hb)) break;
      issue_idx(t + kLA);
      if (a.u != uau) {
        if (a.u == ubu) ua = ub; else tdecode(plan, rc, a.u, ua);
        uau = a.u;
      }
      if (hb && b.u != ubu) {
        tdecode(plan, rc, b.u, ub);
        ubu = b.u;
      }
      cp_async_wait<kLA>();   // chunk t's positions (this lane's); the warp barrier shares them
      __syncwarp();
      const int32_t *pos_s = pos_ring + (t % kNP) * kTChunk;
      int off[kTChunk / 32];
#pragma unroll
      for (int rr = 0; rr < kTChunk / 32; ++rr) {
        const int r = rr * 32 + lane;
        const bool inA = r < a.len, ok = inA || (hb && r < a.len + b.len);
        const int blk_ = inA ? ua.blk : ub.blk, bs_ = inA ? ua.bs : ub.bs, kvh_ = inA ? ua.kvh : ub.kvh;
        const int bt_ = bt_smem ? ((inA ? ua.b : ub.b) - b_first) * ppr : (inA ? ua.bt_row : ub.bt_row) * ppr;
        const int j = inA ? a.j0 + r : r - a.len;
#if DLLM_RTC_IDXLDG
        const int64_t io = inA ? ua.idx_off : ub.idx_off;
        const int pos = j < blk_ ? bs_ + j : (ok ? __ldg(idx + io + (j - blk_)) : 0);
#else
        const int pos = j < blk_ ? bs_ + j : pos_s[r];
#endif
        const int pi = bt_ + (pos >> pshift);
        const int page = ok ? (bt_smem ? bts[pi] : __ldg(plan.block_table + pi)) : 0;
        off[rr] = ok ? (page * hkv + kvh_) * P + (pos & (P - 1)) : -1;
      }
      const int slot = t % kTNT;
      ptx::mbar_wait(b_oempty_t + 8 * slot, ((t / kTNT) & 1) ^ 1);
      int32_t *offs = reinterpret_cast<int32_t *>(gb + kOffOffs) + slot * kTChunk;
#pragma unroll
      for (int rr = 0; rr < kTChunk / 32; ++rr) offs[rr * 32 + lane] = off[rr];
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(b_ofull_t + 8 * slot);
    }
    cp_async_wait<0>();
  } else if (li >= 0) {
    // ============================ loaders ============================
    const int64_t HD = (int64_t)plan.H * D;
    Gen gm(rg);
    for (int t = 0;; ++t) {
      Part a, b;
      bool hb;
      if (!gm.next(plan, rc, a, b, hb)) break;
      // Q rows of the segments that start in this chunk (SW128 K-major, zero rows past the block)
      for (int p = 0; p < (hb ? 2 : 1); ++p) {
        const Part &X = p ? b : a;
        if (!X.first) continue;
        TUnit U;
        tdecode(plan, rc, X.u, U);   // once per segment
        const int seg = X.u - rg.u0, qb = seg & 1;
        ptx::mbar_wait(b_qempty + 8 * qb, ((seg >> 1) & 1) ^ 1);
        const uint32_t sq = sb + kOffQ + qb * kQTile;
        const int row0 = U.rg * kTRows;
        for (int i = li * 32 + lane; i < kTRows * CH; i += kLThreads) {
          const int r = i / CH, c = i - r * CH;
          const bool ok = row0 + r < U.blk;
          const __nv_bfloat16 *src = q_blk + (int64_t)(U.blk_off + (ok ? row0 + r : 0)) * HD + (int64_t)U.h * D + c * 8;
          cp_async16(sq + sw128_off(kTRows, r, c), src, ok ? 16 : 0);
        }
        cp_async_arrive_noinc(b_qfull + 8 * qb);
      }
      const int s = t % NS, slot = t % kTNT;
      ptx::mbar_wait(b_ofull_t + 8 * slot, (t / kTNT) & 1);
      ptx::mbar_wait(b_kvempty + 8 * s, ((t / NS) & 1) ^ 1);
      const int32_t *offs = reinterpret_cast<const int32_t *>(gb + kOffOffs) + slot * kTChunk;
      const uint32_t dk = sb + s * kStage, dv = dk + kTileK;
#pragma unroll 4
      for (int e = li * 32 + lane; e < kTChunk * CH; e += kLThreads) {
        const int r = e >> 4, cc = e & 15;
        const int off = offs[r];
        if (off >= 0) {
          const int64_t goff = (int64_t)off * D + cc * 8;
          const uint32_t so = sw128_off(kTChunk, r, cc);
          cp_async16(dk + so, k_cache + goff, 16);
          cp_async16(dv + so, v_cache + goff, 16);
        }
      }
      cp_async_arrive_noinc(b_kvfull + 8 * s);
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(b_oempty_t + 8 * slot);
#ifdef DLLM_TRACE
      if (t == 0 && li == 0) RTC_CTA(1, rtc_timer());
#endif
      if (li == 0) RTC_CHUNK(1, t);
    }
    cp_async_wait<0>();
  } else if (warp == kMmaWarp) {
    // ============================ MMA issuer ============================
    constexpr uint32_t idesc_s = ptx::idesc_bf16_f32(128, kTRows, false, false);
    constexpr uint32_t idesc_o = ptx::idesc_bf16_f32(128, kTRows, true, true);
    const uint64_t dk0 = ptx::smem_desc_sw128(sb, 16, 1024);                 // K tile (K-major)
    const uint64_t dv0 = ptx::smem_desc_sw128(sb + kTileK, kTChunk * 128, 1024);   // V tile as MN-major A
    const uint64_t dq0 = ptx::smem_desc_sw128(sb + kOffQ, 16, 1024);
    // P^T MN-major SW64: one 32-row atom along N, 8-key groups 512 B apart along K
    const uint64_t dpm0 = ptx::smem_desc(sb, 64 * 8 * 2, 512, ptx::kSwizzle64B);
    Gen g(rg);
    // the previous chunk's P.V, deferred behind this chunk's S^T
    int pv_t = -1, pv_s = 0, pv_oa = 0, pv_ob = 0, pv_sega = 0, pv_segb = 0;
    bool pv_afirst = false, pv_alast = false, pv_hb = false, pv_blast = false;
    auto pv_ready = [&]() -> bool {
      if (!ptx::mbar_test_wait(b_pfull + 8 * (pv_t & 1), (pv_t >> 1) & 1)) return false;
      if (pv_afirst && !ptx::mbar_test_wait(b_ofree + 8 * pv_oa, ((pv_sega >> 1) & 1) ^ 1)) return false;
      if (pv_hb && !ptx::mbar_test_wait(b_ofree + 8 * pv_ob, ((pv_segb >> 1) & 1) ^ 1)) return false;
      return true;
    };
    auto issue_pv = [&]() {
      ptx::mbar_wait(b_pfull + 8 * (pv_t & 1), (pv_t >> 1) & 1);
      if (pv_afirst) ptx::mbar_wait(b_ofree + 8 * pv_oa, ((pv_sega >> 1) & 1) ^ 1);
      if (pv_hb) ptx::mbar_wait(b_ofree + 8 * pv_ob, ((pv_segb >> 1) & 1) ^ 1);
      ptx::tc_fence_after();
      const uint64_t a0 = dv0 + (uint64_t)((pv_s * kStage) >> 4);
      const uint64_t p0 = dpm0 + (uint64_t)((pv_s * kStage) >> 4);
#pragma unroll 1
      for (int k = 0; k < kTChunk / 16; ++k) {
        const uint32_t ao = (uint32_t)((k * 16 * 128) >> 4);
        const uint32_t bo = (uint32_t)((k * 16 * 64) >> 4);
        ptx::mma_ss_elect(tmem + tm_o(pv_oa), a0 + ao, p0 + bo, idesc_o, (!pv_afirst || k > 0) ? 1u : 0u);
      }
      if (pv_hb) {
        const uint64_t p1 = p0 + (uint64_t)(8192 >> 4);
#pragma unroll 1
        for (int k = 0; k < kTChunk / 16; ++k) {
          const uint32_t ao = (uint32_t)((k * 16 * 128) >> 4);
          const uint32_t bo = (uint32_t)((k * 16 * 64) >> 4);
          ptx::mma_ss_elect(tmem + tm_o(pv_ob), a0 + ao, p1 + bo, idesc_o, k > 0 ? 1u : 0u);
        }
      }
      ptx::mma_commit_elect(b_kvempty + 8 * pv_s);
      ptx::mma_commit_elect(b_pvdone);
      RTC_CHUNK(5, pv_t);
      if (pv_alast) ptx::mma_commit_elect(b_ofull + 8 * pv_oa);
      if (pv_hb && pv_blast) ptx::mma_commit_elect(b_ofull + 8 * pv_ob);
      pv_t = -1;
    };
    auto issue_s = [&](int sbuf, int part, int seg, int s) {
      const uint64_t a0 = dk0 + (uint64_t)((s * kStage) >> 4);
      const uint64_t b0 = dq0 + (uint64_t)(((seg & 1) * kQTile) >> 4);
#pragma unroll 1
      for (int k = 0; k < D / 16; ++k) {
        const uint32_t ao = (uint32_t)(((k >> 2) * kTChunk * 128 + (k & 3) * 32) >> 4);
        const uint32_t bo = (uint32_t)(((k >> 2) * kTRows * 128 + (k & 3) * 32) >> 4);
        ptx::mma_ss_elect(tmem + tm_s(sbuf, part), a0 + ao, b0 + bo, idesc_s, k > 0 ? 1u : 0u);
      }
    };
    for (int t = 0;; ++t) {
      Part a, b;
      bool hb;
      if (!g.next(plan, rc, a, b, hb)) break;
      const int s = t % NS, sbuf = t & 1;
      // P.V(t-1) goes out as soon as its P is ready, even when chunk t's K/V rows are
      // still in flight: its stage is released that much earlier
#ifdef DLLM_WATCHDOG
      uint32_t nwd = 0;
#endif
      while (!(ptx::mbar_test_wait(b_kvfull + 8 * s, (t / NS) & 1) &&
               ptx::mbar_test_wait(b_sfree + 8 * sbuf, ((t >> 1) & 1) ^ 1))) {
        if (pv_t >= 0 && pv_ready()) issue_pv();
#ifdef DLLM_WATCHDOG
        if (++nwd == (1u << 22) && lane == 0)
          printf("WATCHDOG MMA cta %d chunk %d: kvfull %d sfree %d pv_t %d (a.u %d j0 %d len %d hb %d)\n", cta, t,
                 (int)ptx::mbar_test_wait(b_kvfull + 8 * s, (t / NS) & 1),
                 (int)ptx::mbar_test_wait(b_sfree + 8 * sbuf, ((t >> 1) & 1) ^ 1), pv_t, a.u, a.j0, a.len, (int)hb);
#endif
      }
      ptx::fence_proxy_async_smem();   // cp.async (generic proxy) data -> tensor core (async proxy)
      ptx::tc_fence_after();
      const int sega = a.u - rg.u0;
      ptx::mbar_wait(b_qfull + 8 * (sega & 1), (sega >> 1) & 1);
      ptx::tc_fence_after();
      issue_s(sbuf, 0, sega, s);
      if (a.last) ptx::mma_commit_elect(b_qempty + 8 * (sega & 1));
      int segb = 0;
      if (hb) {
        segb = b.u - rg.u0;
        ptx::mbar_wait(b_qfull + 8 * (segb & 1), (segb >> 1) & 1);
        ptx::tc_fence_after();
        issue_s(sbuf, 1, segb, s);
        if (b.last) ptx::mma_commit_elect(b_qempty + 8 * (segb & 1));
      }
      ptx::mma_commit_elect(b_sfull + 8 * sbuf);
#ifdef DLLM_TRACE
      if (t == 0) RTC_CTA(2, rtc_timer());
#endif
      RTC_CHUNK(2, t);
      if (pv_t >= 0) issue_pv();
      pv_t = t; pv_s = s;
      pv_sega = sega; pv_oa = sega & 1; pv_afirst = a.first; pv_alast = a.last;
      pv_hb = hb; pv_segb = segb; pv_ob = segb & 1; pv_blast = hb && b.last;
    }
    if (pv_t >= 0) issue_pv();
  } else if (warp < kEpi0) {
    // ============================ softmax (warps 8-11) ============================
    // Thread = one key of the chunk (TMEM lane), 32 query rows (columns).  Every
    // thread keeps the segment's running row maxima m_run[0..31] (identical in all
    // 128 threads).  Common case: no key of the part exceeds its row's running max
    // by more than 2^8 (lazy rescale), decided with one 128-thread barrier-OR, and
    // the part costs one exp2 per score plus four 16-byte P^T stores.  Otherwise
    // the part's row maxima are exchanged and l / O^T are rescaled.
    asm volatile("setmaxnreg.inc.sync.aligned.u32 200;\n" ::: "memory");
    const int sw = warp & 3;   // TMEM lane quarter
    const float sl2 = plan.scale_log2;
    float *red = reinterpret_cast<float *>(gb + kOffRed);
    float *lbuf = reinterpret_cast<float *>(gb + kOffL);
    float *mbuf = reinterpret_cast<float *>(gb + kOffM);
    const uint32_t lane_base = (uint32_t)(sw * 32) << 16;
    const int kc = sw * 32 + lane;   // this thread's key row of the chunk
    float m_run[32], l_part[32];
    Gen g(rg);
    for (int t = 0;; ++t) {
      Part pa, pb;
      bool hb;
      if (!g.next(plan, rc, pa, pb, hb)) break;
      const int sbuf = t & 1;
      ptx::mbar_wait(b_sfull + 8 * sbuf, (t >> 1) & 1);
      ptx::tc_fence_after();
      if (sw == 0) RTC_CHUNK(3, t);
      for (int p = 0; p < (hb ? 2 : 1); ++p) {
        const Part &X = p ? pb : pa;
        const int seg = X.u - rg.u0, ob = seg & 1;
        if (X.first) {
#pragma unroll
          for (int n = 0; n < 32; ++n) { m_run[n] = -INFINITY; l_part[n] = 0.f; }
        }
        const bool valid = kc >= X.row0 && kc < X.row0 + X.len;
        float x[32];
        float dmax = -INFINITY;
        {
          uint32_t r[32];
          DLLM_TMEM_LD32(tmem + lane_base + tm_s(sbuf, p), r);
          ptx::tmem_wait_ld();
#pragma unroll
          for (int n = 0; n < 32; ++n) {
            x[n] = valid ? __uint_as_float(r[n]) * sl2 : -INFINITY;
            dmax = fmaxf(dmax, x[n] - m_run[n]);   // NaN (-inf - -inf) is ignored by fmaxf
          }
        }
        if (p == (hb ? 1 : 0)) {
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(b_sfree + 8 * sbuf);
        }
        const bool rare = ptx::bar_red_or(1, 128, dmax > 8.f);
        if (rare) {
          // part row maxima: warp transpose-reduction (lane j <- max of row j over the
          // warp's 32 keys), the four warps through shared memory, broadcast by shuffles
          float wmx;
          {
            float tmp[32];
#pragma unroll
            for (int n = 0; n < 32; ++n) tmp[n] = x[n];
            wmx = transpose_reduce32<true>(tmp, lane);
          }
          red[sw * 32 + lane] = wmx;
          ptx::named_bar_sync(1, 128);
          // (the next write of `red` happens after the next barrier-OR, i.e. after every
          // warp has read it here)
          const float mc = fmaxf(fmaxf(red[lane], red[32 + lane]), fmaxf(red[64 + lane], red[96 + lane]));
          if (X.first) {
            // a segment's first part: nothing accumulated yet, no rescale factors
#pragma unroll
            for (int n = 0; n < 32; ++n) m_run[n] = __shfl_sync(0xffffffffu, mc, n);
          } else {
            float alpha[32];
#pragma unroll
            for (int n = 0; n < 32; ++n) {
              const float mn = fmaxf(m_run[n], __shfl_sync(0xffffffffu, mc, n));
              alpha[n] = fast_exp2(m_run[n] - mn);
              m_run[n] = mn;
              l_part[n] *= alpha[n];
            }
            // O^T of this segment holds the chunks before t: wait for P.V(t-1), rescale
            ptx::mbar_wait(b_pvdone, (t - 1) & 1);
            ptx::tc_fence_after();
#pragma unroll
            for (int n4 = 0; n4 < 8; ++n4) {
              uint32_t o4[4];
              DLLM_TMEM_LD4(tmem + lane_base + tm_o(ob) + 4 * n4, o4);
              ptx::tmem_wait_ld();
#pragma unroll
              for (int e = 0; e < 4; ++e) o4[e] = __float_as_uint(__uint_as_float(o4[e]) * alpha[4 * n4 + e]);
              DLLM_TMEM_ST4(tmem + lane_base + tm_o(ob) + 4 * n4, o4);
            }
            ptx::tmem_wait_st();
            ptx::tc_fence_before();
          }
        }
        // P^T over the stage's K tile (part p at +8 KB p), MN-major SW64 operand: key
        // kc's 32 row values are one 64-byte row (4 pieces of 16 B), piece j stored at
        // j ^ ((kc >> 1) & 3); keys outside the part get p = 0
        uint8_t *prow = gb + (t % kTNS) * kStage + p * 8192 + kc * 64;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          uint32_t w4[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int n = 8 * j + 2 * q;
            const uint32_t pp = pack_bf16(fast_exp2(x[n] - m_run[n]), fast_exp2(x[n + 1] - m_run[n + 1]));
            l_part[n] += __uint_as_float(pp << 16);
            l_part[n + 1] += __uint_as_float(pp & 0xffff0000u);
            w4[q] = pp;
          }
          *reinterpret_cast<uint4 *>(prow + ((j ^ ((kc >> 1) & 3)) << 4)) = make_uint4(w4[0], w4[1], w4[2], w4[3]);
        }
        if (X.last) {
          // segment end: this warp's partial row sums and the running maxima -> smem
          float mv = m_run[0];
#pragma unroll
          for (int n = 1; n < 32; ++n) mv = lane == n ? m_run[n] : mv;
          const float wsum = transpose_reduce32<false>(l_part, lane);
          ptx::mbar_wait(b_ofree + 8 * ob, ((seg >> 1) & 1) ^ 1);   // segment seg-2's sums consumed
          lbuf[ob * 128 + sw * 32 + lane] = wsum;
          if (sw == 0) mbuf[ob * 32 + lane] = mv;
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(b_lfull + 8 * ob);
        }
      }
      ptx::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(b_pfull + 8 * sbuf);
      if (sw == 0) RTC_CHUNK(4, t);
    }
  } else {
    // ============================ epilogue (warps 12-15) ============================
    // O^T (thread = head-dim lane d, 32 row columns) / l -> bf16 rows in a staging
    // tile -> one 256-byte bulk (TMA) store per row; split units: partial write
    // (non-owner) or merge (owner).
    asm volatile("setmaxnreg.inc.sync.aligned.u32 152;\n" ::: "memory");
    const int ew = warp & 3;
    const int d = ew * 32 + lane;
    const uint32_t lane_base = (uint32_t)(ew * 32) << 16;
    const float *lbuf = reinterpret_cast<const float *>(gb + kOffL);
    const float *mbuf = reinterpret_cast<const float *>(gb + kOffM);
    const int last = rg.empty() ? rg.u0 - 1 : rg.last_unit();
    for (int u = rg.u0; u <= last; ++u) {
      const int seg = u - rg.u0, ob = seg & 1;
      TUnit U;
      tdecode(plan, rc, u, U);
      const bool nonowner = u == rg.u0 && rg.j0 > 0;
      const bool owner_split = !nonowner && u == rg.u1 && rg.j1 > 0;
      ptx::mbar_wait(b_lfull + 8 * ob, (seg >> 1) & 1);
      ptx::mbar_wait(b_ofull + 8 * ob, (seg >> 1) & 1);
      ptx::tc_fence_after();
      float lsum = lbuf[ob * 128 + lane] + lbuf[ob * 128 + 32 + lane] + lbuf[ob * 128 + 64 + lane] +
                   lbuf[ob * 128 + 96 + lane];   // row `lane`
      float mrow = mbuf[ob * 32 + lane];
      float o[32];
      {
        uint32_t r[32];
        DLLM_TMEM_LD32(tmem + lane_base + tm_o(ob), r);
        ptx::tmem_wait_ld();
#pragma unroll
        for (int n = 0; n < 32; ++n) o[n] = __uint_as_float(r[n]);
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(b_ofree + 8 * ob);
      if (nonowner) {
        // a piece of a unit owned by an earlier CTA: unnormalised O^T, m, l -> slot cta
        float *P = ws_part + (int64_t)cta * kPartFloats;
#pragma unroll
        for (int n4 = 0; n4 < 8; ++n4)
          __stcg(reinterpret_cast<float4 *>(P + d * kTRows) + n4,
                 make_float4(o[4 * n4], o[4 * n4 + 1], o[4 * n4 + 2], o[4 * n4 + 3]));
        if (ew == 0) {
          __stcg(P + kTD * kTRows + lane, mrow);
          __stcg(P + kTD * kTRows + kTRows + lane, lsum);
        }
        __threadfence();
        ptx::named_bar_sync(2, 128);
        if (d == 0) st_release(ws_flags + cta, 1);
        continue;
      }
      if (owner_split) {
        // merge the pieces of CTAs cta+1 .. cm (each wrote its slot at its start)
        const int cm = cta_of(plan, U.cost0 + U.nk - 1, ncta);
        for (int c2 = cta + 1; c2 <= cm; ++c2) {
          if (d == 0) {
#ifdef DLLM_WATCHDOG
            uint32_t n = 0;
#endif
            while (ld_acquire(ws_flags + c2) == 0) {
              __nanosleep(64);
#ifdef DLLM_WATCHDOG
              if (++n == (1u << 22)) {
                printf("WATCHDOG reuse cta %d waits for piece of cta %d (cm %d, ncta %d)\n", cta, c2, cm, ncta);
                __trap();
              }
#endif
            }
          }
          ptx::named_bar_sync(2, 128);
          const float *P = ws_part + (int64_t)c2 * kPartFloats;
          const float mj = __ldcg(P + kTD * kTRows + lane), lj = __ldcg(P + kTD * kTRows + kTRows + lane);
          const float mx = fmaxf(mrow, mj);
          const float ai = fast_exp2(mrow - mx), aj = fast_exp2(mj - mx);
          lsum = lsum * ai + lj * aj;
          mrow = mx;
#pragma unroll
          for (int n4 = 0; n4 < 8; ++n4) {
            const float4 v = __ldcg(reinterpret_cast<const float4 *>(P + d * kTRows) + n4);
            const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int n = 4 * n4 + e;
              o[n] = o[n] * __shfl_sync(0xffffffffu, ai, n) + vv[e] * __shfl_sync(0xffffffffu, aj, n);
            }
          }
          ptx::named_bar_sync(2, 128);
          if (d == 0) ws_flags[c2] = 0;   // consumed (the next launch on this workspace is stream-ordered)
        }
      }
      const float inv = lsum > 0.f ? __frcp_rn(lsum) : 0.f;   // row `lane`
      if (ew == 0) ptx::bulk_wait_group_read0();   // previous segment's rows left the staging tile
      ptx::named_bar_sync(2, 128);
      uint8_t *stg = gb + kOffStage + d * 2;
#pragma unroll
      for (int n = 0; n < 32; ++n)
        *reinterpret_cast<__nv_bfloat16 *>(stg + n * (D * 2)) =
            __float2bfloat16_rn(o[n] * __shfl_sync(0xffffffffu, inv, n));
      ptx::fence_proxy_async_smem();
      ptx::named_bar_sync(2, 128);
      const int row0 = U.rg * kTRows;
      const int nrows = min(kTRows, U.blk - row0);
      if (ew == 0 && lane < nrows) {
        ptx::bulk_s2g(out + ((int64_t)(U.blk_off + row0 + lane) * plan.H + U.h) * D, sb + kOffStage + lane * (D * 2),
                      D * 2);
        ptx::bulk_commit_group();
      }
#ifdef DLLM_TRACE
      if (ew == 0 && seg < 8) RTC_CTA(3 + seg, rtc_timer());
#endif
    }
    if (ew == 0) ptx::bulk_wait_group0();
#ifdef DLLM_TRACE
    if (ew == 0) {
      RTC_CTA(11, rtc_timer());
      RTC_CTA(0, t_start);
      uint32_t smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      RTC_CTA(12, (long long)smid);
    }
#endif
  }

  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (warp == kMmaWarp) ptx::tmem_dealloc(tmem, kTmemCols);
}

}  // namespace rtc
}  // namespace dllm
