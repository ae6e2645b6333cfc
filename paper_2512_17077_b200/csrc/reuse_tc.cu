// Reuse sparse attention on tcgen05 (Eq. 4; §4.5):
// the kernel launch around rtc::reuse_tc_body (reuse_tc_body.cuh, where the design
// is described).
#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>

#include "reuse_tc_body.cuh"

#ifdef DLLM_TRACE
extern "C" __attribute__((visibility("default"))) int dllm_trace_rtc_read(long long *cta, long long *chunk) {
  cudaError_t e = cudaMemcpyFromSymbol(cta, dllm::rtc::g_rtc, sizeof(dllm::rtc::g_rtc));
  if (e == cudaSuccess) e = cudaMemcpyFromSymbol(chunk, dllm::rtc::g_rtc_chunk, sizeof(dllm::rtc::g_rtc_chunk));
  return (int)e;
}
#endif

namespace dllm {
namespace {

using namespace rtc;

template <int DP>
__global__ void __launch_bounds__(kTThreads, 1)
reuse_tc_kernel(const __grid_constant__ Plan plan, const __nv_bfloat16 *__restrict__ q_blk,
                const __nv_bfloat16 *__restrict__ k_cache, const __nv_bfloat16 *__restrict__ v_cache,
                const int32_t *__restrict__ idx, __nv_bfloat16 *__restrict__ out) {
  // (griddepcontrol.wait inside the body, after the input-independent prologue)
  reuse_tc_body<DP>(plan, q_blk, k_cache, v_cache, idx, out, (int)blockIdx.x, (int)gridDim.x);
}

int num_sms_tc() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

}  // namespace

// D = 128 on the 128-dim layout; D = 16, 32, 64 on the 64-dim layout (zero-padded rows)
bool reuse_tc_supported(int D) { return D == 128 || D == 64 || D == 32 || D == 16; }

// CTAs for a Reuse plan: one per SM (persistent), at most one per unit
int reuse_tc_grid(const Plan &plan, int max_ctas) {
  // The fewest CTAs that keep the number of static rounds: every CTA gets the same
  // number of units (+-1), and the SMs a partial last round would leave idle are not
  // used at all -- fewer gathers in flight, shorter memory queues: C1 (512 units)
  // runs on 128 CTAs x 4 units in 29.7 us vs 148 CTAs (68 of them with a 4th unit)
  // in 31.7 us; C2 and C4 unchanged (profiles/r02_ab_reuse_balanced_grid.log)
  // (only when the partial last round is at least a quarter full: with a nearly empty
  // one, e.g. C2's 896 units = 6 rounds + 8, dropping 20 SMs from every round cost
  // 8% in a stream of launches, profiles/r02_ab_reuse_balanced_grid.log)
  const int rounds = (plan.total_units + max_ctas - 1) / max_ctas;
  if (rounds <= 0) return 0;
  const int tail = plan.total_units - (rounds - 1) * max_ctas;
  if (rounds > 1 && 4 * tail < max_ctas) return max_ctas;
  return (plan.total_units + rounds - 1) / rounds;
}

template <int DP>
cudaError_t launch_dp(const Plan &plan, const void *q_blk, const void *k_cache, const void *v_cache,
                      const int32_t *idx, void *out, cudaStream_t st) {
  static std::once_flag once;
  static cudaError_t attr = cudaSuccess;
  std::call_once(once, [] {
    attr = cudaFuncSetAttribute(reuse_tc_kernel<DP>, cudaFuncAttributeMaxDynamicSharedMemorySize, RL<DP>::kBytes);
  });
  if (attr != cudaSuccess) return attr;
  const int grid = reuse_tc_grid(plan, num_sms_tc());
  if (grid <= 0) return cudaSuccess;
  return launch_pdl(reuse_tc_kernel<DP>, dim3(grid), dim3(kTThreads), (size_t)RL<DP>::kBytes, st, plan,
                    (const __nv_bfloat16 *)q_blk, (const __nv_bfloat16 *)k_cache, (const __nv_bfloat16 *)v_cache, idx,
                    (__nv_bfloat16 *)out);
}

cudaError_t launch_reuse_tc(const Plan &plan, const void *q_blk, const void *k_cache, const void *v_cache,
                            const int32_t *idx, void *out, void *workspace, cudaStream_t st) {
  (void)workspace;
  if (!reuse_tc_supported(plan.D)) return cudaErrorInvalidValue;
  return plan.D == 128 ? launch_dp<128>(plan, q_blk, k_cache, v_cache, idx, out, st)
                       : launch_dp<64>(plan, q_blk, k_cache, v_cache, idx, out, st);
}

}  // namespace dllm
