// The caller-owned device workspace (dllm_problem.workspace, include/dllm.h):
//   [0, 8)   int32 {claims, CTAs done}: the Refresh kernel's dynamic unit scheduler
//            (self-resetting: the last CTA of a launch zeroes both)
//   [8, 4096) reserved
// Zero-initialised once by the caller; every launch leaves it zeroed again.
#pragma once
#include <stdint.h>

namespace dllm {

constexpr int64_t kWsSchedOff = 0;
constexpr int64_t kWorkspaceBytes = 4096;

inline int32_t *workspace_sched(void *ws) {
  return ws ? reinterpret_cast<int32_t *>(static_cast<char *>(ws) + kWsSchedOff) : nullptr;
}

}  // namespace dllm
