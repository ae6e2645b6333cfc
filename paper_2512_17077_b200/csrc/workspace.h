// The caller-owned device workspace (dllm_problem.workspace, include/dllm.h):
//   [0, 1024)      int32 flags[kMaxCtas]: Reuse split-unit pieces published (1) / consumed (0)
//   [1024, 2048)   int32 scheduler counters (Refresh dynamic unit claims, self-resetting)
//   [4096, ...)    float partials[kMaxCtas][kPartFloats]: unnormalised O^T, m, l of a piece
// Zero-initialised once by the caller; every launch leaves it zeroed again.
#pragma once
#include <stdint.h>

#include "reuse_tc_body.cuh"

namespace dllm {

constexpr int64_t kWsFlagsOff = 0, kWsSchedOff = 1024, kWsPartOff = 4096;
constexpr int64_t kWorkspaceBytes = kWsPartOff + (int64_t)rtc::kMaxCtas * rtc::kPartFloats * 4;

inline void workspace_split(void *ws, float *&part, int32_t *&flags) {
  if (!ws) {
    part = nullptr;
    flags = nullptr;
    return;
  }
  flags = reinterpret_cast<int32_t *>(static_cast<char *>(ws) + kWsFlagsOff);
  part = reinterpret_cast<float *>(static_cast<char *>(ws) + kWsPartOff);
}
inline int32_t *workspace_sched(void *ws) {
  return ws ? reinterpret_cast<int32_t *>(static_cast<char *>(ws) + kWsSchedOff) : nullptr;
}

}  // namespace dllm
