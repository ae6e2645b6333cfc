// Refresh on tcgen05/TMEM (placeholder until the kernel lands).
#include <cuda_runtime.h>
#include "plan.h"
namespace dllm {
bool refresh_tc_supported(int) { return false; }
int refresh_tc_units(int, int, int, int, bool) { return 0; }
cudaError_t launch_refresh_tc(const Plan &, const void *, const void *, const void *, void *, float *,
                              cudaStream_t) { return cudaErrorNotSupported; }
}  // namespace dllm
