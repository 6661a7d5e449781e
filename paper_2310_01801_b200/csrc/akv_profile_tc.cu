// tcgen05/TMA profiling passes (bf16, head dim 128) — placeholder until the
// tensor-core passes land; the SIMT passes in akv_profile.cu serve all shapes.
#include "akv_internal.h"

namespace akv {
bool tc_profile_supported(int N) { (void)N; return false; }
cudaError_t launch_tc_passes(const void*, const void*, const void*, int, int, int, int64_t,
                             const uint8_t*, int64_t, const float*, const float*, float*, double*,
                             double*, float*, float*, cudaStream_t) {
  return cudaErrorNotSupported;
}
}  // namespace akv
