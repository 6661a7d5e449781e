// Internal (non-ABI) declarations shared by the libakv translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

// Records a thread-local error message (printf-style) and returns `code`.
int set_error(int code, const char* fmt, ...);

namespace akv {

// tcgen05/TMA profiling passes for bf16, head dim 128 (akv_profile_tc.cu).
bool tc_profile_supported(int N);
int tc_tiles(int N);  // 128-key tiles of the tensor-core passes (out_part rows per head)
cudaError_t launch_tc_passes(const void* q, const void* k, const void* v, int B, int H, int N,
                             int64_t ld, const uint8_t* cls, int64_t cls_ld, const float* slope,
                             const float* sink, float* lse, double* colsum, double* colsq,
                             float* lastp, float* out_part, cudaStream_t st);
// Set from the environment (AKV_DISABLE_TC=1) at load time: forces the SIMT
// passes, used by the tests to cross-check the two implementations.
extern bool g_disable_tc;

}  // namespace akv
