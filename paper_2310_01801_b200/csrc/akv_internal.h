// Internal (non-ABI) declarations shared by the libakv translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <mutex>

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

// One-time, per-device launch set-up (function attributes such as the
// dynamic shared-memory opt-in are per device context): run(fn) calls
// fn(device) once per device for this object, thread-safe; a failed
// fn is retried by the next call.
constexpr int kMaxDevices = 64;
struct PerDeviceOnce {
  std::mutex mu;
  std::atomic<bool> done[kMaxDevices] = {};
  template <typename F>
  cudaError_t run(F fn) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= kMaxDevices) return cudaErrorInvalidDevice;
    if (done[dev].load(std::memory_order_acquire)) return cudaSuccess;
    std::lock_guard<std::mutex> lock(mu);
    if (done[dev].load(std::memory_order_relaxed)) return cudaSuccess;
    if ((e = fn(dev)) == cudaSuccess) done[dev].store(true, std::memory_order_release);
    return e;
  }
};

// SM count of the current device (cached per device).
cudaError_t current_sm_count(int* out);

}  // namespace akv
