// ABI plumbing of libakv_sm100a.so: thread-local error strings, version,
// device check.
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "../../include/akv.h"
#include "akv_internal.h"

static thread_local char g_err[512] = "";

int set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

namespace akv {
static bool env_disable_tc() {
  const char* s = getenv("AKV_DISABLE_TC");
  return s && s[0] == '1';
}
bool g_disable_tc = env_disable_tc();
}  // namespace akv

extern "C" const char* akv_last_error(void) { return g_err; }

extern "C" const char* akv_version(void) { return "akv-sm100a 0.1.0"; }

extern "C" int akv_device_check(void) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return set_error(AKV_ERR_CUDA, "no CUDA device: %s", cudaGetErrorString(e));
  int major = 0, minor = 0;
  if ((e = cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev)) != cudaSuccess ||
      (e = cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev)) != cudaSuccess)
    return set_error(AKV_ERR_CUDA, "%s", cudaGetErrorString(e));
  if (major != 10 || minor != 0)
    return set_error(AKV_ERR_UNSUPPORTED, "device %d is sm_%d%d; this library is built for sm_100a",
                     dev, major, minor);
  return AKV_OK;
}

// ---------------------------------------------------------------------------
// TMA tensor-map encoding through the driver entry point (no -lcuda needed).
#include <cudaTypedefs.h>

#include "akv_tma.cuh"

namespace akv {
bool encode_tmap_2d_bf16(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols,
                         uint32_t box_cols, uint32_t box_rows, CUtensorMapSwizzle swizzle) {
  // resolved once per process (thread-safe static initialisation)
  static const PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  if (!fn) return false;
  cuuint64_t gdim[2] = {cols, rows};
  cuuint64_t gstride[1] = {cols * 2};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estride[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), gdim, gstride,
                  box, estride, CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}
}  // namespace akv

// Debug hook (not part of the ABI header): enable/disable the tensor-core
// paths at run time (tests cross-check them against the SIMT passes).
extern "C" void akv_debug_set_tc(int enable) { akv::g_disable_tc = !enable; }
