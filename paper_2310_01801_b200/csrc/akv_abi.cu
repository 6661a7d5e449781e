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
  cudaDeviceProp prop;
  e = cudaGetDeviceProperties(&prop, dev);
  if (e != cudaSuccess) return set_error(AKV_ERR_CUDA, "%s", cudaGetErrorString(e));
  if (prop.major != 10 || prop.minor != 0)
    return set_error(AKV_ERR_UNSUPPORTED, "device %s is sm_%d%d; this library is built for sm_100a",
                     prop.name, prop.major, prop.minor);
  return AKV_OK;
}
