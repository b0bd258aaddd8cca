// ABI plumbing: version, thread-local error string, device check.
#include <stdarg.h>
#include "common.cuh"

namespace sphkv {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

}  // namespace sphkv

extern "C" int sphkv_abi_version(void) { return SPHKV_ABI_VERSION; }

extern "C" const char* sphkv_last_error(void) { return sphkv::g_err; }

// 1 when the current device is an sm_100 part this library can run on.
extern "C" int sphkv_device_ok(void) {
  int dev = 0, major = 0, minor = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
  return (major == 10 && minor == 0) ? 1 : 0;
}
