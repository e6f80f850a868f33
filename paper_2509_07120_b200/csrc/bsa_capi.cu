// bsa_capi.cu -- error state and small utilities of the C ABI (include/bsa.h).
#include <cstdarg>
#include <cstdio>

#include "bsa_common.cuh"

namespace bsa {

static thread_local char g_err[1024] = "";

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

}  // namespace bsa

extern "C" {

int bsa_version(void) { return 100; }

const char* bsa_last_error(void) { return bsa::g_err; }

int bsa_device_sm_count(void) {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return -1;
  return n;
}

}  // extern "C"
