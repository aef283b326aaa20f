// C-ABI plumbing shared by every entry point: error strings, device query.
#include "rg_common.cuh"

#include <string.h>

namespace rg {

static thread_local char g_err[512] = {0};

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

void clear_error() { g_err[0] = 0; }

int sm_count() {
  static int cached[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (cached[dev] == 0) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    cached[dev] = v > 0 ? v : 1;
  }
  return cached[dev];
}

}  // namespace rg

extern "C" const char* rg_version(void) { return "rgb200 0.1.0 sm_100a"; }

extern "C" const char* rg_last_error(void) { return rg::g_err; }

extern "C" int rg_device_sm_count(void) { return rg::sm_count(); }
