// C-ABI plumbing: version, thread-local last error, device queries.
#include "common.cuh"

#include <cstring>

namespace sr {

static thread_local char g_last_error[1024] = {0};

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
  va_end(ap);
}

}  // namespace sr

extern "C" {

int sr_version(void) { return 100; }

const char* sr_last_error(void) { return sr::g_last_error; }

int sr_device_sm_count(void) {
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return -1;
  return sms;
}

}  // extern "C"
