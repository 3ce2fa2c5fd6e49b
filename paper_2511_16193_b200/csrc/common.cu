// C-ABI plumbing: version, thread-local last error, device queries.
#include "common.cuh"

#include <atomic>
#include <cstdlib>
#include <cstring>

namespace sr {

static thread_local char g_last_error[1024] = {0};
static std::atomic<long long> g_launches{0};

static bool pdl_from_env() {
  const char* v = getenv("SR_PDL");
  return !(v && v[0] == '0');
}
bool g_pdl = pdl_from_env();

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
  va_end(ap);
}

}  // namespace sr

extern "C" {

int sr_version(void) { return 100; }

long long sr_launch_count(void) { return sr::g_launches.load(); }

const char* sr_last_error(void) { return sr::g_last_error; }

int sr_abi_sizes(int64_t* out, int n) {
  const int64_t sizes[3] = {(int64_t)sizeof(sr_model_desc), (int64_t)sizeof(sr_forward_args),
                            (int64_t)sizeof(sr_seq_info)};
  for (int i = 0; i < n && i < 3; ++i) out[i] = sizes[i];
  return SR_OK;
}

int sr_device_sm_count(void) {
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return -1;
  return sms;
}

}  // extern "C"
