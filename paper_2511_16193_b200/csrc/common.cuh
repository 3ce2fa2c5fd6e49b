// Shared plumbing for the C-ABI: status codes, thread-local error text,
// launch checking.  Every exported entry point returns SR_OK / SR_ERR_CONFIG /
// SR_ERR_RUNTIME (mirroring the reference CLI exit codes, cli.py:55-57) and
// never allocates or synchronizes; the caller owns buffers and the stream.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdarg>

#include "../../include/specrollout_b200.h"

namespace sr {

void set_error(const char* fmt, ...);
void count_launch();

inline int config_error(const char* what) {
  set_error("config: %s", what);
  return SR_ERR_CONFIG;
}

inline int check_launch(const char* kernel) {
  count_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", kernel, cudaGetErrorString(e));
    return SR_ERR_RUNTIME;
  }
  return SR_OK;
}

__host__ __device__ inline int ceil_div(int a, int b) { return (a + b - 1) / b; }

}  // namespace sr

#define SR_CHECK_CUDA(call)                                                   \
  do {                                                                        \
    cudaError_t e_ = (call);                                                  \
    if (e_ != cudaSuccess) {                                                  \
      sr::set_error("%s:%d %s: %s", __FILE__, __LINE__, #call,               \
                    cudaGetErrorString(e_));                                  \
      return SR_ERR_RUNTIME;                                                  \
    }                                                                         \
  } while (0)

#define SR_REQUIRE(cond, msg)                                                 \
  do {                                                                        \
    if (!(cond)) return sr::config_error(msg);                                \
  } while (0)
