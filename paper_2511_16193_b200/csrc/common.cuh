// Shared plumbing for the C-ABI: status codes, thread-local error text,
// launch checking.  Every exported entry point returns SR_OK / SR_ERR_CONFIG /
// SR_ERR_RUNTIME (mirroring the reference CLI exit codes, cli.py:55-57) and
// never allocates or synchronizes; the caller owns buffers and the stream.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdarg>
#include <utility>

#include "../../include/specrollout_b200.h"

// Debug build (SR_EXTRA_NVCC_FLAGS=-DSR_DEBUG_CHECKS python -m
// paper_2511_16193_b200.build): device-side bounds asserts on every index the
// hot path computes from device state (token rows, KV pages, branch slots).
// compute-sanitizer is not available on the GPU pool, so the test suite runs
// against this build instead (scripts/debug_checks.sh).
#ifdef SR_DEBUG_CHECKS
#include <cassert>
#define SR_DCHECK(cond) assert(cond)
#else
#define SR_DCHECK(cond) ((void)0)
#endif

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

// Programmatic dependent launch.  Every kernel is launched with
// programmatic stream serialization and begins (after any prologue that
// touches no predecessor output) with grid_dep_sync(): wait for the previous
// grid in the stream to complete and flush, then allow the next grid to be
// scheduled.  The next kernel's CTA launch and prologue thus overlap this
// kernel's body and tail instead of following its last CTA (within a CUDA
// graph as well as eagerly).  Every kernel waits before any global access,
// so ordering is transitive along the stream.  SR_PDL=0 disables it.
extern bool g_pdl;

__device__ __forceinline__ void grid_dep_sync() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

template <typename... KArgs, typename... Args>
inline void launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                     Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = g_pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);  // error surfaces in check_launch
}

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
