// Small-M GEMM kernels (one per epilogue; gemm_dev.cuh).
#include "gemm_dev.cuh"

namespace sr {
int launch_swap(const GemmPlan& p, int M, cudaStream_t stream) {
  switch (p.epi) {
    case kEpiStoreBf16: return launch_swap_typed<kEpiStoreBf16>(p, M, stream);
    case kEpiStoreF32: return launch_swap_typed<kEpiStoreF32>(p, M, stream);
    case kEpiResidualF32: return launch_swap_typed<kEpiResidualF32>(p, M, stream);
    case kEpiResidualNorm: return launch_swap_typed<kEpiResidualNorm>(p, M, stream);
    case kEpiQkvRope: return launch_swap_typed<kEpiQkvRope>(p, M, stream);
    case kEpiSwiGLU: return launch_swap_typed<kEpiSwiGLU>(p, M, stream);
  }
  return config_error("epilogue has no small-M mode");
}
}  // namespace sr
