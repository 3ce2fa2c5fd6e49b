// CTA-pair GEMM kernels of tile width 112 (gemm_dev.cuh).
#include "gemm_dev.cuh"

namespace sr {
int launch_pair_bn112(const GemmPlan& p, int M, cudaStream_t stream) { return launch_pair_bn<112>(p, M, stream); }
}  // namespace sr
