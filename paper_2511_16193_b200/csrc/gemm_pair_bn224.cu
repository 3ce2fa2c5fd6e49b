// CTA-pair GEMM kernels of tile width 224 (gemm_dev.cuh).
#include "gemm_dev.cuh"

namespace sr {
int launch_pair_bn224(const GemmPlan& p, int M, cudaStream_t stream) { return launch_pair_bn<224>(p, M, stream); }
}  // namespace sr
