// CTA-pair GEMM kernels of tile width 96 (gemm_dev.cuh).
#include "gemm_dev.cuh"

namespace sr {
int launch_pair_bn96(const GemmPlan& p, int M, cudaStream_t stream) { return launch_pair_bn<96>(p, M, stream); }
}  // namespace sr
