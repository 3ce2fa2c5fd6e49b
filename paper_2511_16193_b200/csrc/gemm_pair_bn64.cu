// CTA-pair GEMM kernels of tile width 64 (gemm_dev.cuh).
#include "gemm_dev.cuh"

namespace sr {
int launch_pair_bn64(const GemmPlan& p, int M, cudaStream_t stream) { return launch_pair_bn<64>(p, M, stream); }
}  // namespace sr
