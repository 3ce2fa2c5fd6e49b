// CTA-pair GEMM kernels of tile width 160 (gemm_dev.cuh).
#include "gemm_dev.cuh"

namespace sr {
int launch_pair_bn160(const GemmPlan& p, int M, cudaStream_t stream) { return launch_pair_bn<160>(p, M, stream); }
}  // namespace sr
