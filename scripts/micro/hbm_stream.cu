// HBM streaming with one producer thread per CTA (148 CTAs): S stages of
// 2 x 16 KB, filled by cp.async.bulk (mode 0) or 2D TMA tensor boxes of
// 128 rows x 128 B (mode 1); consumer releases immediately.  Reports TB/s.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2511_16193_b200/csrc -o hbm_stream hbm_stream.cu -lcuda
#include <cuda.h>
#include <cstdio>
#include <cstdint>
#include "sm100.cuh"
using namespace sr::sm100;

template <int S, int MODE>
__global__ void __launch_bounds__(64) stream(const __grid_constant__ CUtensorMap tm, const uint8_t* base,
                                             long long nblocks, int iters) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t full[S], empty[S];
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int it = 0; it < iters; ++it) {
      const int s = it % S;
      mbar_wait(&empty[s], ((it / S) & 1) ^ 1);
      const long long blk = ((long long)it * gridDim.x + blockIdx.x) % nblocks;  // 32 KB blocks, interleaved
      mbar_arrive_expect_tx(&full[s], 32768);
      if (MODE == 0) {
        bulk_load(sm + s * 32768, base + blk * 32768, 16384, &full[s]);
        bulk_load(sm + s * 32768 + 16384, base + blk * 32768 + 16384, 16384, &full[s]);
      } else {
        tma_load_2d(sm + s * 32768, &tm, &full[s], 0, (int)(blk * 256), kEvictFirst);
        tma_load_2d(sm + s * 32768 + 16384, &tm, &full[s], 0, (int)(blk * 256 + 128), kEvictFirst);
      }
    }
  } else if (threadIdx.x == 32) {
    for (int it = 0; it < iters; ++it) {
      const int s = it % S;
      mbar_wait(&full[s], (it / S) & 1);
      mbar_arrive(&empty[s]);
    }
  }
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <int S, int MODE>
void run(const CUtensorMap& tm, uint8_t* buf, long long nblocks) {
  const size_t smem = 1024 + (size_t)S * 32768;
  cudaFuncSetAttribute(stream<S, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int iters = 400;
  stream<S, MODE><<<148, 64, smem>>>(tm, buf, nblocks, 50);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  stream<S, MODE><<<148, 64, smem>>>(tm, buf, nblocks, iters);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("mode %s S=%d: %.2f TB/s (%s)\n", MODE ? "tma2d" : "bulk ", S, 148.0 * iters * 32768 / (ms * 1e-3) / 1e12,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  const long long bytes = 4ll << 30;
  uint8_t* buf; cudaMalloc(&buf, bytes); cudaMemset(buf, 1, bytes);
  void* fn; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  CUtensorMap tm;
  cuuint64_t dims[2] = {64, (cuuint64_t)(bytes / 128)};
  cuuint64_t str[1] = {128};
  cuuint32_t box[2] = {64, 128};
  cuuint32_t es[2] = {1, 1};
  ((EncFn)fn)(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const long long nblocks = bytes / 32768;
  run<2, 0>(tm, buf, nblocks); run<3, 0>(tm, buf, nblocks); run<5, 0>(tm, buf, nblocks); run<6, 0>(tm, buf, nblocks);
  run<2, 1>(tm, buf, nblocks); run<3, 1>(tm, buf, nblocks); run<5, 1>(tm, buf, nblocks); run<6, 1>(tm, buf, nblocks);
  return 0;
}
