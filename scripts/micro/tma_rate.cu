// TMA ingest-rate microbenchmark (B200): per-SM bytes/clk that a single
// producer thread sustains with SWIZZLE_128B 2D tile loads of R rows x 128 B
// into an S-stage ring, consumer releasing stages immediately.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tma_rate tma_rate.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c));
}
#ifndef SPIN
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred P;\nW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W;\n}" ::"r"(su32(b)), "r"(ph) : "memory");
}
#else
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred P;\nW: mbarrier.test_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W;\n}" ::"r"(su32(b)), "r"(ph) : "memory");
}
#endif
__device__ __forceinline__ void bar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void bar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* m, uint64_t* b, int x, int y) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
               ::"r"(su32(dst)), "l"((uint64_t)m), "r"(su32(b)), "r"(x), "r"(y) : "memory");
}

template <int R, int S, int NB>
__global__ void __launch_bounds__(64) ingest(const __grid_constant__ CUtensorMap tm, int rows_total, int kblocks,
                                             int iters, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t full[S], empty[S];
  constexpr uint32_t kBox = R * 128;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) { bar_init(&full[s], 1); bar_init(&empty[s], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const int mblocks = rows_total / R;
  long long t0 = clock64();
  if (threadIdx.x == 0) {
    int st = 0; uint32_t ph = 0;
    for (int it = 0; it < iters; ++it) {
      bar_wait(&empty[st], ph ^ 1);
      bar_expect(&full[st], NB * kBox);
      const int kb = it % kblocks;
      for (int j = 0; j < NB; ++j) {
        const int mb = (blockIdx.x * NB + j + it / kblocks) % mblocks;
        tma2d(sm + (st * NB + j) * kBox, &tm, &full[st], kb * 64, mb * R);
      }
      if (++st == S) { st = 0; ph ^= 1; }
    }
  } else if (threadIdx.x == 32) {
    int st = 0; uint32_t ph = 0;
    for (int it = 0; it < iters; ++it) {
      bar_wait(&full[st], ph);
      bar_arrive(&empty[st]);
      if (++st == S) { st = 0; ph ^= 1; }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) cycles[blockIdx.x] = clock64() - t0;
}

__device__ __forceinline__ void tma3d(void* dst, const CUtensorMap* m, uint64_t* b, int x, int y, int z) {
  asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
               ::"r"(su32(dst)), "l"((uint64_t)m), "r"(su32(b)), "r"(x), "r"(y), "r"(z) : "memory");
}

// 3D map (64-element k chunk, rows, k chunk index): one instruction moves
// R rows x KC*64 k (KC swizzled R x 128 B blocks back to back).
template <int R, int KC, int S>
__global__ void __launch_bounds__(64) ingest3(const __grid_constant__ CUtensorMap tm, int rows_total, int kchunks,
                                              int iters, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t full[S], empty[S];
  constexpr uint32_t kBox = R * 128 * KC;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) { bar_init(&full[s], 1); bar_init(&empty[s], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const int mblocks = rows_total / R;
  const int kblocks = kchunks / KC;
  long long t0 = clock64();
  if (threadIdx.x == 0) {
    int st = 0; uint32_t ph = 0;
    for (int it = 0; it < iters; ++it) {
      bar_wait(&empty[st], ph ^ 1);
      bar_expect(&full[st], kBox);
      const int kb = it % kblocks;
      const int mb = (blockIdx.x + it / kblocks) % mblocks;
      tma3d(sm + st * kBox, &tm, &full[st], 0, mb * R, kb * KC);
      if (++st == S) { st = 0; ph ^= 1; }
    }
  } else if (threadIdx.x == 32) {
    int st = 0; uint32_t ph = 0;
    for (int it = 0; it < iters; ++it) {
      bar_wait(&full[st], ph);
      bar_arrive(&empty[st]);
      if (++st == S) { st = 0; ph ^= 1; }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) cycles[blockIdx.x] = clock64() - t0;
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <int R, int S, int NB>
void run(EncFn enc, void* buf, int rows, int K, int grid, const char* tag) {
  CUtensorMap tm;
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  cuuint64_t str[1] = {(cuuint64_t)K * 2};
  cuuint32_t box[2] = {64, R};
  cuuint32_t es[2] = {1, 1};
  enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const size_t smem = 1024 + (size_t)S * NB * R * 128;
  cudaFuncSetAttribute(ingest<R, S, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  unsigned long long* cyc;
  cudaMalloc(&cyc, grid * 8);
  const int iters = 2000;
  ingest<R, S, NB><<<grid, 64, smem>>>(tm, rows, K / 64, 200, cyc);  // warm L2
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  ingest<R, S, NB><<<grid, 64, smem>>>(tm, rows, K / 64, iters, cyc);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  std::vector<unsigned long long> h(grid);
  cudaMemcpy(h.data(), cyc, grid * 8, cudaMemcpyDeviceToHost);
  double avg = 0; for (auto v : h) avg += v; avg /= grid;
  const double bytes = (double)iters * NB * R * 128;
  printf("%-28s R=%3d S=%2d NB=%d grid=%3d: %7.1f B/clk/SM  %6.2f TB/s chip  %6.0f clk/iter (%s)\n", tag, R, S, NB, grid,
         bytes / avg, bytes * grid / (ms * 1e-3) / 1e12, avg / iters, cudaGetErrorString(cudaGetLastError()));
  cudaFree(cyc);
}

template <int R, int KC, int S>
void run3(EncFn enc, void* buf, int rows, int K, int grid, const char* tag) {
  CUtensorMap tm;
  cuuint64_t dims[3] = {64, (cuuint64_t)rows, (cuuint64_t)K / 64};
  cuuint64_t str[2] = {(cuuint64_t)K * 2, 128};
  cuuint32_t box[3] = {64, R, KC};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("%s: encode failed %d\n", tag, (int)r); return; }
  const size_t smem = 1024 + (size_t)S * R * 128 * KC;
  cudaFuncSetAttribute(ingest3<R, KC, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  unsigned long long* cyc;
  cudaMalloc(&cyc, grid * 8);
  const int iters = 1000;
  ingest3<R, KC, S><<<grid, 64, smem>>>(tm, rows, K / 64, 100, cyc);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  ingest3<R, KC, S><<<grid, 64, smem>>>(tm, rows, K / 64, iters, cyc);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  std::vector<unsigned long long> h(grid);
  cudaMemcpy(h.data(), cyc, grid * 8, cudaMemcpyDeviceToHost);
  double avg = 0; for (auto v : h) avg += v; avg /= grid;
  const double bytes = (double)iters * R * 128 * KC;
  printf("%-28s R=%3d KC=%d S=%2d grid=%3d: %7.1f B/clk/SM  %6.2f TB/s chip  %6.0f clk/iter (%s)\n", tag, R, KC, S, grid,
         bytes / avg, bytes * grid / (ms * 1e-3) / 1e12, avg / iters, cudaGetErrorString(cudaGetLastError()));
  cudaFree(cyc);
}

int main() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  EncFn enc = (EncFn)fn;
  const int rows = 1280, K = 8960;
  void* buf;
  cudaMalloc(&buf, (size_t)rows * K * 2);
  cudaMemset(buf, 0, (size_t)rows * K * 2);
  for (int grid : {120, 148}) {
    run<64, 8, 1>(enc, buf, rows, K, grid, "box 64 rows");
    run<128, 8, 1>(enc, buf, rows, K, grid, "box 128 rows");
    run<256, 6, 1>(enc, buf, rows, K, grid, "box 256 rows");
    run<128, 12, 1>(enc, buf, rows, K, grid, "box 128 rows deep");
    run<64, 8, 2>(enc, buf, rows, K, grid, "2 x box 64");
    run<64, 8, 3>(enc, buf, rows, K, grid, "3 x box 64 (A128+B64)");
    run3<128, 1, 8>(enc, buf, rows, K, grid, "3d 128 rows x 64k");
    run3<128, 2, 6>(enc, buf, rows, K, grid, "3d 128 rows x 128k");
    run3<128, 4, 3>(enc, buf, rows, K, grid, "3d 128 rows x 256k");
    run3<64, 4, 6>(enc, buf, rows, K, grid, "3d 64 rows x 256k");
    run3<256, 2, 3>(enc, buf, rows, K, grid, "3d 256 rows x 128k");
  }
  return 0;
}
