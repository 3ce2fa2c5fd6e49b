// Legacy tensor-path (mma.sync m16n8k16 bf16 -> HMMA) throughput on B200:
// FLOP/clk/SM with W warps per CTA, C CTAs per SM and A independent
// accumulator chains per warp.  Answers whether an mma.sync attention kernel
// is bounded by the legacy tensor pipe rather than by HBM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o hmma_rate hmma_rate.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

template <int A>
__global__ void hmma_loop(int iters, float* out) {
  float c[A][4];
#pragma unroll
  for (int a = 0; a < A; ++a)
#pragma unroll
    for (int i = 0; i < 4; ++i) c[a][i] = 0.0f;
  uint32_t x0 = threadIdx.x, x1 = x0 * 3, x2 = x0 * 5, x3 = x0 * 7, b0 = x0 * 11, b1 = x0 * 13;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int a = 0; a < A; ++a)
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
          "{%0,%1,%2,%3};"
          : "+f"(c[a][0]), "+f"(c[a][1]), "+f"(c[a][2]), "+f"(c[a][3])
          : "r"(x0), "r"(x1), "r"(x2), "r"(x3), "r"(b0), "r"(b1));
  }
  float s = 0.0f;
#pragma unroll
  for (int a = 0; a < A; ++a) s += c[a][0] + c[a][1] + c[a][2] + c[a][3];
  if (s == 12345.0f) out[threadIdx.x] = s;
}

template <int A>
void run(int warps, int ctas_per_sm, int sms) {
  float* out;
  cudaMalloc(&out, 4096);
  const int iters = 20000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  hmma_loop<A><<<sms * ctas_per_sm, warps * 32>>>(100, out);
  cudaEventRecord(e0);
  hmma_loop<A><<<sms * ctas_per_sm, warps * 32>>>(iters, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  int clk_khz;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  const double flops = 2.0 * 16 * 8 * 16 * (double)iters * A * warps * ctas_per_sm * sms;
  const double cycles = ms * 1e-3 * clk_khz * 1e3;
  printf("A=%d warps=%2d ctas/SM=%d: %.1f TFLOP/s, %.0f FLOP/clk/SM (at %d MHz nominal)\n", A, warps,
         ctas_per_sm, flops / ms / 1e9, flops / cycles / sms, clk_khz / 1000);
  cudaFree(out);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int w : {4, 8, 16}) {
    run<1>(w, 1, sms);
    run<2>(w, 1, sms);
    run<4>(w, 1, sms);
    run<8>(w, 1, sms);
  }
  run<4>(8, 2, sms);
  run<8>(8, 2, sms);
  return 0;
}
