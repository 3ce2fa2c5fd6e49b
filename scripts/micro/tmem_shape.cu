// Maps tcgen05.ld.16x256b: which (TMEM lane, column) each thread/register gets.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I../../paper_2511_16193_b200/csrc -o tmem_shape tmem_shape.cu
#include <cstdio>
#include <cstdint>
#include "sm100.cuh"
using namespace sr::sm100;

__global__ void k(int* out) {
  __shared__ uint32_t slot;
  if (threadIdx.x < 32) tmem_alloc<64>(&slot);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tm = slot;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // fill: lane L (= 32w + lane), column c -> value L*1000 + c
  uint32_t v[32];
  for (int c = 0; c < 32; ++c) v[c] = (32 * w + lane) * 1000 + c;
  tmem_st_32x32b_x32(tm + ((uint32_t)(32 * w) << 16), v);
  tmem_st_wait();
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (w == 0) {
    uint32_t r[4];
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(tm));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int i = 0; i < 4; ++i) out[lane * 4 + i] = r[i];
    uint32_t q[8];
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(q[0]), "=r"(q[1]), "=r"(q[2]), "=r"(q[3]), "=r"(q[4]), "=r"(q[5]), "=r"(q[6]), "=r"(q[7])
                 : "r"(tm + 16u));  // column offset 16
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int i = 0; i < 8; ++i) out[128 + lane * 8 + i] = q[i];
    uint32_t h[2];
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(tm + (16u << 16)));  // lane base 16
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int i = 0; i < 4; ++i) out[384 + lane * 4 + i] = r[i];
    (void)h;
  }
  tc_fence_before(); __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc<64>(tm);
}

int main() {
  int* d; cudaMalloc(&d, 4096 * 4);
  k<<<1, 128>>>(d);
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  int h[4096]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("16x256b.x1 @ (lane 0, col 0): thread: (lane,col) of r0..r3\n");
  for (int t = 0; t < 32; ++t) {
    printf("t%2d:", t);
    for (int i = 0; i < 4; ++i) printf(" (%d,%d)", h[t * 4 + i] / 1000, h[t * 4 + i] % 1000);
    printf("\n");
  }
  printf("16x256b.x2 @ col 16:\n");
  for (int t = 0; t < 4; ++t) {
    printf("t%2d:", t);
    for (int i = 0; i < 8; ++i) printf(" (%d,%d)", h[128 + t * 8 + i] / 1000, h[128 + t * 8 + i] % 1000);
    printf("\n");
  }
  printf("16x256b.x1 @ lane 16: t0: (%d,%d) t31: (%d,%d)\n", h[384] / 1000, h[384] % 1000, h[384 + 31 * 4 + 3] / 1000, h[384 + 31 * 4 + 3] % 1000);
  return 0;
}
