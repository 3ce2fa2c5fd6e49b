// Pins the tcgen05 operand layouts the tensor-core attention relies on:
//   S = Q K^T : A = Q [128 x 128] K-major SW128 (2 k-atoms), B = K [64 keys x 128] K-major
//   O = P V   : A = P [128 x 64 keys] K-major SW128,  B = V [64 keys x 128 hd] MN-major SW128
// stored like the bf16 KV cache: [hd atom][key][64 elems], 16-byte chunks ^ (key & 7).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I../../paper_2511_16193_b200/csrc -o umma_mn umma_mn.cu
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include "sm100.cuh"

using namespace sr::sm100;

__device__ uint64_t desc_mn(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)2u << 61;
  return d;
}

// element (r, c) of a [rows][cols] operand stored as [c/64][r][64] with chunk swizzle
__host__ __device__ int sw_off(int r, int c, int rows) {
  return ((c >> 6) * rows + r) * 64 + ((((c & 63) >> 3) ^ (r & 7)) << 3) + (c & 7);
}

__global__ void k_test(const __nv_bfloat16* Q, const __nv_bfloat16* K, const __nv_bfloat16* P,
                       const __nv_bfloat16* V, float* S_out, float* O_out, int variant) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  __nv_bfloat16* sQ = (__nv_bfloat16*)sm;               // 32 KB
  __nv_bfloat16* sK = (__nv_bfloat16*)(sm + 32768);     // 16 KB
  __nv_bfloat16* sP = (__nv_bfloat16*)(sm + 49152);     // 16 KB
  __nv_bfloat16* sV = (__nv_bfloat16*)(sm + 65536);     // 16 KB
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x;
  for (int e = tid; e < 128 * 128; e += blockDim.x) { int r = e / 128, c = e % 128; sQ[sw_off(r, c, 128)] = Q[e]; }
  for (int e = tid; e < 64 * 128; e += blockDim.x) { int r = e / 128, c = e % 128; sK[sw_off(r, c, 64)] = K[e]; }
  for (int e = tid; e < 128 * 64; e += blockDim.x) { int r = e / 64, c = e % 64; sP[sw_off(r, c, 128)] = P[e]; }
  // V[key][hd] stored [hd/64][key][64] (rows = keys)
  for (int e = tid; e < 64 * 128; e += blockDim.x) { int r = e / 128, c = e % 128; sV[sw_off(r, c, 64)] = V[e]; }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (tid < 32) tmem_alloc<256>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = slot;
  if (tid == 0) {
    const uint32_t q0 = smem_u32(sQ), k0 = smem_u32(sK), p0 = smem_u32(sP), v0 = smem_u32(sV);
    // S = Q K^T : M=128, N=64, K=128 (8 steps of 16)
    const uint32_t id_s = umma_idesc_bf16(128, 64);
    for (int j = 0; j < 8; ++j)
      umma_bf16(tm, umma_desc_sw128(q0 + (j >> 2) * 16384 + (j & 3) * 32),
                umma_desc_sw128(k0 + (j >> 2) * 8192 + (j & 3) * 32), id_s, j != 0);
    // O = P V : M=128, N=128, K=64 (4 steps of 16 keys); B MN-major
    const uint32_t id_o = umma_idesc_bf16(128, 128) | (1u << 16);
    for (int j = 0; j < 4; ++j) {
      uint64_t bd;
      const uint32_t addr = v0 + j * 2048;  // 16 keys = two 8-key groups of 1024 B
      if (variant == 0) bd = desc_mn(addr, 8192, 1024);   // LBO = MN atom stride, SBO = 8-key group stride
      else bd = desc_mn(addr, 1024, 8192);                // swapped
      umma_bf16(tm + 128, umma_desc_sw128(p0 + j * 32), bd, id_o, j != 0);
    }
    umma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  const int w = tid >> 5, lane = tid & 31, row = w * 32 + lane;
  for (int c = 0; c < 2; ++c) {
    uint32_t v[32];
    tmem_ld_32x32b_x32(tm + ((uint32_t)(w * 32) << 16) + c * 32, v);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int i = 0; i < 32; ++i) S_out[row * 64 + c * 32 + i] = __uint_as_float(v[i]);
  }
  for (int c = 0; c < 4; ++c) {
    uint32_t v[32];
    tmem_ld_32x32b_x32(tm + ((uint32_t)(w * 32) << 16) + 128 + c * 32, v);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int i = 0; i < 32; ++i) O_out[row * 128 + c * 32 + i] = __uint_as_float(v[i]);
  }
  tc_fence_before();
  __syncthreads();
  if (tid < 32) tmem_dealloc<256>(tm);
}

int main() {
  std::vector<__nv_bfloat16> Q(128 * 128), K(64 * 128), P(128 * 64), V(64 * 128);
  srand(1);
  auto rnd = [] { return (float)(rand() % 17 - 8) / 8.0f; };
  std::vector<float> q(128 * 128), k(64 * 128), p(128 * 64), v(64 * 128);
  for (int i = 0; i < 128 * 128; ++i) { q[i] = rnd(); Q[i] = __float2bfloat16(q[i]); }
  for (int i = 0; i < 64 * 128; ++i) { k[i] = rnd(); K[i] = __float2bfloat16(k[i]); }
  for (int i = 0; i < 128 * 64; ++i) { p[i] = rnd(); P[i] = __float2bfloat16(p[i]); }
  for (int i = 0; i < 64 * 128; ++i) { v[i] = rnd(); V[i] = __float2bfloat16(v[i]); }
  __nv_bfloat16 *dQ, *dK, *dP, *dV; float *dS, *dO;
  cudaMalloc(&dQ, Q.size() * 2); cudaMalloc(&dK, K.size() * 2); cudaMalloc(&dP, P.size() * 2); cudaMalloc(&dV, V.size() * 2);
  cudaMalloc(&dS, 128 * 64 * 4); cudaMalloc(&dO, 128 * 128 * 4);
  cudaMemcpy(dQ, Q.data(), Q.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dK, K.data(), K.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dP, P.data(), P.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dV, V.data(), V.size() * 2, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k_test, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
  for (int variant = 0; variant < 2; ++variant) {
    k_test<<<1, 128, 100000>>>(dQ, dK, dP, dV, dS, dO, variant);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> S(128 * 64), O(128 * 128);
    cudaMemcpy(S.data(), dS, S.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost);
    double es = 0, eo = 0;
    for (int r = 0; r < 128; ++r)
      for (int c = 0; c < 64; ++c) {
        double ref = 0; for (int d = 0; d < 128; ++d) ref += (double)q[r * 128 + d] * k[c * 128 + d];
        es = fmax(es, fabs(ref - S[r * 64 + c]));
      }
    for (int r = 0; r < 128; ++r)
      for (int c = 0; c < 128; ++c) {
        double ref = 0; for (int j = 0; j < 64; ++j) ref += (double)p[r * 64 + j] * v[j * 128 + c];
        eo = fmax(eo, fabs(ref - O[r * 128 + c]));
      }
    printf("variant %d (%s): max|S err| = %g  max|O err| = %g\n", variant, cudaGetErrorString(e), es, eo);
  }
  return 0;
}
