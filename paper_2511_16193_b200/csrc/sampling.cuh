// Keyed sampling noise: the target model's token at temperature T is
//   argmax_v  logit[v] / T + G(seed, request, position, v),
// G = -log(-log(u)) with u from Philox4x32-10 keyed by (seed, request) and
// counted by (position, v / 4).  Because the draw is a pure function of the
// key, speculative verification and plain decoding sample the same token at
// every position (the reference's position-keyed draws, sim.py:313-336, and
// SURVEY §7 "exactness under T=1"); the CPU oracle restates the same stream.
#pragma once
#include <cstdint>

namespace sr {

struct SampleArgs {
  const int32_t* req;   // [rows] request id of each lm_head row (nullptr = greedy)
  const int32_t* pos;   // [rows] position of the token being generated
  uint32_t seed;
  float inv_temp;       // 1 / T; <= 0 means greedy argmax
};

__host__ __device__ __forceinline__ void philox4x32_10(uint32_t c[4], uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint64_t p0 = (uint64_t)0xD2511F53u * c[0];
    const uint64_t p1 = (uint64_t)0xCD9E8D57u * c[2];
    const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    c[0] = hi1 ^ c[1] ^ k0;
    c[1] = lo1;
    c[2] = hi0 ^ c[3] ^ k1;
    c[3] = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
}

// Stream tags (third Philox counter word): the target's sampling noise, and
// the rejection sampler's acceptance uniforms and residual noise.
constexpr uint32_t kTagSample = 0x53414D50u;    // "SAMP"
constexpr uint32_t kTagAccept = 0x41434350u;    // "ACCP"
constexpr uint32_t kTagResidual = 0x52455344u;  // "RESD"

// odd multiple of 2^-24: exactly representable, strictly inside (0, 1)
__host__ __device__ __forceinline__ float unit_open(uint32_t x) {
  return (float)(((x >> 9) << 1) | 1u) * 5.9604644775390625e-8f;
}

// Four Gumbel values for vocabulary ids [4*blk, 4*blk+4) at (req, pos).
__device__ __forceinline__ void gumbel4_tag(uint32_t seed, int req, int pos, int blk, uint32_t tag, float g[4]) {
  uint32_t c[4] = {(uint32_t)pos, (uint32_t)blk, tag, 0u};
  philox4x32_10(c, seed, (uint32_t)req);
#pragma unroll
  for (int i = 0; i < 4; ++i) g[i] = -logf(-logf(unit_open(c[i])));
}

__device__ __forceinline__ void gumbel4(uint32_t seed, int req, int pos, int blk, float g[4]) {
  gumbel4_tag(seed, req, pos, blk, kTagSample, g);
}

// One uniform in (0, 1) keyed by (seed, req, pos) on stream `tag`.
__host__ __device__ __forceinline__ float keyed_uniform(uint32_t seed, int req, int pos, uint32_t tag) {
  uint32_t c[4] = {(uint32_t)pos, 0u, tag, 0u};
  philox4x32_10(c, seed, (uint32_t)req);
  return unit_open(c[0]);
}

}  // namespace sr
