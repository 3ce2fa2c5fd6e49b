// Keyed random streams, bit-identical to the reference's numpy streams.
//
// Reference contract (pkg/src/specrollout/streams.py:16-30): stream(seed, *keys)
// = np.random.default_rng(np.random.SeedSequence([seed, word(k)...])).  The
// hot-path draws are
//   target token  sim.py:313-320  stream(seed, rid, "tokens", pos//256)
//                                 .integers(0, 50257, 256)[pos % 256]
//   accept draw   sim.py:322-336  stream(seed, rid, "accept_draw", method,
//                                 pos//256).random(256)[pos % 256]
// so we restate numpy 2.x's SeedSequence entropy pool (pool size 4, the
// hashmix/mix constants), PCG64 (128-bit LCG, XSL-RR output, numpy seeding via
// generate_state(4, uint64)), next_double ((x >> 11) * 2^-53) and the bounded
// integer path for ranges < 2^32 (Lemire's multiply-shift with rejection over
// buffered 32-bit halves, low half first).  One thread owns one 256-draw chunk.
#pragma once
#include <cstdint>

namespace sr {

#if defined(__CUDACC__)
#define SR_HD __host__ __device__ __forceinline__
#else
#define SR_HD inline
#endif

typedef unsigned __int128 u128;

struct SeedSeqPool {
  uint32_t w[4];
};

constexpr uint32_t kInitA = 0x43b0d7e5u, kMultA = 0x931e8875u;
constexpr uint32_t kInitB = 0x8b51f9ddu, kMultB = 0x58f38dedu;
constexpr uint32_t kMixL = 0xca01f9ddu, kMixR = 0x4973f715u;

SR_HD uint32_t ss_hashmix(uint32_t v, uint32_t& h) {
  v ^= h;
  h *= kMultA;
  v *= h;
  v ^= v >> 16;
  return v;
}

SR_HD uint32_t ss_mix(uint32_t x, uint32_t y) {
  uint32_t r = kMixL * x - kMixR * y;
  return r ^ (r >> 16);
}

// Entropy words are already coerced to uint32 the numpy way (a 64-bit seed is
// 1 or 2 little-endian words, 0 -> one zero word; each key one word).
SR_HD SeedSeqPool ss_pool(const uint32_t* ent, int n) {
  SeedSeqPool p;
  uint32_t h = kInitA;
  for (int i = 0; i < 4; ++i) p.w[i] = ss_hashmix(i < n ? ent[i] : 0u, h);
  for (int s = 0; s < 4; ++s)
    for (int d = 0; d < 4; ++d)
      if (s != d) p.w[d] = ss_mix(p.w[d], ss_hashmix(p.w[s], h));
  for (int s = 4; s < n; ++s)
    for (int d = 0; d < 4; ++d) p.w[d] = ss_mix(p.w[d], ss_hashmix(ent[s], h));
  return p;
}

struct Pcg64 {
  u128 state, inc;
  bool has32;
  uint32_t spare;
};

SR_HD u128 pcg_mult() {
  return ((u128)0x2360ED051FC65DA4ull << 64) | (u128)0x4385DF649FCCF645ull;
}

SR_HD void pcg_step(Pcg64& g) { g.state = g.state * pcg_mult() + g.inc; }

SR_HD uint64_t pcg_next64(Pcg64& g) {
  pcg_step(g);
  uint64_t hi = (uint64_t)(g.state >> 64), lo = (uint64_t)g.state;
  uint64_t x = hi ^ lo;
  unsigned rot = (unsigned)(hi >> 58);
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

SR_HD uint32_t pcg_next32(Pcg64& g) {
  if (g.has32) {
    g.has32 = false;
    return g.spare;
  }
  uint64_t v = pcg_next64(g);
  g.has32 = true;
  g.spare = (uint32_t)(v >> 32);
  return (uint32_t)v;
}

// np.random.default_rng(SeedSequence(ent)): generate_state(4, uint64) then
// pcg64_set_seed(seed = s[0]:s[1], inc = s[2]:s[3]).
SR_HD Pcg64 pcg_from_entropy(const uint32_t* ent, int n) {
  SeedSeqPool p = ss_pool(ent, n);
  uint32_t st[8];
  uint32_t h = kInitB;
  for (int i = 0; i < 8; ++i) {
    uint32_t v = p.w[i & 3];
    v ^= h;
    h *= kMultB;
    v *= h;
    v ^= v >> 16;
    st[i] = v;
  }
  uint64_t s64[4];
  for (int i = 0; i < 4; ++i) s64[i] = (uint64_t)st[2 * i] | ((uint64_t)st[2 * i + 1] << 32);
  u128 seed = ((u128)s64[0] << 64) | (u128)s64[1];
  u128 initseq = ((u128)s64[2] << 64) | (u128)s64[3];
  Pcg64 g;
  g.state = 0;
  g.inc = (initseq << 1) | 1u;
  pcg_step(g);
  g.state += seed;
  pcg_step(g);
  g.has32 = false;
  g.spare = 0;
  return g;
}

SR_HD double pcg_next_double(Pcg64& g) {
  return (double)(pcg_next64(g) >> 11) * (1.0 / 9007199254740992.0);
}

// Generator.integers(0, high) for 1 <= high <= 2^32 (int64 dtype):
// rng = high - 1; buffered Lemire over next_uint32.
SR_HD uint32_t pcg_bounded(Pcg64& g, uint32_t rng) {
  if (rng == 0) return 0;
  if (rng == 0xFFFFFFFFu) return pcg_next32(g);
  const uint32_t excl = rng + 1u;
  uint64_t m = (uint64_t)pcg_next32(g) * excl;
  uint32_t left = (uint32_t)m;
  if (left < excl) {
    const uint32_t thresh = (0xFFFFFFFFu - rng) % excl;
    while (left < thresh) {
      m = (uint64_t)pcg_next32(g) * excl;
      left = (uint32_t)m;
    }
  }
  return (uint32_t)(m >> 32);
}

}  // namespace sr
