// a9 / K4: n-gram (prompt-lookup) drafter over the device token buffer.
//
// Semantics (vLLM 0.22 NgramProposer, ngram_proposer.py:198-285, which the
// paper's n-gram drafter is built on; the reference only prices drafting,
// sim.py:883-892): among earlier occurrences of the context's suffix, take the
// longest match length n <= max_n, ties to the earliest occurrence; if
// n >= min_n propose up to k tokens that follow it.
//
// Formulation used here: for every end position e <= len-2, m(e) = length of
// the backward run where tokens[e-j] == tokens[len-1-j], capped at max_n and
// e+1.  The best match maximizes m(e) and then minimizes e (a length-L match
// ending at e starts at e-L+1, so the smallest e is the earliest start).
// This is exactly the capped-KMP state vLLM tracks, computed data-parallel:
// each CTA stages a 4096-token tile (+max_n halo) in shared memory with
// vectorized coalesced loads, reduces a packed (m, ~e) key with warp
// shuffles, and folds it into a per-request atomicMax; the last CTA of a
// request (arrival counter) writes the proposal and resets the scratch.
#include "common.cuh"

namespace sr {

constexpr int kNgramThreads = 256;
constexpr int kNgramPerThread = 16;
constexpr int kNgramTile = kNgramThreads * kNgramPerThread;  // 4096 end positions
constexpr int kMaxNgram = 16;

__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    unsigned long long x = __shfl_xor_sync(0xffffffffu, v, o);
    v = x > v ? x : v;
  }
  return v;
}

__global__ void __launch_bounds__(kNgramThreads)
ngram_kernel(const int32_t* __restrict__ tokens, int64_t stride, const int32_t* __restrict__ lens,
             int min_n, int max_n, int k, int32_t* __restrict__ out_draft,
             int32_t* __restrict__ out_nd, unsigned long long* __restrict__ keys,
             unsigned int* __restrict__ arrivals) {
  grid_dep_sync();
  const int b = blockIdx.y;
  const int len = lens[b];
  const int32_t* ctx = tokens + (int64_t)b * stride;
  __shared__ int32_t suf[kMaxNgram];
  __shared__ int32_t tile[kMaxNgram + kNgramTile];
  __shared__ unsigned long long warp_best[kNgramThreads / 32];

  if ((int)threadIdx.x < max_n) suf[threadIdx.x] = threadIdx.x < len ? ctx[len - 1 - threadIdx.x] : -1;
  unsigned long long best = 0;
  const int last_end = len - 2;  // the match may not be the suffix itself
  for (int t0 = blockIdx.x * kNgramTile; t0 <= last_end; t0 += gridDim.x * kNgramTile) {
    __syncthreads();
    // halo [t0 - max_n, t0) then the tile [t0, t0 + kNgramTile)
    if ((int)threadIdx.x < max_n) {
      const int p = t0 - max_n + (int)threadIdx.x;
      tile[kMaxNgram - max_n + threadIdx.x] = p >= 0 ? ctx[p] : -1;
    }
    const int span = min(kNgramTile, last_end + 1 - t0);
    if ((((uintptr_t)(ctx + t0)) & 15) == 0) {
      const int4* src = reinterpret_cast<const int4*>(ctx + t0);
      const int vec = span >> 2;
      for (int v = threadIdx.x; v < vec; v += kNgramThreads) {
        int4 q = src[v];
        int* dst = &tile[kMaxNgram + v * 4];
        dst[0] = q.x; dst[1] = q.y; dst[2] = q.z; dst[3] = q.w;
      }
      for (int v = vec * 4 + threadIdx.x; v < span; v += kNgramThreads)
        tile[kMaxNgram + v] = ctx[t0 + v];
    } else {
      for (int v = threadIdx.x; v < span; v += kNgramThreads) tile[kMaxNgram + v] = ctx[t0 + v];
    }
    __syncthreads();
    for (int i = 0; i < kNgramPerThread; ++i) {
      const int off = i * kNgramThreads + threadIdx.x;
      if (off >= span) break;
      const int e = t0 + off;
      const int cap = min(max_n, e + 1);
      int m = 0;
      while (m < cap && tile[kMaxNgram + off - m] == suf[m]) ++m;
      if (m > 0) {
        unsigned long long key = ((unsigned long long)m << 32) | (0xFFFFFFFFu - (unsigned)e);
        best = key > best ? key : best;
      }
    }
  }
  best = warp_max_u64(best);
  if ((threadIdx.x & 31) == 0) warp_best[threadIdx.x >> 5] = best;
  __syncthreads();
  __shared__ bool is_last;
  if (threadIdx.x == 0) {
    unsigned long long blk = 0;
    for (int i = 0; i < kNgramThreads / 32; ++i) blk = warp_best[i] > blk ? warp_best[i] : blk;
    if (blk) atomicMax(&keys[b], blk);
    __threadfence();
    is_last = atomicAdd(&arrivals[b], 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  const unsigned long long key = atomicAdd(&keys[b], 0ull);
  const int L = (int)(key >> 32);
  const int e = (int)(0xFFFFFFFFu - (unsigned)(key & 0xFFFFFFFFull));
  int nd = 0;
  if (len >= min_n && L >= min_n && L > 0) {
    const int start = e + 1;  // tokens following the matched n-gram
    const int64_t room = stride - (int64_t)len, after = (int64_t)len - start;
    nd = (int)(room < after ? room : after);
    nd = min(k, nd);
    nd = max(nd, 0);
    if ((int)threadIdx.x < nd) out_draft[(int64_t)b * k + threadIdx.x] = ctx[start + threadIdx.x];
  }
  if ((int)threadIdx.x >= nd && (int)threadIdx.x < k) out_draft[(int64_t)b * k + threadIdx.x] = -1;
  if (threadIdx.x == 0) {
    out_nd[b] = nd;
    keys[b] = 0ull;
    arrivals[b] = 0u;
  }
}

}  // namespace sr

extern "C" int sr_ngram_propose(int batch, const int32_t* tokens, int64_t stride,
                                const int32_t* lens, int min_n, int max_n, int k,
                                int32_t* out_draft, int32_t* out_ndraft, int64_t* scratch,
                                sr_stream_t stream) {
  SR_REQUIRE(batch >= 0, "negative batch");
  if (batch == 0) return SR_OK;
  SR_REQUIRE(min_n >= 1 && max_n >= min_n && max_n <= sr::kMaxNgram,
             "need 1 <= min_n <= max_n <= 16");
  SR_REQUIRE(k >= 1 && k <= sr::kNgramThreads, "k out of [1, 256]");
  SR_REQUIRE(stride >= 1, "stride must be >= 1");
  SR_REQUIRE(tokens && lens && out_draft && out_ndraft && scratch, "null pointer");
  SR_REQUIRE(batch <= 65535, "batch exceeds grid.y limit");
  const int tiles = (int)((stride + sr::kNgramTile - 1) / sr::kNgramTile);
  dim3 grid(tiles < 8 ? tiles : 8, batch);
  auto* keys = reinterpret_cast<unsigned long long*>(scratch);
  auto* arrivals = reinterpret_cast<unsigned int*>(scratch + batch);
  sr::launch_k(sr::ngram_kernel, grid, sr::kNgramThreads, 0, (cudaStream_t)stream, 
      tokens, stride, lens, min_n, max_n, k, out_draft, out_ndraft, keys, arrivals);
  return sr::check_launch("ngram_kernel");
}
