// a9 / K4: n-gram (prompt-lookup) drafter over the device token buffer.
//
// Semantics (vLLM 0.22 NgramProposer, ngram_proposer.py:198-285, which the
// paper's n-gram drafter is built on; the reference only prices drafting,
// sim.py:883-892): among earlier occurrences of the context's suffix, take the
// longest match length n <= max_n, ties to the earliest occurrence; if
// n >= min_n propose up to k tokens that follow it.
//
// Formulation: for every end position e <= len-2, m(e) = length of the
// backward run where tokens[e-j] == tokens[len-1-j], capped at max_n and e+1.
// The best match maximizes m(e) and then minimizes e (a length-L match ending
// at e starts at e-L+1, so the smallest e is the earliest start) -- exactly
// the capped-KMP state vLLM tracks, computed data-parallel.
//
// HBM-bound design (4 B per context token): every thread streams 16-byte
// chunks (4 tokens) straight from HBM, eight chunks in flight, coalesced
// 512 B per warp-load, issued before the request's length is known (the row
// capacity bounds them).  Only an end position whose token equals the last
// context token can start a match, so each warp ballots that test over its
// 128 positions and skips the chunk when the ballot is empty (almost always,
// for natural or random text); the rare candidates extend their run backward
// from L1.  A CTA streams a 32768-position segment of one request in batches
// of 4096 with the next batch's loads in flight while it scans the current
// one (few registers, so 4 CTAs share an SM and cover each other's latency); a request that spans several segments reduces its best (m, ~e) key
// through a per-request atomicMax, and its last arriving CTA writes the
// proposal and re-zeroes the scratch.
#include "common.cuh"

namespace sr {

constexpr int kNgramThreads = 256;
constexpr int kNgramUnroll = 4;                                  // 16-byte chunks per thread per batch
constexpr int kNgramBatch = kNgramThreads * 4 * kNgramUnroll;    // 4096 positions per batch
constexpr int kNgramBatches = 8;
constexpr int kNgramSegment = kNgramBatch * kNgramBatches;       // 32768 end positions per CTA
constexpr int kMaxNgram = 16;

__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    unsigned long long x = __shfl_xor_sync(0xffffffffu, v, o);
    v = x > v ? x : v;
  }
  return v;
}

// Backward run length at end position e (e >= 0, tokens[e] == suf[0] known).
__device__ __forceinline__ int run_len(const int32_t* __restrict__ ctx, const int32_t* suf, int e, int max_n) {
  const int cap = min(max_n, e + 1);
  int m = 1;
  while (m < cap && __ldg(ctx + e - m) == suf[m]) ++m;
  return m;
}

// One batch of 4 chunks per thread: warp w, chunk u covers positions
// base + (u * 8 + w) * 128 + 4 * lane + [0, 4).  Loads stay inside the row
// (p + 3 < stride) and do not depend on the request's length, so they are
// issued before it arrives; positions past the last end are masked later.
template <bool VEC>
__device__ __forceinline__ void load_batch(const int32_t* __restrict__ ctx, int64_t stride, int base, int4 (&v)[kNgramUnroll]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int u = 0; u < kNgramUnroll; ++u) {
    const int p = base + (u * (kNgramThreads / 32) + warp) * 128 + 4 * lane;
    if (VEC && p + 3 < stride) {
      v[u] = __ldg(reinterpret_cast<const int4*>(ctx + p));
    } else {
      v[u].x = p < stride ? __ldg(ctx + p) : 0;
      v[u].y = p + 1 < stride ? __ldg(ctx + p + 1) : 0;
      v[u].z = p + 2 < stride ? __ldg(ctx + p + 2) : 0;
      v[u].w = p + 3 < stride ? __ldg(ctx + p + 3) : 0;
    }
  }
}

__device__ __forceinline__ void scan_batch(const int32_t* __restrict__ ctx, const int32_t* suf, int s0, int max_n,
                                           int last_end, int base, const int4 (&v)[kNgramUnroll],
                                           unsigned long long& best) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int u = 0; u < kNgramUnroll; ++u) {
    const int p = base + (u * (kNgramThreads / 32) + warp) * 128 + 4 * lane;
    unsigned hit = (v[u].x == s0 ? 1u : 0u) | (v[u].y == s0 ? 2u : 0u) | (v[u].z == s0 ? 4u : 0u) |
                   (v[u].w == s0 ? 8u : 0u);
    const int room = last_end - p + 1;  // end positions of this chunk that may match
    hit &= room >= 4 ? 0xFu : (room > 0 ? (1u << room) - 1u : 0u);
    // warp ballot: does any of the warp's 128 end positions start a match?
    if (__ballot_sync(0xffffffffu, hit != 0) == 0) continue;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (hit & (1u << q)) {
        const int e = p + q;
        const int m = run_len(ctx, suf, e, max_n);
        const unsigned long long key = ((unsigned long long)m << 32) | (0xFFFFFFFFu - (unsigned)e);
        best = key > best ? key : best;
      }
    }
  }
}

template <bool VEC>
__global__ void __launch_bounds__(kNgramThreads, 4)
ngram_kernel(const int32_t* __restrict__ tokens, int64_t stride, const int32_t* __restrict__ lens,
             int min_n, int max_n, int k, int32_t* __restrict__ out_draft,
             int32_t* __restrict__ out_nd, unsigned long long* __restrict__ keys,
             unsigned int* __restrict__ arrivals) {
  grid_dep_sync();
  const int b = blockIdx.y;
  const int32_t* ctx = tokens + (int64_t)b * stride;
  const int seg0 = blockIdx.x * kNgramSegment;
  const int seg_end = (int)((int64_t)seg0 + kNgramSegment < stride ? (int64_t)seg0 + kNgramSegment : stride);
  int4 va[kNgramUnroll], vb[kNgramUnroll];
  load_batch<VEC>(ctx, stride, seg0, va);            // in flight while the length and suffix arrive
  const int len = lens[b];
  __shared__ int32_t suf[kMaxNgram];
  __shared__ unsigned long long warp_best[kNgramThreads / 32];
  if ((int)threadIdx.x < max_n) suf[threadIdx.x] = (int)threadIdx.x < len ? ctx[len - 1 - threadIdx.x] : -1;
  __syncthreads();
  const int s0 = suf[0];
  const int last_end = len - 2;  // the match may not be the suffix itself
  unsigned long long best = 0;
  // two register batches in flight: load batch i+1, then scan batch i
#pragma unroll
  for (int i = 0; i < kNgramBatches; i += 2) {
    const int b0 = seg0 + i * kNgramBatch, b1 = b0 + kNgramBatch;
    if (b0 >= seg_end || b0 > last_end) break;
    if (b1 < seg_end && b1 <= last_end) load_batch<VEC>(ctx, stride, b1, vb);
    scan_batch(ctx, suf, s0, max_n, last_end, b0, va, best);
    if (b1 >= seg_end || b1 > last_end) break;
    const int b2 = b1 + kNgramBatch;
    if (i + 2 < kNgramBatches && b2 < seg_end && b2 <= last_end) load_batch<VEC>(ctx, stride, b2, va);
    scan_batch(ctx, suf, s0, max_n, last_end, b1, vb, best);
  }
  best = warp_max_u64(best);
  if ((threadIdx.x & 31) == 0) warp_best[threadIdx.x >> 5] = best;
  __syncthreads();
  __shared__ bool is_last;
  __shared__ unsigned long long blk_best;
  if (threadIdx.x == 0) {
    unsigned long long blk = 0;
    for (int i = 0; i < kNgramThreads / 32; ++i) blk = warp_best[i] > blk ? warp_best[i] : blk;
    if (gridDim.x == 1) {          // one CTA covers the request: no cross-CTA reduction
      is_last = true;
      blk_best = blk;
    } else {
      if (blk) atomicMax(&keys[b], blk);
      __threadfence();
      is_last = atomicAdd(&arrivals[b], 1u) == gridDim.x - 1;
      if (is_last) {
        __threadfence();
        blk_best = atomicAdd(&keys[b], 0ull);
        keys[b] = 0ull;
        arrivals[b] = 0u;
      }
    }
  }
  __syncthreads();
  if (!is_last) return;
  const unsigned long long key = blk_best;
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
  if (threadIdx.x == 0) out_nd[b] = nd;
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
  // segments sized by the row capacity (stride), so a graph captured once
  // covers every context length the token buffer can hold
  const int segs = (int)((stride + sr::kNgramSegment - 1) / sr::kNgramSegment);
  dim3 grid(segs, batch);
  auto* keys = reinterpret_cast<unsigned long long*>(scratch);
  auto* arrivals = reinterpret_cast<unsigned int*>(scratch + batch);
  const bool vec = stride % 4 == 0 && (reinterpret_cast<uintptr_t>(tokens) & 15) == 0;
  if (vec)
    sr::launch_k(sr::ngram_kernel<true>, grid, sr::kNgramThreads, 0, (cudaStream_t)stream, tokens, stride, lens,
                 min_n, max_n, k, out_draft, out_ndraft, keys, arrivals);
  else
    sr::launch_k(sr::ngram_kernel<false>, grid, sr::kNgramThreads, 0, (cudaStream_t)stream, tokens, stride, lens,
                 min_n, max_n, k, out_draft, out_ndraft, keys, arrivals);
  return sr::check_launch("ngram_kernel");
}

// ---------------------------------------------------------------------------
// Pooled prompt lookup (a fourth drafting method for Best-of-N, configs[4]):
// the request's suffix is matched against its own context (vLLM n-gram
// semantics above) AND every other request's committed tokens -- RL rollouts
// sample each prompt several times, so a group's samples share text.  The
// longest match length n in [min_n, max_n] wins; ties go to the own context,
// then to other requests in index order, then to the earliest end position;
// up to k tokens that follow the match in that row are proposed.  With one
// request it is exactly the n-gram drafter.
//
// One CTA per (row r, request b): stream row r, keep the best (n, rank, e)
// key, atomicMax it into the request's scratch; a second kernel emits the
// proposal and re-zeroes the scratch.  Rows stay hot in L2 across the B
// requests that scan them.
namespace sr {

__global__ void __launch_bounds__(kNgramThreads)
pooled_match_kernel(int B, const int32_t* __restrict__ tokens, int64_t stride, const int32_t* __restrict__ lens,
                    int min_n, int max_n, unsigned long long* __restrict__ keys) {
  grid_dep_sync();
  const int r = blockIdx.x, b = blockIdx.y;
  const int L = lens[b], Lr = lens[r];
  __shared__ int suf[kMaxNgram];
  __shared__ unsigned long long warp_best[kNgramThreads / 32];
  if (L < min_n) return;
  const int32_t* own = tokens + (int64_t)b * stride;
  const int32_t* row = tokens + (int64_t)r * stride;
  if ((int)threadIdx.x < max_n) suf[threadIdx.x] = threadIdx.x < L ? own[L - 1 - threadIdx.x] : -1;  // suf[j] = tokens[L-1-j]
  __syncthreads();
  const int rank = r == b ? 0 : (r < b ? r + 1 : r);  // own context first, then others in index order
  const int lim = (r == b ? L : Lr) - 2;               // a continuation token must follow the match
  const int last = suf[0];
  const int cap_own = L;                                // a match cannot use more suffix tokens than exist
  unsigned long long best = 0ull;
  for (int e = threadIdx.x; e <= lim; e += kNgramThreads) {
    if (row[e] != last) continue;
    int n = 1;
    const int mx = min(min(max_n, e + 1), cap_own);
    while (n < mx && row[e - n] == suf[n]) ++n;
    if (n < min_n) continue;
    const unsigned long long key = ((unsigned long long)n << 56) | ((unsigned long long)(0xFFFFu - rank) << 32) |
                                   (unsigned long long)(0xFFFFFFFFu - (unsigned)e);
    best = key > best ? key : best;
  }
  best = warp_max_u64(best);
  if ((threadIdx.x & 31) == 0) warp_best[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long blk = 0ull;
    for (int i = 0; i < kNgramThreads / 32; ++i) blk = warp_best[i] > blk ? warp_best[i] : blk;
    if (blk) atomicMax(&keys[b], blk);
  }
}

__global__ void pooled_emit_kernel(int B, const int32_t* __restrict__ tokens, int64_t stride,
                                   const int32_t* __restrict__ lens, int min_n, int k, int32_t* __restrict__ out_draft,
                                   int32_t* __restrict__ out_nd, unsigned long long* __restrict__ keys) {
  grid_dep_sync();
  const int b = blockIdx.x;
  const unsigned long long key = keys[b];
  const int L = lens[b];
  int nd = 0;
  const int n = (int)(key >> 56);
  if (key != 0ull && L >= min_n && n >= min_n) {
    const int rank = 0xFFFF - (int)((key >> 32) & 0xFFFFu);
    const int e = (int)(0xFFFFFFFFu - (unsigned)(key & 0xFFFFFFFFull));
    const int r = rank == 0 ? b : (rank <= b ? rank - 1 : rank);
    const int Lr = lens[r];
    const int start = e + 1;
    const int64_t room = stride - (int64_t)L, after = (int64_t)Lr - start;
    nd = (int)(room < after ? room : after);
    nd = max(min(k, nd), 0);
    if ((int)threadIdx.x < nd) out_draft[(int64_t)b * k + threadIdx.x] = tokens[(int64_t)r * stride + start + threadIdx.x];
  }
  __syncthreads();
  if ((int)threadIdx.x >= nd && (int)threadIdx.x < k) out_draft[(int64_t)b * k + threadIdx.x] = -1;
  if (threadIdx.x == 0) {
    out_nd[b] = nd;
    keys[b] = 0ull;  // ready for the next step
  }
}

}  // namespace sr

extern "C" int sr_pooled_ngram_propose(int batch, const int32_t* tokens, int64_t stride, const int32_t* lens,
                                       int min_n, int max_n, int k, int32_t* out_draft, int32_t* out_ndraft,
                                       int64_t* scratch, sr_stream_t stream) {
  SR_REQUIRE(batch >= 0, "negative batch");
  if (batch == 0) return SR_OK;
  SR_REQUIRE(min_n >= 1 && max_n >= min_n && max_n <= sr::kMaxNgram, "need 1 <= min_n <= max_n <= 16");
  SR_REQUIRE(k >= 1 && k <= sr::kNgramThreads, "k out of [1, 256]");
  SR_REQUIRE(stride >= 1 && stride < (int64_t)1 << 31, "stride out of range");
  SR_REQUIRE(tokens && lens && out_draft && out_ndraft && scratch, "null pointer");
  SR_REQUIRE(batch <= 65535, "batch exceeds the 16-bit row rank of the match key");
  auto* keys = reinterpret_cast<unsigned long long*>(scratch);
  cudaStream_t st = (cudaStream_t)stream;
  sr::launch_k(sr::pooled_match_kernel, dim3(batch, batch), sr::kNgramThreads, 0, st, batch, tokens, stride, lens,
               min_n, max_n, keys);
  int rc = sr::check_launch("pooled_match_kernel");
  if (rc) return rc;
  sr::launch_k(sr::pooled_emit_kernel, batch, k < 32 ? 32 : k, 0, st, batch, tokens, stride, lens, min_n, k,
               out_draft, out_ndraft, keys);
  return sr::check_launch("pooled_emit_kernel");
}
