// K3, rejection-sampling mode (distribution-preserving speculative sampling
// for a STOCHASTIC drafter, Leviathan et al. 2023; semantic anchor vLLM 0.22
// v1/sample/rejection_sampler.py:708-760).  The reference only
// models acceptance as a keyed Bernoulli draw (sim.py:322-336); this is the
// model-mode rule for a drafter that samples its window from its own
// distribution q (ModelDrafter, acceptance="rejection"):
//
//   draft d_j ~ q_j is accepted iff u_j < p_j(d_j) / q_j(d_j)
//   at the first rejection j the committed token is drawn from
//   norm(max(0, p_j - q_j)); after a full accept the bonus (if on) is the
//   target's own keyed sample from p_n
//
// with p = softmax(target logits / T), q = softmax(drafter logits / T).  Every
// committed token is then distributed exactly as the target's sample, and a
// draft is accepted with probability sum_v min(p_v, q_v), the optimum over all
// couplings of p and q (the Gumbel-coupled exact-match mode reaches at most
// this).  Randomness is keyed by (seed, request, output position) on separate
// Philox streams (sampling.cuh tags), so a run is reproducible.
//
// Three kernels, HBM-bound over the logit rows they stream:
//   rs_stats:  one CTA per draft slot (j, b): log-sum-exp of p_j and q_j and
//              the draft's log-probabilities -- one pass over both rows
//   rs_sample: 16 CTAs per request, one vocabulary chunk each: acceptance
//              walk, then the chunk of p_a / q_a (residual) or p_n (bonus)
//              -> per-chunk keyed Gumbel-max partial
//   rs_commit: one CTA per request: the walk again, the partials in chunk
//              order, commit, outcome row.
#include "common.cuh"
#include "layers.cuh"
#include "sampling.cuh"

#include <cmath>

namespace sr {

namespace {

constexpr int kThreads = 256;

struct Lse {
  float m, s;
};

__device__ __forceinline__ Lse lse_merge(Lse a, Lse b) {
  const float m = fmaxf(a.m, b.m);
  if (m == -INFINITY) return {m, 0.0f};
  return {m, a.s * __expf(a.m - m) + b.s * __expf(b.m - m)};
}

__device__ __forceinline__ void lse_add(Lse& a, float x) {
  if (x > a.m) {
    a.s = a.s * __expf(a.m - x) + 1.0f;
    a.m = x;
  } else {
    a.s += __expf(x - a.m);
  }
}

template <typename T, typename F>
__device__ __forceinline__ T block_reduce(T v, F op, T* sh) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    T w;
    if constexpr (sizeof(T) == 8) {
      w.m = __shfl_xor_sync(0xffffffffu, v.m, o);
      w.s = __shfl_xor_sync(0xffffffffu, v.s, o);
    }
    v = op(v, w);
  }
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  if (wid == 0) {
    v = lane < (int)(blockDim.x >> 5) ? sh[lane] : T{-INFINITY, 0.0f};
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      T w;
      w.m = __shfl_xor_sync(0xffffffffu, v.m, o);
      w.s = __shfl_xor_sync(0xffffffffu, v.s, o);
      v = op(v, w);
    }
    if (lane == 0) sh[0] = v;
  }
  __syncthreads();
  return sh[0];
}

// (value, index) argmax, lowest index on ties.
struct Best {
  float v;
  int i;
};

__device__ __forceinline__ Best best_of(Best a, Best b) {
  return (b.v > a.v || (b.v == a.v && b.i < a.i)) ? b : a;
}

__device__ Best block_best(Best v, Best* sh) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    Best w{__shfl_xor_sync(0xffffffffu, v.v, o), __shfl_xor_sync(0xffffffffu, v.i, o)};
    v = best_of(v, w);
  }
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  if (wid == 0) {
    v = lane < (int)(blockDim.x >> 5) ? sh[lane] : Best{-INFINITY, 0x7fffffff};
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      Best w{__shfl_xor_sync(0xffffffffu, v.v, o), __shfl_xor_sync(0xffffffffu, v.i, o)};
      v = best_of(v, w);
    }
    if (lane == 0) sh[0] = v;
  }
  __syncthreads();
  return sh[0];
}

// stats[row] = (lse_p, lse_q, log p(d), log q(d)) for every draft slot j < n.
__global__ void __launch_bounds__(kThreads)
rs_stats_kernel(int B, const SeqInfo* __restrict__ seqs, const int32_t* __restrict__ token_ids,
                const float* __restrict__ p, int64_t ldp, const float* __restrict__ q, int64_t ldq, int V,
                float inv_t, float4* __restrict__ stats) {
  grid_dep_sync();
  const int j = blockIdx.x, b = blockIdx.y;
  const SeqInfo sq = seqs[b];
  if (j >= sq.q_len - 1) return;  // only slots that carry a draft
  const int row = sq.q_start + j;
  const float* pr = p + (int64_t)row * ldp;
  const float* qr = q + ((int64_t)j * B + b) * ldq;
  Lse lp{-INFINITY, 0.0f}, lq{-INFINITY, 0.0f};
  int v = threadIdx.x;
  const bool vec = ((ldp | ldq | V) & 3) == 0 && ((reinterpret_cast<uintptr_t>(pr) | reinterpret_cast<uintptr_t>(qr)) & 15) == 0;
  if (vec) {
    // 16-byte streaming loads, two per row in flight; one running-max
    // update per 4 values
    const float4* p4 = reinterpret_cast<const float4*>(pr);
    const float4* q4 = reinterpret_cast<const float4*>(qr);
    const int n4 = V / 4;
    auto add4 = [&](Lse& l, float4 x) {
      x.x *= inv_t; x.y *= inv_t; x.z *= inv_t; x.w *= inv_t;
      const float m4 = fmaxf(fmaxf(x.x, x.y), fmaxf(x.z, x.w));
      if (m4 > l.m) {
        l.s *= __expf(l.m - m4);
        l.m = m4;
      }
      l.s += (__expf(x.x - l.m) + __expf(x.y - l.m)) + (__expf(x.z - l.m) + __expf(x.w - l.m));
    };
    int i = threadIdx.x;
    for (; i + kThreads < n4; i += 2 * kThreads) {
      const float4 a0 = __ldcs(p4 + i), a1 = __ldcs(p4 + i + kThreads);
      const float4 c0 = __ldcs(q4 + i), c1 = __ldcs(q4 + i + kThreads);
      add4(lp, a0); add4(lp, a1);
      add4(lq, c0); add4(lq, c1);
    }
    for (; i < n4; i += kThreads) {
      add4(lp, __ldcs(p4 + i));
      add4(lq, __ldcs(q4 + i));
    }
    v = V;  // scalar loop below has nothing left
  }
  for (; v + 3 * kThreads < V; v += 4 * kThreads) {
    float a[4], c[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      a[u] = __ldg(pr + v + u * kThreads);
      c[u] = __ldg(qr + v + u * kThreads);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      lse_add(lp, a[u] * inv_t);
      lse_add(lq, c[u] * inv_t);
    }
  }
  for (; v < V; v += kThreads) {
    lse_add(lp, __ldg(pr + v) * inv_t);
    lse_add(lq, __ldg(qr + v) * inv_t);
  }
  __shared__ Lse sh[kThreads / 32];
  const Lse tp = block_reduce(lp, lse_merge, sh);
  const Lse tq = block_reduce(lq, lse_merge, sh);
  if (threadIdx.x == 0) {
    const int d = token_ids[row + 1];
    const float Lp = tp.m + __logf(tp.s), Lq = tq.m + __logf(tq.s);
    stats[row] = make_float4(Lp, Lq, pr[d] * inv_t - Lp, qr[d] * inv_t - Lq);
  }
}

// Vocabulary chunks per request for the extra-token pass (rs_sample_kernel).
constexpr int kChunks = 16;

// Acceptance walk shared by the sample and commit kernels: accepted prefix a,
// committed count and whether the extra token is a residual sample.
struct Walk {
  int a, committed, n;
  bool residual;
};

__device__ __forceinline__ Walk rs_walk(const SeqInfo& sq, const float4* __restrict__ stats, int remaining,
                                        uint32_t seed, int bonus) {
  Walk w;
  w.n = sq.q_len - 1;
  const int q0 = sq.q_start, pos0 = sq.ctx_len + 1;
  // u_j < p_j(d) / q_j(d)  (u < min(1, ratio) as u < 1)
  w.a = 0;
  while (w.a < w.n) {
    const float4 st = stats[q0 + w.a];
    const float u = keyed_uniform(seed, sq.request, pos0 + w.a, kTagAccept);
    if (!(u < __expf(st.z - st.w))) break;
    ++w.a;
  }
  if (w.n == 0) w.committed = 1;                   // empty window: a plain decode step
  else if (w.a == w.n) w.committed = w.n + (bonus ? 1 : 0);
  else w.committed = w.a + 1;
  w.committed = min(w.committed, remaining);
  w.residual = w.a < w.n;
  return w;
}

// One vocabulary chunk of the token after the accepted prefix: the residual
// norm(max(0, p - q)) at a rejection (keyed Gumbel-max over log r), the
// target's own keyed sample after a full accept / empty window.  Partial
// (value, index) per (request, chunk); the noise is keyed by 4-token block,
// so chunking does not change any candidate.
__global__ void __launch_bounds__(kThreads)
rs_sample_kernel(int B, const SeqInfo* __restrict__ seqs, const float* __restrict__ p, int64_t ldp,
                 const float* __restrict__ q, int64_t ldq, int V, float inv_t, uint32_t seed,
                 const float4* __restrict__ stats, const int32_t* __restrict__ gen_len,
                 const int32_t* __restrict__ max_new, int bonus, Best* __restrict__ partial) {
  grid_dep_sync();
  const int c = blockIdx.x, b = blockIdx.y;
  const SeqInfo sq = seqs[b];
  const int remaining = max_new[b] - gen_len[b];
  __shared__ Best shb[kThreads / 32];
  if (sq.q_len <= 0 || remaining <= 0) return;
  const Walk w = rs_walk(sq, stats, remaining, seed, bonus);
  if (w.committed <= w.a) return;
  const int row = sq.q_start + w.a, pos = sq.ctx_len + 1 + w.a;
  const float* pr = p + (int64_t)row * ldp;
  const float* qr = q + ((int64_t)w.a * B + b) * ldq;
  const int nblk = (V + 3) / 4;
  const int blk0 = (int)((int64_t)nblk * c / kChunks), blk1 = (int)((int64_t)nblk * (c + 1) / kChunks);
  Best best{-INFINITY, 0x7fffffff};
  if (w.residual) {
    const float4 st = stats[row];
    for (int blk = blk0 + threadIdx.x; blk < blk1; blk += kThreads) {
      float g[4];
      gumbel4_tag(seed, sq.request, pos, blk, kTagResidual, g);
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int v = 4 * blk + t;
        if (v >= V) break;
        const float r = __expf(pr[v] * inv_t - st.x) - __expf(qr[v] * inv_t - st.y);
        if (r > 0.0f) best = best_of(best, Best{__logf(r) + g[t], v});
      }
    }
  } else {
    for (int blk = blk0 + threadIdx.x; blk < blk1; blk += kThreads) {
      float g[4];
      gumbel4(seed, sq.request, pos, blk, g);
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int v = 4 * blk + t;
        if (v >= V) break;
        best = best_of(best, Best{pr[v] * inv_t + g[t], v});
      }
    }
  }
  best = block_best(best, shb);
  if (threadIdx.x == 0) partial[(int64_t)b * kChunks + c] = best;
}

__global__ void __launch_bounds__(kThreads)
rs_commit_kernel(int B, const SeqInfo* __restrict__ seqs, const int32_t* __restrict__ token_ids,
                 const float* __restrict__ p, int64_t ldp, int V, float inv_t, uint32_t seed,
                 const float4* __restrict__ stats, const Best* __restrict__ partial, int32_t* __restrict__ tokens,
                 int64_t tok_stride, int32_t* __restrict__ seq_len, int32_t* __restrict__ gen_len,
                 const int32_t* __restrict__ max_new, int bonus, int32_t* __restrict__ outcome,
                 int32_t* __restrict__ bon) {
  grid_dep_sync();
  const int b = blockIdx.x;
  const SeqInfo sq = seqs[b];
  const int remaining = max_new[b] - gen_len[b];
  int4* orow = reinterpret_cast<int4*>(outcome) + b;
  if (sq.q_len <= 0 || remaining <= 0) {
    if (threadIdx.x == 0) {
      *orow = make_int4(0, 0, 0, 0);
      bon[b] = -1;
    }
    return;
  }
  const Walk w = rs_walk(sq, stats, remaining, seed, bonus);
  const int a = w.a, n = w.n, committed = w.committed, q0 = sq.q_start;
  __shared__ Best shb[kThreads / 32];
  int extra = -1;
  if (committed > a) {
    // chunk partials in chunk order (the argmax with lowest-index ties does
    // not depend on the order anyway)
    Best best{-INFINITY, 0x7fffffff};
    for (int c = 0; c < kChunks; ++c) best = best_of(best, partial[(int64_t)b * kChunks + c]);
    if (best.v == -INFINITY) {
      // residual with p <= q everywhere (p == q up to rounding): the target's
      // own keyed sample, one CTA (rare)
      const int row = q0 + a, pos = sq.ctx_len + 1 + a;
      const float* pr = p + (int64_t)row * ldp;
      for (int blk = threadIdx.x; blk * 4 < V; blk += kThreads) {
        float g[4];
        gumbel4(seed, sq.request, pos, blk, g);
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const int v = 4 * blk + t;
          if (v >= V) break;
          best = best_of(best, Best{pr[v] * inv_t + g[t], v});
        }
      }
      best = block_best(best, shb);
    }
    extra = best.i;
  }
  if (threadIdx.x == 0) {
    const int base = seq_len[b];
    SR_DCHECK(base + committed <= tok_stride);
    int32_t* trow = tokens + (int64_t)b * tok_stride + base;
    const int keep = min(a, committed);
    for (int i = 0; i < keep; ++i) trow[i] = token_ids[q0 + 1 + i];
    if (committed > a) trow[a] = extra;
    *orow = make_int4(n, a, committed, a == n ? 0 : n - a - 1);
    bon[b] = 0;
    seq_len[b] = base + committed;
    gen_len[b] += committed;
  }
}

}  // namespace

}  // namespace sr

extern "C" int sr_accept_rejection(int num_requests, int k, const void* seqs, const int32_t* token_ids,
                                   const float* p_logits, int64_t ldp, const float* q_logits, int64_t ldq,
                                   int vocab, float temperature, uint32_t seed, int32_t* tokens,
                                   int64_t tok_stride, int32_t* seq_len, int32_t* gen_len, const int32_t* max_new,
                                   int bonus_token, float* stats, int32_t* outcome, int32_t* bon,
                                   sr_stream_t stream) {
  SR_REQUIRE(num_requests >= 0 && k >= 0 && vocab > 0 && ldp >= vocab && ldq >= vocab, "bad rejection shape");
  SR_REQUIRE(temperature > 0.0f, "rejection sampling needs temperature > 0");
  if (num_requests == 0) return SR_OK;
  SR_REQUIRE(seqs && token_ids && p_logits && (k == 0 || q_logits) && tokens && seq_len && gen_len && max_new &&
                 stats && outcome && bon,
             "null pointer");
  SR_REQUIRE((reinterpret_cast<uintptr_t>(outcome) & 15) == 0 && (reinterpret_cast<uintptr_t>(stats) & 15) == 0,
             "outcome / stats must be 16-byte aligned");
  const auto* sq = reinterpret_cast<const sr::SeqInfo*>(seqs);
  const float inv_t = 1.0f / temperature;
  cudaStream_t st = (cudaStream_t)stream;
  if (k > 0) {
    sr::launch_k(sr::rs_stats_kernel, dim3(k, num_requests), sr::kThreads, 0, st, num_requests, sq, token_ids,
                 p_logits, ldp, q_logits, ldq, vocab, inv_t, reinterpret_cast<float4*>(stats));
    const int rc = sr::check_launch("rs_stats_kernel");
    if (rc) return rc;
  }
  // chunk partials live behind the per-row stats in the same workspace
  auto* partial = reinterpret_cast<sr::Best*>(stats + (size_t)num_requests * (k + 1) * 4);
  sr::launch_k(sr::rs_sample_kernel, dim3(sr::kChunks, num_requests), sr::kThreads, 0, st, num_requests, sq,
               p_logits, ldp, q_logits, ldq, vocab, inv_t, seed, reinterpret_cast<const float4*>(stats), gen_len,
               max_new, bonus_token, partial);
  int rc = sr::check_launch("rs_sample_kernel");
  if (rc) return rc;
  sr::launch_k(sr::rs_commit_kernel, num_requests, sr::kThreads, 0, st, num_requests, sq, token_ids, p_logits, ldp,
               vocab, inv_t, seed, reinterpret_cast<const float4*>(stats), partial, tokens, tok_stride,
               seq_len, gen_len, max_new, bonus_token, outcome, bon);
  return sr::check_launch("rs_commit_kernel");
}

extern "C" uint64_t sr_accept_rejection_workspace_floats(int num_requests, int k) {
  if (num_requests <= 0 || k < 0) return 0;
  return (uint64_t)num_requests * (k + 1) * 4 + (uint64_t)num_requests * sr::kChunks * 2;
}
