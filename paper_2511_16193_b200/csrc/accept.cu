// K3: acceptance + Best-of-N select + token/KV write-back (model mode), and
// the device-side builder of the next verify batch.
//
// Reference semantics (exact match, sim.py:983-1042): with n drafted tokens
// d_1..d_n verified by target predictions y_0..y_n, the accepted prefix a is
// the number of leading j with d_{j+1} == y_j; a full accept commits n tokens
// (+ y_n when the bonus token is on, sim.py:996-999), a partial accept commits
// the a accepted tokens plus the corrected token y_a (sim.py:1001-1009); n = 0
// is a plain decode step that commits y_0 (sim.py:966-975).  With N drafters
// per prompt (Best-of-N, bon.py:79-139 / sim.py:340-361 first finisher) the
// drafter with the longest accepted prefix wins, ties to the lowest index
// (incumbent first).  Everything stays on device: the host
// reads back only the [B*N, 4] outcome rows.
#include "common.cuh"
#include "layers.cuh"

#include <cuda_bf16.h>

namespace sr {

int model_kv_layout(void* handle, KvLayout* kv, int* dtype);  // model.cu

namespace {

// K3, fused: one CTA per request.  Warp 0 finds every drafter's accepted
// prefix (lane n = drafter n), picks the Best-of-N winner, commits its tokens
// and writes the outcome rows; then, when the winner verified in a drafter
// branch (its window KV sits in the branch buffer, not in the paged cache),
// the whole CTA copies the committed slots' K and V of every layer into the
// cache with 16-byte vector moves (swizzled chunk -> swizzled chunk).
template <typename T>
__global__ void __launch_bounds__(128)
accept_commit_kernel(int B, int N, const SeqInfo* __restrict__ seqs, const int32_t* __restrict__ token_ids,
                     const int32_t* __restrict__ target, int32_t* __restrict__ tokens, int64_t tok_stride,
                     int32_t* __restrict__ seq_len, int32_t* __restrict__ gen_len,
                     const int32_t* __restrict__ max_new, int bonus, int32_t* __restrict__ outcome,
                     int32_t* __restrict__ bon, KvLayout kv) {
  grid_dep_sync();
  const int b = blockIdx.x;
  const int lane = threadIdx.x & 31;
  __shared__ int s_branch, s_ctx, s_req, s_committed;
  if (threadIdx.x < 32) {
    const int remaining = max_new[b] - gen_len[b];
    // per-drafter accepted prefix (lane n handles drafter n)
    int a = -1, n = 0, qs = 0, branch = -1, ctx = 0, req = b;
    if (lane < N) {
      const SeqInfo sq = seqs[b * N + lane];
      branch = sq.branch;
      ctx = sq.ctx_len;
      req = sq.request;
      if (sq.q_len > 0 && remaining > 0) {
        n = sq.q_len - 1;
        qs = sq.q_start;
        a = 0;
        while (a < n && token_ids[qs + a + 1] == target[qs + a]) ++a;
      }
    }
    // longest accepted prefix, lowest drafter index on ties
    int best_a = a, best_n = lane < N ? lane : 0x7fffffff;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const int oa = __shfl_xor_sync(0xffffffffu, best_a, o);
      const int on = __shfl_xor_sync(0xffffffffu, best_n, o);
      if (oa > best_a || (oa == best_a && on < best_n)) { best_a = oa; best_n = on; }
    }
    const int win_n = best_n & 31;
    const int win_q = __shfl_sync(0xffffffffu, qs, win_n);
    const int win_len = __shfl_sync(0xffffffffu, n, win_n);
    const int win_branch = __shfl_sync(0xffffffffu, branch, win_n);
    const int win_ctx = __shfl_sync(0xffffffffu, ctx, win_n);
    const int win_req = __shfl_sync(0xffffffffu, req, win_n);
    int committed = 0;
    if (best_a >= 0) {
      if (win_len == 0) committed = 1;
      else if (best_a == win_len) committed = win_len + (bonus ? 1 : 0);
      else committed = best_a + 1;
      committed = min(committed, remaining);
    }
    const int base = seq_len[b];
    SR_DCHECK(base + committed <= tok_stride);
    for (int i = lane; i < committed; i += 32) tokens[(int64_t)b * tok_stride + base + i] = target[win_q + i];
    if (lane < N) {
      int4 o;
      const bool active = a >= 0;
      const bool win = active && lane == win_n;
      o.x = active ? n : 0;
      o.y = active ? a : 0;
      o.z = win ? committed : 0;
      o.w = !active ? 0 : (win ? (a == n ? 0 : max(n - a - 1, 0)) : n);
      reinterpret_cast<int4*>(outcome)[b * N + lane] = o;
    }
    if (lane == 0) {
      bon[b] = best_a >= 0 ? win_n : -1;
      seq_len[b] = base + committed;
      gen_len[b] += committed;
      // window slots 0..committed-1 are positions ctx .. seq_len_new - 2:
      // exactly the KV the engine invariant (valid below seq_len - 1) adds
      s_branch = best_a >= 0 ? win_branch : -1;
      s_ctx = win_ctx;
      s_req = win_req;
      s_committed = committed;
    }
  }
  __syncthreads();
  if (kv.window == nullptr || s_branch < 0 || s_committed <= 0) return;
  // winner's window KV [layer][branch][K/V][head][slot j][hd] ->
  // paged cache [layer][page][K/V][head][slot][hd] at position ctx + j
  constexpr int kVec = 16 / sizeof(T);             // elements per 16-byte chunk
  const int chunks = kv.head_dim / kVec;           // chunks per KV row
  const int cm = s_committed, nkv = kv.kv_heads, hd = kv.head_dim;
  const int total = kv.layers * 2 * nkv * cm * chunks;
  const int32_t* btab = kv.block_table + (int64_t)s_req * kv.max_pages;
  for (int e = threadIdx.x; e < total; e += blockDim.x) {
    int r = e;
    const int c = r % chunks; r /= chunks;
    const int j = r % cm; r /= cm;
    const int h = r % nkv; r /= nkv;
    const int sel = r & 1;
    const int layer = r >> 1;
    const int pos = s_ctx + j;
    SR_DCHECK(pos / kv.page < kv.max_pages && j < kv.window_max && s_branch < kv.branches);
    const int page = btab[pos / kv.page];
    SR_DCHECK(page >= 0 && page < kv.num_pages);
    const int slot = pos % kv.page;
    const T* src = reinterpret_cast<const T*>(kv.window) + layer * kv.window_layer_elems() +
                   ((((int64_t)s_branch * 2 + sel) * nkv + h) * kv.window_max + j) * hd + kv_phys<T>(j, c * kVec);
    T* dst = reinterpret_cast<T*>(kv.cache) + layer * kv.cache_layer_elems() +
             ((((int64_t)page * 2 + sel) * nkv + h) * kv.page + slot) * hd + kv_phys<T>(slot, c * kVec);
    *reinterpret_cast<int4*>(dst) = *reinterpret_cast<const int4*>(src);
  }
}

// Next verify batch from device state: drafter n of request b gets rows
// [s*(k+1), s*(k+1) + nd + 1): the last committed token then its drafts.
__global__ void build_verify_kernel(int B, int N, int k, const int32_t* __restrict__ tokens, int64_t tok_stride,
                                    const int32_t* __restrict__ seq_len, const int32_t* __restrict__ gen_len,
                                    int32_t* __restrict__ max_new, const int32_t* __restrict__ max_new_cap,
                                    const int32_t* __restrict__ drafts,
                                    const int32_t* __restrict__ ndraft, const int32_t* __restrict__ window,
                                    const int32_t* __restrict__ active_mask, int32_t* __restrict__ token_ids,
                                    int32_t* __restrict__ positions, SeqInfo* __restrict__ seqs) {
  grid_dep_sync();
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= B * N) return;
  const int b = s / N, n = s % N;
  // budgets arrive from the host each step (capture_io); the engine's token
  // row and KV pages were sized for max_new_cap, so clamp in place (thread
  // n == 0 stores; every thread of b computes the same value)
  int mn = max_new[b];
  if (max_new_cap != nullptr) {
    mn = min(mn, max_new_cap[b]);
    if (n == 0) max_new[b] = mn;
  }
  const int remaining = mn - gen_len[b];
  const int L = seq_len[b];
  int nd = 0;
  bool active = remaining > 0;
  if (active) {
    nd = drafts != nullptr ? ndraft[n * B + b] : 0;
    active = nd >= 0;  // ndraft < 0: no window this round (decoupled gap round)
    if (active_mask != nullptr && active_mask[n * B + b] == 0) active = false;  // drafter off for b
    nd = max(0, min(nd, min(k, remaining)));
    if (window != nullptr) nd = min(nd, max(0, window[b]));  // per-request window (reconfiguration)
    // a Best-of-N branch with nothing to propose cannot beat the incumbent
    // (ties go to drafter 0): no window, its outcome row stays zero
    if (n > 0 && nd == 0) active = false;
  }
  SR_DCHECK(!active || (L >= 1 && L + nd <= tok_stride));
  SeqInfo sq;
  sq.q_start = s * (k + 1);
  sq.q_len = active ? nd + 1 : 0;
  sq.request = b;
  sq.ctx_len = L - 1;
  sq.branch = n == 0 ? -1 : b * (N - 1) + (n - 1);
  sq.pad0 = sq.pad1 = sq.pad2 = 0;
  seqs[s] = sq;
  for (int j = 0; j <= k; ++j) {
    const int row = s * (k + 1) + j;
    int tok;
    if (j == 0) tok = tokens[(int64_t)b * tok_stride + L - 1];
    else if (j <= nd) tok = drafts[((int64_t)n * B + b) * k + j - 1];
    else tok = 0;
    token_ids[row] = tok;
    positions[row] = L - 1 + j;
  }
}

// Compacting variant (one CTA): sequences keep their index s = b*N + n, but
// their rows are packed back to back -- q_start = exclusive prefix sum of
// q_len in s order -- so finished requests, gap rounds and unproposed draft
// slots occupy no rows; *live_rows = the packed row count, which the
// forward's GEMMs read to skip dead tiles.  q_start stays non-decreasing in s
// (an empty sequence takes the next live one's start), which the row ->
// sequence binary searches of the forward rely on.
constexpr int kCompactThreads = 1024;

__global__ void __launch_bounds__(kCompactThreads)
build_verify_compact_kernel(int B, int N, int k, const int32_t* __restrict__ tokens, int64_t tok_stride,
                            const int32_t* __restrict__ seq_len, const int32_t* __restrict__ gen_len,
                            int32_t* __restrict__ max_new, const int32_t* __restrict__ max_new_cap,
                            const int32_t* __restrict__ drafts, const int32_t* __restrict__ ndraft,
                            const int32_t* __restrict__ window, const int32_t* __restrict__ active_mask,
                            int32_t* __restrict__ token_ids, int32_t* __restrict__ positions,
                            SeqInfo* __restrict__ seqs, int32_t* __restrict__ live_rows) {
  grid_dep_sync();
  __shared__ int warp_sum[kCompactThreads / 32];
  __shared__ int carry;
  if (threadIdx.x == 0) carry = 0;
  const int S = B * N;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int s0 = 0; s0 < S; s0 += kCompactThreads) {
    const int s = s0 + threadIdx.x;
    int q_len = 0, nd = 0, b = 0, n = 0, L = 0;
    if (s < S) {
      b = s / N;
      n = s % N;
      int mn = max_new[b];
      if (max_new_cap != nullptr) {
        mn = min(mn, max_new_cap[b]);
        if (n == 0) max_new[b] = mn;
      }
      const int remaining = mn - gen_len[b];
      L = seq_len[b];
      bool active = remaining > 0;
      if (active) {
        nd = drafts != nullptr ? ndraft[n * B + b] : 0;
        active = nd >= 0;  // ndraft < 0: no window this round (decoupled gap round)
        if (active_mask != nullptr && active_mask[n * B + b] == 0) active = false;  // drafter off for b
        nd = max(0, min(nd, min(k, remaining)));
        if (window != nullptr) nd = min(nd, max(0, window[b]));
        if (n > 0 && nd == 0) active = false;  // empty BoN branch: cannot beat the incumbent
      }
      q_len = active ? nd + 1 : 0;
    }
    // block-wide exclusive scan of q_len in s order
    int x = q_len;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_sum[wid] = x;
    __syncthreads();
    if (wid == 0) {
      int w = warp_sum[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += y;
      }
      warp_sum[lane] = w;  // inclusive totals of warps 0..lane
    }
    __syncthreads();
    const int start = carry + (wid ? warp_sum[wid - 1] : 0) + x - q_len;
    if (s < S) {
      SeqInfo sq;
      sq.q_start = start;
      sq.q_len = q_len;
      sq.request = b;
      sq.ctx_len = L - 1;
      sq.branch = n == 0 ? -1 : b * (N - 1) + (n - 1);
      sq.pad0 = sq.pad1 = sq.pad2 = 0;
      seqs[s] = sq;
      SR_DCHECK(L >= 1 && L - 1 + q_len <= tok_stride);
      for (int j = 0; j < q_len; ++j) {
        token_ids[start + j] =
            j == 0 ? tokens[(int64_t)b * tok_stride + L - 1] : drafts[((int64_t)n * B + b) * k + j - 1];
        positions[start + j] = L - 1 + j;
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) carry += warp_sum[kCompactThreads / 32 - 1];
    __syncthreads();
  }
  if (threadIdx.x == 0) *live_rows = carry;
}

// Reference-acceptance drafter: proposes the target's own continuation
// truth[g] for output position g when the reference's keyed acceptance draw
// u[g] < p (sim.py:322-336), else a deterministic wrong token, so the
// exact-match verifier accepts exactly the reference's `_verify_prefix` run
// (sim.py:977-981) while every committed token is a real model output.
__global__ void synthetic_draft_kernel(int B, int k, const int32_t* __restrict__ truth, int64_t truth_stride,
                                       const int32_t* __restrict__ truth_len, const double* __restrict__ u,
                                       int64_t u_stride, const double* __restrict__ p,
                                       const int32_t* __restrict__ gen_len, int vocab,
                                       int32_t* __restrict__ drafts, int32_t* __restrict__ ndraft) {
  grid_dep_sync();
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  const int g0 = gen_len[b];
  const int nd = max(0, min(k, truth_len[b] - g0));
  const double pb = p[b];
  for (int j = 0; j < k; ++j) {
    int tok = -1;
    if (j < nd) {
      const int g = g0 + j;
      const int t = truth[(int64_t)b * truth_stride + g];
      tok = u[(int64_t)b * u_stride + g] < pb ? t : (t + 1) % vocab;
    }
    drafts[(int64_t)b * k + j] = tok;
  }
  ndraft[b] = nd;
}

// Draft-model batches (K5).  step 0 = catch-up: the committed tokens the
// drafter has not cached yet, [dkv_len, seq_len), with logits taken at the
// last one (rows [b*(k+2), +k+2)); step j >= 1 = one decode step on the
// previous draft token (row b: forward over the first B rows only).
// The output of step j-1 (prev_out [B]) is filed as draft j-1.
__global__ void draft_batch_kernel(int B, int k, int step, const int32_t* __restrict__ tokens, int64_t tok_stride,
                                   const int32_t* __restrict__ seq_len, const int32_t* __restrict__ gen_len,
                                   const int32_t* __restrict__ max_new, int32_t* __restrict__ dkv_len,
                                   const int32_t* __restrict__ prev_out, int32_t* __restrict__ drafts,
                                   int32_t* __restrict__ ndraft, int32_t* __restrict__ token_ids,
                                   int32_t* __restrict__ positions, SeqInfo* __restrict__ seqs,
                                   int32_t* __restrict__ logit_rows, int32_t* __restrict__ key_pos) {
  grid_dep_sync();
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  const int rows = k + 2;
  const int L = seq_len[b];
  const int want = max(0, min(k, max_new[b] - gen_len[b]));
  if (step >= 1 && step - 1 < k) drafts[(int64_t)b * k + step - 1] = (step - 1 < want) ? prev_out[b] : -1;
  if (step == k) {  // collect only
    ndraft[b] = want;
    return;
  }
  SeqInfo sq;
  sq.q_start = b * rows;
  sq.request = b;
  sq.branch = -1;
  sq.pad0 = sq.pad1 = sq.pad2 = 0;
  if (step == 0) {
    const int d0 = dkv_len[b];
    const int q = want > 0 ? min(L - d0, rows) : 0;
    const int first = L - q;  // clamp: never more than `rows` tokens of catch-up
    sq.q_len = q;
    sq.ctx_len = first;
    for (int j = 0; j < rows; ++j) {
      const int p = first + j;
      token_ids[b * rows + j] = (j < q) ? tokens[(int64_t)b * tok_stride + p] : 0;
      positions[b * rows + j] = (j < q) ? p : 0;
    }
    logit_rows[b] = b * rows + max(q - 1, 0);
    if (key_pos != nullptr) key_pos[b] = L;  // the draft's output position
    if (q > 0) dkv_len[b] = L;
  } else {
    // decode steps: one row per request, packed at row b (the forward runs
    // over B rows, not B * (k + 2))
    const int p = L - 1 + step;
    sq.q_start = b;
    sq.q_len = step < want ? 1 : 0;
    sq.ctx_len = p;
    token_ids[b] = prev_out[b];
    positions[b] = p;
    logit_rows[b] = b;
    if (key_pos != nullptr) key_pos[b] = p + 1;
  }
  seqs[b] = sq;
}

}  // namespace

// Host-facing step result: per request its outcome row then the token
// slots [seq_before, seq_before + w) (clamped to the row), one thread per cell.
__global__ void pack_results_kernel(int B, int N, int w, const int32_t* __restrict__ outcome,
                                    const int32_t* __restrict__ tokens, int64_t tok_stride,
                                    const int32_t* __restrict__ seq_before, int32_t* __restrict__ out) {
  grid_dep_sync();
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  const int cols = 4 * N + w;
  if (e >= B * cols) return;
  const int b = e / cols, c = e % cols;
  int v;
  if (c < 4 * N) {
    v = outcome[(int64_t)b * 4 * N + c];   // drafter c / 4's outcome row
  } else {
    const int64_t pos = min((int64_t)seq_before[b] + (c - 4 * N), tok_stride - 1);
    v = tokens[(int64_t)b * tok_stride + pos];
  }
  out[e] = v;
}

// Host-facing step prologue: this step's request budgets straight from the
// caller's pinned host buffer (zero-copy over the host link; build_verify
// clamps them to each slot's capacity) and the pre-step lengths the result
// pack reads.  One kernel instead of two copy-engine nodes in the step graph.
__global__ void io_begin_kernel(int B, const int32_t* __restrict__ budget_host, int32_t* __restrict__ max_new,
                                const int32_t* __restrict__ seq_len, int32_t* __restrict__ seq_before) {
  grid_dep_sync();
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  max_new[b] = budget_host[b];
  seq_before[b] = seq_len[b];
}

}  // namespace sr

extern "C" int sr_io_begin(int num_requests, const int32_t* budget_host, int32_t* max_new, const int32_t* seq_len,
                           int32_t* seq_before, sr_stream_t stream) {
  SR_REQUIRE(num_requests >= 0, "negative request count");
  if (num_requests == 0) return SR_OK;
  SR_REQUIRE(budget_host && max_new && seq_len && seq_before, "null pointer");
  void* dev = nullptr;
  SR_REQUIRE(cudaHostGetDevicePointer(&dev, const_cast<int32_t*>(budget_host), 0) == cudaSuccess,
             "budget_host must be pinned (page-locked) host memory");
  sr::launch_k(sr::io_begin_kernel, sr::ceil_div(num_requests, 256), 256, 0, (cudaStream_t)stream, num_requests,
               reinterpret_cast<const int32_t*>(dev), max_new, seq_len, seq_before);
  return sr::check_launch("io_begin_kernel");
}

extern "C" int sr_pack_results(int num_requests, int num_drafters, int width, const int32_t* outcome,
                               const int32_t* tokens, int64_t tok_stride, const int32_t* seq_before, int32_t* out,
                               sr_stream_t stream) {
  SR_REQUIRE(num_requests >= 0 && num_drafters >= 1 && width >= 0 && tok_stride > 0, "bad result shape");
  if (num_requests == 0) return SR_OK;
  SR_REQUIRE(outcome && tokens && seq_before && out, "null pointer");
  // `out` may be pinned host memory: the kernel then writes it zero-copy
  cudaPointerAttributes pa{};
  const bool known = cudaPointerGetAttributes(&pa, out) == cudaSuccess;
  cudaGetLastError();  // clear a failed query
  SR_REQUIRE(known && pa.type != cudaMemoryTypeUnregistered,
             "result buffer must be device memory or pinned (page-locked) host memory");
  if (pa.type == cudaMemoryTypeHost) {
    void* dev = nullptr;
    SR_REQUIRE(cudaHostGetDevicePointer(&dev, out, 0) == cudaSuccess, "result buffer: host memory must be pinned");
    out = reinterpret_cast<int32_t*>(dev);
  }
  const int n = num_requests * (4 * num_drafters + width);
  sr::launch_k(sr::pack_results_kernel, sr::ceil_div(n, 256), 256, 0, (cudaStream_t)stream, num_requests,
               num_drafters, width, outcome, tokens, tok_stride, seq_before, out);
  return sr::check_launch("pack_results_kernel");
}

extern "C" int sr_accept_commit(void* model, int num_requests, int num_drafters, const void* seqs,
                                const int32_t* token_ids, const int32_t* target, int32_t* tokens,
                                int64_t tok_stride, int32_t* seq_len, int32_t* gen_len,
                                const int32_t* max_new, int bonus_token, int32_t* outcome,
                                int32_t* bon, sr_stream_t stream) {
  SR_REQUIRE(num_requests >= 0, "negative request count");
  if (num_requests == 0) return SR_OK;
  SR_REQUIRE(num_drafters >= 1 && num_drafters <= 32, "num_drafters out of [1, 32]");
  SR_REQUIRE(seqs && token_ids && target && tokens && seq_len && gen_len && max_new && outcome && bon,
             "null pointer");
  SR_REQUIRE((reinterpret_cast<uintptr_t>(outcome) & 15) == 0, "outcome rows must be 16-byte aligned");
  sr::KvLayout kv{};
  int dtype = 1;
  if (num_drafters > 1 && model != nullptr) {
    const int rc = sr::model_kv_layout(model, &kv, &dtype);
    if (rc) return rc;
    SR_REQUIRE(kv.window != nullptr, "drafter branches need a window buffer");
  }
  const auto* sq = reinterpret_cast<const sr::SeqInfo*>(seqs);
  if (dtype == 1)
    sr::launch_k(sr::accept_commit_kernel<__nv_bfloat16>, num_requests, 128, 0, (cudaStream_t)stream,
                 num_requests, num_drafters, sq, token_ids, target, tokens, tok_stride, seq_len, gen_len, max_new,
                 bonus_token, outcome, bon, kv);
  else
    sr::launch_k(sr::accept_commit_kernel<float>, num_requests, 128, 0, (cudaStream_t)stream, num_requests,
                 num_drafters, sq, token_ids, target, tokens, tok_stride, seq_len, gen_len, max_new, bonus_token,
                 outcome, bon, kv);
  return sr::check_launch("accept_commit_kernel");
}

extern "C" int sr_synthetic_draft(int num_requests, int k, const int32_t* truth, int64_t truth_stride,
                                  const int32_t* truth_len, const double* uniforms, int64_t u_stride,
                                  const double* accept_p, const int32_t* gen_len, int vocab, int32_t* drafts,
                                  int32_t* ndraft, sr_stream_t stream) {
  SR_REQUIRE(num_requests >= 0 && k >= 1 && vocab >= 2, "bad synthetic draft shape");
  if (num_requests == 0) return SR_OK;
  SR_REQUIRE(truth && truth_len && uniforms && accept_p && gen_len && drafts && ndraft, "null pointer");
  sr::launch_k(sr::synthetic_draft_kernel, sr::ceil_div(num_requests, 128), 128, 0, (cudaStream_t)stream, 
      num_requests, k, truth, truth_stride, truth_len, uniforms, u_stride, accept_p, gen_len, vocab, drafts,
      ndraft);
  return sr::check_launch("synthetic_draft_kernel");
}

extern "C" int sr_draft_model_batch(int num_requests, int k, int step, const int32_t* tokens, int64_t tok_stride,
                                    const int32_t* seq_len, const int32_t* gen_len, const int32_t* max_new,
                                    int32_t* dkv_len, const int32_t* prev_out, int32_t* drafts, int32_t* ndraft,
                                    int32_t* token_ids, int32_t* positions, void* seqs, int32_t* logit_rows,
                                    int32_t* key_pos, sr_stream_t stream) {
  SR_REQUIRE(num_requests >= 0 && k >= 1 && step >= 0 && step <= k, "bad draft step");
  if (num_requests == 0) return SR_OK;
  SR_REQUIRE(tokens && seq_len && gen_len && max_new && dkv_len && drafts && ndraft && token_ids && positions &&
                 seqs && logit_rows && (step == 0 || prev_out),
             "null pointer");
  sr::launch_k(sr::draft_batch_kernel, sr::ceil_div(num_requests, 128), 128, 0, (cudaStream_t)stream, 
      num_requests, k, step, tokens, tok_stride, seq_len, gen_len, max_new, dkv_len, prev_out, drafts, ndraft,
      token_ids, positions, reinterpret_cast<sr::SeqInfo*>(seqs), logit_rows, key_pos);
  return sr::check_launch("draft_batch_kernel");
}

extern "C" int sr_build_verify_batch(int num_requests, int num_drafters, int k, const int32_t* tokens,
                                     int64_t tok_stride, const int32_t* seq_len, const int32_t* gen_len,
                                     int32_t* max_new, const int32_t* max_new_cap, const int32_t* drafts,
                                     const int32_t* ndraft,
                                     const int32_t* window, const int32_t* active, int32_t* token_ids,
                                     int32_t* positions, void* seqs, int32_t* live_rows, sr_stream_t stream) {
  SR_REQUIRE(num_requests >= 0 && num_drafters >= 1 && k >= 0, "bad batch shape");
  if (num_requests == 0) return SR_OK;
  SR_REQUIRE(tokens && seq_len && gen_len && max_new && token_ids && positions && seqs, "null pointer");
  SR_REQUIRE(drafts == nullptr || ndraft != nullptr, "drafts without ndraft");
  const int S = num_requests * num_drafters;
  if (live_rows != nullptr) {
    sr::launch_k(sr::build_verify_compact_kernel, 1, sr::kCompactThreads, 0, (cudaStream_t)stream, num_requests,
                 num_drafters, k, tokens, tok_stride, seq_len, gen_len, max_new, max_new_cap, drafts, ndraft, window,
                 active, token_ids, positions, reinterpret_cast<sr::SeqInfo*>(seqs), live_rows);
    return sr::check_launch("build_verify_compact_kernel");
  }
  sr::launch_k(sr::build_verify_kernel, sr::ceil_div(S, 128), 128, 0, (cudaStream_t)stream, 
      num_requests, num_drafters, k, tokens, tok_stride, seq_len, gen_len, max_new, max_new_cap, drafts, ndraft,
      window, active, token_ids, positions, reinterpret_cast<sr::SeqInfo*>(seqs));
  return sr::check_launch("build_verify_kernel");
}
