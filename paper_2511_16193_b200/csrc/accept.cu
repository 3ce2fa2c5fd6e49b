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

namespace {

__global__ void accept_commit_kernel(int B, int N, const SeqInfo* __restrict__ seqs,
                                     const int32_t* __restrict__ token_ids,
                                     const int32_t* __restrict__ target, int32_t* __restrict__ tokens,
                                     int64_t tok_stride, int32_t* __restrict__ seq_len,
                                     int32_t* __restrict__ gen_len, const int32_t* __restrict__ max_new,
                                     int bonus, int32_t* __restrict__ outcome,
                                     int32_t* __restrict__ bon) {
  grid_dep_sync();
  const int b = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (b >= B) return;
  const int remaining = max_new[b] - gen_len[b];
  // per-drafter accepted prefix (lane n handles drafter n)
  int a = -1, n = 0, qs = 0;
  if (lane < N) {
    const SeqInfo sq = seqs[b * N + lane];
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
  const int win_n = best_n;
  const int win_q = __shfl_sync(0xffffffffu, qs, win_n & 31);
  const int win_len = __shfl_sync(0xffffffffu, n, win_n & 31);
  int committed = 0;
  if (best_a >= 0) {
    if (win_len == 0) committed = 1;
    else if (best_a == win_len) committed = win_len + (bonus ? 1 : 0);
    else committed = best_a + 1;
    committed = min(committed, remaining);
  }
  const int base = seq_len[b];
  for (int i = lane; i < committed; i += 32) tokens[(int64_t)b * tok_stride + base + i] = target[win_q + i];
  if (lane < N) {
    int32_t* o = outcome + (int64_t)(b * N + lane) * 4;
    const bool active = a >= 0;
    const bool win = active && lane == win_n;
    o[0] = active ? n : 0;
    o[1] = active ? a : 0;
    o[2] = win ? committed : 0;
    o[3] = !active ? 0 : (win ? (a == n ? 0 : max(n - a - 1, 0)) : n);
  }
  if (lane == 0) {
    bon[b] = best_a >= 0 ? win_n : -1;
    seq_len[b] = base + committed;
    gen_len[b] += committed;
  }
}

// Copy the winning drafter-branch window KV (slots [0, committed)) into the
// paged cache at positions [ctx_len, ctx_len + committed), every layer.
template <typename T>
__global__ void kv_commit_kernel(int N, const SeqInfo* __restrict__ seqs, const int32_t* __restrict__ outcome,
                                 const int32_t* __restrict__ bon, KvLayout kv) {
  grid_dep_sync();
  const int b = blockIdx.x, layer = blockIdx.y;
  const int w = bon[b];
  if (w < 0) return;
  const SeqInfo sq = seqs[b * N + w];
  if (sq.branch < 0) return;  // the winner wrote its KV in place
  const int committed = outcome[(int64_t)(b * N + w) * 4 + 2];
  const int hd = kv.head_dim, nkv = kv.kv_heads;
  const T* wbase = reinterpret_cast<const T*>(kv.window) + layer * kv.window_layer_elems() +
                   (int64_t)sq.branch * 2 * nkv * kv.window_max * hd;
  T* cbase = reinterpret_cast<T*>(kv.cache) + layer * kv.cache_layer_elems();
  const int32_t* btab = kv.block_table + (int64_t)sq.request * kv.max_pages;
  const int per_slot = 2 * nkv * hd;
  for (int e = threadIdx.x; e < committed * per_slot; e += blockDim.x) {
    const int j = e / per_slot, r = e % per_slot;
    const int kvsel = r / (nkv * hd), h = (r / hd) % nkv, d = r % hd;
    const int pos = sq.ctx_len + j;
    const int page = btab[pos / kv.page];
    const int slot = pos % kv.page;
    cbase[(((int64_t)page * 2 + kvsel) * nkv + h) * kv.page * hd + (int64_t)slot * hd + kv_phys<T>(slot, d)] =
        wbase[((int64_t)kvsel * nkv + h) * kv.window_max * hd + (int64_t)j * hd + kv_phys<T>(j, d)];
  }
}

// Next verify batch from device state: drafter n of request b gets rows
// [s*(k+1), s*(k+1) + nd + 1): the last committed token then its drafts.
__global__ void build_verify_kernel(int B, int N, int k, const int32_t* __restrict__ tokens, int64_t tok_stride,
                                    const int32_t* __restrict__ seq_len, const int32_t* __restrict__ gen_len,
                                    int32_t* __restrict__ max_new, const int32_t* __restrict__ max_new_cap,
                                    const int32_t* __restrict__ drafts,
                                    const int32_t* __restrict__ ndraft, const int32_t* __restrict__ window,
                                    int32_t* __restrict__ token_ids, int32_t* __restrict__ positions,
                                    SeqInfo* __restrict__ seqs) {
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
    nd = max(0, min(nd, min(k, remaining)));
    if (window != nullptr) nd = min(nd, max(0, window[b]));  // per-request window (reconfiguration)
  }
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
// last one; step j >= 1 = one decode step on the previous draft token.
// The output of step j-1 (prev_out [B]) is filed as draft j-1.
__global__ void draft_batch_kernel(int B, int k, int step, const int32_t* __restrict__ tokens, int64_t tok_stride,
                                   const int32_t* __restrict__ seq_len, const int32_t* __restrict__ gen_len,
                                   const int32_t* __restrict__ max_new, int32_t* __restrict__ dkv_len,
                                   const int32_t* __restrict__ prev_out, int32_t* __restrict__ drafts,
                                   int32_t* __restrict__ ndraft, int32_t* __restrict__ token_ids,
                                   int32_t* __restrict__ positions, SeqInfo* __restrict__ seqs,
                                   int32_t* __restrict__ logit_rows) {
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
    if (q > 0) dkv_len[b] = L;
  } else {
    const int p = L - 1 + step;
    sq.q_len = step < want ? 1 : 0;
    sq.ctx_len = p;
    token_ids[b * rows] = prev_out[b];
    positions[b * rows] = p;
    logit_rows[b] = b * rows;
  }
  seqs[b] = sq;
}

}  // namespace

int kv_commit(int B, int N, const SeqInfo* seqs, const int32_t* outcome, const int32_t* bon,
              const KvLayout& kv, int dtype, cudaStream_t s) {
  if (B == 0 || N <= 1) return SR_OK;
  dim3 grid(B, kv.layers);
  if (dtype == 1)
    sr::launch_k(kv_commit_kernel<__nv_bfloat16>, grid, 256, 0, s, N, seqs, outcome, bon, kv);
  else
    sr::launch_k(kv_commit_kernel<float>, grid, 256, 0, s, N, seqs, outcome, bon, kv);
  return check_launch("kv_commit_kernel");
}

// Host-facing step result: per request its outcome row then the token
// slots [seq_before, seq_before + w) (clamped to the row), one thread per cell.
__global__ void pack_results_kernel(int B, int w, const int32_t* __restrict__ outcome,
                                    const int32_t* __restrict__ tokens, int64_t tok_stride,
                                    const int32_t* __restrict__ seq_before, int32_t* __restrict__ out) {
  grid_dep_sync();
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  const int cols = 4 + w;
  if (e >= B * cols) return;
  const int b = e / cols, c = e % cols;
  int v;
  if (c < 4) {
    v = outcome[(int64_t)b * 4 + c];
  } else {
    const int64_t pos = min((int64_t)seq_before[b] + (c - 4), tok_stride - 1);
    v = tokens[(int64_t)b * tok_stride + pos];
  }
  out[e] = v;
}

}  // namespace sr

extern "C" int sr_pack_results(int num_requests, int width, const int32_t* outcome, const int32_t* tokens,
                               int64_t tok_stride, const int32_t* seq_before, int32_t* out, sr_stream_t stream) {
  SR_REQUIRE(num_requests >= 0 && width >= 0 && tok_stride > 0, "bad result shape");
  if (num_requests == 0) return SR_OK;
  SR_REQUIRE(outcome && tokens && seq_before && out, "null pointer");
  const int n = num_requests * (4 + width);
  sr::launch_k(sr::pack_results_kernel, sr::ceil_div(n, 256), 256, 0, (cudaStream_t)stream, num_requests, width,
               outcome, tokens, tok_stride, seq_before, out);
  return sr::check_launch("pack_results_kernel");
}

extern "C" int sr_accept_commit(int num_requests, int num_drafters, const void* seqs,
                                const int32_t* token_ids, const int32_t* target, int32_t* tokens,
                                int64_t tok_stride, int32_t* seq_len, int32_t* gen_len,
                                const int32_t* max_new, int bonus_token, int32_t* outcome,
                                int32_t* bon, sr_stream_t stream) {
  SR_REQUIRE(num_requests >= 0, "negative request count");
  if (num_requests == 0) return SR_OK;
  SR_REQUIRE(num_drafters >= 1 && num_drafters <= 32, "num_drafters out of [1, 32]");
  SR_REQUIRE(seqs && token_ids && target && tokens && seq_len && gen_len && max_new && outcome && bon,
             "null pointer");
  sr::launch_k(sr::accept_commit_kernel, sr::ceil_div(num_requests, 8), 256, 0, (cudaStream_t)stream, 
      num_requests, num_drafters, reinterpret_cast<const sr::SeqInfo*>(seqs), token_ids, target, tokens,
      tok_stride, seq_len, gen_len, max_new, bonus_token, outcome, bon);
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
                                    sr_stream_t stream) {
  SR_REQUIRE(num_requests >= 0 && k >= 1 && step >= 0 && step <= k, "bad draft step");
  if (num_requests == 0) return SR_OK;
  SR_REQUIRE(tokens && seq_len && gen_len && max_new && dkv_len && drafts && ndraft && token_ids && positions &&
                 seqs && logit_rows && (step == 0 || prev_out),
             "null pointer");
  sr::launch_k(sr::draft_batch_kernel, sr::ceil_div(num_requests, 128), 128, 0, (cudaStream_t)stream, 
      num_requests, k, step, tokens, tok_stride, seq_len, gen_len, max_new, dkv_len, prev_out, drafts, ndraft,
      token_ids, positions, reinterpret_cast<sr::SeqInfo*>(seqs), logit_rows);
  return sr::check_launch("draft_batch_kernel");
}

extern "C" int sr_build_verify_batch(int num_requests, int num_drafters, int k, const int32_t* tokens,
                                     int64_t tok_stride, const int32_t* seq_len, const int32_t* gen_len,
                                     int32_t* max_new, const int32_t* max_new_cap, const int32_t* drafts,
                                     const int32_t* ndraft,
                                     const int32_t* window, int32_t* token_ids, int32_t* positions,
                                     void* seqs, sr_stream_t stream) {
  SR_REQUIRE(num_requests >= 0 && num_drafters >= 1 && k >= 0, "bad batch shape");
  if (num_requests == 0) return SR_OK;
  SR_REQUIRE(tokens && seq_len && gen_len && max_new && token_ids && positions && seqs, "null pointer");
  SR_REQUIRE(drafts == nullptr || ndraft != nullptr, "drafts without ndraft");
  const int S = num_requests * num_drafters;
  sr::launch_k(sr::build_verify_kernel, sr::ceil_div(S, 128), 128, 0, (cudaStream_t)stream, 
      num_requests, num_drafters, k, tokens, tok_stride, seq_len, gen_len, max_new, max_new_cap, drafts, ndraft,
      window,
      token_ids, positions, reinterpret_cast<sr::SeqInfo*>(seqs));
  return sr::check_launch("build_verify_kernel");
}
