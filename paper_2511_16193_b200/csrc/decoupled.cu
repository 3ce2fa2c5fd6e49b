// Round bookkeeping of decoupled speculation (pipeline depth 2; reference
// sim.py:860-917 begin_round decoupled branch, sim.py:1051-1092
// _end_decoupled) as native kernels, one thread per request: the drafter
// side's window placement and decision folding, the verifier side's decision
// packing and successor admission.  With these, a decoupled round on either
// GPU is only library kernels plus the NCCL exchange.
//
// Per request b, the drafter keeps a mirror of the committed tokens plus the
// window in flight (inflight[b] drafted tokens after seq_len[b]); each round
// it drafts the successor window behind the in-flight one.  The verifier's
// decision for the in-flight window is (verified, accepted a, committed c,
// the committed tokens).  A window survives only if its predecessor was
// fully accepted; a rejected predecessor discards it (depth-2 waste,
// sim.py:1074-1080) and the request's next round is a fresh window from the
// corrected position.  An empty window that committed the target's token
// leaves its successor misaligned by one, so it counts as rejected.
#include "common.cuh"

namespace sr {

namespace {

__device__ __forceinline__ bool full_accept(bool verified, int accepted, int proposed, int committed) {
  return verified && accepted == proposed && (proposed > 0 || committed == 0);
}

// Before drafting: the successor's first output position and its context.
__global__ void draft_prep_kernel(int B, const int32_t* __restrict__ seq_len, const int32_t* __restrict__ gen_len,
                                  const int32_t* __restrict__ inflight, int32_t* __restrict__ g0,
                                  int32_t* __restrict__ ctx) {
  grid_dep_sync();
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  g0[b] = gen_len[b] + inflight[b];
  ctx[b] = seq_len[b] + inflight[b];
}

// After drafting: cap the window at the remaining budget, append it behind
// the in-flight window in the token mirror, and stage it for the verifier.
__global__ void draft_post_kernel(int B, int k, int64_t stride, const int32_t* __restrict__ max_new,
                                  const int32_t* __restrict__ g0, const int32_t* __restrict__ ctx,
                                  const int32_t* __restrict__ drafts, int32_t* __restrict__ nd,
                                  int32_t* __restrict__ tokens, int32_t* __restrict__ out_drafts,
                                  int32_t* __restrict__ out_nd) {
  grid_dep_sync();
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  const int room = max(0, max_new[b] - g0[b]);
  const int n = min(nd[b], room);
  nd[b] = n;
  out_nd[b] = n;
  int32_t* row = tokens + (int64_t)b * stride;
  for (int j = 0; j < k; ++j) {
    const int d = drafts[(int64_t)b * k + j];
    out_drafts[(int64_t)b * k + j] = d;
    const int64_t p = min((int64_t)ctx[b] + j, stride - 1);
    if (j < n) row[p] = d;
  }
}

// Fold the verifier's decision for the in-flight window into the mirror.
__global__ void draft_apply_kernel(int B, int k, int64_t stride, const int32_t* __restrict__ in_verified,
                                   const int32_t* __restrict__ in_accepted, const int32_t* __restrict__ in_committed,
                                   const int32_t* __restrict__ in_ctoks, const int32_t* __restrict__ out_nd,
                                   int32_t* __restrict__ inflight, int32_t* __restrict__ tokens,
                                   int32_t* __restrict__ seq_len, int32_t* __restrict__ gen_len,
                                   int32_t* __restrict__ dkv_len) {
  grid_dep_sync();
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  const bool verified = in_verified[b] > 0;
  const int a = in_accepted[b], c = in_committed[b], fl = inflight[b];
  const bool part = verified && !full_accept(verified, a, fl, c);
  if (part) {  // accepted prefix + corrected token (the drafts after it were wrong)
    const int64_t p = min((int64_t)seq_len[b] + a, stride - 1);
    tokens[(int64_t)b * stride + p] = in_ctoks[(int64_t)b * (k + 1) + min(a, k)];
  }
  const int adv = verified ? c : 0;
  const int L = seq_len[b] + adv;
  seq_len[b] = L;
  gen_len[b] += adv;
  // the model drafter's KV from the corrected token on was computed on
  // rejected tokens: recompute from there next window
  if (dkv_len != nullptr && part) dkv_len[b] = min(dkv_len[b], L - 1);
  inflight[b] = part ? 0 : out_nd[b];
}

// Verifier, after K3: the decision sent back (verified, accepted, committed,
// the k + 1 committed-token slots) from the outcome row and the token buffer.
__global__ void verify_post_kernel(int B, int k, int64_t stride, const int32_t* __restrict__ outcome,
                                   const int32_t* __restrict__ bon, const int32_t* __restrict__ tokens,
                                   const int32_t* __restrict__ seq_before, int32_t* __restrict__ rows,
                                   int32_t* __restrict__ out_verified, int32_t* __restrict__ out_accepted,
                                   int32_t* __restrict__ out_committed, int32_t* __restrict__ out_ctoks) {
  grid_dep_sync();
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  const int4 o = reinterpret_cast<const int4*>(outcome)[b];
  reinterpret_cast<int4*>(rows)[b] = o;
  out_verified[b] = bon[b] >= 0 ? 1 : 0;
  out_accepted[b] = o.y;
  out_committed[b] = o.z;
  for (int j = 0; j <= k; ++j) {
    const int64_t p = min((int64_t)seq_before[b] + j, stride - 1);
    out_ctoks[(int64_t)b * (k + 1) + j] = tokens[(int64_t)b * stride + p];
  }
}

// Verifier, after the exchange: admit the drafter's new windows as pending
// unless their predecessor was rejected (then charge them as waste).
__global__ void verify_receive_kernel(int B, int k, const int32_t* __restrict__ out_verified,
                                      const int32_t* __restrict__ out_accepted,
                                      const int32_t* __restrict__ out_committed, const int32_t* __restrict__ in_drafts,
                                      const int32_t* __restrict__ in_nd, int32_t* __restrict__ rows,
                                      int32_t* __restrict__ pending, int32_t* __restrict__ pending_nd) {
  grid_dep_sync();
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  const bool verified = out_verified[b] > 0;
  const int nd = in_nd[b];
  const bool full = full_accept(verified, out_accepted[b], rows[(int64_t)b * 4], out_committed[b]);
  const bool part = verified && !full;
  for (int j = 0; j < k; ++j) pending[(int64_t)b * k + j] = in_drafts[(int64_t)b * k + j];
  pending_nd[b] = ((!verified || full) && nd >= 0) ? nd : -1;
  if (part) rows[(int64_t)b * 4 + 3] += nd;
}

}  // namespace

}  // namespace sr

#define SR_GRID(B) sr::ceil_div((B), 128), 128, 0, (cudaStream_t)stream

extern "C" int sr_decoupled_draft_prep(int B, const int32_t* seq_len, const int32_t* gen_len, const int32_t* inflight,
                                       int32_t* g0, int32_t* ctx, sr_stream_t stream) {
  SR_REQUIRE(B >= 0, "negative batch");
  if (B == 0) return SR_OK;
  SR_REQUIRE(seq_len && gen_len && inflight && g0 && ctx, "null pointer");
  sr::launch_k(sr::draft_prep_kernel, SR_GRID(B), B, seq_len, gen_len, inflight, g0, ctx);
  return sr::check_launch("draft_prep_kernel");
}

extern "C" int sr_decoupled_draft_post(int B, int k, int64_t stride, const int32_t* max_new, const int32_t* g0,
                                       const int32_t* ctx, const int32_t* drafts, int32_t* nd, int32_t* tokens,
                                       int32_t* out_drafts, int32_t* out_nd, sr_stream_t stream) {
  SR_REQUIRE(B >= 0 && k >= 1 && stride > 0, "bad shape");
  if (B == 0) return SR_OK;
  SR_REQUIRE(max_new && g0 && ctx && drafts && nd && tokens && out_drafts && out_nd, "null pointer");
  sr::launch_k(sr::draft_post_kernel, SR_GRID(B), B, k, stride, max_new, g0, ctx, drafts, nd, tokens, out_drafts,
               out_nd);
  return sr::check_launch("draft_post_kernel");
}

extern "C" int sr_decoupled_draft_apply(int B, int k, int64_t stride, const int32_t* in_verified,
                                        const int32_t* in_accepted, const int32_t* in_committed,
                                        const int32_t* in_ctoks, const int32_t* out_nd, int32_t* inflight,
                                        int32_t* tokens, int32_t* seq_len, int32_t* gen_len, int32_t* dkv_len,
                                        sr_stream_t stream) {
  SR_REQUIRE(B >= 0 && k >= 1 && stride > 0, "bad shape");
  if (B == 0) return SR_OK;
  SR_REQUIRE(in_verified && in_accepted && in_committed && in_ctoks && out_nd && inflight && tokens && seq_len &&
                 gen_len,
             "null pointer");
  sr::launch_k(sr::draft_apply_kernel, SR_GRID(B), B, k, stride, in_verified, in_accepted, in_committed, in_ctoks,
               out_nd, inflight, tokens, seq_len, gen_len, dkv_len);
  return sr::check_launch("draft_apply_kernel");
}

extern "C" int sr_decoupled_verify_post(int B, int k, int64_t stride, const int32_t* outcome, const int32_t* bon,
                                        const int32_t* tokens, const int32_t* seq_before, int32_t* rows,
                                        int32_t* out_verified, int32_t* out_accepted, int32_t* out_committed,
                                        int32_t* out_ctoks, sr_stream_t stream) {
  SR_REQUIRE(B >= 0 && k >= 0 && stride > 0, "bad shape");
  if (B == 0) return SR_OK;
  SR_REQUIRE(outcome && bon && tokens && seq_before && rows && out_verified && out_accepted && out_committed &&
                 out_ctoks,
             "null pointer");
  SR_REQUIRE((reinterpret_cast<uintptr_t>(outcome) & 15) == 0 && (reinterpret_cast<uintptr_t>(rows) & 15) == 0,
             "outcome / rows must be 16-byte aligned");
  sr::launch_k(sr::verify_post_kernel, SR_GRID(B), B, k, stride, outcome, bon, tokens, seq_before, rows,
               out_verified, out_accepted, out_committed, out_ctoks);
  return sr::check_launch("verify_post_kernel");
}

extern "C" int sr_decoupled_verify_receive(int B, int k, const int32_t* out_verified, const int32_t* out_accepted,
                                           const int32_t* out_committed, const int32_t* in_drafts,
                                           const int32_t* in_nd, int32_t* rows, int32_t* pending,
                                           int32_t* pending_nd, sr_stream_t stream) {
  SR_REQUIRE(B >= 0 && k >= 1, "bad shape");
  if (B == 0) return SR_OK;
  SR_REQUIRE(out_verified && out_accepted && out_committed && in_drafts && in_nd && rows && pending && pending_nd,
             "null pointer");
  sr::launch_k(sr::verify_receive_kernel, SR_GRID(B), B, k, out_verified, out_accepted, out_committed, in_drafts,
               in_nd, rows, pending, pending_nd);
  return sr::check_launch("verify_receive_kernel");
}
