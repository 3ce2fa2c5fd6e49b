/*
 * specrollout_b200 -- C ABI of the B200 speculative-rollout hot path.
 *
 * The reference (arxiv 2511.16193 "SpecActor", package `specrollout`) has no
 * FFI: its boundary is the Python API (pkg/src/specrollout/__init__.py:4-52).
 * Each entry point below replaces one reference function on the rollout hot
 * path; the replaced function is cited per declaration.
 *
 * Conventions
 *   - All array arguments are DEVICE pointers owned by the caller, unless the
 *     comment says "host".  Layouts are row-major, int32 unless stated.
 *   - No entry point allocates device memory or synchronizes the device; all
 *     work is enqueued on `stream` (a cudaStream_t; NULL = legacy default).
 *   - Return SR_OK (0), SR_ERR_CONFIG (2, bad shape/argument -> ConfigError)
 *     or SR_ERR_RUNTIME (3, CUDA failure -> DeviceError).  These mirror the
 *     reference CLI exit codes (pkg/src/specrollout/cli.py:55-57).
 *     sr_last_error() returns the calling thread's last message.
 */
#ifndef SPECROLLOUT_B200_H_
#define SPECROLLOUT_B200_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SR_OK 0
#define SR_ERR_CONFIG 2
#define SR_ERR_RUNTIME 3

typedef struct CUstream_st* sr_stream_t;

/* Library version (major*10000 + minor*100 + patch). */
int sr_version(void);

/* Last error message of the calling thread ("" if none). */
const char* sr_last_error(void);

/* Number of SMs of the current device (for grid sizing by callers). */
int sr_device_sm_count(void);

/* sizeof(sr_model_desc), sizeof(sr_forward_args), sizeof(sr_seq_info) into
 * out[0..n) -- lets bindings verify their struct mirrors (no GPU needed). */
int sr_abi_sizes(int64_t* out, int n);

/* Kernels launched by this library since load (bench evidence). */
long long sr_launch_count(void);

/* ---------------------------------------------------------------------------
 * a1/a2  Keyed draws.  Replaces `streams.stream` + `_Sim.true_token`
 * (sim.py:313-320, generate_true_sequence sim.py:45-56) and
 * `_Sim.accept_draw` (sim.py:322-336).
 *
 * Stream s has entropy words words[s*max_words .. +num_words[s]) (uint32,
 * coerced like numpy's SeedSequence: the 64-bit seed is 1-2 little-endian
 * words, each key one word, strings as CRC-32).  Draw i of stream s goes to
 * out[s*per_stream + i].
 *   sr_keyed_tokens:   Generator.integers(0, high)  (int32 output, high<=2^31)
 *   sr_keyed_uniforms: Generator.random()           (float64 output)
 * ------------------------------------------------------------------------- */
int sr_keyed_tokens(int num_streams, const uint32_t* words, const int32_t* num_words,
                    int max_words, int64_t high, int per_stream, int32_t* out,
                    sr_stream_t stream);
int sr_keyed_uniforms(int num_streams, const uint32_t* words, const int32_t* num_words,
                      int max_words, int per_stream, double* out, sr_stream_t stream);

/* ---------------------------------------------------------------------------
 * a3/a4/a5  Window verification in reference ("truth") mode.  Replaces
 * `_Executor._verify_prefix` (sim.py:977-981), `_apply_outcome`
 * (sim.py:983-1042) and `_Sim.commit` (sim.py:340-353) for a batch of W
 * windows (one executor round).
 *
 * win: [4, W]  rows: request row, start position, n drafted (0 = plain
 *              decode step: commit the target token at start), depth-2
 *              successor size charged as waste on a partial accept.
 * truth:      [R, row_stride]      target tokens by absolute position.
 * uniforms:   [R, M, row_stride]   acceptance uniforms (float64).
 * accept_p:   [R, M]               latent acceptance probability (float64).
 * method:     column of uniforms/accept_p used by all W windows.
 * true_len:   [R]
 * seq:        [R, row_stride]      committed-token buffer, -1 = empty;
 *                                  accepted tokens are written here.
 * high:       [R]                  committed-high watermark, advanced here.
 * out:        [4, W]  accepted, committed, wasted, committed-high after the
 *             window (-1 = conflicting commit; reference AssertionError).
 * A request row may appear at most once per call.
 * ------------------------------------------------------------------------- */
int sr_verify_windows(int num_windows, const int32_t* win, int method, int num_methods,
                      int row_stride, const int32_t* truth, const double* uniforms,
                      const double* accept_p, const int32_t* true_len, int bonus_token,
                      int32_t* seq, int32_t* high, int32_t* out, sr_stream_t stream);

/* ---------------------------------------------------------------------------
 * a9  n-gram drafter (drafting is only priced in the reference, sim.py:883-892;
 * proposal semantics follow vLLM 0.22 NgramProposer,
 * vllm/v1/spec_decode/ngram_proposer.py:198-285): longest suffix n-gram with
 * n in [min_n, max_n] that re-occurs earlier in the context, earliest
 * occurrence on ties, propose up to k following tokens.
 *
 * tokens: [B, stride] context (prompt + committed output), lens: [B].
 * out_draft: [B, k] (unused slots = -1), out_ndraft: [B].
 * scratch: >= 2*B int64 words, zeroed once by the caller before first use
 *          (the kernel leaves it zeroed again).
 * ------------------------------------------------------------------------- */
int sr_ngram_propose(int batch, const int32_t* tokens, int64_t stride, const int32_t* lens,
                     int min_n, int max_n, int k, int32_t* out_draft, int32_t* out_ndraft,
                     int64_t* scratch, sr_stream_t stream);

/* Pooled prompt lookup (a fourth Best-of-N drafting method, configs[4]): the
 * suffix of request b is matched against its own context (sr_ngram_propose
 * semantics) and every other request's committed tokens; the longest match
 * in [min_n, max_n] wins, ties to the own context, then other requests in
 * index order, then the earliest end position; up to k following tokens of
 * that row are proposed (none past the row's length or b's capacity).  With
 * batch 1 it equals sr_ngram_propose.  scratch: batch int64 (zero on entry,
 * left zero). */
int sr_pooled_ngram_propose(int batch, const int32_t* tokens, int64_t stride, const int32_t* lens, int min_n,
                            int max_n, int k, int32_t* out_draft, int32_t* out_ndraft, int64_t* scratch,
                            sr_stream_t stream);

/* ---------------------------------------------------------------------------
 * K1 building block: C = A[M,K] . W[N,K]^T with a fused epilogue (the
 * projections of the target model's verification forward; no reference
 * counterpart -- the reference has no model).
 *   dtype 1: bf16 A/W on tcgen05 tensor cores (TMA + TMEM).  bn selects the
 *            tile: 128|256 one CTA per 128-row tile; -w a CTA pair
 *            (cta_group::2) per 256 x w tile, w a multiple of 16 in [64, 256];
 *            -(1024 + w) two such pairs per cluster sharing A by TMA
 *            multicast; 0 chooses from (M, N, K)
 *   dtype 0: fp32 A/W on CUDA cores (parity path), bn ignored
 * epilogue 0: C = acc + bias (bf16; f32 when dtype 0)
 *          1: C(f32) += acc                      (residual stream)
 *          2: C[M, N/2] = silu(gate) * up, W rows interleaved per 32:
 *             16 gate rows then the 16 matching up rows
 *          3: C(f32) = acc + bias                (logits)
 *          4: (bf16 only) fused vocabulary argmax: per (row, N tile of bn
 *             columns) C(f32)[M, tiles] = max, aux[M, tiles] = its lowest
 *             column index; logits never reach HBM
 * ------------------------------------------------------------------------- */
int sr_gemm(int dtype, int M, int N, int K, const void* A, int lda, const void* W, int ldw,
            void* C, int ldc, int epilogue, const float* bias, int bn, int32_t* aux,
            sr_stream_t stream);

/* K ranges the bf16 projection (N, K, epilogue) is split into: its small-M
 * mode (live rows <= 128; weights as the 256-row UMMA side, tokens as N)
 * spreads (weight tile, K range) units over the SMs and sums the ranges'
 * fp32 partials in order, and the large-M mode sums one TMEM accumulator
 * per range in the same order, so a row's bits do not depend on how many
 * rows a launch carries.  Depends on the shape and the SM count only. */
int sr_gemm_splits(int N, int K, int epilogue);

/* Live-row threshold of the small-M mode for GEMM plans (sr_gemm, models)
 * created afterwards: -1 = per shape (default: the weight bytes decide),
 * 0 = off, 1..128.  Either mode gives the same bits. */
int sr_set_gemm_swap_max_m(int max_m);

/* ---------------------------------------------------------------------------
 * K1+K2+K6  Verification forward of the target model (Qwen2-style decoder:
 * RMSNorm, RoPE, GQA with QKV bias, SwiGLU, tied or untied lm_head).  The
 * reference only *prices* verification (`_Executor._verify_cost`,
 * sim.py:781-792; `true_token` stands in for the model's output,
 * sim.py:313-320); this computes the target tokens for real.
 *
 * Weights layout (device, `dtype` unless noted f32):
 *   embed, lm_head [vocab, hidden] (lm_head may alias embed); final_norm f32
 *   layer_weights: HOST array of layers*7 device pointers, per layer:
 *     ln1 f32 [hidden]; w_qkv [(q+2kv)*hd, hidden]; b_qkv f32 [(q+2kv)*hd]
 *       (bf16: the q and k rows of w_qkv / b_qkv pair-interleaved per head,
 *       row 2i = dim i, row 2i+1 = dim i + hd/2 -- RoPE runs in the GEMM
 *       epilogue; needs head_dim % 32 == 0);
 *     w_o [hidden, q*hd]; ln2 f32 [hidden];
 *     w_gu [2*inter, hidden], rows interleaved per 32 (16 gate, 16 up);
 *     w_down [hidden, inter]
 * KV cache: [layers, num_pages, 2 (K,V), kv_heads, 64, head_dim], paged
 *   through block_table [max_requests, max_pages_per_req] (int32 page ids).
 *   Zero-initialise it: attention streams whole pages, and the slots past a
 *   sequence's last key must hold finite values (their weight is exactly 0).
 * window_kv: [layers, max_branches, 2, kv_heads, window_max, head_dim] holds
 *   the in-flight KV of Best-of-N drafter branches >= 1 (branch 0 writes its
 *   window straight into the paged cache).
 * ------------------------------------------------------------------------- */
typedef struct sr_seq_info {
  int32_t q_start;  /* first token row of the sequence in the batch */
  int32_t q_len;    /* window positions (k+1 verify, 1 decode, P prefill; 0 = idle) */
  int32_t request;  /* block_table / token-buffer row */
  int32_t ctx_len;  /* keys already committed in the paged cache */
  int32_t branch;   /* -1: KV in place; >= 0: window_kv branch slot */
  int32_t pad0, pad1, pad2;
} sr_seq_info;

typedef struct sr_model_desc {
  int32_t hidden, intermediate, layers, q_heads, kv_heads, head_dim, vocab;
  int32_t dtype;            /* 0 fp32 (CUDA-core parity path), 1 bf16 (tcgen05) */
  float rms_eps;
  int32_t max_pos;          /* rows of rope_cos / rope_sin [max_pos, head_dim/2] f32 */
  int32_t num_pages, page_size, max_requests, max_pages_per_req;
  int32_t max_branches, window_max;
  int32_t max_tokens;       /* token rows per forward */
  int32_t max_seqs;         /* sequences per forward */
  int32_t max_key;          /* largest key position any forward touches */
  int32_t logits_capacity;  /* fp32 logit rows the workspace holds (0 = argmax only) */
  const void* embed;
  const void* lm_head;
  const float* final_norm;
  const void* const* layer_weights;
  const float* rope_cos;
  const float* rope_sin;
  void* kv_cache;
  const int32_t* block_table;
  void* window_kv;
  void* workspace;
  uint64_t workspace_bytes;
} sr_model_desc;

typedef struct sr_forward_args {
  int32_t num_tokens, num_seqs;
  int32_t max_q_len;        /* host upper bound of q_len over the sequences */
  int32_t max_key;          /* host upper bound of ctx_len + q_len - 1 */
  int32_t output;           /* 0: argmax ids (int32 [rows]); 1: fp32 logits [rows, vocab];
                               2: keyed sample at `temperature` (int32 [rows]) */
  int32_t num_logit_rows;   /* rows of logit_rows (ignored when it is NULL) */
  const int32_t* token_ids; /* [num_tokens] */
  const int32_t* positions; /* [num_tokens] */
  const sr_seq_info* seqs;  /* [num_seqs] device */
  const int32_t* logit_rows;/* optional token rows to project (e.g. last prompt token) */
  void* out;
  float* out_val;           /* optional max logit per row (argmax output) */
  float temperature;        /* output 2: T > 0 */
  uint32_t seed;            /* output 2: sampling stream seed */
  const int32_t* live_rows; /* optional device int: the batch's rows [0, *live_rows) are live
                               (sr_build_verify_batch compaction); the bf16 GEMMs skip the rest.
                               Must be written >= 2 kernel launches before the forward on its
                               stream (the GEMMs read it before their dependency wait). */
} sr_forward_args;

/* Keyed Gumbel-max sampling of fp32 logit rows:
 *   id = argmax_v logits[r, v] / T + G(seed, req[r], pos[r], v)
 * with G from Philox4x32-10 keyed by (seed, request), counter (position, v/4).
 * The draw is a pure function of (seed, request, position), so speculative and
 * plain decoding sample identical tokens.  Same noise as the
 * fused lm_head epilogue of sr_model_forward(output = 2). */
int sr_sample_rows(const float* logits, int rows, int vocab, int ld, const int32_t* req, const int32_t* pos,
                   uint32_t seed, float temperature, int32_t* ids, sr_stream_t stream);

/* K2 alone: paged GQA attention of the verify rows described by seqs over
 * one layer of the KV cache (layouts as above; bf16 rows pre-swizzled in
 * 16-byte chunks by slot & 7).  q, out [M, q_heads, head_dim]; partials is
 * fp32 scratch for multi-split blocks. */
int sr_paged_attention(int dtype, const void* q, const void* seqs, int num_seqs, int max_q_len, int max_key,
                       int q_heads, int kv_heads, int head_dim, int layer, int layers, void* kv_cache,
                       int num_pages, const int32_t* block_table, int max_pages, void* window, int branches,
                       int window_max, float* partials, uint64_t partial_floats, void* out,
                       sr_stream_t stream);

/* KV split size of K2 in 64-key tiles (default 32).  Part of the numerics:
 * keep it fixed for a model so verify and decode stay bit-identical. */
int sr_set_attention_split(int tiles);

/* K2 kernel for head_dim 128: 0 = mma.sync (default), 1 = tcgen05/TMEM
 * (attn_tc_kernel).  Part of the numerics like the split size: set it once
 * per process, before any forward. */
int sr_set_attention_tc(int on);

uint64_t sr_model_workspace_bytes(const sr_model_desc* desc);
int sr_model_create(const sr_model_desc* desc, void** handle);
int sr_model_destroy(void* handle);
int sr_model_forward(void* handle, const sr_forward_args* args, sr_stream_t stream);

/* Launch timing: while enabled, every forward brackets its launches with
 * CUDA events on the launching stream.  A call with ms_out/count_out set
 * waits for the recorded work and returns per-category totals over
 * [qkv, o, gate_up, down, lm_head, attention, other, attention_combine]
 * (8 entries), then
 * clears the record and sets the enable state for the following forwards. */
int sr_model_profile(void* handle, int enable, float* ms_out, int32_t* count_out);

/* ---------------------------------------------------------------------------
 * K3  Acceptance + Best-of-N + write-back (model mode), ONE kernel.  Replaces
 * `_verify_prefix` / `_apply_outcome` / `commit` (sim.py:977-1042, 340-353)
 * with real tokens, and the Best-of-N first-finisher (sim.py:340-361) with an
 * in-forward longest-accepted-prefix select over N drafters per request.
 *
 * seqs [B*N] (drafter n of request b is sequence b*N+n); token_ids [M] are
 * the verify inputs (slot j+1 holds draft d_{j+1}); target [M] the target
 * model's token per row.  Commits into tokens [B, tok_stride] at seq_len,
 * advances seq_len / gen_len (capped by max_new), and writes outcome
 * [B*N, 4] (16-byte aligned) = (proposed, accepted, committed, wasted) and
 * bon [B] (winner, -1 = request inactive).  When the winner verified in a
 * drafter branch (N > 1), its committed slots' KV is copied from the
 * model's branch window into the paged cache in the same kernel; `model`
 * (the sr_model_create handle) NULL skips that write-back (N == 1, or every
 * sequence verified in place, branch < 0).
 * ------------------------------------------------------------------------- */
int sr_accept_commit(void* model, int num_requests, int num_drafters, const void* seqs,
                     const int32_t* token_ids, const int32_t* target, int32_t* tokens, int64_t tok_stride,
                     int32_t* seq_len, int32_t* gen_len, const int32_t* max_new, int bonus_token,
                     int32_t* outcome, int32_t* bon, sr_stream_t stream);

/* ---------------------------------------------------------------------------
 * K3, rejection-sampling mode (distribution-preserving speculative sampling,
 * Leviathan et al.; semantics of vLLM 0.22 rejection_sampler.py:708-760,
 * SURVEY §8c) for ONE stochastic drafter per request (N = 1): the model-mode
 * counterpart of the reference's keyed acceptance draw (sim.py:322-336) when
 * the drafter samples its window from its own distribution q.
 *
 * p_logits [M, ldp] f32: the target's verify-row logits (row q_start + j).
 * q_logits f32: the drafter's logits behind draft j of request b at
 *   q_logits + (j * B + b) * ldq  ([k, B, ldq]).
 * Draft j is accepted iff u < p_j(d)/q_j(d) (u keyed by seed, request,
 * position); the first rejected slot commits a sample of
 * norm(max(0, p_j - q_j)); a full accept commits the bonus (if on) as the
 * target's keyed sample of p_n; an empty window commits the keyed sample of
 * p_0.  p, q = softmax(logits / temperature).  Commits, outcome rows and bon
 * as sr_accept_commit.  stats: f32 workspace [M, 4] (16-byte aligned).
 * ------------------------------------------------------------------------- */
int sr_accept_rejection(int num_requests, int k, const void* seqs, const int32_t* token_ids,
                        const float* p_logits, int64_t ldp, const float* q_logits, int64_t ldq, int vocab,
                        float temperature, uint32_t seed, int32_t* tokens, int64_t tok_stride,
                        int32_t* seq_len, int32_t* gen_len, const int32_t* max_new, int bonus_token,
                        float* stats, int32_t* outcome, int32_t* bon, sr_stream_t stream);

/* Floats of the `stats` workspace sr_accept_rejection needs: per verify row
 * (lse_p, lse_q, log p(d), log q(d)), then 16 per-request vocabulary-chunk
 * (value, index) partials of the extra-token sample. */
uint64_t sr_accept_rejection_workspace_floats(int num_requests, int k);

/* Host-facing step prologue (RolloutEngine.capture_io): max_new[b] =
 * budget_host[b] read zero-copy from PINNED host memory (clamped later to the
 * slot capacity by sr_build_verify_batch) and seq_before[b] = seq_len[b].
 * Replaces the H2D copy of the reference-facing step's inputs
 * (sim.py:983-1042 budgets per request). */
int sr_io_begin(int num_requests, const int32_t* budget_host, int32_t* max_new, const int32_t* seq_len,
                int32_t* seq_before, sr_stream_t stream);

/* Host-facing step result (RolloutEngine.capture_io): out [B, 4N + width] =
 * the N drafters' outcome rows of request b (4N ints) then
 * tokens[b, seq_before[b] + j] for j < width (clamped to the row) -- the
 * committed window of the step.  `out` may be device memory or pinned host
 * memory (written zero-copy: the step's D2H without a copy-engine node). */
int sr_pack_results(int num_requests, int num_drafters, int width, const int32_t* outcome,
                    const int32_t* tokens, int64_t tok_stride, const int32_t* seq_before, int32_t* out,
                    sr_stream_t stream);

/* Reference-acceptance drafter: for output position
 * g = gen_len[b] + j propose truth[b, g] (the target's own greedy token) when
 * uniforms[b, g] < accept_p[b] -- the reference's keyed `accept_draw`
 * (sim.py:322-336) -- else (truth + 1) % vocab.  Exact-match verification then
 * accepts exactly the reference's `_verify_prefix` run (sim.py:977-981).
 * drafts [B, k] (-1 padded), ndraft [B] = min(k, truth_len - gen_len). */
int sr_synthetic_draft(int num_requests, int k, const int32_t* truth, int64_t truth_stride,
                       const int32_t* truth_len, const double* uniforms, int64_t u_stride,
                       const double* accept_p, const int32_t* gen_len, int vocab, int32_t* drafts,
                       int32_t* ndraft, sr_stream_t stream);

/* K5 small-model drafter batches (drafting methods `draft-0.5b`/`draft-1.5b`,
 * scenarios.py:25-29, priced per token at sim.py:883-892).  Step 0: rows
 * [b*(k+2), +k+2) belong to request b; steps >= 1: row b (run the forward
 * over the first B rows).  step 0: catch-up of the committed tokens the
 * drafter has not cached, [dkv_len, seq_len) (advances dkv_len), logits at
 * the last one; step j in [1, k): decode the previous draft; step k: file the
 * last output and write ndraft.  prev_out [B] is the previous forward's
 * output and becomes draft (step-1).  drafts [B, k], ndraft [B].  key_pos
 * [B] (optional): the output position of each request's logit row (the
 * sampling key of a drafter that samples its own window, sr_sample_rows). */
int sr_draft_model_batch(int num_requests, int k, int step, const int32_t* tokens, int64_t tok_stride,
                         const int32_t* seq_len, const int32_t* gen_len, const int32_t* max_new,
                         int32_t* dkv_len, const int32_t* prev_out, int32_t* drafts, int32_t* ndraft,
                         int32_t* token_ids, int32_t* positions, void* seqs, int32_t* logit_rows,
                         int32_t* key_pos, sr_stream_t stream);

/* Next verify batch from device state: for drafter n of request b, rows
 * [(b*N+n)*(k+1), +nd+1) = last committed token then the drafts.  drafts
 * [N, B, k] / ndraft [N, B] are drafter-major (each drafter kernel writes its
 * own [B, k] block); both NULL = plain decode; ndraft < 0 = the request has
 * no window this round (decoupled gap round, sim.py:1076-1080).  window
 * [B] (optional): per-request window w_r <= k, the mixed-window batch of
 * request-level reconfiguration (planner.py:223-272); NULL = k for all.
 * max_new_cap [B] (optional): max_new is clamped to it IN PLACE first --
 * the token row and KV pages of request b hold max_new_cap[b] outputs, and a
 * retired request (cap = gen_len) stays retired whatever budget the host
 * copies in.
 * active [N, B] (optional): drafter n proposes for request b only where
 * active[n*B + b] != 0 (Best-of-N drafters assigned to tail requests on
 * drain, bon.py:79-139); NULL = every drafter for every request.
 * live_rows (optional, device int): COMPACT the batch instead -- sequence
 * s = b*N+n keeps its SeqInfo slot but its rows are packed back to back
 * (q_start = exclusive prefix sum of q_len over s), so finished requests and
 * unproposed draft slots take no rows; *live_rows = rows used.  Pass it on to
 * sr_forward_args.live_rows and the GEMMs skip the dead tiles. */
int sr_build_verify_batch(int num_requests, int num_drafters, int k, const int32_t* tokens,
                          int64_t tok_stride, const int32_t* seq_len, const int32_t* gen_len,
                          int32_t* max_new, const int32_t* max_new_cap, const int32_t* drafts,
                          const int32_t* ndraft,
                          const int32_t* window, const int32_t* active, int32_t* token_ids,
                          int32_t* positions, void* seqs, int32_t* live_rows, sr_stream_t stream);

/* ---------------------------------------------------------------------------
 * a6  Decoupled speculation round bookkeeping (pipeline depth 2; replaces the
 * decoupled branch of `_Executor.begin_round` sim.py:860-917 and
 * `_end_decoupled` sim.py:1051-1092 for the per-request state), one thread
 * per request.  Drafter side: prep (successor's first output position g0
 * and context length ctx behind the in-flight window), post (cap the drafted
 * window at the remaining budget, append it to the token mirror, stage it
 * for the verifier), apply (fold the verifier's decision: accepted prefix +
 * corrected token, advance, roll a model drafter's KV length back, the new
 * in-flight count).  Verifier side: post (after K3: the decision rows and the
 * k+1 committed-token slots to send back), receive (admit the drafter's new
 * windows as pending, or drop them and charge their size as depth-2 waste
 * when the predecessor was rejected).  dkv_len may be NULL.
 * ------------------------------------------------------------------------- */
int sr_decoupled_draft_prep(int B, const int32_t* seq_len, const int32_t* gen_len, const int32_t* inflight,
                            int32_t* g0, int32_t* ctx, sr_stream_t stream);
int sr_decoupled_draft_post(int B, int k, int64_t stride, const int32_t* max_new, const int32_t* g0,
                            const int32_t* ctx, const int32_t* drafts, int32_t* nd, int32_t* tokens,
                            int32_t* out_drafts, int32_t* out_nd, sr_stream_t stream);
int sr_decoupled_draft_apply(int B, int k, int64_t stride, const int32_t* in_verified, const int32_t* in_accepted,
                             const int32_t* in_committed, const int32_t* in_ctoks, const int32_t* out_nd,
                             int32_t* inflight, int32_t* tokens, int32_t* seq_len, int32_t* gen_len,
                             int32_t* dkv_len, sr_stream_t stream);
int sr_decoupled_verify_post(int B, int k, int64_t stride, const int32_t* outcome, const int32_t* bon,
                             const int32_t* tokens, const int32_t* seq_before, int32_t* rows, int32_t* out_verified,
                             int32_t* out_accepted, int32_t* out_committed, int32_t* out_ctoks, sr_stream_t stream);
int sr_decoupled_verify_receive(int B, int k, const int32_t* out_verified, const int32_t* out_accepted,
                                const int32_t* out_committed, const int32_t* in_drafts, const int32_t* in_nd,
                                int32_t* rows, int32_t* pending, int32_t* pending_nd, sr_stream_t stream);

#ifdef __cplusplus
}
#endif

#endif /* SPECROLLOUT_B200_H_ */
