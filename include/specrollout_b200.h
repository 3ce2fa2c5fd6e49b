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

/* ---------------------------------------------------------------------------
 * K1 building block: C = A[M,K] . W[N,K]^T with a fused epilogue (the
 * projections of the target model's verification forward; no reference
 * counterpart -- the reference has no model).
 *   dtype 1: bf16 A/W on tcgen05 tensor cores (TMA + TMEM), bn = 128|256|0
 *   dtype 0: fp32 A/W on CUDA cores (parity path), bn ignored
 * epilogue 0: C = acc + bias (bf16; f32 when dtype 0)
 *          1: C(f32) += acc                      (residual stream)
 *          2: C[M, N/2] = silu(gate) * up, W rows interleaved per 32:
 *             16 gate rows then the 16 matching up rows
 *          3: C(f32) = acc + bias                (logits)
 * ------------------------------------------------------------------------- */
int sr_gemm(int dtype, int M, int N, int K, const void* A, int lda, const void* W, int ldw,
            void* C, int ldc, int epilogue, const float* bias, int bn, sr_stream_t stream);

#ifdef __cplusplus
}
#endif

#endif /* SPECROLLOUT_B200_H_ */
