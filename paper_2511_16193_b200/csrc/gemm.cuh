// K1 verify GEMMs: D[M,N] = A[M,K] . W[N,K]^T with fused epilogues.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cstdint>

#include "sampling.cuh"

namespace sr {

enum GemmEpilogue : int {
  kEpiStoreBf16 = 0,    // C bf16 = acc (+ bias)
  kEpiResidualF32 = 1,  // C f32 += acc            (residual stream)
  kEpiSwiGLU = 2,       // C bf16 [M, N/2] = silu(gate) * up; W rows interleaved
                        //   in blocks of 32: 16 gate rows then 16 up rows
  kEpiStoreF32 = 3,     // C f32 = acc (+ bias)     (logits)
  kEpiArgmax = 4,       // per (row, N tile): max value -> C f32 [M, tiles],
                        //   its lowest column index -> aux [M, tiles]
  kEpiResidualNorm = 5, // C f32 += acc, then RMSNorm producer side (NormArgs):
                        //   h[row, col] = bf16(C * w[col]), ssq[row, n tile] = sum C^2
  kEpiQkvRope = 6,      // qkv projection + bias, RoPE on q/k, q -> q_out, k/v -> paged KV
                        //   cache (RopeArgs); q/k weight rows pair-interleaved (d, d + hd/2)
};

// RoPE + KV scatter fused into the qkv GEMM epilogue (kEpiQkvRope).  The q and
// k rows of W_qkv (and the bias) are stored pair-interleaved per head --
// output column 2i holds dim i, column 2i+1 dim i + hd/2 -- so every 32-column
// epilogue chunk holds 16 complete rotation pairs of one head.  Per row the
// epilogue needs the position and where the row's K/V live (a paged-cache
// slot or a drafter-branch window slot), precomputed once per forward
// (kv_rows): kv_dst = element offset of the row's K block (kv head 0) inside
// this layer's cache or window, kv_info = slot | window << 16, or -1 for a
// padding row (no writes).
struct RopeArgs {
  const int32_t* pos = nullptr;      // [M]
  const int64_t* kv_dst = nullptr;   // [M]
  const int32_t* kv_info = nullptr;  // [M]
  const float* cos = nullptr;        // [max_pos, hd / 2]
  const float* sin = nullptr;
  __nv_bfloat16* q_out = nullptr;    // [M, nq, hd]
  __nv_bfloat16* cache = nullptr;    // this layer's paged cache
  __nv_bfloat16* window = nullptr;   // this layer's branch windows
  int nq = 0, nkv = 0, hd = 0, page = 64, window_max = 0;
};

// Fused RMSNorm.  norm(x) W = r (x o w) W with r = rsqrt(mean(x^2) + eps) per
// row, so the residual GEMM that produces x (kEpiResidualNorm) writes
// bf16(x o w) as the next GEMM's A operand plus partial sums of x^2 per
// 128-column group, and the consuming GEMM scales each accumulator row by r
// (summing the partials in column order) before its bias / SwiGLU / argmax.
// No separate normalization pass touches the residual stream.  A group's
// partial has one fixed form, whatever tile or GEMM mode produced it: per
// 32-column chunk s_q = fma chain over columns 4q..4q+3 (q = 0..7), chunk =
// ((s0 + s1) + (s2 + s3)) + ((s4 + s5) + (s6 + s7)); group = the chunks
// summed in column order.  Producer tiles are 128 or 256 wide.
constexpr int kSsqCols = 128;
struct NormArgs {
  const float* ssq_in = nullptr;  // consumer: [M, parts_in] (nullptr: no row scaling)
  int parts_in = 0;
  float hdim = 0.0f, eps = 0.0f;
  __nv_bfloat16* h_out = nullptr;  // producer (kEpiResidualNorm): [M, ld_h]
  const float* w = nullptr;        // norm weights [N]
  float* ssq_out = nullptr;        // [M, ceil(N / kSsqCols)]
  int ld_h = 0;
};

// Host: encode a 2D bf16 tensor map (inner dim contiguous) with 128B swizzle.
int make_tmap_kv_pages(CUtensorMap* map, const void* cache, uint64_t blocks);
int make_tmap_bf16(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer,
                   uint64_t row_bytes, uint32_t box_inner, uint32_t box_outer);

// Small-M ("swap") mode of the CTA-pair kernel, taken on device when the live
// row count is <= max_m: the pair computes C^T = W A^T -- 256 weight rows as
// the UMMA M side (128 per CTA), the <= 128 live tokens as N -- so a launch
// streams weights on many SMs instead of padding tokens to 256-row tiles.
// Long-K projections split K into `splits` contiguous ranges (one pair per
// (256-row weight tile, range)); fp32 partials go through `ws` and the last
// pair to arrive on a tile sums them in range order.  The pair mode keeps
// one TMEM accumulator per range and sums them in the same order, so both
// modes produce identical bits for every row (batch invariance across
// live-row counts).  `splits` is a function of (N, K) only.
constexpr int kSwapRows = 128;
// The small-M mode's tensor maps live in device memory (a 640-byte block per
// plan, uploaded once) so the kernel parameter block stays small: launch
// cost grows with it.
struct SwapMaps {
  CUtensorMap w;         // W [N, K] as (64, rows, K / 64), box (64, 128, 2)
  CUtensorMap x[4];      // A [cap, K], box (64, 16 (g + 1), 2): token rows per CTA
};
struct SwapArgs {
  const SwapMaps* maps = nullptr;  // device copy of the plan's maps
  float* ws = nullptr;   // [splits][kSwapRows][N] fp32 partials
  int32_t* cnt = nullptr;  // [2 ceil(N / 256)] arrival counters, zero between launches
  int splits = 1;
  int max_m = 0;         // 0: swap mode off
  int flags = 1;         // bit 0: stage the first weight blocks before griddepcontrol.wait
#ifdef SR_GEMM_TRACE
  unsigned long long* trace = nullptr;  // measurement builds: per-CTA phase stamps
#endif
};

struct GemmPlan {
  CUtensorMap a, b;
  SwapArgs sw;
  SwapMaps sw_maps;   // host copy; the owner uploads it and sets sw.maps
  int M, N, K, bn, epi;
  bool pair;          // CTA-pair (cta_group::2, 256-row tiles) kernel
  int mc;             // pairs per cluster sharing (multicasting) A: 1 | 2
  int kc;             // 64-wide k chunks per pipeline stage (pair kernel): 1 | 2
  void* c;
  int ldc;
  const float* bias;
  int32_t* aux;
  SampleArgs sample;  // argmax epilogue: keyed Gumbel sampling when inv_temp > 0
  NormArgs norm;      // fused RMSNorm (consumer scaling / producer outputs)
  RopeArgs rope;      // fused RoPE + KV scatter (kEpiQkvRope)
  const int32_t* m_live = nullptr;  // device live-row count (compacted batch); nullptr = M
};

// Build a plan (tensor maps) once; launch many times (graph-capturable).
// bn > 0: single-CTA kernel with that tile width (128 | 256); bn < 0: CTA-pair
// kernel with width -bn (multiple of 16, <= 256), or width -bn - 1024 with
// two pairs per cluster multicasting A (bn < -1024); bn == 0: choose from
// (M, N, K) -- M is the plan's capacity, so the choice (and hence the
// accumulation order) never depends on how many rows a launch carries.
int gemm_bf16_plan(GemmPlan* plan, int M, int N, int K, const __nv_bfloat16* A, int lda,
                   const __nv_bfloat16* W, int ldw, void* C, int ldc, int epi,
                   const float* bias, int bn, int32_t* aux = nullptr);
// Launch with the plan's tensor maps; m_override >= 0 replaces plan.M (rows
// beyond it are computed from stale memory and discarded).
int gemm_bf16_launch(const GemmPlan& plan, cudaStream_t stream, int m_override = -1);
int gemm_num_n_tiles(int N, int bn);
// Workspace (bytes) the plan's swap mode needs: partials + counters.
size_t gemm_swap_ws_floats(const GemmPlan& plan);
size_t gemm_swap_cnt_ints(const GemmPlan& plan);
// Number of K ranges a (N, K) projection is split into (see SwapArgs).
int gemm_splits(int N, int K, int epi);

// fp32 parity path (CUDA cores, fixed k order): same epilogues, f32 activations.
int gemm_f32(int M, int N, int K, const float* A, int lda, const float* W, int ldw, void* C,
             int ldc, int epi, const float* bias, cudaStream_t stream);

}  // namespace sr
