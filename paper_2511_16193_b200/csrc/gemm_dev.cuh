#pragma once
// K1: verify-forward GEMMs on the 5th-gen tensor cores (device code; included
// by gemm.cu and the per-tile-width translation units gemm_pair_bn*.cu).
//
// The target model's verification forward over B prompts x N drafters x
// (k+1) positions is a dense contraction of the M verify
// rows with every weight matrix.  This kernel is a persistent,
// warp-specialized tcgen05 GEMM:
//
//   warp 0      TMA producer: 128x64 activation tile + BNx64 weight tile per
//               stage into 128B-swizzled smem, mbarrier expect_tx.
//   warp 1      TMEM owner + MMA issuer: one thread issues
//               tcgen05.mma.cta_group::1.kind::f16 (M=128, N=BN, K=16) x4 per
//               stage into a double-buffered fp32 TMEM accumulator and
//               commits smem slots / finished accumulators to mbarriers.
//   warps 2..5  epilogue: tcgen05.ld 32x32b.x32 -> registers -> fused
//               bias / residual-add / SwiGLU / cast -> global.
//
// Tiles are walked M-fastest so the CTAs resident at once share weight
// tiles through L2 (weights are the dominant HBM stream at small M).  The
// accumulation order over K is fixed by the tile config, which depends only
// on (N, K): a row's result is independent of M and of its position in the
// batch, which makes speculative verify and plain decode bit-identical.
#include "common.cuh"
#include "gemm.cuh"
#include "layers.cuh"
#include "sampling.cuh"
#include "sm100.cuh"

#include <cudaTypedefs.h>
#include <cstdlib>

namespace sr {

int num_sms();


namespace {

constexpr int kBM = 128, kBK = 64;
constexpr int kThreads = 192;

// Measurement builds (-DSR_GEMM_TRACE): %globaltimer stamps per CTA and
// event of the last launch, read back with sr_debug_gemm_trace.
#ifdef SR_GEMM_TRACE
#define GT(ev) (sw.trace ? (void)(sw.trace[blockIdx.x * 8 + (ev)] = sm100::global_timer_ns()) : (void)0)
#else
#define GT(ev) ((void)0)
#endif

template <int BN>
struct GemmCfg {
  static constexpr int kStages = BN == 256 ? 4 : 6;
  static constexpr uint32_t kABytes = kBM * kBK * 2;
  static constexpr uint32_t kBBytes = BN * kBK * 2;
  static constexpr uint32_t kStageBytes = kABytes + kBBytes;
  static constexpr uint32_t kTmemCols = 2 * BN;  // two accumulator buffers
  static constexpr size_t kSmem = 1024 + (size_t)kStages * kStageBytes + 256;
};

__device__ __forceinline__ float bf16_lo(uint32_t v) { return __uint_as_float(v << 16); }

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

__device__ __forceinline__ float silu(float g) { return g / (1.0f + __expf(-g)); }

// Epilogue for W (16 or 32) consecutive accumulator columns [col, col+W) of one row.
// Element offset of dim d of KV row `slot` (rows [slot][hd], bf16 chunk swizzle).
__device__ __forceinline__ int64_t kv_elem(int slot, int d, int hd) {
  return (int64_t)slot * hd + kv_phys<__nv_bfloat16>(slot, d);
}

__device__ __forceinline__ uint4 pack8_bf16(const float* f) {
  uint4 w;
  w.x = pack_bf16(f[0], f[1]);
  w.y = pack_bf16(f[2], f[3]);
  w.z = pack_bf16(f[4], f[5]);
  w.w = pack_bf16(f[6], f[7]);
  return w;
}

// Per-row inputs of the RoPE epilogue, loaded before the accumulator is ready.
struct RopeRow {
  int info = -1, pos = 0;
  int64_t dst = 0;
};

__device__ __forceinline__ RopeRow rope_row(const RopeArgs& ra, int row, int M) {
  RopeRow r;
  if (row < M) {
    r.info = ra.kv_info[row];
    r.pos = ra.pos[row];
    r.dst = ra.kv_dst[row];
  }
  return r;
}

// cos / sin of the 16 rotation pairs a q/k chunk at column `col` needs for
// this row (loaded one chunk ahead of their use).
struct RopeTab {
  float4 c[4], s[4];
};

__device__ __forceinline__ RopeTab rope_tab(const RopeArgs& ra, const RopeRow& rr, int col) {
  RopeTab tb;
  const int hd = ra.hd, half = hd >> 1;
  if (rr.info >= 0 && col < (ra.nq + ra.nkv) * hd) {
    const int d0 = (col % hd) >> 1;
    const float4* c4 = reinterpret_cast<const float4*>(ra.cos + (int64_t)rr.pos * half + d0);
    const float4* s4 = reinterpret_cast<const float4*>(ra.sin + (int64_t)rr.pos * half + d0);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      tb.c[q] = c4[q];
      tb.s[q] = s4[q];
    }
  } else {
#pragma unroll
    for (int q = 0; q < 4; ++q) tb.c[q] = tb.s[q] = make_float4(0, 0, 0, 0);
  }
  return tb;
}

// The rotation with explicit rounding (no contraction choice left to the
// compiler): both GEMM modes and their epilogue layouts round identically.
__device__ __forceinline__ float rope_y1(float x1, float x2, float c, float s) {
  return __fmaf_rn(x1, c, -__fmul_rn(x2, s));
}
__device__ __forceinline__ float rope_y2(float x1, float x2, float c, float s) {
  return __fmaf_rn(x2, c, __fmul_rn(x1, s));
}

// kEpiQkvRope for one 32-column chunk of one row (see RopeArgs).
__device__ __forceinline__ void qkv_rope_chunk(const float* f, int row, int col, const RopeArgs& ra,
                                               const RopeRow& rr, const RopeTab& tb) {
  const int info = rr.info;
  if (info < 0) return;  // padding row of the verify batch
  const int hd = ra.hd, half = hd >> 1;
  const int hq = ra.nq * hd, hk = ra.nkv * hd;
  const bool win = (info >> 16) & 1;
  const int slot = info & 0xFFFF;
  const int rows = win ? ra.window_max : ra.page;
  __nv_bfloat16* kbase = (win ? ra.window : ra.cache) + rr.dst;
  if (col < hq + hk) {
    const int hc = col % hd, d0 = hc >> 1;  // 16 pairs (d0 + i, d0 + i + half)
    float y1[16], y2[16];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float4 c = tb.c[q], s = tb.s[q];
      const float cs[4] = {c.x, c.y, c.z, c.w}, sn[4] = {s.x, s.y, s.z, s.w};
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = 4 * q + u;
        const float x1 = f[2 * i], x2 = f[2 * i + 1];
        y1[i] = rope_y1(x1, x2, cs[u], sn[u]);
        y2[i] = rope_y2(x1, x2, cs[u], sn[u]);
      }
    }
    if (col < hq) {
      __nv_bfloat16* q = ra.q_out + ((int64_t)row * ra.nq + col / hd) * hd;
      *reinterpret_cast<uint4*>(q + d0) = pack8_bf16(y1);
      *reinterpret_cast<uint4*>(q + d0 + 8) = pack8_bf16(y1 + 8);
      *reinterpret_cast<uint4*>(q + d0 + half) = pack8_bf16(y2);
      *reinterpret_cast<uint4*>(q + d0 + half + 8) = pack8_bf16(y2 + 8);
    } else {
      __nv_bfloat16* k = kbase + (int64_t)((col - hq) / hd) * rows * hd;
      *reinterpret_cast<uint4*>(k + kv_elem(slot, d0, hd)) = pack8_bf16(y1);
      *reinterpret_cast<uint4*>(k + kv_elem(slot, d0 + 8, hd)) = pack8_bf16(y1 + 8);
      *reinterpret_cast<uint4*>(k + kv_elem(slot, d0 + half, hd)) = pack8_bf16(y2);
      *reinterpret_cast<uint4*>(k + kv_elem(slot, d0 + half + 8, hd)) = pack8_bf16(y2 + 8);
    }
    return;
  }
  // V: natural column order, 32 dims of one head
  const int vc = col - hq - hk, hc = vc % hd;
  __nv_bfloat16* vb = kbase + (int64_t)ra.nkv * rows * hd + (int64_t)(vc / hd) * rows * hd;
#pragma unroll
  for (int q = 0; q < 4; ++q) *reinterpret_cast<uint4*>(vb + kv_elem(slot, hc + 8 * q, hd)) = pack8_bf16(f + 8 * q);
}

// kSsqCols partial form (gemm.cuh): fma chain over 4 columns, then a fixed tree.
__device__ __forceinline__ float quad_ssq(float4 a) {
  float s = a.x * a.x;
  s = fmaf(a.y, a.y, s);
  s = fmaf(a.z, a.z, s);
  return fmaf(a.w, a.w, s);
}
__host__ __device__ __forceinline__ int ssq_parts(int N) { return (N + kSsqCols - 1) / kSsqCols; }
// Add a 32-column chunk's partial to its 128-column group; the group's last
// chunk (or the row's) writes it.  gss starts at 0 (0 + c0 == c0 exactly).
__device__ __forceinline__ void ssq_accum(float& gss, float chunk, int col, int N, float* row_parts, bool ok) {
  gss += chunk;
  if ((col + 32) % kSsqCols == 0 || col + 32 >= N) {
    if (ok) row_parts[col / kSsqCols] = gss;
    gss = 0.0f;
  }
}
__device__ __forceinline__ float tree8(const float (&s)[8]) {
  return ((s[0] + s[1]) + (s[2] + s[3])) + ((s[4] + s[5]) + (s[6] + s[7]));
}

template <int EPI, int W = 32>
__device__ __forceinline__ void epilogue_chunk(const uint32_t* v, int row, int col, int M, int N, void* C,
                                               int ldc, const float* bias, const NormArgs& na, float& ss,
                                               const RopeArgs& ra, const RopeRow& rr = RopeRow{}) {
  if (row >= M) return;
  if constexpr (EPI == kEpiArgmax) return;  // handled in the tile loop
  if constexpr (EPI == kEpiQkvRope) {
    static_assert(EPI != kEpiQkvRope || W == 32, "RoPE chunks are 16 pairs");
    float f[W];
#pragma unroll
    for (int i = 0; i < W; ++i) f[i] = __uint_as_float(v[i]);
    if (bias != nullptr) {  // 32 consecutive floats, 128-byte aligned: eight 16-byte loads
      const float4* b4 = reinterpret_cast<const float4*>(bias + col);
#pragma unroll
      for (int q = 0; q < W / 4; ++q) {
        const float4 b = b4[q];
        f[4 * q] += b.x; f[4 * q + 1] += b.y; f[4 * q + 2] += b.z; f[4 * q + 3] += b.w;
      }
    }
    qkv_rope_chunk(f, row, col, ra, rr, rope_tab(ra, rr, col));
    return;
  }
  float f[W];
#pragma unroll
  for (int i = 0; i < W; ++i) f[i] = __uint_as_float(v[i]);
  const bool full = col + W <= N;
  if constexpr (EPI == kEpiStoreBf16 || EPI == kEpiStoreF32) {
    if (bias != nullptr) {
#pragma unroll
      for (int i = 0; i < W; ++i) f[i] += (col + i < N) ? bias[col + i] : 0.0f;
    }
  }
  if constexpr (EPI == kEpiStoreBf16) {
    __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(C) + (int64_t)row * ldc + col;
    if (full) {
#pragma unroll
      for (int q = 0; q < W / 8; ++q) {
        uint4 w;
        w.x = pack_bf16(f[8 * q + 0], f[8 * q + 1]);
        w.y = pack_bf16(f[8 * q + 2], f[8 * q + 3]);
        w.z = pack_bf16(f[8 * q + 4], f[8 * q + 5]);
        w.w = pack_bf16(f[8 * q + 6], f[8 * q + 7]);
        reinterpret_cast<uint4*>(out)[q] = w;
      }
    } else {
      for (int i = 0; i < W && col + i < N; ++i) out[i] = __float2bfloat16_rn(f[i]);
    }
  } else if constexpr (EPI == kEpiStoreF32) {
    float* out = reinterpret_cast<float*>(C) + (int64_t)row * ldc + col;
    if (full) {
#pragma unroll
      for (int q = 0; q < W / 4; ++q)
        reinterpret_cast<float4*>(out)[q] = make_float4(f[4 * q], f[4 * q + 1], f[4 * q + 2], f[4 * q + 3]);
    } else {
      for (int i = 0; i < W && col + i < N; ++i) out[i] = f[i];
    }
  } else if constexpr (EPI == kEpiResidualF32) {
    float* out = reinterpret_cast<float*>(C) + (int64_t)row * ldc + col;
    if (full) {
#pragma unroll
      for (int q = 0; q < W / 4; ++q) {
        float4 r = reinterpret_cast<float4*>(out)[q];
        r.x += f[4 * q]; r.y += f[4 * q + 1]; r.z += f[4 * q + 2]; r.w += f[4 * q + 3];
        reinterpret_cast<float4*>(out)[q] = r;
      }
    } else {
      for (int i = 0; i < W && col + i < N; ++i) out[i] += f[i];
    }
  } else if constexpr (EPI == kEpiResidualNorm) {
    // ss = this 32-column chunk's partial sum of squares (kSsqCols form)
    static_assert(EPI != kEpiResidualNorm || W == 32, "norm partials are per 32-column chunk");
    float* out = reinterpret_cast<float*>(C) + (int64_t)row * ldc + col;
    __nv_bfloat16* hr = na.h_out + (int64_t)row * na.ld_h + col;
    float sq[8];
    if (full) {
#pragma unroll
      for (int q = 0; q < W / 8; ++q) {
        float4 a = reinterpret_cast<float4*>(out)[2 * q];
        float4 b = reinterpret_cast<float4*>(out)[2 * q + 1];
        a.x += f[8 * q]; a.y += f[8 * q + 1]; a.z += f[8 * q + 2]; a.w += f[8 * q + 3];
        b.x += f[8 * q + 4]; b.y += f[8 * q + 5]; b.z += f[8 * q + 6]; b.w += f[8 * q + 7];
        reinterpret_cast<float4*>(out)[2 * q] = a;
        reinterpret_cast<float4*>(out)[2 * q + 1] = b;
        sq[2 * q] = quad_ssq(a);
        sq[2 * q + 1] = quad_ssq(b);
        const float4 wa = reinterpret_cast<const float4*>(na.w + col)[2 * q];
        const float4 wb = reinterpret_cast<const float4*>(na.w + col)[2 * q + 1];
        uint4 hv;
        hv.x = pack_bf16(a.x * wa.x, a.y * wa.y);
        hv.y = pack_bf16(a.z * wa.z, a.w * wa.w);
        hv.z = pack_bf16(b.x * wb.x, b.y * wb.y);
        hv.w = pack_bf16(b.z * wb.z, b.w * wb.w);
        reinterpret_cast<uint4*>(hr)[q] = hv;
      }
    } else {
#pragma unroll
      for (int q = 0; q < 8; ++q) sq[q] = 0.0f;
      for (int i = 0; i < W && col + i < N; ++i) {
        const float xn = out[i] + f[i];
        out[i] = xn;
        sq[i >> 2] = fmaf(xn, xn, sq[i >> 2]);
        hr[i] = __float2bfloat16_rn(xn * na.w[col + i]);
      }
    }
    ss = tree8(sq);
  } else if constexpr (EPI == kEpiSwiGLU) {
    static_assert(EPI != kEpiSwiGLU || W == 32, "SwiGLU pairs 16 gate + 16 up columns");
    // columns [col, col+16) are gate, [col+16, col+32) the matching up rows
    __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(C) + (int64_t)row * ldc + col / 2;
    if (full) {
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        uint4 w;
        w.x = pack_bf16(silu(f[8 * q + 0]) * f[16 + 8 * q + 0], silu(f[8 * q + 1]) * f[16 + 8 * q + 1]);
        w.y = pack_bf16(silu(f[8 * q + 2]) * f[16 + 8 * q + 2], silu(f[8 * q + 3]) * f[16 + 8 * q + 3]);
        w.z = pack_bf16(silu(f[8 * q + 4]) * f[16 + 8 * q + 4], silu(f[8 * q + 5]) * f[16 + 8 * q + 5]);
        w.w = pack_bf16(silu(f[8 * q + 6]) * f[16 + 8 * q + 6], silu(f[8 * q + 7]) * f[16 + 8 * q + 7]);
        reinterpret_cast<uint4*>(out)[q] = w;
      }
    }
  }
}

// Vocabulary argmax over W accumulator columns; with sampling on, each logit
// is scaled by 1/T and perturbed by its keyed Gumbel noise first (keyed
// Gumbel-max = exact sample of softmax(logits / T)).  Strict '>' in column
// order keeps the lowest index on ties.
template <int W>
__device__ __forceinline__ void argmax_chunk(const uint32_t* v, int col, int N, int row, int M,
                                             const SampleArgs& sa, float& best, int& best_idx) {
  if (sa.inv_temp > 0.0f) {
    if (row >= M) return;
    const int rq = sa.req[row], ps = sa.pos[row];
#pragma unroll
    for (int i = 0; i < W; i += 4) {
      float g[4];
      gumbel4(sa.seed, rq, ps, (col + i) >> 2, g);
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const float f = __uint_as_float(v[i + t]) * sa.inv_temp + g[t];
        if (col + i + t < N && f > best) { best = f; best_idx = col + i + t; }
      }
    }
    return;
  }
#pragma unroll
  for (int i = 0; i < W; ++i) {
    const float f = __uint_as_float(v[i]);
    if (col + i < N && f > best) { best = f; best_idx = col + i; }
  }
}

template <int EPI>
__device__ __forceinline__ void epilogue32(const uint32_t (&v)[32], int row, int col, int M, int N, void* C,
                                           int ldc, const float* bias, const NormArgs& na, float& ss,
                                           const RopeArgs& ra) {
  RopeRow rr;
  if constexpr (EPI == kEpiQkvRope) rr = rope_row(ra, row, M);
  epilogue_chunk<EPI, 32>(v, row, col, M, N, C, ldc, bias, na, ss, ra, rr);
}

// Consumer side of the fused RMSNorm: r = rsqrt(sum of the row's partials
// (tile order) / H + eps), the same expression rmsnorm_kernel evaluates.
__device__ __forceinline__ float norm_row_scale(const NormArgs& na, int row, int M) {
  if (na.ssq_in == nullptr || row >= M) return 1.0f;
  const float* p = na.ssq_in + (int64_t)row * na.parts_in;
  const int parts = na.parts_in;
  float s = 0.0f;
  int t = 0;
  if ((parts & 3) == 0 && ((reinterpret_cast<uintptr_t>(p) & 15) == 0)) {
    // 16-byte loads, several in flight; the sum stays sequential in t
#pragma unroll 4
    for (; t < parts; t += 4) {
      const float4 q = *reinterpret_cast<const float4*>(p + t);
      s += q.x; s += q.y; s += q.z; s += q.w;
    }
  }
  for (; t < parts; ++t) s += p[t];
  return rsqrtf(s / na.hdim + na.eps);
}

template <int W>
__device__ __forceinline__ void scale_chunk(uint32_t* v, float r) {
#pragma unroll
  for (int i = 0; i < W; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * r);
}

// Live-row count of a compacted verify batch (sr_build_verify_batch writes
// it): tiles are walked over min(capacity, live) rows, so the rows of
// finished requests and unproposed draft slots cost nothing.  Read before
// griddepcontrol.wait, bypassing L1: the value is written by a kernel at
// least two launches earlier in the stream, which has completed (and
// flushed) before the immediately preceding kernel passes its own wait --
// and this grid cannot start before that.  The tile schedule (and so every
// row's accumulation order) does not depend on it: only the tile count does.
__device__ __forceinline__ int live_rows(int cap, const int32_t* m_live) {
  if (m_live == nullptr) return cap;
  const int v = __ldcg(m_live);
  return v < cap ? (v > 0 ? v : 0) : cap;
}

template <int BN, int EPI>
__global__ void __launch_bounds__(kThreads, 1)
gemm_tcgen05_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    int M_cap, const int32_t* __restrict__ m_live, int N, int K, void* C, int ldc,
                    const float* __restrict__ bias, int32_t* __restrict__ aux, SampleArgs sa, NormArgs na,
                    RopeArgs ra) {
  using Cfg = GemmCfg<BN>;
  const int M = live_rows(M_cap, m_live);
  constexpr int S = Cfg::kStages;
  extern __shared__ uint8_t smem_raw[];
  // 1 KB-aligned by pointer arithmetic on the __shared__ array (an integer
  // round trip would make every derived access generic)
  uint8_t* smem = smem_raw + ((1024u - (sm100::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;
  uint8_t* sB = smem + S * Cfg::kABytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * Cfg::kStageBytes);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int num_m = (M + kBM - 1) / kBM, num_n = (N + BN - 1) / BN;
  const int num_tiles = num_m * num_n;
  const int num_kb = (K + kBK - 1) / kBK;

  if (warp == 0 && lane == 0) {
    sm100::tma_prefetch_desc(&tmA);
    sm100::tma_prefetch_desc(&tmB);
    for (int s = 0; s < S; ++s) {
      sm100::mbar_init(&full[s], 1);
      sm100::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      sm100::mbar_init(&tfull[a], 1);
      sm100::mbar_init(&tempty[a], 128);
    }
    sm100::fence_barrier_init();
  }
  if (warp == 1) sm100::tmem_alloc<Cfg::kTmemCols>(tmem_slot);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // the first tile's first weight blocks before griddepcontrol.wait
  const int pre = (warp == 0 && (int)blockIdx.x < num_tiles) ? (num_kb < S ? num_kb : S) : 0;
  if (pre > 0) {
    if (sm100::elect_one()) {
      for (int kb = 0; kb < pre; ++kb) {
        sm100::mbar_arrive_expect_tx(&full[kb], Cfg::kStageBytes);
        sm100::tma_load_2d(sB + kb * Cfg::kBBytes, &tmB, &full[kb], kb * kBK, ((int)blockIdx.x / num_m) * BN,
                           sm100::kEvictNormal);
      }
    }
    __syncwarp();
  }
  grid_dep_sync();  // prologue above touched no predecessor output

  if (warp == 0) {
    {
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        const int m_blk = tile % num_m, n_blk = tile / num_m;
        for (int kb = 0; kb < num_kb; ++kb) {
          const bool staged_b = tile == (int)blockIdx.x && kb < pre;
          sm100::mbar_wait(&empty[stage], phase ^ 1);
          if (sm100::elect_one()) {
            if (!staged_b) sm100::mbar_arrive_expect_tx(&full[stage], Cfg::kStageBytes);
            sm100::tma_load_2d(sA + stage * Cfg::kABytes, &tmA, &full[stage], kb * kBK, m_blk * kBM,
                               sm100::kEvictLast);
            if (!staged_b)
              sm100::tma_load_2d(sB + stage * Cfg::kBBytes, &tmB, &full[stage], kb * kBK, n_blk * BN,
                                 sm100::kEvictNormal);
          }
          __syncwarp();
          if (++stage == S) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    {
      constexpr uint32_t idesc = sm100::umma_idesc_bf16(kBM, BN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        sm100::mbar_wait(&tempty[acc], acc_phase ^ 1);
        sm100::tc_fence_after();
        const uint32_t d = tmem_base + acc * BN;
        for (int kb = 0; kb < num_kb; ++kb) {
          sm100::mbar_wait(&full[stage], phase);
          sm100::tc_fence_after();
          const uint32_t a0 = sm100::smem_u32(sA + stage * Cfg::kABytes);
          const uint32_t b0 = sm100::smem_u32(sB + stage * Cfg::kBBytes);
          if (sm100::elect_one()) {
#pragma unroll
            for (int k = 0; k < kBK / 16; ++k) {
              sm100::umma_bf16(d, sm100::umma_desc_sw128(a0 + k * 32), sm100::umma_desc_sw128(b0 + k * 32),
                               idesc, (kb | k) != 0);
            }
            sm100::umma_commit(&empty[stage]);
          }
          __syncwarp();
          if (++stage == S) { stage = 0; phase ^= 1; }
        }
        if (sm100::elect_one()) sm100::umma_commit(&tfull[acc]);
        __syncwarp();
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else {
    const int quad = warp & 3;  // TMEM lane quadrant this warp may access
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
      const int m_blk = tile % num_m, n_blk = tile / num_m;
      sm100::mbar_wait(&tfull[acc], acc_phase);
      sm100::tc_fence_after();
      const int row = m_blk * kBM + quad * 32 + lane;
      const uint32_t taddr = tmem_base + ((uint32_t)(quad * 32) << 16) + acc * BN;
      float best = -INFINITY;
      int best_idx = 0x7fffffff;
      float ss = 0.0f, gss = 0.0f;
      const float rs = norm_row_scale(na, row, M);
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t v[32];
        sm100::tmem_ld_32x32b_x32(taddr + c * 32, v);
        sm100::tmem_ld_wait();
        if (na.ssq_in != nullptr) scale_chunk<32>(v, rs);
        const int col = n_blk * BN + c * 32;
        if constexpr (EPI == kEpiArgmax) {
          argmax_chunk<32>(v, col, N, row, M, sa, best, best_idx);
        } else {
          if (col < N) {
            epilogue32<EPI>(v, row, col, M, N, C, ldc, bias, na, ss, ra);
            if constexpr (EPI == kEpiResidualNorm)
              ssq_accum(gss, ss, col, N, na.ssq_out + (int64_t)row * ssq_parts(N), row < M);
          }
        }
      }
      if constexpr (EPI == kEpiArgmax) {
        if (row < M) {
          const int tiles_n = (N + BN - 1) / BN;
          reinterpret_cast<float*>(C)[(int64_t)row * tiles_n + n_blk] = best;
          aux[(int64_t)row * tiles_n + n_blk] = best_idx;
        }
      }
      sm100::tc_fence_before();
      sm100::mbar_arrive(&tempty[acc]);
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  }
  __syncthreads();
  if (warp == 1) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc<Cfg::kTmemCols>(tmem_base);
  }
}

// ---------------------------------------------------------------------------
// CTA-pair variant (cta_group::2): the pair computes a 256 x BN tile; each CTA
// stages its own 128 activation rows and BN/2 weight rows per k-block, the
// leader issues tcgen05.mma.cta_group::2 (M=256) reading both CTAs' shared
// memory, and each CTA's TMEM holds its 128 accumulator rows.  Per SM this
// halves the weight bytes per MAC, the bound of the 1-CTA kernel.
//
// KC = k chunks (64 wide, one 128-byte swizzle atom per row) per pipeline
// stage.  With KC = 2 each operand is staged by ONE 3D TMA instruction
// (chunk as the outer box dimension) per 128 k: measured on B200, a stage
// costs ~280 clk of TMA issue + barrier turnaround regardless of size up to
// ~32 KB, plus ~100 clk per extra instruction (scripts/micro/tma_rate.cu),
// so 64-k stages with two instructions (~400 clk) starve a 256 x 128 MMA
// (256 clk) while 128-k stages (~450 clk vs 512 clk of MMA) do not.


template <int BN, int KC = 1>
struct PairCfg {
  static constexpr int kBNH = BN / 2;
  // residual epilogues (o, down) stage each warp's 32x32 fp32 chunk through
  // shared memory so global stores are row-contiguous (full 32-byte sectors)
  static constexpr uint32_t kStageRow = 36;  // floats per staged row (pad 4: conflict-free)
  static constexpr uint32_t kEpiStageBytes = 4 * 32 * kStageRow * 4;
  static constexpr uint32_t kAChunk = kBM * kBK * 2;   // 128 rows x 128 B
  static constexpr uint32_t kBChunk = kBNH * kBK * 2;
  static constexpr uint32_t kABytes = KC * kAChunk;
  static constexpr uint32_t kBBytes = KC * kBChunk;
  static constexpr uint32_t kStageBytes = kABytes + kBBytes;
  static constexpr int kStages = (212992 / kStageBytes) < 8 ? (212992 / kStageBytes) : 8;
  // 512: room for the per-K-range accumulators (SwapArgs::splits)
  static constexpr uint32_t kTmemCols = 512;
  static constexpr int kChunk = BN % 32 == 0 ? 32 : 16;
  static constexpr size_t kSmem = 1024 + (size_t)kStages * kStageBytes + 256;
};

// residual epilogues stage through shared memory when the staging area fits
// next to the ring (every shape the planner picks except 160-wide tiles)
template <int BN, int EPI, int KC>
constexpr bool kStagedEpi = (EPI == kEpiResidualF32 || EPI == kEpiResidualNorm) && BN % 32 == 0 &&
                            PairCfg<BN, KC>::kSmem + PairCfg<BN, KC>::kEpiStageBytes <= 232448;

template <int CW>
__device__ __forceinline__ void tmem_ld_chunk(uint32_t taddr, uint32_t* v) {
  if constexpr (CW == 32) sm100::tmem_ld_32x32b_x32(taddr, *reinterpret_cast<uint32_t(*)[32]>(v));
  else sm100::tmem_ld_32x32b_x16(taddr, v);
}

// v holds K range 0's accumulator chunk (loaded, waited); add ranges
// 1..splits-1 in order -- the same left fold swap_gemm applies to its fp32
// partials, so both modes round identically.
// one range per TMEM round trip (register-lean: the residual path keeps its
// whole residual slice in registers)
template <int CW>
__device__ __forceinline__ void add_splits1(uint32_t taddr, int splits, int stride, uint32_t* v) {
  for (int r = 1; r < splits; ++r) {
    uint32_t t[CW];
    tmem_ld_chunk<CW>(taddr + (uint32_t)(r * stride), t);
    sm100::tmem_ld_wait();
#pragma unroll
    for (int i = 0; i < CW; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) + __uint_as_float(t[i]));
  }
}

template <int CW>
__device__ __forceinline__ void add_splits(uint32_t taddr, int splits, int stride, uint32_t* v) {
  for (int r = 1; r < splits; r += 2) {  // two ranges per TMEM round trip
    uint32_t t[CW], t2[CW];
    tmem_ld_chunk<CW>(taddr + (uint32_t)(r * stride), t);
    if (r + 1 < splits) tmem_ld_chunk<CW>(taddr + (uint32_t)((r + 1) * stride), t2);
    sm100::tmem_ld_wait();
#pragma unroll
    for (int i = 0; i < CW; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) + __uint_as_float(t[i]));
    if (r + 1 < splits) {
#pragma unroll
      for (int i = 0; i < CW; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) + __uint_as_float(t2[i]));
    }
  }
}

// Epilogues the small-M (swap) mode runs: the row-major 32-column chunk
// epilogues, reached through a per-warp 32 x 32 transpose.
template <int EPI>
constexpr bool kSwapEpi = EPI == kEpiStoreBf16 || EPI == kEpiStoreF32 || EPI == kEpiResidualF32 || EPI == kEpiSwiGLU ||
                          EPI == kEpiResidualNorm || EPI == kEpiQkvRope;


__device__ __forceinline__ void epi_bar_sync() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

// Column-major epilogue of the small-M mode: lane = output column
// col0 + lane, v[i] = token row0 + i.  Every store instruction covers one
// row's 32 consecutive columns (coalesced).  The arithmetic and rounding are
// those of the row-major chunk epilogues (epilogue_chunk, qkv_rope_chunk,
// the kSsqCols partial form), so both GEMM modes write identical bits.
// Cross-lane data (a row's scale / RoPE destination, SwiGLU and RoPE
// partners, the norm partial over the warp's 32 columns) goes through the
// warp's shared scratch, not shuffles: swap_gemm is not inlined, and a
// shuffle in a function the compiler cannot prove converged is wrapped in
// a slow collective sequence.
// One lane's token row inputs for the small-M epilogue (loaded before the
// accumulator is ready): RMSNorm row scale, RoPE position / KV destination.
struct SwapRow {
  float rs = 1.0f;
  int info = -1, pos = 0;
  long long dst = 0;
};

template <int EPI>
__device__ __forceinline__ SwapRow swap_row(const NormArgs& na, const RopeArgs& ra, int row, int M) {
  SwapRow r;
  if (na.ssq_in != nullptr) r.rs = norm_row_scale(na, row, M);
  if constexpr (EPI == kEpiQkvRope) {
    const RopeRow rr = rope_row(ra, row, M);
    r.info = rr.info;
    r.pos = rr.info >= 0 ? rr.pos : 0;  // padding rows: any valid table row
    r.dst = rr.dst;
  }
  return r;
}

struct SwapScratch {
  float t[32 * 33];      // [token][column] (+1 pad)
  float rs[32];          // per token: RMSNorm row scale
  int info[32], pos[32];
  long long dst[32];
};

template <int EPI>
__device__ __forceinline__ void swap_epilogue(uint32_t (&v)[32], int row0, int col0, int lane, int M, int N,
                                              void* C, int ldc, const float* __restrict__ bias, const NormArgs na,
                                              const RopeArgs ra, int parts, int quad, float* red,
                                              SwapScratch& xs, const SwapRow& me, const float* res_pre) {
  // (the argument structs are copies: their fields stay in registers across
  // the global stores below instead of being reloaded behind each store)
  const int n = col0 + lane;
  const bool col_ok = n < N;
  const int my_row = row0 + lane;  // per-row inputs are loaded by lane, read back per token
  if (na.ssq_in != nullptr) {
    xs.rs[lane] = me.rs;
    __syncwarp();
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * xs.rs[i]);
    __syncwarp();
  }
  const float b = (bias != nullptr && col_ok) ? bias[n] : 0.0f;
  if constexpr (EPI == kEpiStoreF32 || EPI == kEpiStoreBf16) {
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      float f = __uint_as_float(v[i]);
      if (bias != nullptr) f += b;
      if (row0 + i < M && col_ok) {
        if constexpr (EPI == kEpiStoreF32) reinterpret_cast<float*>(C)[(int64_t)(row0 + i) * ldc + n] = f;
        else reinterpret_cast<__nv_bfloat16*>(C)[(int64_t)(row0 + i) * ldc + n] = __float2bfloat16_rn(f);
      }
    }
  } else if constexpr (EPI == kEpiResidualF32 || EPI == kEpiResidualNorm) {
    // the residual rows, all in flight (clamped addresses, no branches)
    float res[32];
    const int nl = col_ok ? n : N - 1;
    float* cbase = reinterpret_cast<float*>(C) + nl;
    if (res_pre != nullptr) {
#pragma unroll
      for (int i = 0; i < 32; ++i) res[i] = res_pre[i];
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i) res[i] = cbase[(int64_t)(row0 + i < M ? row0 + i : M - 1) * ldc];
    }
    if constexpr (EPI == kEpiResidualF32) {
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (row0 + i < M && col_ok) cbase[(int64_t)(row0 + i) * ldc] = res[i] + __uint_as_float(v[i]);
      return;
    }
    const float wn = col_ok ? na.w[n] : 0.0f;
    __nv_bfloat16* const hbase = na.h_out + n;
    const int64_t ld_h = na.ld_h;
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      float a = 0.0f;
      if (row0 + i < M && col_ok) {
        a = res[i] + __uint_as_float(v[i]);
        cbase[(int64_t)(row0 + i) * ldc] = a;
        hbase[(int64_t)(row0 + i) * ld_h] = __float2bfloat16_rn(a * wn);
      }
      xs.t[i * 33 + lane] = a;
    }
    __syncwarp();
    // lane = token: this warp's 32-column chunk partial in the kSsqCols form
    {
      const float* tr = xs.t + lane * 33;
      float sq[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) sq[q] = quad_ssq(make_float4(tr[4 * q], tr[4 * q + 1], tr[4 * q + 2], tr[4 * q + 3]));
      red[quad * 32 + lane] = tree8(sq);
    }
    __syncwarp();
    // the group (this CTA's 128 columns = 4 warps' chunks) in column order
    epi_bar_sync();
    if (quad == 0) {
      float* const ssq_out = na.ssq_out;
      const float gsum = ((red[lane] + red[32 + lane]) + red[64 + lane]) + red[96 + lane];
      if (row0 + lane < M && col0 < N) ssq_out[(int64_t)(row0 + lane) * parts + col0 / kSsqCols] = gsum;
    }
    epi_bar_sync();
  } else if constexpr (EPI == kEpiSwiGLU) {
    // the warp's 32 columns are one interleave block: lanes 0-15 gate, 16-31 up
    const bool ok = col0 + 32 <= N;  // N % 32 == 0 (plan)
#pragma unroll
    for (int i = 0; i < 32; ++i) xs.t[i * 33 + lane] = __uint_as_float(v[i]);
    __syncwarp();
    if (lane < 16 && ok) {
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (row0 + i < M)
          reinterpret_cast<__nv_bfloat16*>(C)[(int64_t)(row0 + i) * ldc + col0 / 2 + lane] =
              __float2bfloat16_rn(silu(__uint_as_float(v[i])) * xs.t[i * 33 + lane + 16]);
    }
    __syncwarp();
  } else if constexpr (EPI == kEpiQkvRope) {
    const int hd = ra.hd, half = hd >> 1;
    const int nq = ra.nq, nkv = ra.nkv, page = ra.page, window_max = ra.window_max;
    const int hq = nq * hd, hk = nkv * hd;
    __nv_bfloat16* const q_out = ra.q_out;
    __nv_bfloat16* const cache = ra.cache;
    __nv_bfloat16* const window = ra.window;
    const float* const cos_t = ra.cos;
    const float* const sin_t = ra.sin;
    xs.info[lane] = me.info;
    xs.pos[lane] = me.pos;
    xs.dst[lane] = me.dst;
#pragma unroll
    for (int i = 0; i < 32; ++i) xs.t[i * 33 + lane] = __uint_as_float(v[i]) + b;
    __syncwarp();
    const int pidx = (col0 % hd) / 2 + (lane >> 1);  // rotation pair of this column (q / k)
    const bool odd = lane & 1;
    const bool rot = col0 < hq + hk;
    // cos / sin of every token's position, all in flight before the stores
    float cs[32], sn_[32];
    if (rot) {
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        cs[i] = cos_t[(int64_t)xs.pos[i] * half + pidx];
        sn_[i] = sin_t[(int64_t)xs.pos[i] * half + pidx];
      }
    }
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const int info = xs.info[i];
      if (info < 0 || row0 + i >= M || !col_ok) continue;  // padding row of the verify batch
      const float x = xs.t[i * 33 + lane];
      const bool win = (info >> 16) & 1;
      const int slot = info & 0xFFFF;
      const int rows = win ? window_max : page;
      __nv_bfloat16* kbase = (win ? window : cache) + xs.dst[i];
      if (rot) {
        const float xp = xs.t[i * 33 + (lane ^ 1)];  // the pair partner
        const float x1 = odd ? xp : x, x2 = odd ? x : xp;
        const float y = odd ? rope_y2(x1, x2, cs[i], sn_[i]) : rope_y1(x1, x2, cs[i], sn_[i]);
        const int dim = pidx + (odd ? half : 0);
        if (col0 < hq) {
          q_out[((int64_t)(row0 + i) * nq + col0 / hd) * hd + dim] = __float2bfloat16_rn(y);
        } else {
          __nv_bfloat16* k = kbase + (int64_t)((col0 - hq) / hd) * rows * hd;
          k[kv_elem(slot, dim, hd)] = __float2bfloat16_rn(y);
        }
      } else {
        const int vc = n - hq - hk;
        __nv_bfloat16* vb = kbase + (int64_t)nkv * rows * hd + (int64_t)(vc / hd) * rows * hd;
        vb[kv_elem(slot, vc % hd, hd)] = __float2bfloat16_rn(x);
      }
    }
    __syncwarp();
  }
}

// Small-M mode of the pair kernel (SwapArgs): C^T[n, m] = sum_k W[n, k] A[m, k].
// Unit u = (256-row weight tile u / splits, K range u % splits); CTA rank r
// of the pair stages W rows tile*256 + 128 r .. +127 as the UMMA A operand
// and tokens r*NT/2 .. +NT/2 as its half of the B operand (NT = live rows
// rounded up to 32), so its TMEM holds its 128 output columns (lanes) x NT
// tokens.  Epilogue warps read 32 tokens x 32 columns per step, transpose
// them through shared memory and run the row-major chunk epilogue (thread =
// token row, 32 consecutive columns) -- the same code and rounding as the
// pair mode.  With splits > 1 each unit stores its fp32 partial; the last
// of a tile's `splits` units (arrival counter) sums them in range order.
template <int EPI>
__device__ __forceinline__ void swap_gemm(uint32_t ring_bytes, const SwapArgs sw, int M, int N, int K, void* C,
                                          int ldc, const float* __restrict__ bias, const NormArgs na,
                                          const RopeArgs ra) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (sm100::smem_u32(smem_raw) & 1023u)) & 1023u);
  constexpr int KC = 2;
  constexpr int kMaxStages = 12;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t crank = sm100::cluster_ctarank();
  const uint32_t rank = crank & 1;
  const uint32_t lead = crank & ~1u;
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  const int splits = sw.splits > 1 ? sw.splits : 1;
  const int chunks = (K + kBK - 1) / kBK;
  const int cs = splits > 1 ? chunks / splits : chunks;  // 64-k chunks per range
  const int stages_per_unit = (cs + KC - 1) / KC;
  const int tiles = (N + 255) / 256;
  const int units = tiles * splits;
  const int NT = (M + 31) & ~31;  // 32..128 tokens (UMMA N)
  const int nth = NT >> 1;        // token rows staged per CTA
  const CUtensorMap* wmap = &sw.maps->w;
  const CUtensorMap* xmap = &sw.maps->x[(nth >> 4) - 1];
  const uint32_t wbytes = KC * 16384u, xbytes = KC * (uint32_t)nth * 128u, stage_bytes = wbytes + xbytes;
  // the last KB of the ring: the norm-group reduction scratch [4 warps][32 rows]
  // ring tail: the norm-group scratch [4 warps][32 rows] and the epilogue
  // warps' exchange scratch
  constexpr uint32_t kScratch = (1024 + 4 * sizeof(SwapScratch) + 1023) & ~1023u;
  float* red = reinterpret_cast<float*>(smem + ring_bytes - kScratch);
  SwapScratch* xsc = reinterpret_cast<SwapScratch*>(smem + ring_bytes - kScratch + 1024);
  int nst = (int)((ring_bytes - kScratch) / stage_bytes);
  nst = nst < kMaxStages ? nst : kMaxStages;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + ring_bytes);
  uint64_t* empty = full + kMaxStages;
  uint64_t* tfull = empty + kMaxStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  volatile int* last_flag = reinterpret_cast<volatile int*>(tmem_slot + 1);

  if (warp == 0 && lane == 0) {
    GT(0);
    sm100::tma_prefetch_desc(wmap);
    sm100::tma_prefetch_desc(xmap);
    for (int s = 0; s < nst; ++s) {
      sm100::mbar_init(&full[s], 1);
      sm100::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      sm100::mbar_init(&tfull[a], 1);
      sm100::mbar_init(&tempty[a], 8);  // 4 epilogue warps x 2 CTAs
    }
    sm100::fence_barrier_init();
  }
  if (warp == 1) sm100::tmem_alloc_pair<512>(tmem_slot);
  sm100::tc_fence_before();
  sm100::cluster_sync();
  sm100::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // weights of the first unit before griddepcontrol.wait (see the pair mode)
  const int pre = (warp == 0 && pair < units && (sw.flags & 1)) ? (stages_per_unit < nst ? stages_per_unit : nst) : 0;
  if (pre > 0) {
    const int tile0 = pair / splits, range0 = pair - tile0 * splits;
    if (sm100::elect_one()) {
      for (int j = 0; j < pre; ++j) {
        if (rank == 0) sm100::mbar_arrive_expect_tx(&full[j], 2 * stage_bytes);
        sm100::tma_load_3d_pair(smem + j * stage_bytes, wmap, &full[j], 0, tile0 * 256 + (int)rank * 128,
                                range0 * cs + j * KC, sm100::kEvictNormal);
      }
    }
    __syncwarp();
  }
  grid_dep_sync();
  if (threadIdx.x == 0) GT(1);

  if (warp == 0) {
    int stage = 0;
    uint32_t phase = 0;
    for (int u = pair; u < units; u += npairs) {
      const int tile = u / splits, range = u - tile * splits;
      const int wrow = tile * 256 + (int)rank * 128;
      for (int j = 0; j < stages_per_unit; ++j) {
        const int c0 = range * cs + j * KC;
        const bool staged_w = u == pair && j < pre;
        sm100::mbar_wait(&empty[stage], phase ^ 1);
        if (sm100::elect_one()) {
          uint8_t* st = smem + stage * stage_bytes;
          if (!staged_w) {
            if (rank == 0) sm100::mbar_arrive_expect_tx(&full[stage], 2 * stage_bytes);
            sm100::tma_load_3d_pair(st, wmap, &full[stage], 0, wrow, c0, sm100::kEvictNormal);
          }
          sm100::tma_load_3d_pair(st + wbytes, xmap, &full[stage], 0, (int)rank * nth, c0, sm100::kEvictLast);
        }
        __syncwarp();
        if (++stage == nst) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {
      const uint32_t idesc = sm100::umma_idesc_bf16(2 * kBM, (uint32_t)NT);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int u = pair; u < units; u += npairs) {
        sm100::mbar_wait(&tempty[acc], acc_phase ^ 1);
        sm100::tc_fence_after();
        const uint32_t d = tmem_base + acc * 128;
        for (int j = 0; j < stages_per_unit; ++j) {
          const int kin = cs - j * KC < KC ? cs - j * KC : KC;  // chunks of this stage in the range
          sm100::mbar_wait(&full[stage], phase);
          sm100::tc_fence_after();
          if (j == 0 && u == pair && lane == 0) GT(2);
          const uint32_t w0 = sm100::smem_u32(smem + stage * stage_bytes);
          const uint32_t x0 = w0 + wbytes;
          if (sm100::elect_one()) {
            for (int k = 0; k < kin * 4; ++k)
              sm100::umma_bf16_pair(d, sm100::umma_desc_sw128(w0 + (k >> 2) * 16384u + (k & 3) * 32),
                                    sm100::umma_desc_sw128(x0 + (k >> 2) * (uint32_t)nth * 128u + (k & 3) * 32),
                                    idesc, (j | k) != 0);
            sm100::umma_commit_pair(&empty[stage], (uint16_t)(0x3u << lead));
          }
          __syncwarp();
          if (++stage == nst) { stage = 0; phase ^= 1; }
        }
        if (sm100::elect_one()) sm100::umma_commit_pair(&tfull[acc], (uint16_t)(0x3u << lead));
        __syncwarp();
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else {
    const int quad = warp & 3;
    const uint32_t leader_tempty = sm100::mapa_shared(sm100::smem_u32(tempty), lead);
    const int parts = ssq_parts(N);
    const int groups = NT >> 5;
    int acc = 0;
    uint32_t acc_phase = 0;
    SwapRow rows[4];       // this lane's token in each 32-token group
    float res0[32];        // residual epilogues: group 0's residual rows
    bool have_res0 = false;
    auto finish = [&](uint32_t (&v)[32], int g, int col0) {
      swap_epilogue<EPI>(v, g * 32, col0, lane, M, N, C, ldc, bias, na, ra, parts, quad, red, xsc[quad],
                         rows[g], g == 0 && have_res0 ? res0 : nullptr);
    };
    for (int u = pair; u < units; u += npairs) {
      const int tile = u / splits, range = u - tile * splits;
      const int col0 = tile * 256 + (int)rank * 128 + quad * 32;  // this warp's 32 output columns
      const int n = col0 + lane;                                   // this lane's column
      const uint32_t taddr = tmem_base + ((uint32_t)(quad * 32) << 16) + acc * 128;
      // row inputs and group 0's residual while the mainloop runs
#pragma unroll
      for (int g = 0; g < 4; ++g)
        if (g < groups) rows[g] = swap_row<EPI>(na, ra, g * 32 + lane, M);
      if constexpr (EPI == kEpiResidualF32 || EPI == kEpiResidualNorm) {
        const float* cb = reinterpret_cast<const float*>(C) + (n < N ? n : N - 1);
#pragma unroll
        for (int i = 0; i < 32; ++i) res0[i] = cb[(int64_t)(i < M ? i : M - 1) * ldc];
        have_res0 = true;
      }
      sm100::mbar_wait(&tfull[acc], acc_phase);
      sm100::tc_fence_after();
      if (warp == 2 && lane == 0 && u == pair) GT(3);
      if (splits == 1) {
        for (int g = 0; g < groups; ++g) {
          uint32_t v[32];
          sm100::tmem_ld_32x32b_x32(taddr + g * 32, v);
          sm100::tmem_ld_wait();
          finish(v, g, col0);
        }
        sm100::tc_fence_before();
        __syncwarp();
        if (lane == 0) sm100::mbar_arrive_cluster(leader_tempty + acc * 8);
      } else {
        // partial of this range: [range][token][n] (a warp stores one
        // 128-byte row segment per token)
        float* part = sw.ws + (size_t)range * kSwapRows * N + n;
        for (int g = 0; g < groups; ++g) {
          uint32_t v[32];
          sm100::tmem_ld_32x32b_x32(taddr + g * 32, v);
          sm100::tmem_ld_wait();
          if (n < N) {  // token rows >= M land in unused rows of the range's slab
#pragma unroll
            for (int i = 0; i < 32; ++i) part[(size_t)(g * 32 + i) * N] = __uint_as_float(v[i]);
          }
        }
        sm100::tc_fence_before();
        __syncwarp();
        if (lane == 0) sm100::mbar_arrive_cluster(leader_tempty + acc * 8);
        // release the CTA's partial (bar.sync orders the 128 threads' stores
        // before one thread's gpu-scope fence + arrival); the last arrival
        // acquires every range's partial the same way
        epi_bar_sync();
        if (warp == 2 && lane == 0) {
          int32_t* cnt = sw.cnt + tile * 2 + rank;
          asm volatile("fence.acq_rel.gpu;" ::: "memory");
          const int prev = atomicAdd(cnt, 1);
          const int last = prev == splits - 1;
          if (last) {
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
            *cnt = 0;  // next launch (stream-ordered after this grid)
          }
          *last_flag = last;
        }
        epi_bar_sync();
        const int last = *last_flag;
        epi_bar_sync();  // flag read before the next unit rewrites it
        if (warp == 2 && lane == 0 && u == pair) GT(4);
        if (last) {
          for (int g = 0; g < groups; ++g) {
            // every range's 32 tokens of this column in flight at once (one
            // 128-byte segment per warp and token), then the left fold in
            // range order
            // (unpredicated loads: a load inside a per-element branch is
            // waited on before the branch reconverges, serializing them)
            float t[4][32];
            const float* base = sw.ws + (n < N ? n : N - 1) + (size_t)g * 32 * N;
#pragma unroll
            for (int r = 0; r < 4; ++r) {
              if (r < splits) {
#pragma unroll
                for (int i = 0; i < 32; ++i) t[r][i] = base[((size_t)r * kSwapRows + i) * N];
              } else {
#pragma unroll
                for (int i = 0; i < 32; ++i) t[r][i] = 0.0f;
              }
            }
            uint32_t v[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              float a = t[0][i];
#pragma unroll
              for (int r = 1; r < 4; ++r)
                if (r < splits) a += t[r][i];
              v[i] = __float_as_uint(a);
            }
            if (warp == 2 && lane == 0 && u == pair && g == 0) GT(7);
            finish(v, g, col0);
          }
        }
      }
      if (warp == 2 && lane == 0 && u == pair) GT(5);
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  }
  sm100::tc_fence_before();
  sm100::cluster_sync();
  if (threadIdx.x == 0) GT(6);
  if (warp == 1) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc_pair<512>(tmem_base);
  }
}

// MC = 2: a cluster of two pairs computes two horizontally adjacent tiles
// (n blocks 2j, 2j+1) of the same 256 rows.  Both pairs need the same
// activation rows, so each CTA loads half of its 128-row A block and
// multicasts it to itself and its counterpart in the other pair: A's L2->SM
// traffic halves, the bound of the small-N verify GEMMs (o, down, qkv).  A
// stage is reusable only when both pairs' MMAs have drained it, so the
// leaders' commits are multicast to all four CTAs' empty barriers (count 2).
// XM: the plan splits K into ranges (one TMEM accumulator per range, summed
// in order); plain plans (XM false) compile none of it.
template <int BN, int EPI, int MC, int KC, bool XM>
__global__ void __cluster_dims__(2 * MC, 1, 1) __launch_bounds__(kThreads, 1)
gemm_pair_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                 int M_cap, const int32_t* __restrict__ m_live, int N, int K, void* C, int ldc,
                 const float* __restrict__ bias, int32_t* __restrict__ aux, SampleArgs sa, NormArgs na,
                 RopeArgs ra, SwapArgs sw) {
  static_assert(MC == 1 || KC == 1 || KC == MC, "A multicast splits rows (KC 1) or k chunks (KC == MC)");
  const int M = live_rows(M_cap, m_live);
  using Cfg = PairCfg<BN, KC>;
  constexpr int S = Cfg::kStages;
  constexpr int CW = Cfg::kChunk;
  extern __shared__ uint8_t smem_raw[];
  // 1 KB-aligned by pointer arithmetic on the __shared__ array (an integer
  // round trip would make every derived access generic)
  uint8_t* smem = smem_raw + ((1024u - (sm100::smem_u32(smem_raw) & 1023u)) & 1023u);
  if constexpr (kSwapEpi<EPI>) {
    // dual launch (SwapArgs flags bit 1): the small-M kernel launched beside
    // this one computes live row counts <= max_m; exit after the wait
    if ((sw.flags & 2) && M >= 1 && M <= sw.max_m) {
      grid_dep_sync();
      return;
    }
  }
  // K ranges summed in order (SwapArgs): one TMEM accumulator per range
  const int n_split = XM && sw.splits > 1 ? sw.splits : 1;
  const int split_chunks = n_split > 1 ? (K / kBK) / n_split : (1 << 30);
  const int nacc = 2 * n_split * BN <= 512 ? 2 : 1;
  uint8_t* sA = smem;
  uint8_t* sB = smem + S * Cfg::kABytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * Cfg::kStageBytes);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t crank = sm100::cluster_ctarank();
  const uint32_t rank = crank & 1;        // position inside the pair
  const uint32_t q = crank >> 1;          // pair inside the cluster
  const uint32_t lead = crank & ~1u;      // this pair's MMA-issuing CTA
  const int pair = blockIdx.x / (2 * MC), npairs = gridDim.x / (2 * MC);
  const int num_m = (M + 2 * kBM - 1) / (2 * kBM), num_n = (N + BN - 1) / BN;
  const int num_tiles = num_m * ((num_n + MC - 1) / MC);
  const int num_kb = (K + KC * kBK - 1) / (KC * kBK);

  if (warp == 0 && lane == 0) {
    sm100::tma_prefetch_desc(&tmA);
    sm100::tma_prefetch_desc(&tmB);
    for (int s = 0; s < S; ++s) {
      sm100::mbar_init(&full[s], 1);
      sm100::mbar_init(&empty[s], MC);  // one commit per pair reading this CTA's loads
    }
    for (int a = 0; a < 2; ++a) {
      sm100::mbar_init(&tfull[a], 1);
      sm100::mbar_init(&tempty[a], 8);  // 4 epilogue warps x 2 CTAs
    }
    sm100::fence_barrier_init();
  }
  // TMEM: two accumulators of BN columns, times the K ranges
  const bool tmem_wide = (XM && n_split > 1) || 2 * BN > 256;
  if (warp == 1) {
    if (tmem_wide) sm100::tmem_alloc_pair<512>(tmem_slot);
    else sm100::tmem_alloc_pair<256>(tmem_slot);
  }
  sm100::tc_fence_before();
  sm100::cluster_sync();
  sm100::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // after the barrier area (kSmem's trailing 256 B); launched with
  // kEpiStageBytes more dynamic smem when kStagedEpi
  float* epi_stage = reinterpret_cast<float*>(smem + S * Cfg::kStageBytes + 256);
  // Weights do not depend on the preceding kernel: the producer stages the
  // first tile's first weight blocks before griddepcontrol.wait, so they
  // stream in while the predecessor drains (activations follow the wait).
  const int pre = (warp == 0 && pair < num_tiles && (sw.flags & 1)) ? (num_kb < S ? num_kb : S) : 0;
  if (pre > 0) {
    const int brow0 = ((pair / num_m) * MC + (int)q) * BN + (int)rank * Cfg::kBNH;
    if (sm100::elect_one()) {
      for (int kb = 0; kb < pre; ++kb) {
        if (rank == 0) sm100::mbar_arrive_expect_tx(&full[kb], 2 * Cfg::kStageBytes);
        if constexpr (KC > 1)
          sm100::tma_load_3d_pair(sB + kb * Cfg::kBBytes, &tmB, &full[kb], 0, brow0, kb * KC, sm100::kEvictNormal);
        else
          sm100::tma_load_2d_pair(sB + kb * Cfg::kBBytes, &tmB, &full[kb], kb * kBK, brow0, sm100::kEvictNormal);
      }
    }
    __syncwarp();
  }
  grid_dep_sync();  // prologue above touched no predecessor output

  if (warp == 0) {
    {
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = pair; tile < num_tiles; tile += npairs) {
        const int m_blk = tile % num_m, n_blk = (tile / num_m) * MC + (int)q;
        const int arow = m_blk * 2 * kBM + (int)rank * kBM;
        const int brow = n_blk * BN + (int)rank * Cfg::kBNH;
        for (int kb = 0; kb < num_kb; ++kb) {
          const bool staged_b = tile == pair && kb < pre;  // weights already in flight
          sm100::mbar_wait(&empty[stage], phase ^ 1);
          if (sm100::elect_one()) {
          if (rank == 0 && !staged_b) sm100::mbar_arrive_expect_tx(&full[stage], 2 * Cfg::kStageBytes);
          if constexpr (MC > 1 && KC == MC) {
            // chunk q of this stage's A for both pairs (same rows, same layout)
            sm100::tma_load_2d_pair_mc(sA + stage * Cfg::kABytes + q * Cfg::kAChunk, &tmA, &full[stage],
                                       (kb * KC + (int)q) * kBK, arow,
                                       (uint16_t)((1u << crank) | (1u << (crank ^ 2u))), sm100::kEvictLast);
          } else if constexpr (KC > 1) {
            sm100::tma_load_3d_pair(sA + stage * Cfg::kABytes, &tmA, &full[stage], 0, arow, kb * KC,
                                    sm100::kEvictLast);
          } else if constexpr (MC == 1) {
            sm100::tma_load_2d_pair(sA + stage * Cfg::kABytes, &tmA, &full[stage], kb * kBK, arow,
                                    sm100::kEvictLast);
          } else {
            sm100::tma_load_2d_pair_mc(sA + stage * Cfg::kABytes + q * (Cfg::kABytes / 2), &tmA,
                                       &full[stage], kb * kBK, arow + (int)q * (kBM / 2),
                                       (uint16_t)((1u << crank) | (1u << (crank ^ 2u))), sm100::kEvictLast);
          }
          if (!staged_b) {
            if constexpr (KC > 1)
              sm100::tma_load_3d_pair(sB + stage * Cfg::kBBytes, &tmB, &full[stage], 0, brow, kb * KC,
                                      sm100::kEvictNormal);
            else
              sm100::tma_load_2d_pair(sB + stage * Cfg::kBBytes, &tmB, &full[stage], kb * kBK, brow,
                                      sm100::kEvictNormal);
          }
          }
          __syncwarp();
          if (++stage == S) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {
      constexpr uint32_t idesc = sm100::umma_idesc_bf16(2 * kBM, BN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int tile = pair; tile < num_tiles; tile += npairs) {
        sm100::mbar_wait(&tempty[acc], acc_phase ^ 1);
        sm100::tc_fence_after();
        const uint32_t d = tmem_base + acc * n_split * BN;
        int range = 0, in_range = 0;  // K range of the next 64-k chunk, chunks into it
        for (int kb = 0; kb < num_kb; ++kb) {
          // per 64-k chunk of this stage: its K range (accumulator) and whether it starts one
          uint32_t dk[KC], fresh[KC];
#pragma unroll
          for (int j = 0; j < KC; ++j) {
            if constexpr (XM) {
              dk[j] = d + (uint32_t)(range * BN);
              fresh[j] = in_range == 0;
              if (++in_range == split_chunks) { in_range = 0; ++range; }
            } else {
              dk[j] = d;
              fresh[j] = kb == 0 && j == 0;
            }
          }
          sm100::mbar_wait(&full[stage], phase);
          sm100::tc_fence_after();
          const uint32_t a0 = sm100::smem_u32(sA + stage * Cfg::kABytes);
          const uint32_t b0 = sm100::smem_u32(sB + stage * Cfg::kBBytes);
          if (sm100::elect_one()) {
#pragma unroll
            for (int k = 0; k < KC * kBK / 16; ++k)
              sm100::umma_bf16_pair(dk[k >> 2], sm100::umma_desc_sw128(a0 + (k >> 2) * Cfg::kAChunk + (k & 3) * 32),
                                    sm100::umma_desc_sw128(b0 + (k >> 2) * Cfg::kBChunk + (k & 3) * 32),
                                    idesc, !((k & 3) == 0 && fresh[k >> 2]));
            sm100::umma_commit_pair(&empty[stage], MC == 1 ? 0x3 : 0xF);
          }
          __syncwarp();
          if (++stage == S) { stage = 0; phase ^= 1; }
        }
        if (sm100::elect_one()) sm100::umma_commit_pair(&tfull[acc], (uint16_t)(0x3u << lead));
        __syncwarp();
        if (++acc == nacc) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else {
    const int quad = warp & 3;
    const uint32_t leader_tempty = sm100::mapa_shared(sm100::smem_u32(tempty), lead);
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int tile = pair; tile < num_tiles; tile += npairs) {
      const int m_blk = tile % num_m, n_blk = (tile / num_m) * MC + (int)q;
      const int row = m_blk * 2 * kBM + (int)rank * kBM + quad * 32 + lane;
      const uint32_t taddr = tmem_base + ((uint32_t)(quad * 32) << 16) + acc * n_split * BN;
      if constexpr ((EPI == kEpiResidualF32 || EPI == kEpiResidualNorm) && BN <= 128) {
        // Residual epilogue: the warps are idle during the mainloop, so pull
        // this row's residual slice into registers before the accumulator is
        // ready; the add + store then never waits on a global load.
        float res[BN];
        float* xr = reinterpret_cast<float*>(C) + (int64_t)row * ldc + n_blk * BN;
        const bool row_ok = row < M;
        const bool vec = row_ok && n_blk * BN + BN <= N;
#pragma unroll
        for (int q = 0; q < BN / 4; ++q) {
          float4 r4 = make_float4(0, 0, 0, 0);
          if (vec) r4 = reinterpret_cast<const float4*>(xr)[q];
          res[4 * q] = r4.x; res[4 * q + 1] = r4.y; res[4 * q + 2] = r4.z; res[4 * q + 3] = r4.w;
        }
        sm100::mbar_wait(&tfull[acc], acc_phase);
        sm100::tc_fence_after();
        float gss = 0.0f;
        float* row_parts = na.ssq_out + (int64_t)row * ssq_parts(N);
#pragma unroll
        for (int c = 0; c < BN / CW; ++c) {
          uint32_t v[CW];
          tmem_ld_chunk<CW>(taddr + c * CW, v);
          sm100::tmem_ld_wait();
          if constexpr (XM) add_splits1<CW>(taddr + c * CW, n_split, BN, v);
          const int col = n_blk * BN + c * CW;
          if constexpr (kStagedEpi<BN, EPI, KC>) {
            if (n_blk * BN + BN <= N) {  // warp-uniform: full-width tile
              // 1) thread = row: x_new = residual + acc, sum of squares in column order
              float* T = epi_stage + quad * 32 * Cfg::kStageRow;
              float sq[8];
#pragma unroll
              for (int q = 0; q < 8; ++q) {
                float4 xn;
                xn.x = res[c * CW + 4 * q] + __uint_as_float(v[4 * q]);
                xn.y = res[c * CW + 4 * q + 1] + __uint_as_float(v[4 * q + 1]);
                xn.z = res[c * CW + 4 * q + 2] + __uint_as_float(v[4 * q + 2]);
                xn.w = res[c * CW + 4 * q + 3] + __uint_as_float(v[4 * q + 3]);
                if constexpr (EPI == kEpiResidualNorm) sq[q] = quad_ssq(xn);
                *reinterpret_cast<float4*>(T + lane * Cfg::kStageRow + 4 * q) = xn;
              }
              if constexpr (EPI == kEpiResidualNorm) ssq_accum(gss, tree8(sq), col, N, row_parts, row_ok);
              __syncwarp();
              // 2) lane = (row it*4 + lane/8, columns 4*(lane%8)..+3): each
              //    store instruction writes four full 128-byte row segments
              const int qq = lane & 7;
              const int row0 = row - lane;
              float4 wv = make_float4(0, 0, 0, 0);
              if constexpr (EPI == kEpiResidualNorm) wv = reinterpret_cast<const float4*>(na.w + col)[qq];
#pragma unroll
              for (int it = 0; it < 8; ++it) {
                const int r = it * 4 + (lane >> 3);
                const float4 xv = *reinterpret_cast<const float4*>(T + r * Cfg::kStageRow + 4 * qq);
                if (row0 + r < M) {
                  reinterpret_cast<float4*>(reinterpret_cast<float*>(C) + (int64_t)(row0 + r) * ldc + col)[qq] = xv;
                  if constexpr (EPI == kEpiResidualNorm) {
                    uint2 hv;
                    hv.x = pack_bf16(xv.x * wv.x, xv.y * wv.y);
                    hv.y = pack_bf16(xv.z * wv.z, xv.w * wv.w);
                    reinterpret_cast<uint2*>(na.h_out + (int64_t)(row0 + r) * na.ld_h + col)[qq] = hv;
                  }
                }
              }
              __syncwarp();  // T is rewritten by the next chunk
              continue;
            }
          }
          if (vec) {
            float sq[8];
#pragma unroll
            for (int q = 0; q < CW / 8; ++q) {
              float xn[8];
#pragma unroll
              for (int i = 0; i < 8; ++i) xn[i] = res[c * CW + 8 * q + i] + __uint_as_float(v[8 * q + i]);
              reinterpret_cast<float4*>(xr)[c * CW / 4 + 2 * q] = make_float4(xn[0], xn[1], xn[2], xn[3]);
              reinterpret_cast<float4*>(xr)[c * CW / 4 + 2 * q + 1] = make_float4(xn[4], xn[5], xn[6], xn[7]);
              if constexpr (EPI == kEpiResidualNorm) {
                sq[(2 * q) & 7] = quad_ssq(make_float4(xn[0], xn[1], xn[2], xn[3]));
                sq[(2 * q + 1) & 7] = quad_ssq(make_float4(xn[4], xn[5], xn[6], xn[7]));
                const float4 wa = reinterpret_cast<const float4*>(na.w + col)[2 * q];
                const float4 wb = reinterpret_cast<const float4*>(na.w + col)[2 * q + 1];
                uint4 hv;
                hv.x = pack_bf16(xn[0] * wa.x, xn[1] * wa.y);
                hv.y = pack_bf16(xn[2] * wa.z, xn[3] * wa.w);
                hv.z = pack_bf16(xn[4] * wb.x, xn[5] * wb.y);
                hv.w = pack_bf16(xn[6] * wb.z, xn[7] * wb.w);
                reinterpret_cast<uint4*>(na.h_out + (int64_t)row * na.ld_h + col)[q] = hv;
              }
            }
            if constexpr (EPI == kEpiResidualNorm) ssq_accum(gss, tree8(sq), col, N, row_parts, true);
          } else if (row_ok && col < N) {
            float ss = 0.0f;
            epilogue_chunk<EPI, CW>(v, row, col, M, N, C, ldc, bias, na, ss, ra);
            if constexpr (EPI == kEpiResidualNorm) ssq_accum(gss, ss, col, N, row_parts, true);
          }
        }
        sm100::tc_fence_before();
        __syncwarp();
        if (lane == 0) sm100::mbar_arrive_cluster(leader_tempty + acc * 8);
        if (++acc == nacc) { acc = 0; acc_phase ^= 1; }
        continue;
      }
      if constexpr (kStagedEpi<BN, EPI, KC> && BN > 128) {
        // Wide residual tiles (7B / 32B o and down): the row's residual does
        // not fit in registers, so it is read in the store layout instead --
        // lane = (row it*4 + lane/8, 4 columns): coalesced 128-byte row
        // segments, one chunk ahead of its use.  The sum of squares
        // accumulates per lane and reduces over the row's 8 lanes at the end
        // (fixed order).
        if (n_blk * BN + BN <= N) {
          float* T = epi_stage + quad * 32 * Cfg::kStageRow;
          const int qq = lane & 7, row0 = row - lane;
          float4 xres[8], xnext[8];
          float ssp[8], gsp[8];
#pragma unroll
          for (int it = 0; it < 8; ++it) gsp[it] = 0.0f;
          auto load_res = [&](int c, float4 (&dst)[8]) {
#pragma unroll
            for (int it = 0; it < 8; ++it) {
              const int r = it * 4 + (lane >> 3);
              dst[it] = row0 + r < M ? reinterpret_cast<const float4*>(reinterpret_cast<const float*>(C) +
                                                                         (int64_t)(row0 + r) * ldc + n_blk * BN +
                                                                         c * 32)[qq]
                                     : make_float4(0, 0, 0, 0);
            }
          };
          load_res(0, xres);
          sm100::mbar_wait(&tfull[acc], acc_phase);
          sm100::tc_fence_after();
#pragma unroll 1
          for (int c = 0; c < BN / 32; ++c) {
            uint32_t v[32];
            sm100::tmem_ld_32x32b_x32(taddr + c * 32, v);
            if (c + 1 < BN / 32) load_res(c + 1, xnext);
            sm100::tmem_ld_wait();
            if constexpr (XM) add_splits<32>(taddr + c * 32, n_split, BN, v);
            const int col = n_blk * BN + c * 32;
#pragma unroll
            for (int it = 0; it < 8; ++it) ssp[it] = 0.0f;
#pragma unroll
            for (int q = 0; q < 8; ++q)
              *reinterpret_cast<float4*>(T + lane * Cfg::kStageRow + 4 * q) =
                  make_float4(__uint_as_float(v[4 * q]), __uint_as_float(v[4 * q + 1]),
                              __uint_as_float(v[4 * q + 2]), __uint_as_float(v[4 * q + 3]));
            __syncwarp();
            float4 wv = make_float4(0, 0, 0, 0);
            if constexpr (EPI == kEpiResidualNorm) wv = reinterpret_cast<const float4*>(na.w + col)[qq];
#pragma unroll
            for (int it = 0; it < 8; ++it) {
              const int r = it * 4 + (lane >> 3);
              const float4 a = *reinterpret_cast<const float4*>(T + r * Cfg::kStageRow + 4 * qq);
              float4 xv = xres[it];
              xv.x += a.x; xv.y += a.y; xv.z += a.z; xv.w += a.w;
              if (row0 + r < M) {
                reinterpret_cast<float4*>(reinterpret_cast<float*>(C) + (int64_t)(row0 + r) * ldc + col)[qq] = xv;
                if constexpr (EPI == kEpiResidualNorm) {
                  ssp[it] = quad_ssq(xv);
                  uint2 hv;
                  hv.x = pack_bf16(xv.x * wv.x, xv.y * wv.y);
                  hv.y = pack_bf16(xv.z * wv.z, xv.w * wv.w);
                  reinterpret_cast<uint2*>(na.h_out + (int64_t)(row0 + r) * na.ld_h + col)[qq] = hv;
                }
              }
            }
            if constexpr (EPI == kEpiResidualNorm) {
              // chunk partial of row (it*4 + lane/8): lane qq holds columns
              // 4qq..4qq+3; the butterfly is the kSsqCols tree
#pragma unroll
              for (int it = 0; it < 8; ++it) {
                float s_ = ssp[it];
                s_ += __shfl_xor_sync(0xffffffffu, s_, 1);
                s_ += __shfl_xor_sync(0xffffffffu, s_, 2);
                s_ += __shfl_xor_sync(0xffffffffu, s_, 4);
                const int r = it * 4 + (lane >> 3);
                ssq_accum(gsp[it], s_, col, N, na.ssq_out + (int64_t)(row0 + r) * ssq_parts(N), qq == 0 && row0 + r < M);
              }
            }
            __syncwarp();
#pragma unroll
            for (int it = 0; it < 8; ++it) xres[it] = xnext[it];
          }
          sm100::tc_fence_before();
          __syncwarp();
          if (lane == 0) sm100::mbar_arrive_cluster(leader_tempty + acc * 8);
          if (++acc == nacc) { acc = 0; acc_phase ^= 1; }
          continue;
        }
      }
      if constexpr (EPI == kEpiQkvRope) {
        // RoPE epilogue: the row's KV destination and the first chunk's
        // cos/sin are loaded while the mainloop runs; each later chunk's
        // tables one chunk ahead of their use
        static_assert(EPI != kEpiQkvRope || CW == 32, "RoPE chunks are 32 columns");
        const RopeRow rq = rope_row(ra, row, M);
        const float rsq = norm_row_scale(na, row, M);
        RopeTab tb = rope_tab(ra, rq, n_blk * BN);
        sm100::mbar_wait(&tfull[acc], acc_phase);
        sm100::tc_fence_after();
#pragma unroll 1
        for (int c = 0; c < BN / 32; ++c) {
          uint32_t v[32];
          sm100::tmem_ld_32x32b_x32(taddr + c * 32, v);
          const int col = n_blk * BN + c * 32;
          RopeTab tn;
          if (c + 1 < BN / 32) tn = rope_tab(ra, rq, col + 32);
          sm100::tmem_ld_wait();
          if constexpr (XM) add_splits<32>(taddr + c * 32, n_split, BN, v);
          if (na.ssq_in != nullptr) scale_chunk<32>(v, rsq);
          if (row < M && col < N) {
            float f[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) f[i] = __uint_as_float(v[i]);
            if (bias != nullptr) {
              const float4* b4 = reinterpret_cast<const float4*>(bias + col);
#pragma unroll
              for (int q = 0; q < 8; ++q) {
                const float4 b = b4[q];
                f[4 * q] += b.x; f[4 * q + 1] += b.y; f[4 * q + 2] += b.z; f[4 * q + 3] += b.w;
              }
            }
            qkv_rope_chunk(f, row, col, ra, rq, tb);
          }
          if (c + 1 < BN / 32) tb = tn;
        }
        sm100::tc_fence_before();
        __syncwarp();
        if (lane == 0) sm100::mbar_arrive_cluster(leader_tempty + acc * 8);
        if (++acc == nacc) { acc = 0; acc_phase ^= 1; }
        continue;
      }
      const float rs = norm_row_scale(na, row, M);
      sm100::mbar_wait(&tfull[acc], acc_phase);
      sm100::tc_fence_after();
      float best = -INFINITY;
      int best_idx = 0x7fffffff;
      float gss = 0.0f;
#pragma unroll 1
      for (int c = 0; c < BN / CW; ++c) {
        uint32_t v[CW];
        tmem_ld_chunk<CW>(taddr + c * CW, v);
        sm100::tmem_ld_wait();
        if constexpr (XM) add_splits<CW>(taddr + c * CW, n_split, BN, v);
        if (na.ssq_in != nullptr) scale_chunk<CW>(v, rs);
        const int col = n_blk * BN + c * CW;
        if constexpr (EPI == kEpiArgmax) {
          argmax_chunk<CW>(v, col, N, row, M, sa, best, best_idx);
        } else {
          if (col < N) {
            float ss = 0.0f;
            epilogue_chunk<EPI, CW>(v, row, col, M, N, C, ldc, bias, na, ss, ra);
            if constexpr (EPI == kEpiResidualNorm)
              ssq_accum(gss, ss, col, N, na.ssq_out + (int64_t)row * ssq_parts(N), row < M);
          }
        }
      }
      if constexpr (EPI == kEpiArgmax) {
        if (row < M && n_blk < num_n) {
          const int tiles_n = (N + BN - 1) / BN;
          reinterpret_cast<float*>(C)[(int64_t)row * tiles_n + n_blk] = best;
          aux[(int64_t)row * tiles_n + n_blk] = best_idx;
        }
      }
      sm100::tc_fence_before();
      __syncwarp();
      if (lane == 0) sm100::mbar_arrive_cluster(leader_tempty + acc * 8);
      if (++acc == nacc) { acc = 0; acc_phase ^= 1; }
    }
  }
  sm100::tc_fence_before();
  sm100::cluster_sync();
  if (warp == 1) {
    sm100::tc_fence_after();
    if (tmem_wide) sm100::tmem_dealloc_pair<512>(tmem_base);
    else sm100::tmem_dealloc_pair<256>(tmem_base);
  }
}

// Small-M mode as its own kernel (SwapArgs): launched alone when the host
// knows the launch carries <= max_m rows, or beside the pair kernel (dual
// launch) when only the device knows the live row count; each exits after
// griddepcontrol.wait when the other one owns the launch.
constexpr uint32_t kSwapRing = 200 * 1024;

template <int EPI>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
gemm_swap_kernel(int M_cap, const int32_t* __restrict__ m_live, int N, int K, void* C, int ldc,
                 const float* __restrict__ bias, NormArgs na, RopeArgs ra, SwapArgs sw) {
  const int M = live_rows(M_cap, m_live);
  if (!(M >= 1 && M <= sw.max_m)) {
    grid_dep_sync();
    return;
  }
  swap_gemm<EPI>(kSwapRing, sw, M, N, K, C, ldc, bias, na, ra);
}

template <int EPI>
int launch_swap_typed(const GemmPlan& p, int M, cudaStream_t stream) {
  auto kern = gemm_swap_kernel<EPI>;
  constexpr size_t smem = 1024 + kSwapRing + 256;
  static bool attr_set = false;
  if (!attr_set) {
    SR_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr_set = true;
  }
  const int units = ((p.N + 255) / 256) * p.sw.splits;
  const int slots = num_sms() / 2;
  const int pairs = units < slots ? units : slots;
  sr::launch_k(kern, 2 * pairs, kThreads, smem, stream, M, p.m_live, p.N, p.K, p.c, p.ldc, p.bias, p.norm, p.rope,
               p.sw);
  return check_launch("gemm_swap_kernel");
}

template <int BN, int EPI, int MC, int KC, bool XM>
int launch_pair_mc(const GemmPlan& p, int M, cudaStream_t stream) {
  using Cfg = PairCfg<BN, KC>;
  auto kern = gemm_pair_kernel<BN, EPI, MC, KC, XM>;
  constexpr size_t smem = Cfg::kSmem + (kStagedEpi<BN, EPI, KC> ? Cfg::kEpiStageBytes : 0);
  static_assert(smem <= 232448, "pair GEMM shared memory exceeds 227 KB");
  static bool attr_set = false;
  if (!attr_set) {
    SR_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr_set = true;
  }
  const int tiles = ((M + 2 * kBM - 1) / (2 * kBM)) * (((p.N + BN - 1) / BN + MC - 1) / MC);
  const int slots = num_sms() / (2 * MC);
  const int clusters = tiles < slots ? tiles : slots;
  sr::launch_k(kern, 2 * MC * clusters, kThreads, smem, stream, p.a, p.b, M, p.m_live, p.N, p.K, p.c, p.ldc,
               p.bias, p.aux, p.sample, p.norm, p.rope, p.sw);
  return check_launch("gemm_pair_kernel");
}

template <int BN, int EPI>
int launch_pair_typed(const GemmPlan& p, int M, cudaStream_t stream) {
  const bool xm = p.sw.splits > 1;
  if constexpr (kSwapEpi<EPI>) {
    if (xm) {  // K ranges / small-M mode: KC 2 only (gemm_bf16_plan)
      if (p.kc != 2) return config_error("K-range / small-M GEMM plans need 128-k stages");
      return p.mc == 2 ? launch_pair_mc<BN, EPI, 2, 2, true>(p, M, stream)
                       : launch_pair_mc<BN, EPI, 1, 2, true>(p, M, stream);
    }
  }
  if (xm) return config_error("K ranges / small-M mode on an epilogue that has neither");
  if (p.mc == 2) {
    return p.kc == 2 ? launch_pair_mc<BN, EPI, 2, 2, false>(p, M, stream)
                     : launch_pair_mc<BN, EPI, 2, 1, false>(p, M, stream);
  }
  return p.kc == 2 ? launch_pair_mc<BN, EPI, 1, 2, false>(p, M, stream)
                   : launch_pair_mc<BN, EPI, 1, 1, false>(p, M, stream);
}

template <int BN>
int launch_pair_bn(const GemmPlan& p, int M, cudaStream_t stream) {
  switch (p.epi) {
    case kEpiStoreBf16: return launch_pair_typed<BN, kEpiStoreBf16>(p, M, stream);
    case kEpiResidualF32: return launch_pair_typed<BN, kEpiResidualF32>(p, M, stream);
    case kEpiResidualNorm:
      if constexpr (BN % 32 == 0) return launch_pair_typed<BN, kEpiResidualNorm>(p, M, stream);
      return config_error("residual+norm epilogue needs a tile width that is a multiple of 32");
    case kEpiQkvRope:
      if constexpr (BN % 32 == 0) return launch_pair_typed<BN, kEpiQkvRope>(p, M, stream);
      return config_error("RoPE epilogue needs a tile width that is a multiple of 32");
    case kEpiStoreF32: return launch_pair_typed<BN, kEpiStoreF32>(p, M, stream);
    case kEpiArgmax: return launch_pair_typed<BN, kEpiArgmax>(p, M, stream);
    case kEpiSwiGLU:
      if constexpr (BN % 32 == 0) return launch_pair_typed<BN, kEpiSwiGLU>(p, M, stream);
      return config_error("SwiGLU needs a tile width that is a multiple of 32");
  }
  return config_error("unknown epilogue");
}

}  // namespace

// one per tile width (gemm_pair_bn<BN>.cu); the small-M kernels (gemm_swap.cu)
int launch_swap(const GemmPlan& p, int M, cudaStream_t stream);
int launch_pair_bn64(const GemmPlan& p, int M, cudaStream_t stream);
int launch_pair_bn96(const GemmPlan& p, int M, cudaStream_t stream);
int launch_pair_bn112(const GemmPlan& p, int M, cudaStream_t stream);
int launch_pair_bn128(const GemmPlan& p, int M, cudaStream_t stream);
int launch_pair_bn160(const GemmPlan& p, int M, cudaStream_t stream);
int launch_pair_bn192(const GemmPlan& p, int M, cudaStream_t stream);
int launch_pair_bn224(const GemmPlan& p, int M, cudaStream_t stream);
int launch_pair_bn256(const GemmPlan& p, int M, cudaStream_t stream);

}  // namespace sr
