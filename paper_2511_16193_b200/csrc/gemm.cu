// K1: verify-forward GEMMs on the 5th-gen tensor cores.
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

namespace {

constexpr int kBM = 128, kBK = 64;
constexpr int kThreads = 192;

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
        y1[i] = x1 * cs[u] - x2 * sn[u];
        y2[i] = x2 * cs[u] + x1 * sn[u];
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
    float* out = reinterpret_cast<float*>(C) + (int64_t)row * ldc + col;
    __nv_bfloat16* hr = na.h_out + (int64_t)row * na.ld_h + col;
    if (full) {
#pragma unroll
      for (int q = 0; q < W / 8; ++q) {
        float4 a = reinterpret_cast<float4*>(out)[2 * q];
        float4 b = reinterpret_cast<float4*>(out)[2 * q + 1];
        a.x += f[8 * q]; a.y += f[8 * q + 1]; a.z += f[8 * q + 2]; a.w += f[8 * q + 3];
        b.x += f[8 * q + 4]; b.y += f[8 * q + 5]; b.z += f[8 * q + 6]; b.w += f[8 * q + 7];
        reinterpret_cast<float4*>(out)[2 * q] = a;
        reinterpret_cast<float4*>(out)[2 * q + 1] = b;
        ss = fmaf(a.x, a.x, ss); ss = fmaf(a.y, a.y, ss); ss = fmaf(a.z, a.z, ss); ss = fmaf(a.w, a.w, ss);
        ss = fmaf(b.x, b.x, ss); ss = fmaf(b.y, b.y, ss); ss = fmaf(b.z, b.z, ss); ss = fmaf(b.w, b.w, ss);
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
      for (int i = 0; i < W && col + i < N; ++i) {
        const float xn = out[i] + f[i];
        out[i] = xn;
        ss = fmaf(xn, xn, ss);
        hr[i] = __float2bfloat16_rn(xn * na.w[col + i]);
      }
    }
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
  float s = 0.0f;
  for (int t = 0; t < na.parts_in; ++t) s += p[t];
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
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
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
  grid_dep_sync();  // prologue above touched no predecessor output

  if (warp == 0) {
    {
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        const int m_blk = tile % num_m, n_blk = tile / num_m;
        for (int kb = 0; kb < num_kb; ++kb) {
          sm100::mbar_wait(&empty[stage], phase ^ 1);
          if (sm100::elect_one()) {
            sm100::mbar_arrive_expect_tx(&full[stage], Cfg::kStageBytes);
            sm100::tma_load_2d(sA + stage * Cfg::kABytes, &tmA, &full[stage], kb * kBK, m_blk * kBM,
                               sm100::kEvictLast);
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
      float ss = 0.0f;
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
          if (col < N) epilogue32<EPI>(v, row, col, M, N, C, ldc, bias, na, ss, ra);
        }
      }
      if constexpr (EPI == kEpiArgmax) {
        if (row < M) {
          const int tiles_n = (N + BN - 1) / BN;
          reinterpret_cast<float*>(C)[(int64_t)row * tiles_n + n_blk] = best;
          aux[(int64_t)row * tiles_n + n_blk] = best_idx;
        }
      }
      if constexpr (EPI == kEpiResidualNorm) {
        if (row < M) na.ssq_out[(int64_t)row * num_n + n_blk] = ss;
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
  static constexpr uint32_t kTmemCols = 2 * BN <= 256 ? 256 : 512;
  static constexpr int kChunk = BN % 32 == 0 ? 32 : 16;
  static constexpr size_t kSmem = 1024 + (size_t)kStages * kStageBytes + 256;
};

// residual epilogues stage through shared memory when the staging area fits
// next to the ring (every shape the planner picks except 160-wide tiles)
template <int BN, int EPI, int KC>
constexpr bool kStagedEpi = (EPI == kEpiResidualF32 || EPI == kEpiResidualNorm) && BN % 32 == 0 &&
                            PairCfg<BN, KC>::kSmem + PairCfg<BN, KC>::kEpiStageBytes <= 232448;

// MC = 2: a cluster of two pairs computes two horizontally adjacent tiles
// (n blocks 2j, 2j+1) of the same 256 rows.  Both pairs need the same
// activation rows, so each CTA loads half of its 128-row A block and
// multicasts it to itself and its counterpart in the other pair: A's L2->SM
// traffic halves, the bound of the small-N verify GEMMs (o, down, qkv).  A
// stage is reusable only when both pairs' MMAs have drained it, so the
// leaders' commits are multicast to all four CTAs' empty barriers (count 2).
template <int BN, int EPI, int MC, int KC>
__global__ void __cluster_dims__(2 * MC, 1, 1) __launch_bounds__(kThreads, 1)
gemm_pair_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                 int M_cap, const int32_t* __restrict__ m_live, int N, int K, void* C, int ldc,
                 const float* __restrict__ bias, int32_t* __restrict__ aux, SampleArgs sa, NormArgs na,
                 RopeArgs ra) {
  static_assert(MC == 1 || KC == 1 || KC == MC, "A multicast splits rows (KC 1) or k chunks (KC == MC)");
  const int M = live_rows(M_cap, m_live);
  using Cfg = PairCfg<BN, KC>;
  constexpr int S = Cfg::kStages;
  constexpr int CW = Cfg::kChunk;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
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
  if (warp == 1) sm100::tmem_alloc_pair<Cfg::kTmemCols>(tmem_slot);
  sm100::tc_fence_before();
  sm100::cluster_sync();
  sm100::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // after the barrier area (kSmem's trailing 256 B); launched with
  // kEpiStageBytes more dynamic smem when kStagedEpi
  float* epi_stage = reinterpret_cast<float*>(smem + S * Cfg::kStageBytes + 256);
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
          sm100::mbar_wait(&empty[stage], phase ^ 1);
          if (sm100::elect_one()) {
          if (rank == 0) sm100::mbar_arrive_expect_tx(&full[stage], 2 * Cfg::kStageBytes);
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
          if constexpr (KC > 1)
            sm100::tma_load_3d_pair(sB + stage * Cfg::kBBytes, &tmB, &full[stage], 0, brow, kb * KC,
                                    sm100::kEvictNormal);
          else
            sm100::tma_load_2d_pair(sB + stage * Cfg::kBBytes, &tmB, &full[stage], kb * kBK, brow,
                                    sm100::kEvictNormal);
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
        const uint32_t d = tmem_base + acc * BN;
        for (int kb = 0; kb < num_kb; ++kb) {
          sm100::mbar_wait(&full[stage], phase);
          sm100::tc_fence_after();
          const uint32_t a0 = sm100::smem_u32(sA + stage * Cfg::kABytes);
          const uint32_t b0 = sm100::smem_u32(sB + stage * Cfg::kBBytes);
          if (sm100::elect_one()) {
#pragma unroll
            for (int k = 0; k < KC * kBK / 16; ++k)
              sm100::umma_bf16_pair(d, sm100::umma_desc_sw128(a0 + (k >> 2) * Cfg::kAChunk + (k & 3) * 32),
                                    sm100::umma_desc_sw128(b0 + (k >> 2) * Cfg::kBChunk + (k & 3) * 32),
                                    idesc, (kb | k) != 0);
            sm100::umma_commit_pair(&empty[stage], MC == 1 ? 0x3 : 0xF);
          }
          __syncwarp();
          if (++stage == S) { stage = 0; phase ^= 1; }
        }
        if (sm100::elect_one()) sm100::umma_commit_pair(&tfull[acc], (uint16_t)(0x3u << lead));
        __syncwarp();
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
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
      const uint32_t taddr = tmem_base + ((uint32_t)(quad * 32) << 16) + acc * BN;
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
        float ss = 0.0f;
#pragma unroll
        for (int c = 0; c < BN / CW; ++c) {
          uint32_t v[CW];
          if constexpr (CW == 32) sm100::tmem_ld_32x32b_x32(taddr + c * CW, *reinterpret_cast<uint32_t(*)[32]>(v));
          else sm100::tmem_ld_32x32b_x16(taddr + c * CW, v);
          sm100::tmem_ld_wait();
          const int col = n_blk * BN + c * CW;
          if constexpr (kStagedEpi<BN, EPI, KC>) {
            if (n_blk * BN + BN <= N) {  // warp-uniform: full-width tile
              // 1) thread = row: x_new = residual + acc, sum of squares in column order
              float* T = epi_stage + quad * 32 * Cfg::kStageRow;
#pragma unroll
              for (int q = 0; q < 8; ++q) {
                float xn[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                  xn[i] = res[c * CW + 4 * q + i] + __uint_as_float(v[4 * q + i]);
                  if constexpr (EPI == kEpiResidualNorm) ss = fmaf(xn[i], xn[i], ss);
                }
                *reinterpret_cast<float4*>(T + lane * Cfg::kStageRow + 4 * q) =
                    make_float4(xn[0], xn[1], xn[2], xn[3]);
              }
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
#pragma unroll
            for (int q = 0; q < CW / 8; ++q) {
              float xn[8];
#pragma unroll
              for (int i = 0; i < 8; ++i) xn[i] = res[c * CW + 8 * q + i] + __uint_as_float(v[8 * q + i]);
              reinterpret_cast<float4*>(xr)[c * CW / 4 + 2 * q] = make_float4(xn[0], xn[1], xn[2], xn[3]);
              reinterpret_cast<float4*>(xr)[c * CW / 4 + 2 * q + 1] = make_float4(xn[4], xn[5], xn[6], xn[7]);
              if constexpr (EPI == kEpiResidualNorm) {
#pragma unroll
                for (int i = 0; i < 8; ++i) ss = fmaf(xn[i], xn[i], ss);
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
          } else if (row_ok && col < N) {
            epilogue_chunk<EPI, CW>(v, row, col, M, N, C, ldc, bias, na, ss, ra);
          }
        }
        if constexpr (EPI == kEpiResidualNorm) {
          if (row_ok && n_blk < num_n) na.ssq_out[(int64_t)row * num_n + n_blk] = ss;
        }
        sm100::tc_fence_before();
        __syncwarp();
        if (lane == 0) sm100::mbar_arrive_cluster(leader_tempty + acc * 8);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
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
          float ssp[8];
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
#pragma unroll
          for (int it = 0; it < 8; ++it) ssp[it] = 0.0f;
          sm100::mbar_wait(&tfull[acc], acc_phase);
          sm100::tc_fence_after();
#pragma unroll 1
          for (int c = 0; c < BN / 32; ++c) {
            uint32_t v[32];
            sm100::tmem_ld_32x32b_x32(taddr + c * 32, v);
            if (c + 1 < BN / 32) load_res(c + 1, xnext);
            sm100::tmem_ld_wait();
            const int col = n_blk * BN + c * 32;
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
                  ssp[it] = fmaf(xv.x, xv.x, ssp[it]);
                  ssp[it] = fmaf(xv.y, xv.y, ssp[it]);
                  ssp[it] = fmaf(xv.z, xv.z, ssp[it]);
                  ssp[it] = fmaf(xv.w, xv.w, ssp[it]);
                  uint2 hv;
                  hv.x = pack_bf16(xv.x * wv.x, xv.y * wv.y);
                  hv.y = pack_bf16(xv.z * wv.z, xv.w * wv.w);
                  reinterpret_cast<uint2*>(na.h_out + (int64_t)(row0 + r) * na.ld_h + col)[qq] = hv;
                }
              }
            }
            __syncwarp();
#pragma unroll
            for (int it = 0; it < 8; ++it) xres[it] = xnext[it];
          }
          if constexpr (EPI == kEpiResidualNorm) {
#pragma unroll
            for (int it = 0; it < 8; ++it) {
              float s_ = ssp[it];
              s_ += __shfl_xor_sync(0xffffffffu, s_, 1);
              s_ += __shfl_xor_sync(0xffffffffu, s_, 2);
              s_ += __shfl_xor_sync(0xffffffffu, s_, 4);
              const int r = it * 4 + (lane >> 3);
              if (qq == 0 && row0 + r < M) na.ssq_out[(int64_t)(row0 + r) * num_n + n_blk] = s_;
            }
          }
          sm100::tc_fence_before();
          __syncwarp();
          if (lane == 0) sm100::mbar_arrive_cluster(leader_tempty + acc * 8);
          if (++acc == 2) { acc = 0; acc_phase ^= 1; }
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
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        continue;
      }
      const float rs = norm_row_scale(na, row, M);
      sm100::mbar_wait(&tfull[acc], acc_phase);
      sm100::tc_fence_after();
      float best = -INFINITY;
      int best_idx = 0x7fffffff;
      float ss = 0.0f;
#pragma unroll 1
      for (int c = 0; c < BN / CW; ++c) {
        uint32_t v[CW];
        if constexpr (CW == 32) sm100::tmem_ld_32x32b_x32(taddr + c * CW, *reinterpret_cast<uint32_t(*)[32]>(v));
        else sm100::tmem_ld_32x32b_x16(taddr + c * CW, v);
        sm100::tmem_ld_wait();
        if (na.ssq_in != nullptr) scale_chunk<CW>(v, rs);
        const int col = n_blk * BN + c * CW;
        if constexpr (EPI == kEpiArgmax) {
          argmax_chunk<CW>(v, col, N, row, M, sa, best, best_idx);
        } else {
          if (col < N) epilogue_chunk<EPI, CW>(v, row, col, M, N, C, ldc, bias, na, ss, ra);
        }
      }
      if constexpr (EPI == kEpiResidualNorm) {
        if (row < M && n_blk < num_n) na.ssq_out[(int64_t)row * num_n + n_blk] = ss;
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
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  }
  sm100::tc_fence_before();
  sm100::cluster_sync();
  if (warp == 1) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc_pair<Cfg::kTmemCols>(tmem_base);
  }
}

PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (fn == nullptr) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

int g_num_sms = 0;
int g_pair_kc = [] {
  const char* v = getenv("SR_GEMM_KC");
  return (v && v[0] == '1') ? 1 : 2;
}();

int num_sms() {
  if (g_num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  return g_num_sms;
}

template <int BN, int EPI>
int launch_typed(const GemmPlan& p, int M, cudaStream_t stream) {
  using Cfg = GemmCfg<BN>;
  auto kern = gemm_tcgen05_kernel<BN, EPI>;
  static bool attr_set = false;
  if (!attr_set) {
    SR_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::kSmem));
    attr_set = true;
  }
  const int tiles = ((M + kBM - 1) / kBM) * ((p.N + BN - 1) / BN);
  const int grid = tiles < num_sms() ? tiles : num_sms();
  sr::launch_k(kern, grid, kThreads, Cfg::kSmem, stream, p.a, p.b, M, p.m_live, p.N, p.K, p.c, p.ldc, p.bias, p.aux,
               p.sample, p.norm, p.rope);
  return check_launch("gemm_tcgen05_kernel");
}

template <int BN>
int launch_bn(const GemmPlan& p, int M, cudaStream_t stream) {
  switch (p.epi) {
    case kEpiStoreBf16: return launch_typed<BN, kEpiStoreBf16>(p, M, stream);
    case kEpiResidualF32: return launch_typed<BN, kEpiResidualF32>(p, M, stream);
    case kEpiResidualNorm: return launch_typed<BN, kEpiResidualNorm>(p, M, stream);
    case kEpiQkvRope: return launch_typed<BN, kEpiQkvRope>(p, M, stream);
    case kEpiSwiGLU: return launch_typed<BN, kEpiSwiGLU>(p, M, stream);
    case kEpiStoreF32: return launch_typed<BN, kEpiStoreF32>(p, M, stream);
    case kEpiArgmax: return launch_typed<BN, kEpiArgmax>(p, M, stream);
  }
  return config_error("unknown epilogue");
}


template <int BN, int EPI, int MC, int KC>
int launch_pair_mc(const GemmPlan& p, int M, cudaStream_t stream) {
  using Cfg = PairCfg<BN, KC>;
  auto kern = gemm_pair_kernel<BN, EPI, MC, KC>;
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
               p.bias, p.aux, p.sample, p.norm, p.rope);
  return check_launch("gemm_pair_kernel");
}

template <int BN, int EPI>
int launch_pair_typed(const GemmPlan& p, int M, cudaStream_t stream) {
  if (p.mc == 2) {
    return p.kc == 2 ? launch_pair_mc<BN, EPI, 2, 2>(p, M, stream) : launch_pair_mc<BN, EPI, 2, 1>(p, M, stream);
  }
  return p.kc == 2 ? launch_pair_mc<BN, EPI, 1, 2>(p, M, stream) : launch_pair_mc<BN, EPI, 1, 1>(p, M, stream);
}

template <int BN>
int launch_pair_bn(const GemmPlan& p, int M, cudaStream_t stream) {
  switch (p.epi) {
    case kEpiStoreBf16: return launch_pair_typed<BN, kEpiStoreBf16>(p, M, stream);
    case kEpiResidualF32: return launch_pair_typed<BN, kEpiResidualF32>(p, M, stream);
    case kEpiResidualNorm: return launch_pair_typed<BN, kEpiResidualNorm>(p, M, stream);
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

int launch_pair(const GemmPlan& p, int M, cudaStream_t stream) {
  switch (p.bn) {
    case 64: return launch_pair_bn<64>(p, M, stream);
    case 96: return launch_pair_bn<96>(p, M, stream);
    case 112: return launch_pair_bn<112>(p, M, stream);
    case 128: return launch_pair_bn<128>(p, M, stream);
    case 160: return launch_pair_bn<160>(p, M, stream);
    case 192: return launch_pair_bn<192>(p, M, stream);
    case 224: return launch_pair_bn<224>(p, M, stream);
    case 256: return launch_pair_bn<256>(p, M, stream);
  }
  return config_error("unsupported pair tile width (64|96|112|128|160|192|224|256)");
}

// Pair tile (width, pairs per cluster).  Measured on B200 (scripts/
// gemm_probe.py) the pair kernel is MMA-bound once operands are staged 128 k
// per TMA instruction: a 64-k block of a 256 x BN tile costs ~1.64 ns * BN,
// plus ~1.5 us per tile of fill/drain.  Minimize waves x per-tile time over
// widths that are multiples of 32 (16-column epilogue chunks measured
// slower).  Two pairs per cluster multicasting A save ~3% when the grid is a
// single wave with an even tile count per row block, and lose badly
// (cluster-of-4 residency) over several waves.
// tuning probe: cap the pair tile width (SR_PAIR_BN_MAX, default 256)
int g_pair_bn_max = [] {
  const char* v = getenv("SR_PAIR_BN_MAX");
  const int b = v ? atoi(v) : 256;
  return b >= 64 && b <= 256 ? b : 256;
}();

void choose_pair_tile(int M, int N, int K, int epi, int* bn_out, int* mc_out) {
  static const int cands[] = {256, 224, 192, 160, 128, 96, 64};
  const int num_m = (M + 255) / 256;
  const int kb = (K + 63) / 64;
  const int pairs = num_sms() / 2;
  int best = g_pair_bn_max;
  double best_t = 1e30;
  for (int bn : cands) {
    if (bn > g_pair_bn_max) continue;
    if ((epi == kEpiSwiGLU || epi == kEpiQkvRope) && bn % 32 != 0) continue;
    const int tiles = num_m * ((N + bn - 1) / bn);
    const int waves = (tiles + pairs - 1) / pairs;
    const double t = waves * ((double)kb * bn + 900.0);
    if (t < best_t * 0.999) { best_t = t; best = bn; }
  }
  const int num_n = (N + best - 1) / best;
  const int clusters = num_m * (num_n / 2);
  *bn_out = best;
  // A multicast couples the rings of two pairs; with the 3-stage ring of the
  // widest tiles that stalls both (7B o / down: 2x slower), so only <= 160.
  *mc_out = (num_n % 2 == 0 && clusters <= num_sms() / 4 && best <= 160) ? 2 : 1;
}
}  // namespace

int make_tmap_bf16(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer,
                   uint64_t row_bytes, uint32_t box_inner, uint32_t box_outer) {
  auto enc = tmap_encoder();
  if (enc == nullptr) {
    set_error("cuTensorMapEncodeTiled unavailable (driver too old?)");
    return SR_ERR_RUNTIME;
  }
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {row_bytes};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d): inner=%llu outer=%llu stride=%llu", (int)r,
              (unsigned long long)inner, (unsigned long long)outer, (unsigned long long)row_bytes);
    return SR_ERR_CONFIG;
  }
  return SR_OK;
}

// [rows, K] bf16 viewed as (64-element k chunk, row, chunk index): a box of
// (64, box_rows, box_chunks) lands as box_chunks swizzled [box_rows x 128 B]
// blocks back to back -- the K-major SW128 layout UMMA reads per 16-k step.
int make_tmap_bf16_3d(CUtensorMap* map, const void* base, uint64_t K, uint64_t rows, uint64_t row_bytes,
                      uint32_t box_rows, uint32_t box_chunks) {
  auto enc = tmap_encoder();
  if (enc == nullptr) {
    set_error("cuTensorMapEncodeTiled unavailable (driver too old?)");
    return SR_ERR_RUNTIME;
  }
  cuuint64_t dims[3] = {(cuuint64_t)kBK, rows, K / kBK};
  cuuint64_t strides[2] = {row_bytes, (cuuint64_t)kBK * 2};
  cuuint32_t box[3] = {(cuuint32_t)kBK, box_rows, box_chunks};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled (3d) failed (%d): K=%llu rows=%llu", (int)r, (unsigned long long)K,
              (unsigned long long)rows);
    return SR_ERR_CONFIG;
  }
  return SR_OK;
}

int gemm_bf16_plan(GemmPlan* p, int M, int N, int K, const __nv_bfloat16* A, int lda,
                   const __nv_bfloat16* W, int ldw, void* C, int ldc, int epi,
                   const float* bias, int bn, int32_t* aux) {
  SR_REQUIRE(M >= 0 && N > 0 && K > 0, "bad GEMM shape");
  SR_REQUIRE(epi != kEpiArgmax || aux != nullptr, "argmax epilogue needs an index buffer");
  SR_REQUIRE(lda % 8 == 0 && ldw % 8 == 0 && lda >= K && ldw >= K, "lda/ldw must be >= K and multiples of 8");
  SR_REQUIRE(epi == kEpiArgmax || ldc % 8 == 0, "ldc must be a multiple of 8");
  SR_REQUIRE(((uintptr_t)A & 15) == 0 && ((uintptr_t)W & 15) == 0 && ((uintptr_t)C & 15) == 0,
             "A, W, C must be 16-byte aligned");
  bool pair;
  int mc = 1;
  if (bn == 0) {
    pair = M >= 256;
    // gate_up at M = 256j + (<= 128) rows (e.g. 64 prompts x 5 = 320): the
    // last 256-row pair block would be mostly padding; 128-row single-CTA
    // tiles waste less (7B 99 -> 90 us, 32B 200 -> 190 us at M = 320)
    if (pair && epi == kEpiSwiGLU && M % 256 != 0 && M % 256 <= 128) pair = false;
    if (pair) choose_pair_tile(M, N, K, epi, &bn, &mc);
    else bn = N >= 4096 ? 256 : 128;
  } else if (bn < 0) {
    pair = true;
    bn = -bn;
    if (bn > 1024) { mc = 2; bn -= 1024; }
  } else {
    pair = false;
    SR_REQUIRE(bn == 128 || bn == 256, "single-CTA bn must be 128 or 256");
  }
  if (pair) SR_REQUIRE(bn % 16 == 0 && bn >= 64 && bn <= 256, "pair bn must be a multiple of 16 in [64, 256]");
  SR_REQUIRE(epi != kEpiSwiGLU || (N % 32 == 0 && bn % 32 == 0), "SwiGLU needs N and bn multiples of 32");
  SR_REQUIRE(epi != kEpiQkvRope || (N % 32 == 0 && bn % 32 == 0), "qkv RoPE needs N and bn multiples of 32");
  p->M = M; p->N = N; p->K = K; p->bn = bn; p->epi = epi; p->c = C; p->ldc = ldc; p->bias = bias;
  p->aux = aux;
  p->pair = pair;
  p->mc = mc;
  p->kc = (pair && K % kBK == 0 && g_pair_kc == 2) ? 2 : 1;
  p->sample = SampleArgs{nullptr, nullptr, 0u, 0.0f};
  p->m_live = nullptr;
  const int mrows = M > 0 ? M : 1;
  if (p->kc > 1) {
    int rc = mc == 2 ? make_tmap_bf16(&p->a, A, (uint64_t)K, (uint64_t)mrows, (uint64_t)lda * 2, kBK, kBM)
                     : make_tmap_bf16_3d(&p->a, A, (uint64_t)K, (uint64_t)mrows, (uint64_t)lda * 2, kBM, p->kc);
    if (rc) return rc;
    return make_tmap_bf16_3d(&p->b, W, (uint64_t)K, (uint64_t)N, (uint64_t)ldw * 2, bn / 2, p->kc);
  }
  int rc = make_tmap_bf16(&p->a, A, (uint64_t)K, (uint64_t)mrows, (uint64_t)lda * 2, kBK,
                          mc == 2 ? kBM / 2 : kBM);
  if (rc) return rc;
  return make_tmap_bf16(&p->b, W, (uint64_t)K, (uint64_t)N, (uint64_t)ldw * 2, kBK, pair ? bn / 2 : bn);
}

int gemm_bf16_launch(const GemmPlan& p, cudaStream_t stream, int m_override) {
  const int M = m_override >= 0 ? m_override : p.M;
  SR_REQUIRE(p.epi != kEpiResidualNorm ||
                 (p.norm.h_out != nullptr && p.norm.w != nullptr && p.norm.ssq_out != nullptr && p.N % 8 == 0),
             "residual+norm epilogue needs NormArgs (h_out, w, ssq_out) and N % 8 == 0");
  SR_REQUIRE(p.epi != kEpiQkvRope ||
                 (p.rope.pos != nullptr && p.rope.kv_dst != nullptr && p.rope.kv_info != nullptr &&
                  p.rope.cos != nullptr && p.rope.q_out != nullptr && p.rope.cache != nullptr &&
                  p.rope.hd % 32 == 0 && p.N == (p.rope.nq + 2 * p.rope.nkv) * p.rope.hd),
             "qkv RoPE epilogue needs RopeArgs and head_dim % 32 == 0");
  if (M == 0) return SR_OK;
  if (p.pair) return launch_pair(p, M, stream);
  return p.bn == 256 ? launch_bn<256>(p, M, stream) : launch_bn<128>(p, M, stream);
}

int gemm_num_n_tiles(int N, int bn) { return (N + bn - 1) / bn; }

// ---------------------------------------------------------------------------
// fp32 parity GEMM (CUDA cores).  64x64 tile, 256 threads, 4x4 per thread,
// k ascending in steps of 16: deterministic and batch invariant.

namespace {

constexpr int kFT = 64, kFK = 16;

template <int EPI>
__global__ void __launch_bounds__(256)
gemm_f32_kernel(int M, int N, int K, const float* __restrict__ A, int lda,
                const float* __restrict__ W, int ldw, float* __restrict__ C, int ldc,
                const float* __restrict__ bias) {
  grid_dep_sync();
  __shared__ float sa[kFK][kFT + 4];
  __shared__ float sw[kFK][kFT + 4];
  const int m0 = blockIdx.y * kFT, n0 = blockIdx.x * kFT;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += kFK) {
    for (int i = threadIdx.x; i < kFT * kFK; i += 256) {
      const int r = i / kFK, kk = i % kFK;
      sa[kk][r] = (m0 + r < M && k0 + kk < K) ? A[(int64_t)(m0 + r) * lda + k0 + kk] : 0.0f;
      sw[kk][r] = (n0 + r < N && k0 + kk < K) ? W[(int64_t)(n0 + r) * ldw + k0 + kk] : 0.0f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < kFK; ++kk) {
      float a[4], w[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) { a[i] = sa[kk][ty * 4 + i]; w[i] = sw[kk][tx * 4 + i]; }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], w[j], acc[i][j]);
    }
    __syncthreads();
  }
  // stage the 64x64 tile so the SwiGLU epilogue can pair gate column c with
  // up column c+16 (held by another thread)
  __shared__ float tile[kFT][kFT + 1];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) tile[ty * 4 + i][tx * 4 + j] = acc[i][j];
  __syncthreads();
  for (int e = threadIdx.x; e < kFT * kFT; e += 256) {
    const int r = e / kFT, cidx = e % kFT;
    const int row = m0 + r, col = n0 + cidx;
    if (row >= M || col >= N) continue;
    const float v = tile[r][cidx];
    if constexpr (EPI == kEpiSwiGLU) {
      if ((col & 31) >= 16) continue;
      const float up = tile[r][cidx + 16];
      C[(int64_t)row * ldc + (col >> 5) * 16 + (col & 15)] = v / (1.0f + expf(-v)) * up;
    } else if constexpr (EPI == kEpiResidualF32) {
      C[(int64_t)row * ldc + col] += v;
    } else {
      C[(int64_t)row * ldc + col] = v + (bias != nullptr ? bias[col] : 0.0f);
    }
  }
}

}  // namespace

int gemm_f32(int M, int N, int K, const float* A, int lda, const float* W, int ldw, void* C,
             int ldc, int epi, const float* bias, cudaStream_t stream) {
  SR_REQUIRE(M >= 0 && N > 0 && K > 0, "bad GEMM shape");
  if (M == 0) return SR_OK;
  dim3 grid((N + kFT - 1) / kFT, (M + kFT - 1) / kFT);
  float* c = reinterpret_cast<float*>(C);
  switch (epi) {
    case kEpiStoreBf16:
    case kEpiStoreF32:
      sr::launch_k(gemm_f32_kernel<kEpiStoreF32>, grid, 256, 0, stream, M, N, K, A, lda, W, ldw, c, ldc, bias);
      break;
    case kEpiResidualF32:
      sr::launch_k(gemm_f32_kernel<kEpiResidualF32>, grid, 256, 0, stream, M, N, K, A, lda, W, ldw, c, ldc, bias);
      break;
    case kEpiSwiGLU:
      sr::launch_k(gemm_f32_kernel<kEpiSwiGLU>, grid, 256, 0, stream, M, N, K, A, lda, W, ldw, c, ldc, bias);
      break;
    default:
      return config_error("unknown epilogue");
  }
  return check_launch("gemm_f32_kernel");
}

}  // namespace sr

extern "C" int sr_gemm(int dtype, int M, int N, int K, const void* A, int lda, const void* W,
                       int ldw, void* C, int ldc, int epilogue, const float* bias, int bn,
                       int32_t* aux, sr_stream_t stream) {
  SR_REQUIRE(epilogue >= 0 && epilogue <= sr::kEpiArgmax,
             "epilogue must be 0..4 (the fused-norm epilogue is internal to sr_model_forward)");
  if (dtype == 1) {
    sr::GemmPlan plan;
    int rc = sr::gemm_bf16_plan(&plan, M, N, K, reinterpret_cast<const __nv_bfloat16*>(A), lda,
                                reinterpret_cast<const __nv_bfloat16*>(W), ldw, C, ldc, epilogue,
                                bias, bn, aux);
    if (rc) return rc;
    return sr::gemm_bf16_launch(plan, (cudaStream_t)stream);
  }
  SR_REQUIRE(dtype == 0, "dtype must be 0 (f32) or 1 (bf16)");
  SR_REQUIRE(epilogue != sr::kEpiArgmax, "argmax epilogue is bf16-only; use sr_argmax_rows");
  return sr::gemm_f32(M, N, K, reinterpret_cast<const float*>(A), lda,
                      reinterpret_cast<const float*>(W), ldw, C, ldc, epilogue, bias,
                      (cudaStream_t)stream);
}
