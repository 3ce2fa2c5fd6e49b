// K2: verification attention over the paged KV cache.
//
// One CTA = (sequence, kv head, query block of 32 rows, KV split).  Rows are
// (window position j, group head g) pairs, r = j*G + g, so all query heads
// sharing a kv head read each K/V tile once (GQA).  Keys are walked in
// tiles of 64 *absolute* positions (tile t = keys [64t, 64t+64)); a key comes
// from the paged cache when it is committed (pos < ctx_len) or written in
// place, else from the drafter-branch window buffer.  Splits are fixed
// 2048-key ranges (sr_set_attention_split) merged by a combine kernel in
// split order.  Because the
// tiling depends only on absolute positions, a query's arithmetic is the
// same in a 5-position verify window and in a 1-position decode step: the
// speculative and plain paths produce bit-identical logits.
//
// Per tile: 3-stage cp.async ring (16-byte, XOR-swizzled) for K/V; warp w
// owns keys 16w..16w+15 of each tile: S = Q K^T with mma.sync m16n8k16 bf16,
// warp-level online softmax in registers (quad shuffles, exp2), P re-used as
// the A fragment of O += P V without touching shared memory.  The 4 warps'
// states merge once per CTA.  HBM-bound: the kernel's algorithmic bytes are
// the K/V tiles it reads.
#include "common.cuh"
#include "layers.cuh"
#include "sm100.cuh"

#include <cuda_bf16.h>

#include <algorithm>
#include <type_traits>
#include <cstdio>
#include <cstdlib>

namespace sr {

namespace {

#ifndef SR_ATTN_PROBE
#define SR_ATTN_PROBE 0
#endif

constexpr int kKT = 64;          // keys per tile (= page size)
constexpr int kRows = 32;        // query rows per CTA
constexpr int kMaxLayers = 128;  // per-layer work-claim counters
constexpr int kStages = 3;       // cp.async ring depth
constexpr int kAttnThreads = 256;  // 8 warps: (m-tile, 16-key slice) pairs

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(smem)),
               "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void mma_bf16(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// 2^x on the SFU (ex2.approx.ftz: ~2 ulp, -inf -> +0).  Used for every
// softmax exponent of the bf16 path, so verify and decode stay bit-identical.
__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// [rows][HD] bf16 tile, 16-byte chunks XOR-swizzled by (row & 7).
template <int HD>
__device__ __forceinline__ uint32_t swz(int row, int chunk) {
  return (uint32_t)(row * HD * 2 + ((chunk ^ (row & 7)) << 4));
}

struct AttnArgs {
  const __nv_bfloat16* q;  // [M, nq, HD]
  const SeqInfo* seqs;
  KvLayout kv;
  int layer, nq, G;
  float scale_log2;
  float* part_o;   // [S*nkv, qblocks, splits, 64, HD]
  float* part_ml;  // [S*nkv, qblocks, splits, 64, 2]
  int qblocks, splits;
  int split_tiles;     // tiles per KV split (fixed per model: batch invariance)
  __nv_bfloat16* out;  // [M, nq, HD]
  int* order;          // work items, longest first (attn_plan_kernel)
  int* counters;       // [0] items in order, [1 + layer] work-claim counter of a layer
  int n_slots;         // S*nkv * qblocks * splits
};

int g_split_tiles = [] {  // 2048-key splits (SR_ATTN_SPLIT overrides, for tuning)
  // SR_ATTN_SPLIT counts 64-key TILES, like sr_set_attention_split, and gets
  // the same [4, 1024] check: hist[] in attn_plan_kernel holds 1025 entries
  // and the workspace bound assumes >= 4 tiles per split.  Out-of-range
  // values are ignored (with a warning) rather than clamped silently.
  const char* v = getenv("SR_ATTN_SPLIT");
  if (!v) return 32;
  const int t = atoi(v);
  if (t < 4 || t > 1024) {
    fprintf(stderr, "specrollout_b200: SR_ATTN_SPLIT=%s ignored (64-key tiles, must be in [4, 1024])\n", v);
    return 32;
  }
  return t;
}();

__device__ __forceinline__ int block_max_key(const SeqInfo& sq, int r0, int rows, int G) {
  return sq.ctx_len + (r0 + rows - 1) / G;
}

// FA2-style split-K inside the CTA: warp w owns keys [16w, 16w+16) of every
// 64-key tile, keeps its own online-softmax state and O accumulator in
// registers (no block barrier inside the math), and the 4 warps merge in a
// fixed order at the end.  One __syncthreads per tile guards the 3-stage
// cp.async ring.
template <int HD>
__global__ void __launch_bounds__(kAttnThreads, 2)
attn_bf16_kernel(AttnArgs A) {
  grid_dep_sync();
  constexpr int CH = HD / 8;       // 16-byte chunks per row
  constexpr int NO = HD / 8;       // n8 tiles of O per m-tile
  constexpr uint32_t kTileBytes = kKT * HD * 2;
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* sQ = smem;                              // [kRows][HD]
  uint8_t* sKV = sQ + kRows * HD * 2;              // [stages][K tile, V tile]

  const int nkv = A.kv.kv_heads;
  const int G = A.G;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // K/V ring: stage = [K tile | V tile]; full[stage] completes when both land.
  // Stage/parity follow a CTA-global tile counter so the ring runs across items.
  __shared__ __align__(8) uint64_t full[kStages];
  __shared__ int s_item;
  if (tid == 0) {
    for (int i = 0; i < kStages; ++i) sm100::mbar_init(&full[i], 1);
    sm100::fence_barrier_init();
  }
  uint32_t gi = 0;
  for (;;) {
  __syncthreads();  // previous item fully consumed (smem reusable)
  if (tid == 0) s_item = atomicAdd(&A.counters[1 + A.layer], 1);
  __syncthreads();
  if (s_item >= A.counters[0]) break;
  const int packed = A.order[s_item];
  const int sp = packed % A.splits;
  const int qb = (packed / A.splits) % A.qblocks;
  const int z = packed / (A.splits * A.qblocks);
  const int s = z / nkv, h = z % nkv;
  const SeqInfo sq = A.seqs[s];
  const int rows_total = sq.q_len * G;
  const int r0 = qb * kRows;
  const int rows = min(kRows, rows_total - r0);
  const int max_key = block_max_key(sq, r0, rows, G);
  const int ntiles = max_key / kKT + 1;
  const int t_begin = sp * A.split_tiles, t_end = min(ntiles, t_begin + A.split_tiles);
  const int mtv = (rows + 15) / 16;

  const __nv_bfloat16* cache = reinterpret_cast<const __nv_bfloat16*>(A.kv.cache) +
                               (int64_t)A.layer * A.kv.cache_layer_elems();
  const __nv_bfloat16* win = reinterpret_cast<const __nv_bfloat16*>(A.kv.window) +
                             (int64_t)A.layer * A.kv.window_layer_elems();
  const int32_t* btab = A.kv.block_table + (int64_t)sq.request * A.kv.max_pages;
  const int psz = A.kv.page;
  SR_DCHECK(max_key / psz < A.kv.max_pages || sq.branch >= 0);

  for (int e = tid; e < kRows * CH; e += kAttnThreads) {
    const int r = e / CH, c = e % CH;
    uint8_t* dst = sQ + swz<HD>(r, c);
    if (r < rows) {
      const int gr = r0 + r, j = gr / G, g = gr % G;
      cp_async16(dst, A.q + ((int64_t)(sq.q_start + j) * A.nq + h * G + g) * HD + c * 8);
    } else {
      *reinterpret_cast<uint4*>(dst) = make_uint4(0, 0, 0, 0);
    }
  }

  // Called by all threads (uniform control flow).
  auto load_tile = [&](int t, int stage) {
    if (t >= t_end) return;
    uint8_t* k_dst = sKV + stage * 2 * kTileBytes;
    uint8_t* v_dst = k_dst + kTileBytes;
    const int last = t * kKT + kKT - 1;
    if (sq.branch < 0 || last < sq.ctx_len) {
      // a page of the paged cache: K and V of head h are two contiguous 16 KB
      // blocks stored pre-swizzled -> two TMA bulk copies, no thread work.
      // Slots past max_key (the tail of the last page) hold stale finite
      // values (the cache is zero-initialised, sr_model_desc): their scores
      // are masked to -inf, so p = 0 and 0 * v adds exactly nothing.
      if (tid == 0) {
#if SR_ATTN_PROBE == 2  // measurement build: compute only, no K/V traffic
        sm100::mbar_arrive(&full[stage]);
        return;
#endif
        const __nv_bfloat16* kb = cache + ((int64_t)btab[t] * 2 * nkv + h) * psz * HD;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        sm100::mbar_arrive_expect_tx(&full[stage], 2 * kTileBytes);
        // KV pages are read once per layer: evict-first keeps them from
        // displacing the weights prefetched into L2 for the next GEMMs
        sm100::bulk_load_hint(k_dst, kb, kTileBytes, &full[stage], sm100::kEvictFirst);
        sm100::bulk_load_hint(v_dst, kb + (int64_t)nkv * psz * HD, kTileBytes, &full[stage], sm100::kEvictFirst);
      }
      return;
    }
    // tile reaching drafter-branch window keys: synchronous swizzle-aware copy
    for (int e = tid; e < kKT * CH; e += kAttnThreads) {
      const int r = e / CH, pc = e % CH;        // destination row, physical chunk
      const int kp = t * kKT + r;
      const uint32_t off = (uint32_t)(r * HD * 2 + pc * 16);
      uint4 kv4 = make_uint4(0, 0, 0, 0), vv4 = make_uint4(0, 0, 0, 0);
      if (kp <= max_key) {
        const __nv_bfloat16* ksrc;
        int64_t vstep;
        int src_chunk;
        if (sq.branch < 0 || kp < sq.ctx_len) {
          const int page = btab[kp / psz];
          ksrc = cache + (((int64_t)page * 2 * nkv + h) * psz + kp % psz) * HD;
          vstep = (int64_t)nkv * psz * HD;
          src_chunk = pc;  // page slot == tile row: same swizzle
        } else {
          const int j = kp - sq.ctx_len;
          ksrc = win + (((int64_t)sq.branch * 2 * nkv + h) * A.kv.window_max + j) * HD;
          vstep = (int64_t)nkv * A.kv.window_max * HD;
          src_chunk = (pc ^ (r & 7)) ^ (j & 7);  // logical chunk re-swizzled by window slot
        }
        kv4 = *reinterpret_cast<const uint4*>(ksrc + src_chunk * 8);
        vv4 = *reinterpret_cast<const uint4*>(ksrc + vstep + src_chunk * 8);
      }
      *reinterpret_cast<uint4*>(k_dst + off) = kv4;
      *reinterpret_cast<uint4*>(v_dst + off) = vv4;
    }
    if (tid == 0) sm100::mbar_arrive(&full[stage]);
  };

  // warp (mw, kw): m-tile mw (rows 16mw..), keys [16kw, 16kw+16) of each tile
  const int mw = warp >> 2, kw = warp & 3;
  const bool active = mw < mtv;
  float o[NO][4];
  float m_run[2] = {-INFINITY, -INFINITY}, l_run[2] = {0.0f, 0.0f};
#pragma unroll
  for (int nt = 0; nt < NO; ++nt)
#pragma unroll
    for (int i = 0; i < 4; ++i) o[nt][i] = 0.0f;
  // query position of this thread's rows g=lane/4 and g+8 (causal mask)
  int qpos[2];
#pragma unroll
  for (int hi = 0; hi < 2; ++hi) {
    const int r = mw * 16 + (lane >> 2) + hi * 8;
    qpos[hi] = r < rows ? sq.ctx_len + (r0 + r) / G : -1;  // -1: padding row, all masked
  }
  const int min_qpos = sq.ctx_len + r0 / G;  // first query row of the block
  load_tile(t_begin, gi % kStages);
  load_tile(t_begin + 1, (gi + 1) % kStages);
  cp_async_commit();
  cp_async_wait<0>();  // Q block
  // ldmatrix addresses, hoisted: a fragment row r reads logical chunk
  // 2kk + b, stored at physical chunk (2kk + b) ^ (r & 7).  With kk = 4u + j
  // that is 8u + ((2j + b) ^ (r & 7)), so four per-thread offsets (j) plus an
  // immediate 128u bytes address every k step.
  const int mi = lane >> 3, x7 = lane & 7;
  uint32_t qo[4], ko[4], vo[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    qo[j] = (uint32_t)__cvta_generic_to_shared(sQ) + (mw * 16 + (mi & 1) * 8 + x7) * HD * 2 +
            (((2 * j + (mi >> 1)) ^ x7) << 4);
    ko[j] = (kw * 16 + (mi >> 1) * 8 + x7) * HD * 2 + (((2 * j + (mi & 1)) ^ x7) << 4);
    vo[j] = (kw * 16 + (mi & 1) * 8 + x7) * HD * 2 + (((2 * j + (mi >> 1)) ^ x7) << 4);
  }
  const float sl2 = A.scale_log2;

  // One 64-key tile for this warp's 16 rows x 16 keys; MASK: some key of the
  // slice may lie past a row's query position (the block's last tiles).
  auto tile_math = [&](auto mask_tag, uint32_t k_base, int key0) {
    constexpr bool MASK = decltype(mask_tag)::value;
    const uint32_t v_base = k_base + kTileBytes;
    // S = Q K^T for this warp's 16 keys
    float sacc[2][4] = {{0, 0, 0, 0}, {0, 0, 0, 0}};
#pragma unroll
    for (int kk = 0; kk < HD / 16; ++kk) {
      uint32_t a0, a1, a2, a3, b0, b1, b2, b3;
      ldsm_x4(qo[kk & 3] + (kk >> 2) * 128, a0, a1, a2, a3);
      ldsm_x4(k_base + ko[kk & 3] + (kk >> 2) * 128, b0, b1, b2, b3);
      mma_bf16(sacc[0], a0, a1, a2, a3, b0, b1);
      mma_bf16(sacc[1], a0, a1, a2, a3, b2, b3);
    }
    float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int hi = i >> 1;
        if constexpr (MASK) {
          const int kp = key0 + nt * 8 + 2 * (lane & 3) + (i & 1);
          if (kp > qpos[hi]) sacc[nt][i] = -INFINITY;
        }
        mx[hi] = fmaxf(mx[hi], sacc[nt][i]);
      }
    uint32_t pa[4];
    bool rescale = false;
    float alpha[2];
#pragma unroll
    for (int hi = 0; hi < 2; ++hi) {
      mx[hi] = fmaxf(mx[hi], __shfl_xor_sync(0xffffffffu, mx[hi], 1));
      mx[hi] = fmaxf(mx[hi], __shfl_xor_sync(0xffffffffu, mx[hi], 2));
      // lazy rescaling (FA4): keep the reference max m_run (raw score units)
      // unless the new max exceeds it by more than 8 in log2 units; p can
      // then reach 2^8, harmless in fp32/bf16.  The decision depends only on
      // this row's keys in tile order, so it is batch invariant.
      const float m_old = m_run[hi];
      const bool up = mx[hi] != -INFINITY && (m_old == -INFINITY || (mx[hi] - m_old) * sl2 > 8.0f);
      alpha[hi] = 1.0f;
      if (up) {
        alpha[hi] = m_old == -INFINITY ? 0.0f : fast_exp2((m_old - mx[hi]) * sl2);
        m_run[hi] = mx[hi];
        rescale = true;
      }
      const float m_ref = m_run[hi];
      const float neg = m_ref == -INFINITY ? 0.0f : -m_ref * sl2;
      float p[4];
#pragma unroll
      for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int c = 0; c < 2; ++c) p[nt * 2 + c] = fast_exp2(fmaf(sacc[nt][hi * 2 + c], sl2, neg));
      const float rs = ((p[0] + p[1]) + p[2]) + p[3];
      l_run[hi] = l_run[hi] * alpha[hi] + rs;
      __nv_bfloat162 lo = __floats2bfloat162_rn(p[0], p[1]);
      __nv_bfloat162 hi2 = __floats2bfloat162_rn(p[2], p[3]);
      pa[hi] = *reinterpret_cast<uint32_t*>(&lo);       // a0 (row g) / a1 (row g+8)
      pa[2 + hi] = *reinterpret_cast<uint32_t*>(&hi2);  // a2 / a3
    }
    if (__any_sync(0xffffffffu, rescale)) {
#pragma unroll
      for (int nt = 0; nt < NO; ++nt) {
        o[nt][0] *= alpha[0];
        o[nt][1] *= alpha[0];
        o[nt][2] *= alpha[1];
        o[nt][3] *= alpha[1];
      }
    }
    // O += P V over the warp's 16 keys
#pragma unroll
    for (int np = 0; np < NO / 2; ++np) {
      uint32_t b0, b1, b2, b3;
      ldsm_x4_t(v_base + vo[np & 3] + (np >> 2) * 128, b0, b1, b2, b3);
      mma_bf16(o[2 * np], pa[0], pa[1], pa[2], pa[3], b0, b1);
      mma_bf16(o[2 * np + 1], pa[0], pa[1], pa[2], pa[3], b2, b3);
    }
  };

  const uint32_t kv_base = (uint32_t)__cvta_generic_to_shared(sKV);
  for (int t = t_begin; t < t_end; ++t) {
    const uint32_t g = gi + (uint32_t)(t - t_begin);
    const int stage = g % kStages;
    sm100::mbar_wait(&full[stage], (g / kStages) & 1u);
    __syncthreads();  // tile t (incl. plain smem stores) visible; tile t-1's slot is free
    load_tile(t + 2, (g + 2) % kStages);
#if SR_ATTN_PROBE == 1  // measurement build: K/V traffic only, no math
    continue;
#endif
    if (!active) continue;
    const int key0 = t * kKT + kw * 16;
    const uint32_t k_base = kv_base + stage * 2 * kTileBytes;
    if (key0 + 15 > min_qpos) tile_math(std::true_type{}, k_base, key0);
    else tile_math(std::false_type{}, k_base, key0);
  }
  __syncthreads();

  // ---- merge the 4 key-slice warps of each m-tile (fixed order) via smem
  constexpr int OP = HD + 8;                                 // padded row (bank spread)
  float* sO = reinterpret_cast<float*>(sKV);                 // [4][kRows][OP]
  float* sML = sO + 4 * kRows * OP;                          // [4][kRows][2]
  if (active) {
#pragma unroll
    for (int hi = 0; hi < 2; ++hi) {
      float l = l_run[hi];
      l += __shfl_xor_sync(0xffffffffu, l, 1);
      l += __shfl_xor_sync(0xffffffffu, l, 2);
      const int r = mw * 16 + (lane >> 2) + hi * 8;
      if ((lane & 3) == 0) {
        const float m = m_run[hi];
        sML[(kw * kRows + r) * 2] = m == -INFINITY ? -INFINITY : m * A.scale_log2;
        sML[(kw * kRows + r) * 2 + 1] = l;
      }
#pragma unroll
      for (int nt = 0; nt < NO; ++nt) {
        const int col = nt * 8 + 2 * (lane & 3);
        *reinterpret_cast<float2*>(&sO[(kw * kRows + r) * OP + col]) =
            make_float2(o[nt][hi * 2], o[nt][hi * 2 + 1]);
      }
    }
  }
  __syncthreads();
  const int64_t pidx = ((int64_t)z * A.qblocks + qb) * A.splits + sp;
  float* po = A.part_o + pidx * kRows * HD;
  float* pml = A.part_ml + pidx * kRows * 2;
  // A block whose keys fit one split finishes here: out = O / l is exactly
  // what the combine computes for a single split (weight exp2(0) = 1).
  const bool single = ntiles <= A.split_tiles;
  // per row: warp weights, M, l, 1/l and the output row (token * nq + head)
  float* sW = sML + 4 * kRows * 2;  // [kRows][4] weights, [kRows] M, [kRows] l, [kRows] 1/l
  int* sOutRow = reinterpret_cast<int*>(sW + 7 * kRows);
  if (tid < rows) {
    const int r = tid;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < 4; ++w) M = fmaxf(M, sML[(w * kRows + r) * 2]);
    const float Mu = M == -INFINITY ? 0.0f : M;
    float l = 0.0f;
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const float wt = fast_exp2(sML[(w * kRows + r) * 2] - Mu);
      sW[r * 4 + w] = wt;
      l += wt * sML[(w * kRows + r) * 2 + 1];
    }
    sW[4 * kRows + r] = M;
    sW[5 * kRows + r] = l;
    sW[6 * kRows + r] = 1.0f / l;
    const int gr = r0 + r, j = gr / G, g = gr % G;
    sOutRow[r] = (sq.q_start + j) * A.nq + h * G + g;
  }
  __syncthreads();
  // 8 consecutive head-dim elements per thread: 16-byte stores
  for (int e = tid; e < rows * (HD / 8); e += kAttnThreads) {
    const int r = e / (HD / 8), d0 = (e % (HD / 8)) * 8;
    float acc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = 0.0f;
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const float wt = sW[r * 4 + w];
      const float4 a = *reinterpret_cast<const float4*>(&sO[(w * kRows + r) * OP + d0]);
      const float4 b = *reinterpret_cast<const float4*>(&sO[(w * kRows + r) * OP + d0 + 4]);
      acc[0] += wt * a.x; acc[1] += wt * a.y; acc[2] += wt * a.z; acc[3] += wt * a.w;
      acc[4] += wt * b.x; acc[5] += wt * b.y; acc[6] += wt * b.z; acc[7] += wt * b.w;
    }
    if (single) {
      const float inv = sW[6 * kRows + r];
      uint4 pk;
      uint32_t* pw = reinterpret_cast<uint32_t*>(&pk);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        __nv_bfloat162 v2 = __floats2bfloat162_rn(acc[2 * i] * inv, acc[2 * i + 1] * inv);
        pw[i] = *reinterpret_cast<uint32_t*>(&v2);
      }
      *reinterpret_cast<uint4*>(A.out + (int64_t)sOutRow[r] * HD + d0) = pk;
      continue;
    }
    *reinterpret_cast<float4*>(&po[r * HD + d0]) = make_float4(acc[0], acc[1], acc[2], acc[3]);
    *reinterpret_cast<float4*>(&po[r * HD + d0 + 4]) = make_float4(acc[4], acc[5], acc[6], acc[7]);
    if (d0 == 0) {
      pml[r * 2] = sW[4 * kRows + r];
      pml[r * 2 + 1] = sW[5 * kRows + r];
    }
  }
  gi += (uint32_t)(t_end - t_begin);
  }  // item loop
}

// Work list of the persistent attention kernel: every non-empty (sequence x
// kv head, query block, split) item, ordered by decreasing tile count
// (counting sort), so the 2-per-SM persistent CTAs claim the longest items
// first (LPT).  Processing order does not change any item's arithmetic.  The
// list depends only on the sequence table, so a forward builds it once (layer
// 0) and every layer claims from its own zeroed counter.
__global__ void __launch_bounds__(1024) attn_plan_kernel(AttnArgs A) {
  grid_dep_sync();
  __shared__ int hist[1025];
  __shared__ int base[1025];
  const int T = A.split_tiles;
  for (int i = threadIdx.x; i <= T; i += blockDim.x) hist[i] = 0;
  __syncthreads();
  const int nkv = A.kv.kv_heads;
  auto tiles_of = [&](int packed) {
    const int sp = packed % A.splits;
    const int qb = (packed / A.splits) % A.qblocks;
    const int z = packed / (A.splits * A.qblocks);
    const SeqInfo sq = A.seqs[z / nkv];
    const int rows_total = sq.q_len * A.G;
    const int r0 = qb * kRows;
    if (r0 >= rows_total) return 0;
    const int rows = min(kRows, rows_total - r0);
    const int ntiles = block_max_key(sq, r0, rows, A.G) / kKT + 1;
    return max(0, min(ntiles, sp * T + T) - sp * T);
  };
  for (int i = threadIdx.x; i < A.n_slots; i += blockDim.x) atomicAdd(&hist[tiles_of(i)], 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int t = T; t >= 1; --t) { base[t] = acc; acc += hist[t]; }
    A.counters[0] = acc;
  }
  for (int i = threadIdx.x; i < kMaxLayers; i += blockDim.x) A.counters[1 + i] = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < A.n_slots; i += blockDim.x) {
    const int t = tiles_of(i);
    if (t > 0) A.order[atomicAdd(&base[t], 1)] = i;
  }
}

// Multi-split blocks only: one thread per (row, head-dim) output element,
// splits merged in split order.
template <int HD>
__global__ void __launch_bounds__(256)
attn_combine_kernel(AttnArgs A) {
  grid_dep_sync();
  const int nkv = A.kv.kv_heads;
  const int qb = blockIdx.y, z = blockIdx.z;
  const int s = z / nkv, h = z % nkv;
  const SeqInfo sq = A.seqs[s];
  const int G = A.G;
  const int rows_total = sq.q_len * G;
  const int r0 = qb * kRows;
  if (r0 >= rows_total) return;
  const int rows = min(kRows, rows_total - r0);
  const int ntiles = block_max_key(sq, r0, rows, G) / kKT + 1;
  if (ntiles <= A.split_tiles) return;  // written directly by the attention kernel
  const int nsplit = (ntiles + A.split_tiles - 1) / A.split_tiles;
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= rows * HD) return;
  const int r = e / HD, d = e % HD;
  const int64_t base = ((int64_t)z * A.qblocks + qb) * A.splits;
  float M = -INFINITY;
  for (int sp = 0; sp < nsplit; ++sp) M = fmaxf(M, A.part_ml[((base + sp) * kRows + r) * 2]);
  float den = 0.0f, num = 0.0f;
  for (int sp = 0; sp < nsplit; ++sp) {
    const float w = fast_exp2(A.part_ml[((base + sp) * kRows + r) * 2] - M);
    den += w * A.part_ml[((base + sp) * kRows + r) * 2 + 1];
    num += w * A.part_o[((base + sp) * kRows + r) * HD + d];
  }
  const int gr = r0 + r, j = gr / G, g = gr % G;
  const float inv = 1.0f / den;  // same form as the single-split path of attn_bf16_kernel
  A.out[((int64_t)(sq.q_start + j) * A.nq + h * G + g) * HD + d] = __float2bfloat16_rn(num * inv);
}

// fp32 parity attention: one warp per (token, q head), keys in position
// order with an fp32 online softmax (no splits).
__global__ void attn_f32_kernel(const float* __restrict__ q, const SeqInfo* __restrict__ seqs, KvLayout kv,
                                int layer, int nq, int G, float scale, float* __restrict__ out) {
  grid_dep_sync();
  const SeqInfo sq = seqs[blockIdx.y];
  const int item = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (item >= sq.q_len * nq) return;
  const int j = item / nq, qh = item % nq, h = qh / G;
  const int hd = kv.head_dim, nkv = kv.kv_heads, psz = kv.page;
  const int tok = sq.q_start + j, qpos = sq.ctx_len + j;
  const float* qv = q + ((int64_t)tok * nq + qh) * hd;
  const float* cache = reinterpret_cast<const float*>(kv.cache) + (int64_t)layer * kv.cache_layer_elems();
  const float* win = reinterpret_cast<const float*>(kv.window) + (int64_t)layer * kv.window_layer_elems();
  const int32_t* btab = kv.block_table + (int64_t)sq.request * kv.max_pages;
  float m = -INFINITY, l = 0.0f;
  float acc[4] = {0, 0, 0, 0};  // head_dim <= 128: lane owns dims lane, lane+32, ...
  for (int kp = 0; kp <= qpos; ++kp) {
    const float* k;
    int64_t vstep;
    if (sq.branch < 0 || kp < sq.ctx_len) {
      const int page = btab[kp / psz];
      SR_DCHECK(kp / psz < kv.max_pages && page >= 0 && page < kv.num_pages);
      k = cache + (((int64_t)page * 2 * nkv + h) * psz + kp % psz) * hd;
      vstep = (int64_t)nkv * psz * hd;
    } else {
      k = win + (((int64_t)sq.branch * 2 * nkv + h) * kv.window_max + (kp - sq.ctx_len)) * hd;
      vstep = (int64_t)nkv * kv.window_max * hd;
    }
    float dot = 0.0f;
    for (int d = lane; d < hd; d += 32) dot = fmaf(qv[d], k[d], dot);
#pragma unroll
    for (int o = 16; o; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
    const float sc = dot * scale;
    const float m_new = fmaxf(m, sc);
    const float alpha = expf(m - m_new), p = expf(sc - m_new);
    l = l * alpha + p;
    for (int i = 0, d = lane; d < hd; ++i, d += 32) acc[i] = acc[i] * alpha + p * k[vstep + d];
    m = m_new;
  }
  float* o = out + ((int64_t)tok * nq + qh) * hd;
  for (int i = 0, d = lane; d < hd; ++i, d += 32) o[d] = acc[i] / l;
}

template <int HD>
size_t attn_smem() {
  const size_t ring = (size_t)kStages * 2 * kKT * HD * 2;
  const size_t merge = (size_t)4 * kRows * (HD + 8 + 2) * 4 + (size_t)8 * kRows * 4;
  return (size_t)kRows * HD * 2 + (ring > merge ? ring : merge);
}

}  // namespace

size_t attention_partial_floats(int num_seqs, int kv_heads, int qblocks, int splits, int hd) {
  return (size_t)num_seqs * kv_heads * qblocks * splits * kRows * (hd + 2);
}

// Partial-buffer bound for a model: sum over sequences of query blocks is at
// most max_seqs + max_tokens*G/kRows; splits cover keys [0, max_key].
size_t attention_workspace_floats(int max_seqs, int max_tokens, int G, int kv_heads, int max_key, int hd) {
  const int qblocks = max_seqs + (max_tokens * G + kRows - 1) / kRows;
  const int splits = ceil_div(max_key / kKT + 1, 4);  // bound for any split size >= 4 tiles
  const size_t slots = (size_t)qblocks * kv_heads * splits;
  return attention_partial_floats(1, kv_heads, qblocks, splits, hd) + (slots + 1 + kMaxLayers + 63) / 64 * 64;
}

int attention_bf16(const __nv_bfloat16* q, const SeqInfo* seqs, int num_seqs, int max_q_len, int max_key,
                   const KvLayout& kv, int layer, int nq, float* partials, size_t partial_floats,
                   __nv_bfloat16* out, cudaStream_t stream, int phase, bool plan) {
  if (num_seqs == 0) return SR_OK;
  const int hd = kv.head_dim, G = nq / kv.kv_heads;
  SR_REQUIRE(hd == 64 || hd == 128, "bf16 attention supports head_dim 64 or 128");
  SR_REQUIRE(kv.page == kKT, "paged cache page size must be 64 tokens");
  SR_REQUIRE(layer >= 0 && layer < kMaxLayers, "attention supports at most 128 layers");
  AttnArgs a;
  a.q = q; a.seqs = seqs; a.kv = kv; a.layer = layer; a.nq = nq; a.G = G; a.out = out;
  a.scale_log2 = 1.4426950408889634f / sqrtf((float)hd);
  a.qblocks = ceil_div(max_q_len * G, kRows);
  a.split_tiles = g_split_tiles;
  a.splits = ceil_div(max_key / kKT + 1, a.split_tiles);
  a.n_slots = num_seqs * kv.kv_heads * a.qblocks * a.splits;
  // partial workspace = [counters (1 + kMaxLayers) + item list (n_slots), 256 B aligned | O | (m, l)]
  const size_t list_floats = ((size_t)a.n_slots + 1 + kMaxLayers + 63) / 64 * 64;
  const size_t need = list_floats + attention_partial_floats(num_seqs, kv.kv_heads, a.qblocks, a.splits, hd);
  SR_REQUIRE(need <= partial_floats, "attention partial workspace too small");
  a.counters = reinterpret_cast<int*>(partials);
  a.order = a.counters + 1 + kMaxLayers;
  a.part_o = partials + list_floats;
  a.part_ml = a.part_o + (size_t)num_seqs * kv.kv_heads * a.qblocks * a.splits * kRows * hd;
  if (phase == 0) {
    if (plan) {
      sr::launch_k(attn_plan_kernel, 1, 1024, 0, stream, a);
      int rc = check_launch("attn_plan_kernel");
      if (rc) return rc;
    }
    // persistent: two CTAs per SM (smem/register limited), longest items first
    int sms = 0, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int grid = std::min(a.n_slots, 2 * (sms > 0 ? sms : 148));
    if (hd == 128) {
      static bool set = false;
      if (!set) {
        SR_CHECK_CUDA(cudaFuncSetAttribute(attn_bf16_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)attn_smem<128>()));
        set = true;
      }
      sr::launch_k(attn_bf16_kernel<128>, grid, kAttnThreads, attn_smem<128>(), stream, a);
    } else {
      static bool set = false;
      if (!set) {
        SR_CHECK_CUDA(cudaFuncSetAttribute(attn_bf16_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)attn_smem<64>()));
        set = true;
      }
      sr::launch_k(attn_bf16_kernel<64>, grid, kAttnThreads, attn_smem<64>(), stream, a);
    }
    return check_launch("attn_bf16_kernel");
  }
  if (a.splits <= 1) return SR_OK;  // every block finished in the main kernel
  const dim3 cgrid(ceil_div(kRows * hd, 256), a.qblocks, num_seqs * kv.kv_heads);
  if (hd == 128) sr::launch_k(attn_combine_kernel<128>, cgrid, 256, 0, stream, a);
  else sr::launch_k(attn_combine_kernel<64>, cgrid, 256, 0, stream, a);
  return check_launch("attn_combine_kernel");
}

int attention_f32(const float* q, const SeqInfo* seqs, int num_seqs, int max_q_len, const KvLayout& kv,
                  int layer, int nq, float* out, cudaStream_t stream) {
  if (num_seqs == 0) return SR_OK;
  SR_REQUIRE(kv.head_dim <= 128, "fp32 attention supports head_dim <= 128");
  const int G = nq / kv.kv_heads;
  dim3 grid(ceil_div(max_q_len * nq, 8), num_seqs);
  sr::launch_k(attn_f32_kernel, grid, 256, 0, stream, q, seqs, kv, layer, nq, G, 1.0f / sqrtf((float)kv.head_dim), out);
  return check_launch("attn_f32_kernel");
}

}  // namespace sr

extern "C" int sr_set_attention_split(int tiles) {
  SR_REQUIRE(tiles >= 4 && tiles <= 1024, "split tiles out of [4, 1024]");
  sr::g_split_tiles = tiles;
  return SR_OK;
}

extern "C" int sr_paged_attention(int dtype, const void* q, const void* seqs, int num_seqs, int max_q_len,
                                  int max_key, int q_heads, int kv_heads, int head_dim, int layer,
                                  int layers, void* kv_cache, int num_pages, const int32_t* block_table,
                                  int max_pages, void* window, int branches, int window_max, float* partials,
                                  uint64_t partial_floats, void* out, sr_stream_t stream) {
  SR_REQUIRE(q_heads > 0 && kv_heads > 0 && q_heads % kv_heads == 0, "bad head counts");
  SR_REQUIRE(layer >= 0 && layer < layers, "layer out of range");
  sr::KvLayout kv;
  kv.cache = kv_cache;
  kv.block_table = block_table;
  kv.max_pages = max_pages;
  kv.page = 64;
  kv.num_pages = num_pages;
  kv.window = window;
  kv.window_max = window_max;
  kv.branches = branches;
  kv.kv_heads = kv_heads;
  kv.head_dim = head_dim;
  kv.layers = layers;
  const auto* sq = reinterpret_cast<const sr::SeqInfo*>(seqs);
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == 1) {
    int rc = sr::attention_bf16(reinterpret_cast<const __nv_bfloat16*>(q), sq, num_seqs, max_q_len, max_key, kv,
                                layer, q_heads, partials, partial_floats, reinterpret_cast<__nv_bfloat16*>(out), st, 0, true);
    if (rc) return rc;
    return sr::attention_bf16(reinterpret_cast<const __nv_bfloat16*>(q), sq, num_seqs, max_q_len, max_key, kv,
                              layer, q_heads, partials, partial_floats, reinterpret_cast<__nv_bfloat16*>(out), st, 1, true);
  }
  SR_REQUIRE(dtype == 0, "dtype must be 0 or 1");
  return sr::attention_f32(reinterpret_cast<const float*>(q), sq, num_seqs, max_q_len, kv, layer, q_heads,
                           reinterpret_cast<float*>(out), st);
}
