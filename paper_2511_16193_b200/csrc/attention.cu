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

#include <cuda.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <type_traits>
#include <cstdio>
#include <cstdlib>

namespace sr {

int make_tmap_kv_pages(CUtensorMap* map, const void* cache, uint64_t blocks);  // gemm.cu

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
  int early;           // the work list is from an earlier launch: claim + stream context pages before the wait
};

// SR_ATTN_TC=1 runs head_dim 128 on the tcgen05 kernel (attn_tc_kernel).  It
// is exact and faster on long contexts but slower on the bench's short verify
// items, so the mma.sync kernel stays the default.
// The choice is process-wide: verify and decode must use the same kernel.
bool g_attn_tc = [] {
  const char* v = getenv("SR_ATTN_TC");
  return v && v[0] == '1';
}();

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
  // Programmatic dependent launch: the previous kernel (this layer's qkv
  // GEMM) writes Q and the window's K/V, nothing else this kernel reads.  When
  // the work list comes from an earlier launch (layers >= 1 of a forward), a
  // CTA claims its first item and streams that item's first pages that hold
  // only context keys (written by earlier steps) before waiting, so their
  // latency hides behind the GEMM's tail.
  uint32_t pre_issued = 0;  // first-item tiles (bit p: t_begin + p) already in flight
  bool pre_claimed = false;
  if (A.early) {
    __syncthreads();  // barrier init visible
    if (tid == 0) {
      const int i = atomicAdd(&A.counters[1 + A.layer], 1);
      s_item = i;
      if (i < A.counters[0]) {
        const int pk = A.order[i];
        const int sp0 = pk % A.splits;
        const int qb0 = (pk / A.splits) % A.qblocks;
        const int z0 = pk / (A.splits * A.qblocks);
        const SeqInfo sq0 = A.seqs[z0 / nkv];
        const int rows0 = min(kRows, sq0.q_len * G - qb0 * kRows);
        const int tb = sp0 * A.split_tiles;
        const int te = min(block_max_key(sq0, qb0 * kRows, rows0, G) / kKT + 1, tb + A.split_tiles);
        const __nv_bfloat16* cache0 = reinterpret_cast<const __nv_bfloat16*>(A.kv.cache) +
                                      (int64_t)A.layer * A.kv.cache_layer_elems();
        const int32_t* bt0 = A.kv.block_table + (int64_t)sq0.request * A.kv.max_pages;
        constexpr uint32_t kTB = kKT * HD * 2;
        for (int p = 0; p < 2; ++p) {
          const int t = tb + p;
          if (t >= te || t * kKT + kKT - 1 >= sq0.ctx_len) break;  // window keys: after the wait
          const int stage = p;  // gi == 0
          uint8_t* k_dst = sKV + stage * 2 * kTB;
          const __nv_bfloat16* kb = cache0 + ((int64_t)bt0[t] * 2 * nkv + z0 % nkv) * A.kv.page * HD;
          sm100::mbar_arrive_expect_tx(&full[stage], 2 * kTB);
          sm100::bulk_load_hint(k_dst, kb, kTB, &full[stage], sm100::kEvictFirst);
          sm100::bulk_load_hint(k_dst + kTB, kb + (int64_t)nkv * A.kv.page * HD, kTB, &full[stage],
                                sm100::kEvictFirst);
          pre_issued |= 1u << p;
        }
      }
    }
    pre_claimed = true;
  }
  grid_dep_sync();
  for (;;) {
  __syncthreads();  // previous item fully consumed (smem reusable)
  if (tid == 0 && !pre_claimed) s_item = atomicAdd(&A.counters[1 + A.layer], 1);
  pre_claimed = false;
  __syncthreads();
  if (s_item >= A.counters[0]) break;
  // only thread 0 issues (and skips) bulk copies; a pre-issued tile is a
  // cache page, which the other threads' load_tile leaves to thread 0 anyway
  const uint32_t issued = pre_issued;
  pre_issued = 0;
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
  if (!(issued & 1u)) load_tile(t_begin, gi % kStages);
  if (!(issued & 2u)) load_tile(t_begin + 1, (gi + 1) % kStages);
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

// ---------------------------------------------------------------------------
// K2 on the 5th-generation tensor cores (head_dim 128).
//
// Same work items, key tiling, splits and combine as attn_bf16_kernel, but
// both products run as tcgen05.mma with TMEM accumulators, transposed so the
// keys (not the ~30 query rows of a GQA item) fill the 128-row MMA side:
//   S^T[128 keys x 32 rows] = K_blk[128 x 128 hd] . Q^T          (A = K, K-major)
//   O^T[128 hd x 32 rows]  += V_blk^T[128 hd x 128 keys] . P^T    (A = V, B = P^T, MN-major)
// Keys move in blocks of 128 absolute positions (two 64-key pages).  A page
// of K or V (64 slots x 128 head dims, rows already XOR-swizzled by slot in
// HBM) lands by ONE 5D TMA box as [8-slot group][dim half][8 slots][128 B]:
// SWIZZLE_128B atoms the UMMA descriptors read in place (group stride 2 KB).
//
// Warp roles (320 threads, one persistent CTA per SM):
//   warp 0    producer: claims items (atomic counter over the longest-first
//             list) one item ahead, Q tile by cp.async, K/V pages by TMA into
//             a 3-stage ring (drafter-branch window keys by lane copies);
//             the item's block-table slice sits in the warp's lanes
//   warp 1    MMA issuer (one elected lane) with two cursors: S^T(g) as soon
//             as block g's K/V and an S slot are in, PV(g') as soon as the
//             softmax of g' is written -- neither waits for the other
//   warps 2-9 two softmax warpgroups taking alternate items, so one group's
//             item epilogue and first-block max overlap the other's stream;
//             thread = one key (TMEM lane) holding its 32 row scores;
//             lazy-rescaled online softmax (FA4: the reference max moves only
//             when a score exceeds it by 2^8, found by one barrier.red.or);
//             P^T as bf16 into the group's shared buffer; per-row sums kept
//             per key thread and reduced once per item; the epilogue reads
//             O^T (thread = head dim) from TMEM.
// Every row's arithmetic depends only on its own scores in block order, so a
// query gives the same bits in a verify window and as a single decode step.
// ---------------------------------------------------------------------------

#if SR_ATTN_PROBE == 4  // measurement build: per-block event times of CTA 0 (printed at exit)
__device__ unsigned long long g_tc_trace[8][64];
#define TC_TRACE(ev, blk) do { if (blockIdx.x == 0 && (blk) < 64) g_tc_trace[ev][blk] = sm100::global_timer_ns(); } while (0)
#else
#define TC_TRACE(ev, blk) do { } while (0)
#endif

// mbarrier wait that, in probe builds (SR_ATTN_PROBE), names itself if it
// stalls (a protocol bug reports role, barrier and phase before the trap)
__device__ __forceinline__ void tc_wait(uint64_t* bar, uint32_t phase, int tag) {
#if SR_ATTN_PROBE == 0
  (void)tag;  // release builds: the plain watchdog wait (no printf path in the kernel)
  sm100::mbar_wait(bar, phase);
  return;
#endif
  if (sm100::mbar_try_wait(bar, phase)) return;
  const uint64_t t0 = sm100::global_timer_ns();
  bool said = false;
  while (!sm100::mbar_try_wait(bar, phase)) {
    const uint64_t dt = sm100::global_timer_ns() - t0;
    if (!said && dt > 2000000000ull) {
      printf("attn_tc stall: cta %d thread %d tag %d phase %u\n", blockIdx.x, threadIdx.x, tag, phase);
      said = true;
    }
    if (dt > 4000000000ull) __trap();
  }
}

// Softmax warpgroups taking items round-robin.  Two overlap one item's
// epilogue with the next item's stream but cap registers at 168 (per-SMSP
// register files) and measured slower (58 vs 46 us on the bench shape), so
// one is the default.
#ifndef SR_ATTN_TC_GROUPS
#define SR_ATTN_TC_GROUPS 1
#endif
constexpr int kTcGroups = SR_ATTN_TC_GROUPS;
constexpr int kTcThreads = 64 + 128 * kTcGroups;
constexpr int kTcStages = 3;
constexpr uint32_t kTcStageBytes = 65536;                 // K [2 pages][8 groups][2 halves][8 keys][128 B] | V same
constexpr uint32_t kTcQOff = kTcStages * kTcStageBytes;    // Q [2][2 halves][32 rows][128 B]
constexpr uint32_t kTcPOff = kTcQOff + 2 * 8192;           // P^T [2 groups][128 keys][32 rows x bf16], MN-major SW64
constexpr uint32_t kTcMiscOff = kTcPOff + 2 * 8192;        // barriers and small per-CTA state

// Everything small lives behind the big buffers: no static shared memory, so
// the dynamic window starts 1024-aligned (SWIZZLE_128B atoms) and the CTA
// fits the 227 KB per-block limit (which includes the 1 KB system reserve).
struct TcMisc {
  uint64_t kv_full[kTcStages], kv_empty[kTcStages];
  uint64_t item_full[2], item_empty[2], q_full[2], q_empty[2];
  uint64_t s_full[2], s_empty[2], p_full[2], p_empty[2], o_full[2], o_empty[2];
  int item[2], item_g[2];  // item slot n & 1 (= softmax group): packed id, first global block
  int mma_items[4];        // MMA warp: packed ids between its PV and S cursors
  uint32_t tmem;
  float red[2][4][32];
  int orow[2][32];
};
constexpr uint32_t kTcSmem = kTcMiscOff + (uint32_t)((sizeof(TcMisc) + 127) / 128 * 128);

__device__ __forceinline__ void tma_load_5d(void* smem_dst, const CUtensorMap* desc, uint64_t* bar, int c4,
                                            uint64_t hint) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %3, %3, %3, %4}], [%2], %5;" ::"r"(sm100::smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(desc)), "r"(sm100::smem_u32(bar)), "r"(0), "r"(c4), "l"(hint)
      : "memory");
}

// K-major SWIZZLE_128B operand whose 8-row groups are SBO bytes apart.
__device__ __forceinline__ uint64_t desc_k_sbo(uint32_t addr, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFFu);
  d |= (uint64_t)1u << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)2u << 61;
  return d;
}

// MN-major SWIZZLE_64B operand: 64-byte rows (32 MN elements) per k, 8-row
// atoms of 512 B (16-byte chunk c of row k at c ^ ((k >> 1) & 3)).
__device__ __forceinline__ uint64_t desc_mn_sw64(uint32_t addr) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFFu);
  d |= (uint64_t)(4096u >> 4) << 16;  // LBO: next 32-wide MN atom (unused at N = 32)
  d |= (uint64_t)(512u >> 4) << 32;   // SBO: next 8-key group
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)4u << 61;            // SWIZZLE_64B
  return d;
}

// OR of a predicate over one softmax warpgroup (named barrier 1 + group).
__device__ __forceinline__ bool group_any(bool p, int grp) {
  uint32_t r;
  asm volatile(
      "{\n\t.reg .pred a, b;\n\t"
      "setp.ne.u32 a, %1, 0;\n\t"
      "bar.red.or.pred b, %2, 128, a;\n\t"
      "selp.u32 %0, 1, 0, b;\n\t}"
      : "=r"(r)
      : "r"((uint32_t)p), "r"(1 + grp)
      : "memory");
  return r != 0;
}
__device__ __forceinline__ void group_bar(int grp) { asm volatile("bar.sync %0, 128;" ::"r"(1 + grp) : "memory"); }

// Transposed butterfly over a warp: v[32] per lane in, lane l ends with
// op(v[l] over all 32 lanes) in v[0] (fixed tree order).
template <bool MAX>
__device__ __forceinline__ float warp_transpose_reduce(float (&v)[32], int lane) {
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) {
    const bool up = lane & m;
#pragma unroll
    for (int i = 0; i < m; ++i) {
      const float send = up ? v[i] : v[i + m];
      const float keep = up ? v[i + m] : v[i];
      const float got = __shfl_xor_sync(0xffffffffu, send, m);
      v[i] = MAX ? fmaxf(keep, got) : keep + got;
    }
  }
  return v[0];
}

struct TcItem {
  int s, h, qb, sp, z, rows, r0, t_begin, t_end, ntiles;
  SeqInfo sq;
};

__device__ __forceinline__ TcItem tc_item(const AttnArgs& A, int packed) {
  TcItem I;
  const int nkv = A.kv.kv_heads;
  I.sp = packed % A.splits;
  I.qb = (packed / A.splits) % A.qblocks;
  I.z = packed / (A.splits * A.qblocks);
  I.s = I.z / nkv;
  I.h = I.z % nkv;
  I.sq = A.seqs[I.s];
  I.r0 = I.qb * kRows;
  I.rows = min(kRows, I.sq.q_len * A.G - I.r0);
  I.ntiles = block_max_key(I.sq, I.r0, I.rows, A.G) / kKT + 1;
  I.t_begin = I.sp * A.split_tiles;
  I.t_end = min(I.ntiles, I.t_begin + A.split_tiles);
  return I;
}
__device__ __forceinline__ int tc_blocks(const TcItem& I) { return (I.t_end + 1) / 2 - (I.t_begin >> 1); }

__global__ void __launch_bounds__(kTcThreads, 1)
attn_tc_kernel(const __grid_constant__ CUtensorMap tm_kv, AttnArgs A) {
  grid_dep_sync();
  extern __shared__ __align__(1024) uint8_t sm[];
  if ((sm100::smem_u32(sm) & 1023) != 0) __trap();  // SWIZZLE_128B atoms need a 1024-aligned window
  TcMisc& M = *reinterpret_cast<TcMisc*>(sm + kTcMiscOff);
  uint64_t* kv_full = M.kv_full;
  uint64_t* kv_empty = M.kv_empty;
  uint64_t* item_full = M.item_full;
  uint64_t* item_empty = M.item_empty;
  uint64_t* q_full = M.q_full;
  uint64_t* q_empty = M.q_empty;
  uint64_t* s_full = M.s_full;
  uint64_t* s_empty = M.s_empty;
  uint64_t* p_full = M.p_full;
  uint64_t* p_empty = M.p_empty;
  uint64_t* o_full = M.o_full;
  uint64_t* o_empty = M.o_empty;
  int* s_item = M.item;
  int* s_item_g = M.item_g;
  int* s_mma_items = M.mma_items;
  auto& s_red = M.red;
  auto& s_orow = M.orow;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int i = 0; i < kTcStages; ++i) {
      sm100::mbar_init(&kv_full[i], 1);
      sm100::mbar_init(&kv_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      sm100::mbar_init(&item_full[i], 1);
      sm100::mbar_init(&item_empty[i], 5);  // MMA lane + the group's 4 warps
      sm100::mbar_init(&q_full[i], 1);
      sm100::mbar_init(&q_empty[i], 1);
      sm100::mbar_init(&s_full[i], 1);
      sm100::mbar_init(&s_empty[i], 4);
      sm100::mbar_init(&p_full[i], 4);
      sm100::mbar_init(&p_empty[i], 1);
      sm100::mbar_init(&o_full[i], 1);
      sm100::mbar_init(&o_empty[i], 4);
    }
    sm100::fence_barrier_init();
  }
  if (warp == 1) sm100::tmem_alloc<128>(&M.tmem);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = M.tmem;  // cols [0,64): S^T per group, [64,128): O^T per group
  const int nkv = A.kv.kv_heads;
  const float sl2 = A.scale_log2;

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    const __nv_bfloat16* cache = reinterpret_cast<const __nv_bfloat16*>(A.kv.cache) +
                                 (int64_t)A.layer * A.kv.cache_layer_elems();
    const __nv_bfloat16* win = reinterpret_cast<const __nv_bfloat16*>(A.kv.window) +
                               (int64_t)A.layer * A.kv.window_layer_elems();
    const int psz = A.kv.page;
    const int64_t layer_blocks = (int64_t)A.layer * A.kv.num_pages * 2 * nkv;
    if (lane == 0) sm100::tma_prefetch_desc(&tm_kv);
    // Item n is claimed (and its Q tile requested) while item n-1's first
    // block is being issued, so neither the claim nor the Q latency sits
    // between two items' K/V streams.
    auto claim = [&](uint32_t n, uint32_t g0) -> int {
      const int slot = n & 1;
      tc_wait(&item_empty[slot], ((n >> 1) & 1) ^ 1, 1);
      int pk = -1;
      if (lane == 0) {
        const int i = atomicAdd(&A.counters[1 + A.layer], 1);
        pk = i < A.counters[0] ? A.order[i] : -1;
        s_item[slot] = pk;
        s_item_g[slot] = (int)g0;
      }
      pk = __shfl_sync(0xffffffffu, pk, 0);
      if (lane == 0) sm100::mbar_arrive(&item_full[slot]);
      if (pk < 0) {
        // the other softmax group waits on the other slot: end it there too
        const uint32_t n2 = n + 1;
        tc_wait(&item_empty[n2 & 1], ((n2 >> 1) & 1) ^ 1, 2);
        if (lane == 0) {
          s_item[n2 & 1] = -1;
          s_item_g[n2 & 1] = (int)g0;
          sm100::mbar_arrive(&item_full[n2 & 1]);
        }
        return pk;
      }
      // Q tile [2 halves][32 rows][128 B], chunk c of row r at ((c & 7) ^ (r & 7))
      const TcItem I = tc_item(A, pk);
      const int qbuf = n & 1;
      uint8_t* sQ = sm + kTcQOff + qbuf * 8192;
      tc_wait(&q_empty[qbuf], ((n >> 1) & 1) ^ 1, 3);
#pragma unroll 4
      for (int e = lane; e < kRows * 16; e += 32) {
        const int r = e >> 4, c = e & 15;
        uint8_t* dst = sQ + (c >> 3) * 4096 + r * 128 + (((c & 7) ^ (r & 7)) << 4);
        if (r < I.rows) {
          const int gr = I.r0 + r, j = gr / A.G, gg = gr % A.G;
          cp_async16(dst, A.q + ((int64_t)(I.sq.q_start + j) * A.nq + I.h * A.G + gg) * 128 + c * 8);
        } else {
          *reinterpret_cast<uint4*>(dst) = make_uint4(0, 0, 0, 0);
        }
      }
      cp_async_commit();
      return pk;
    };
    uint32_t it = 0, g = 0;
    int packed = claim(0, 0);
    while (packed >= 0) {
      const TcItem I = tc_item(A, packed);
      const int32_t* btab = A.kv.block_table + (int64_t)I.sq.request * A.kv.max_pages;
      const int max_key = block_max_key(I.sq, I.r0, I.rows, A.G);
      const int qbuf = it & 1;
      // lane j holds page t_begin + j of this item (items span <= 32 tiles)
      const int bt_lane = I.t_begin + lane < I.t_end ? __ldg(btab + I.t_begin + lane) : 0;
      const uint32_t g_next = g + tc_blocks(I);
      int next = -1;
      for (int b = I.t_begin >> 1; 2 * b < I.t_end; ++b, ++g) {
        const int st = g % kTcStages;
        tc_wait(&kv_empty[st], ((g / kTcStages) & 1) ^ 1, 4);
        if (lane == 0) TC_TRACE(0, g);  // producer: stage free
        uint8_t* sK = sm + st * kTcStageBytes;
        uint8_t* sV = sK + 32768;
        uint32_t tx = 0;
        int tma_pages = 0;  // bit p: page p of the block comes from the paged cache by TMA
        for (int p = 0; p < 2 && 2 * b + p < I.t_end; ++p) {
          const int t = 2 * b + p;
          const int last = t * kKT + kKT - 1;
          if (I.sq.branch < 0 || last < I.sq.ctx_len) {
            tma_pages |= 1 << p;
            tx += 32768;
            continue;
          }
          // tile reaching drafter-branch window keys: lane copies, same layout
          for (int e = lane; e < kKT * 16; e += 32) {
            const int r = e >> 4, pc = e & 15;  // key slot, destination physical chunk
            const int hh = pc >> 3;
            const int c = hh * 8 + ((pc & 7) ^ (r & 7));  // logical chunk held there
            const int kp = t * kKT + r;
            uint4 kv4 = make_uint4(0, 0, 0, 0), vv4 = make_uint4(0, 0, 0, 0);
            if (kp <= max_key) {
              const __nv_bfloat16* ksrc;
              int64_t vstep;
              int src_chunk;
              if (kp < I.sq.ctx_len) {
                ksrc = cache + (((int64_t)btab[kp / psz] * 2 * nkv + I.h) * psz + kp % psz) * 128;
                vstep = (int64_t)nkv * psz * 128;
                src_chunk = pc;  // page slot == key slot: same swizzle
              } else {
                const int j = kp - I.sq.ctx_len;
                ksrc = win + (((int64_t)I.sq.branch * 2 * nkv + I.h) * A.kv.window_max + j) * 128;
                vstep = (int64_t)nkv * A.kv.window_max * 128;
                src_chunk = (c & 8) | ((c & 7) ^ (j & 7));
              }
              kv4 = *reinterpret_cast<const uint4*>(ksrc + src_chunk * 8);
              vv4 = *reinterpret_cast<const uint4*>(ksrc + vstep + src_chunk * 8);
            }
            const uint32_t off = p * 16384 + (r >> 3) * 2048 + hh * 1024 + (r & 7) * 128 + (pc & 7) * 16;
            *reinterpret_cast<uint4*>(sK + off) = kv4;
            *reinterpret_cast<uint4*>(sV + off) = vv4;
          }
        }
        if (tma_pages != 3) sm100::fence_proxy_async();
        int pg[2];  // the block's pages, from the item's block-table slice in lane registers
        pg[0] = __shfl_sync(0xffffffffu, bt_lane, 2 * b - I.t_begin);
        pg[1] = __shfl_sync(0xffffffffu, bt_lane, min(2 * b + 1 - I.t_begin, 31));
        __syncwarp();
        if (lane == 0) {
          if (tx) sm100::mbar_arrive_expect_tx(&kv_full[st], tx);
          else sm100::mbar_arrive(&kv_full[st]);
          for (int p = 0; p < 2; ++p) {
            if (!(tma_pages >> p & 1)) continue;
            const int64_t blk = layer_blocks + (int64_t)pg[p] * 2 * nkv + I.h;
            // KV pages are read once per layer: evict-first keeps the next
            // GEMMs' weights in L2
            tma_load_5d(sK + p * 16384, &tm_kv, &kv_full[st], (int)blk, sm100::kEvictFirst);
            tma_load_5d(sV + p * 16384, &tm_kv, &kv_full[st], (int)(blk + nkv), sm100::kEvictFirst);
          }
        }
        if (b == (I.t_begin >> 1)) {
          // this item's Q (requested one item ago) is in: publish it, then
          // claim the next item and request its Q
          cp_async_wait<0>();
          sm100::fence_proxy_async();
          __syncwarp();
          if (lane == 0) sm100::mbar_arrive(&q_full[qbuf]);
          next = claim(it + 1, g_next);
        }
      }
      packed = next;
      ++it;
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t id_s = sm100::umma_idesc_bf16(128, kRows);
    // O^T += V^T P^T: A (V^T) and B (P^T) both MN-major
    constexpr uint32_t id_o = sm100::umma_idesc_bf16(128, kRows) | (1u << 15) | (1u << 16);
    const uint32_t sbase = sm100::smem_u32(sm);
    // lane 0's view of a barrier, made warp-uniform (the waits that follow
    // return at once and give every lane its acquire)
    auto ready = [&](uint64_t* bar, uint32_t ph) {
      return __shfl_sync(0xffffffffu, (int)sm100::mbar_try_wait(bar, ph), 0) != 0;
    };
    // S cursor: item its (packed ps, block i_s of ns), global block gs
    // PV cursor: item itp (packed pp, block i_p of np), global block gp
    uint32_t its = 0, gs = 0, itp = 0, gp = 0;
    int ps = 0, ns = 0, i_s = 0, tb_s = 0, te_s = 0;
    bool s_have = false, s_end = false;
    int pp = 0, np_ = 0, i_p = 0, tb_p = 0, te_p = 0;
    bool p_have = false;
    uint32_t pcount[2] = {0, 0};  // blocks whose PV was issued, per softmax group
    uint32_t scount[2] = {0, 0};  // blocks whose S^T was issued, per softmax group (its S slot's phase)
    for (;;) {
      // ---- S side: next item descriptor, then S^T of block gs
      if (!s_have && !s_end && gs - gp < 3) {
        const int slot = its & 1;
        if (ready(&item_full[slot], (its >> 1) & 1)) {
          tc_wait(&item_full[slot], (its >> 1) & 1, 5);
          ps = s_item[slot];
          __syncwarp();
          if (lane == 0) sm100::mbar_arrive(&item_empty[slot]);
          if (ps < 0) {
            s_end = true;
          } else {
            const TcItem I = tc_item(A, ps);
            ns = tc_blocks(I);
            tb_s = I.t_begin;
            te_s = I.t_end;
            i_s = 0;
            if (lane == 0) s_mma_items[its & 3] = ps;
            __syncwarp();
            tc_wait(&q_full[slot], (its >> 1) & 1, 6);
            s_have = true;
          }
        }
      }
      if (s_have) {
        // S slot = the item's softmax group: each group consumes its slot in
        // order, so no waiter can run a phase ahead on a shared barrier
        const uint32_t st = gs % kTcStages, sb = kTcGroups == 1 ? (gs & 1) : its % kTcGroups;
        if (ready(&kv_full[st], (gs / kTcStages) & 1) && ready(&s_empty[sb], (scount[sb] & 1) ^ 1)) {
          tc_wait(&kv_full[st], (gs / kTcStages) & 1, 7);
          tc_wait(&s_empty[sb], (scount[sb] & 1) ^ 1, 8);
          if (lane == 0) TC_TRACE(1, gs);  // MMA: data landed
          sm100::tc_fence_after();
          const uint32_t qb = its & 1;  // Q buffer: by item parity
          if (sm100::elect_one()) {
            const uint32_t k0 = sbase + st * kTcStageBytes;
            const uint32_t q0 = sbase + kTcQOff + qb * 8192;
#pragma unroll
            for (int ks = 0; ks < 8; ++ks)
              sm100::umma_bf16(tmem + sb * 32, desc_k_sbo(k0 + (ks >> 2) * 1024 + (ks & 3) * 32, 2048),
                               sm100::umma_desc_sw128(q0 + (ks >> 2) * 4096 + (ks & 3) * 32), id_s, ks ? 1u : 0u);
            sm100::umma_commit(&s_full[sb]);
            TC_TRACE(2, gs);  // MMA: S issued
            if (i_s == ns - 1) sm100::umma_commit(&q_empty[qb]);
          }
          __syncwarp();
          ++scount[sb];
          ++gs;
          if (++i_s == ns) {
            s_have = false;
            ++its;
          }
        }
      }
      // ---- PV side: O^T += V^T P^T of block gp once its softmax is written
      if (gp < gs) {
        if (!p_have) {
          pp = s_mma_items[itp & 3];
          const TcItem I = tc_item(A, pp);
          np_ = tc_blocks(I);
          tb_p = I.t_begin;
          te_p = I.t_end;
          i_p = 0;
          p_have = true;
        }
        const uint32_t grp = itp % kTcGroups;
        const uint32_t ouse = itp / kTcGroups;  // the group's item count: its O^T buffer phase
        if (ready(&p_full[grp], pcount[grp] & 1) && (i_p > 0 || ready(&o_empty[grp], (ouse & 1) ^ 1))) {
          tc_wait(&p_full[grp], pcount[grp] & 1, 9);
          if (i_p == 0) tc_wait(&o_empty[grp], (ouse & 1) ^ 1, 10);
          if (lane == 0) TC_TRACE(6, gp);  // MMA: PV issue
          sm100::tc_fence_after();
          const int b = (tb_p >> 1) + i_p;
          const int pages = min(2, te_p - 2 * b);
          if (sm100::elect_one()) {
            const uint32_t v0 = sbase + (gp % kTcStages) * kTcStageBytes + 32768;
            const uint32_t p0 = sbase + kTcPOff + grp * 8192;
            for (int ks = 0; ks < 4 * pages; ++ks)
              sm100::umma_bf16(tmem + 64 + grp * 32, sm100::umma_desc_sw128_mn(v0 + ks * 4096, 1024, 2048),
                               desc_mn_sw64(p0 + ks * 1024), id_o, (i_p == 0 && ks == 0) ? 0u : 1u);
            sm100::umma_commit(&kv_empty[gp % kTcStages]);
            sm100::umma_commit(&p_empty[grp]);
            if (i_p == np_ - 1) sm100::umma_commit(&o_full[grp]);
          }
          __syncwarp();
          ++pcount[grp];
          ++gp;
          if (++i_p == np_) {
            p_have = false;
            ++itp;
          }
        }
      } else if (s_end) {
        break;
      }
    }
  } else {
    // ------------------------------------------------------------ softmax groups + epilogue
    const int grp = (warp - 2) >> 2;   // warps 2-5: group 0, 6-9: group 1 (items round-robin)
    const int qd = warp & 3;           // TMEM lane quadrant this warp may access
    const int kk = qd * 32 + lane;     // key within the block / head dim in the epilogue
    const int gt = kk;                 // thread index within the group (TMEM lane order)
    const uint32_t lane_base = (uint32_t)(qd * 32) << 16;
    uint8_t* sP = sm + kTcPOff + grp * 8192;
    // P^T is MN-major SWIZZLE_64B: key kk owns the 64-byte row kk, its 32 rows'
    // probabilities are logical 16-byte chunks 0..3 stored at chunk ^ ((kk >> 1) & 3)
    uint8_t* p_row = sP + kk * 64;
    const int kx = (kk >> 1) & 3;
    uint32_t it = grp, pc = 0;
    for (;;) {
      const int slot = it & 1;
      tc_wait(&item_full[slot], (it >> 1) & 1, 11);
      const int packed = s_item[slot];
      uint32_t g = (uint32_t)s_item_g[slot];
      __syncwarp();
      if (lane == 0) sm100::mbar_arrive(&item_empty[slot]);
      if (packed < 0) break;
      const TcItem I = tc_item(A, packed);
      const int G = A.G;
      if (gt < kRows) {
        const int r = gt;
        const int gr = I.r0 + r, j = gr / G, gg = gr % G;
        s_orow[grp][r] = r < I.rows ? (I.sq.q_start + j) * A.nq + I.h * G + gg : -1;
      }
      // per row r (uniform across the group): neg = -(running max) in log2
      // units; padding rows get -inf (every exponent -inf, never a trigger).
      // `unset`: live rows that have not seen a key yet (their threshold is
      // -inf instead of the 2^8 headroom).
      float neg[kRows], lsum[kRows];
      uint32_t unset = I.rows >= 32 ? 0xffffffffu : ((1u << I.rows) - 1u);
#pragma unroll
      for (int r = 0; r < kRows; ++r) neg[r] = r < I.rows ? 0.0f : -INFINITY, lsum[r] = 0.0f;
      const int min_qpos = I.sq.ctx_len + I.r0 / G;
      const int b0 = I.t_begin >> 1, nb = tc_blocks(I);
      for (int i = 0; i < nb; ++i, ++g, ++pc) {
        // one group: S double-buffered by block parity; two groups: one slot
        // each (a shared slot would let a group wait a phase ahead)
        const uint32_t sb = kTcGroups == 1 ? (g & 1) : grp;
        tc_wait(&s_full[sb], kTcGroups == 1 ? (g >> 1) & 1 : pc & 1, 12);
        if (gt == 0) TC_TRACE(3, g);  // softmax: S ready
        sm100::tc_fence_after();
        uint32_t raw[32];
        sm100::tmem_ld_32x32b_x32(tmem + lane_base + sb * 32, raw);
        sm100::tmem_ld_wait();
        sm100::tc_fence_before();
        __syncwarp();
        if (lane == 0) sm100::mbar_arrive(&s_empty[sb]);
        float e[kRows];  // exponents s * log2(e) / sqrt(hd) - running max
#pragma unroll
        for (int r = 0; r < kRows; ++r) e[r] = fmaf(__uint_as_float(raw[r]), sl2, neg[r]);
        const int kb = (b0 + i) * 128;
        if (kb + 127 > min_qpos) {
          // causal edge inside this block: row r sees key kp iff r0 + r >= (kp - ctx) * G
          const int rmin = max(0, (kb + kk - I.sq.ctx_len) * G - I.r0);
#pragma unroll
          for (int r = 0; r < kRows; ++r) e[r] = r < rmin ? -INFINITY : e[r];
        }
        bool trig = false;
        if (unset == 0) {
#pragma unroll
          for (int r = 0; r < kRows; ++r) trig |= e[r] > 8.0f;
        } else {
#pragma unroll
          for (int r = 0; r < kRows; ++r) trig |= e[r] > ((unset >> r & 1) ? -INFINITY : 8.0f);
        }
        if (i == 0 || group_any(trig, grp)) {  // first block: every live max is unset
          // exact column maxima of this block's exponents
          float v[32];
#pragma unroll
          for (int r = 0; r < kRows; ++r) v[r] = e[r];
          const float wm = warp_transpose_reduce<true>(v, lane);
          s_red[grp][qd][lane] = wm;
          group_bar(grp);
          const float bm = fmaxf(fmaxf(s_red[grp][0][lane], s_red[grp][1][lane]),
                                 fmaxf(s_red[grp][2][lane], s_red[grp][3][lane]));
          group_bar(grp);  // s_red reusable
          if (gt == 0) TC_TRACE(7, g);  // softmax: column maxima known
          uint32_t ov[32];
          const uint32_t oaddr = tmem + lane_base + 64 + grp * 32;
          if (i > 0) {  // O^T is rescaled below: the previous block's PV must be complete
            tc_wait(&p_empty[grp], (pc - 1) & 1, 13);
            sm100::tc_fence_after();
            sm100::tmem_ld_32x32b_x32(oaddr, ov);
            sm100::tmem_ld_wait();
          }
          // branch-free per-row update (the decisions are uniform across the
          // group; divergent-looking branches would cost a convergence
          // barrier per row)
#pragma unroll
          for (int r = 0; r < kRows; ++r) {
            const float em = __shfl_sync(0xffffffffu, bm, r);
            const bool was_unset = unset >> r & 1;
            const bool up = em != -INFINITY && (was_unset || em > 8.0f);
            const float a = was_unset ? 0.0f : fast_exp2(-em);
            const float sub = up ? em : 0.0f;
            neg[r] -= sub;
            e[r] -= sub;
            lsum[r] = up ? lsum[r] * a : lsum[r];
            ov[r] = up ? __float_as_uint(__uint_as_float(ov[r]) * a) : ov[r];
            unset &= up ? ~(1u << r) : 0xffffffffu;
          }
          if (i > 0) {
            sm100::tmem_st_32x32b_x32(oaddr, ov);
            sm100::tmem_st_wait();
          }
        }
        uint32_t pw[16];
#pragma unroll
        for (int r = 0; r < kRows; r += 2) {
          const float p0 = fast_exp2(e[r]);
          const float p1 = fast_exp2(e[r + 1]);
          lsum[r] += p0;
          lsum[r + 1] += p1;
          const __nv_bfloat162 pk = __floats2bfloat162_rn(p0, p1);
          pw[r >> 1] = *reinterpret_cast<const uint32_t*>(&pk);
        }
        // the group's P^T buffer is free once its previous block's PV completed
        if (pc > 0) tc_wait(&p_empty[grp], (pc - 1) & 1, 14);
        if (gt == 0) TC_TRACE(4, g);  // softmax: P buffer free
#pragma unroll
        for (int c = 0; c < 4; ++c)
          *reinterpret_cast<uint4*>(p_row + ((c ^ kx) << 4)) = make_uint4(pw[4 * c], pw[4 * c + 1], pw[4 * c + 2], pw[4 * c + 3]);
        sm100::fence_proxy_async();
        sm100::tc_fence_before();
        __syncwarp();
        if (lane == 0) sm100::mbar_arrive(&p_full[grp]);
        if (gt == 0) TC_TRACE(5, g);  // softmax: P written
      }
      // ---- epilogue: row sums across the 128 key threads, O^T from TMEM
      const float lrow = warp_transpose_reduce<false>(lsum, lane);
      s_red[grp][qd][lane] = lrow;
      group_bar(grp);
      // lane r: row r's sum (fixed quadrant order) and its reciprocal
      const float ltot = ((s_red[grp][0][lane] + s_red[grp][1][lane]) + s_red[grp][2][lane]) + s_red[grp][3][lane];
      const float linv = 1.0f / ltot;
      tc_wait(&o_full[grp], (it / kTcGroups) & 1, 15);
      sm100::tc_fence_after();
      uint32_t ov[32];
      sm100::tmem_ld_32x32b_x32(tmem + lane_base + 64 + grp * 32, ov);
      sm100::tmem_ld_wait();
      sm100::tc_fence_before();
      __syncwarp();
      if (lane == 0) sm100::mbar_arrive(&o_empty[grp]);
      const int64_t pidx = ((int64_t)I.z * A.qblocks + I.qb) * A.splits + I.sp;
      const int d = kk;
      if (I.ntiles <= A.split_tiles) {
        // single split: out = O / l (the combine's form for one split).  The
        // group's P^T buffer is idle here (its PVs have all completed): it
        // transposes the bf16 rows so the stores are 16-byte vectors.
        __nv_bfloat16* sT = reinterpret_cast<__nv_bfloat16*>(sP);  // [32 rows][128]
#pragma unroll
        for (int r = 0; r < kRows; ++r)
          sT[r * 128 + d] = __float2bfloat16_rn(__uint_as_float(ov[r]) * __shfl_sync(0xffffffffu, linv, r));
        group_bar(grp);
#pragma unroll
        for (int e = gt; e < kRows * 16; e += 128) {
          const int r = e >> 4, c = e & 15;
          const int orow = s_orow[grp][r];
          if (orow >= 0)
            *reinterpret_cast<uint4*>(A.out + (int64_t)orow * 128 + c * 8) =
                *reinterpret_cast<const uint4*>(sT + r * 128 + c * 8);
        }
      } else {
        float* po = A.part_o + pidx * kRows * 128;
#pragma unroll
        for (int r = 0; r < kRows; ++r)
          if (r < I.rows) po[r * 128 + d] = __uint_as_float(ov[r]);
        if (qd == 0 && lane < I.rows) {
          float nl = 0.0f;
#pragma unroll
          for (int r = 0; r < kRows; ++r) nl = r == lane ? neg[r] : nl;
          float* pml = A.part_ml + pidx * kRows * 2;
          pml[lane * 2] = (unset >> lane & 1) ? -INFINITY : -nl;
          pml[lane * 2 + 1] = ltot;
        }
      }
      group_bar(grp);  // s_red, s_orow and the P^T buffer reusable by the next item
      it += kTcGroups;
    }
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 1) sm100::tmem_dealloc<128>(tmem);
#if SR_ATTN_PROBE == 4
  if (blockIdx.x == 0 && tid == 0) {
    const unsigned long long t0 = g_tc_trace[0][0];
    for (int b = 0; b < 64 && g_tc_trace[0][b]; ++b)
      printf("TRACE %d %lld %lld %lld %lld %lld %lld %lld %lld\n", b, (long long)(g_tc_trace[0][b] - t0),
             (long long)(g_tc_trace[1][b] - t0), (long long)(g_tc_trace[2][b] - t0), (long long)(g_tc_trace[3][b] - t0),
             (long long)(g_tc_trace[4][b] - t0), (long long)(g_tc_trace[5][b] - t0), (long long)(g_tc_trace[6][b] - t0),
             (long long)(g_tc_trace[7][b] ? g_tc_trace[7][b] - t0 : 0));
    for (int e = 0; e < 8; ++e) for (int b = 0; b < 64; ++b) g_tc_trace[e][b] = 0;
  }
#endif
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
  a.early = (phase == 0 && !plan) ? 1 : 0;
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
    if (hd == 128 && g_attn_tc && a.split_tiles % 2 == 0 && a.split_tiles <= 32) {
      // tcgen05 path: 128-key blocks (split boundaries stay block aligned; an
      // item's block-table slice fits the producer warp's lanes)
      static bool set_tc = false;
      if (!set_tc) {
        SR_CHECK_CUDA(cudaFuncSetAttribute(attn_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)kTcSmem));
        set_tc = true;
      }
      CUtensorMap tm;
      const uint64_t blocks = (uint64_t)kv.layers * kv.num_pages * 2 * kv.kv_heads;
      const int trc = make_tmap_kv_pages(&tm, kv.cache, blocks);
      if (trc) return trc;
      const char* gv = getenv("SR_ATTN_TC_GRID");  // fewer CTAs, more items each (tests)
      const int grid_cap = gv ? std::max(1, atoi(gv)) : 1 << 30;
      const int tgrid = std::min(std::min(a.n_slots, sms > 0 ? sms : 148), grid_cap);
      sr::launch_k(attn_tc_kernel, tgrid, kTcThreads, (size_t)kTcSmem, stream, tm, a);
      const cudaError_t le = cudaPeekAtLastError();
      if (le != cudaSuccess) {
        cudaFuncAttributes fa;
        cudaFuncGetAttributes(&fa, attn_tc_kernel);
        cudaGetLastError();
        set_error("attn_tc_kernel: %s (regs %d, max threads %d, static smem %zu, max dyn smem %d, requested %u x %d)",
                  cudaGetErrorString(le), fa.numRegs, fa.maxThreadsPerBlock, fa.sharedSizeBytes,
                  fa.maxDynamicSharedSizeBytes, kTcSmem, kTcThreads);
        return SR_ERR_RUNTIME;
      }
      return SR_OK;
    }
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

extern "C" int sr_set_attention_tc(int on) {
  SR_REQUIRE(on == 0 || on == 1, "attention kernel selector must be 0 or 1");
  sr::g_attn_tc = on != 0;
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
