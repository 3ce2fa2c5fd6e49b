// K2: verification attention over the paged KV cache.
//
// One CTA = (sequence, kv head, query block of 64 rows, KV split).  Rows are
// (window position j, group head g) pairs, r = j*G + g, so all query heads
// sharing a kv head read each K/V tile once (GQA).  Keys are walked in
// tiles of 64 *absolute* positions (tile t = keys [64t, 64t+64)); a key comes
// from the paged cache when it is committed (pos < ctx_len) or written in
// place, else from the drafter-branch window buffer.  Splits are fixed
// 1024-key ranges merged by a combine kernel in split order.  Because the
// tiling depends only on absolute positions, a query's arithmetic is the
// same in a 5-position verify window and in a 1-position decode step: the
// speculative and plain paths produce bit-identical logits.
//
// Per tile: cp.async (16-byte, XOR-swizzled) double-buffered K/V staging;
// S = Q K^T with mma.sync m16n8k16 bf16 (warp w owns keys 16w..16w+15);
// fp32 online softmax in shared memory (2 threads per row, exp2); O += P V
// with mma.sync (warp w owns head-dim columns w*HD/4..).  HBM-bound: the
// kernel's algorithmic bytes are the K/V tiles it reads.
#include "common.cuh"
#include "layers.cuh"

#include <cuda_bf16.h>

namespace sr {

namespace {

constexpr int kKT = 64;          // keys per tile (= page size)
constexpr int kRows = 64;        // query rows per CTA
constexpr int kSplitTiles = 16;  // tiles per KV split (1024 keys)
constexpr int kAttnThreads = 128;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(smem)),
               "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait0() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

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
};

__device__ __forceinline__ int block_max_key(const SeqInfo& sq, int r0, int rows, int G) {
  return sq.ctx_len + (r0 + rows - 1) / G;
}

template <int HD>
__global__ void __launch_bounds__(kAttnThreads)
attn_bf16_kernel(AttnArgs A) {
  constexpr int CH = HD / 8;                 // 16-byte chunks per row
  constexpr int NT = HD / 32;                // n8 tiles of O per warp
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* sQ = smem;
  uint8_t* sK = sQ + kRows * HD * 2;         // [2][64][HD]
  uint8_t* sV = sK + 2 * kKT * HD * 2;       // [2][64][HD]
  float* sS = reinterpret_cast<float*>(sV + 2 * kKT * HD * 2);   // [64][68]
  __nv_bfloat16* sP = reinterpret_cast<__nv_bfloat16*>(sS + kRows * 68);  // [64][72]
  float* sAlpha = reinterpret_cast<float*>(sP + kRows * 72);
  float* sM = sAlpha + kRows;
  float* sL = sM + kRows;

  const int nkv = A.kv.kv_heads;
  const int sp = blockIdx.x, qb = blockIdx.y;
  const int s = blockIdx.z / nkv, h = blockIdx.z % nkv;
  const SeqInfo sq = A.seqs[s];
  const int G = A.G;
  const int rows_total = sq.q_len * G;
  const int r0 = qb * kRows;
  if (r0 >= rows_total) return;
  const int rows = min(kRows, rows_total - r0);
  const int max_key = block_max_key(sq, r0, rows, G);
  const int ntiles = max_key / kKT + 1;
  const int t_begin = sp * kSplitTiles, t_end = min(ntiles, t_begin + kSplitTiles);
  if (t_begin >= t_end) return;
  const int mtv = (rows + 15) / 16;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  const __nv_bfloat16* cache = reinterpret_cast<const __nv_bfloat16*>(A.kv.cache) +
                               (int64_t)A.layer * A.kv.cache_layer_elems();
  const __nv_bfloat16* win = reinterpret_cast<const __nv_bfloat16*>(A.kv.window) +
                             (int64_t)A.layer * A.kv.window_layer_elems();
  const int32_t* btab = A.kv.block_table + (int64_t)sq.request * A.kv.max_pages;
  const int psz = A.kv.page;

  // ---- Q block -> smem (zeros for padding rows)
  for (int e = tid; e < kRows * CH; e += kAttnThreads) {
    const int r = e / CH, c = e % CH;
    uint8_t* dst = sQ + swz<HD>(r, c);
    if (r < rows) {
      const int gr = r0 + r, j = gr / G, g = gr % G;
      const __nv_bfloat16* src = A.q + ((int64_t)(sq.q_start + j) * A.nq + h * G + g) * HD + c * 8;
      cp_async16(dst, src);
    } else {
      *reinterpret_cast<uint4*>(dst) = make_uint4(0, 0, 0, 0);
    }
  }
  if (tid < kRows) {
    sM[tid] = -INFINITY;
    sL[tid] = 0.0f;
  }

  auto load_tile = [&](int t, int stage) {
    uint8_t* k_dst = sK + stage * kKT * HD * 2;
    uint8_t* v_dst = sV + stage * kKT * HD * 2;
    for (int e = tid; e < kKT * CH; e += kAttnThreads) {
      const int r = e / CH, c = e % CH;
      const int kp = t * kKT + r;
      const uint32_t off = swz<HD>(r, c);
      if (kp > max_key) {
        *reinterpret_cast<uint4*>(k_dst + off) = make_uint4(0, 0, 0, 0);
        *reinterpret_cast<uint4*>(v_dst + off) = make_uint4(0, 0, 0, 0);
        continue;
      }
      const __nv_bfloat16* ksrc;
      int64_t vstep;
      if (sq.branch < 0 || kp < sq.ctx_len) {
        const int page = btab[kp / psz];
        ksrc = cache + (((int64_t)page * 2 * nkv + h) * psz + kp % psz) * HD;
        vstep = (int64_t)nkv * psz * HD;
      } else {
        ksrc = win + (((int64_t)sq.branch * 2 * nkv + h) * A.kv.window_max + (kp - sq.ctx_len)) * HD;
        vstep = (int64_t)nkv * A.kv.window_max * HD;
      }
      cp_async16(k_dst + off, ksrc + c * 8);
      cp_async16(v_dst + off, ksrc + vstep + c * 8);
    }
    cp_async_commit();
  };

  float o[4][NT][4];
#pragma unroll
  for (int mt = 0; mt < 4; ++mt)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int i = 0; i < 4; ++i) o[mt][nt][i] = 0.0f;

  load_tile(t_begin, 0);
  const uint32_t q_base = (uint32_t)__cvta_generic_to_shared(sQ);
  for (int t = t_begin; t < t_end; ++t) {
    const int stage = (t - t_begin) & 1;
    cp_async_wait0();
    __syncthreads();  // tile t (and Q) visible; previous P/alpha consumers done
    if (t + 1 < t_end) load_tile(t + 1, stage ^ 1);
    const uint32_t k_base = (uint32_t)__cvta_generic_to_shared(sK + stage * kKT * HD * 2);
    const uint32_t v_base = (uint32_t)__cvta_generic_to_shared(sV + stage * kKT * HD * 2);

    // ---- S = Q K^T for keys [16w, 16w+16)
#pragma unroll
    for (int mt = 0; mt < 4; ++mt) {
      if (mt >= mtv) break;
      float acc[2][4] = {{0, 0, 0, 0}, {0, 0, 0, 0}};
#pragma unroll
      for (int kk = 0; kk < HD / 16; ++kk) {
        uint32_t a0, a1, a2, a3, b0, b1, b2, b3;
        {
          const int mi = lane >> 3;
          const int row = mt * 16 + (mi & 1) * 8 + (lane & 7);
          ldsm_x4(q_base + swz<HD>(row, kk * 2 + (mi >> 1)), a0, a1, a2, a3);
        }
        {
          const int mi = lane >> 3;
          const int key = warp * 16 + (mi >> 1) * 8 + (lane & 7);
          ldsm_x4(k_base + swz<HD>(key, kk * 2 + (mi & 1)), b0, b1, b2, b3);
        }
        mma_bf16(acc[0], a0, a1, a2, a3, b0, b1);
        mma_bf16(acc[1], a0, a1, a2, a3, b2, b3);
      }
#pragma unroll
      for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int r = mt * 16 + (lane >> 2) + (i >> 1) * 8;
          const int col = warp * 16 + nt * 8 + 2 * (lane & 3) + (i & 1);
          const int kp = t * kKT + col;
          const int qpos = sq.ctx_len + (r0 + r) / G;
          const bool ok = r < rows && kp <= qpos;
          sS[r * 68 + col] = ok ? acc[nt][i] * A.scale_log2 : -INFINITY;
        }
    }
    __syncthreads();

    // ---- online softmax: 2 threads per row
    {
      const int r = tid >> 1, half = tid & 1;
      if (r < mtv * 16) {
        const float* srow = sS + r * 68 + half * 32;
        float mx = -INFINITY;
#pragma unroll
        for (int c = 0; c < 32; ++c) mx = fmaxf(mx, srow[c]);
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
        const float m_old = sM[r];
        const float m_new = fmaxf(m_old, mx);
        const float m_use = m_new == -INFINITY ? 0.0f : m_new;
        float sum = 0.0f;
        __nv_bfloat16* prow = sP + r * 72 + half * 32;
#pragma unroll
        for (int c = 0; c < 32; ++c) {
          const float p = exp2f(srow[c] - m_use);
          prow[c] = __float2bfloat16_rn(p);
          sum += p;
        }
        sum += __shfl_xor_sync(0xffffffffu, sum, 1);
        const float alpha = exp2f(m_old - m_use);
        const float l_old = sL[r];
        __syncwarp();
        if (half == 0) {
          sM[r] = m_new;
          sL[r] = l_old * alpha + sum;
          sAlpha[r] = alpha;
        }
      }
    }
    __syncthreads();

    // ---- O = alpha * O + P V for head-dim columns [w*HD/4, (w+1)*HD/4)
    const uint32_t p_base = (uint32_t)__cvta_generic_to_shared(sP);
#pragma unroll
    for (int mt = 0; mt < 4; ++mt) {
      if (mt >= mtv) break;
      const float a_lo = sAlpha[mt * 16 + (lane >> 2)], a_hi = sAlpha[mt * 16 + (lane >> 2) + 8];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        o[mt][nt][0] *= a_lo; o[mt][nt][1] *= a_lo;
        o[mt][nt][2] *= a_hi; o[mt][nt][3] *= a_hi;
      }
#pragma unroll
      for (int kk = 0; kk < kKT / 16; ++kk) {
        uint32_t a0, a1, a2, a3;
        {
          const int mi = lane >> 3;
          const int row = mt * 16 + (mi & 1) * 8 + (lane & 7);
          const int col = kk * 16 + (mi >> 1) * 8;
          ldsm_x4(p_base + (uint32_t)(row * 72 + col) * 2, a0, a1, a2, a3);
        }
#pragma unroll
        for (int np = 0; np < NT / 2; ++np) {
          uint32_t b0, b1, b2, b3;
          const int mi = lane >> 3;
          const int key = kk * 16 + (mi & 1) * 8 + (lane & 7);
          const int dim0 = warp * (HD / 4) + np * 16 + (mi >> 1) * 8;
          ldsm_x4_t(v_base + swz<HD>(key, dim0 / 8), b0, b1, b2, b3);
          mma_bf16(o[mt][2 * np], a0, a1, a2, a3, b0, b1);
          mma_bf16(o[mt][2 * np + 1], a0, a1, a2, a3, b2, b3);
        }
      }
    }
  }
  __syncthreads();

  // ---- partials
  const int64_t pidx = ((int64_t)blockIdx.z * A.qblocks + qb) * A.splits + sp;
  float* po = A.part_o + pidx * kRows * HD;
#pragma unroll
  for (int mt = 0; mt < 4; ++mt) {
    if (mt >= mtv) break;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const int col = warp * (HD / 4) + nt * 8 + 2 * (lane & 3);
      const int r = mt * 16 + (lane >> 2);
      *reinterpret_cast<float2*>(po + r * HD + col) = make_float2(o[mt][nt][0], o[mt][nt][1]);
      *reinterpret_cast<float2*>(po + (r + 8) * HD + col) = make_float2(o[mt][nt][2], o[mt][nt][3]);
    }
  }
  if (tid < kRows) {
    float* pml = A.part_ml + pidx * kRows * 2;
    pml[tid * 2] = sM[tid];
    pml[tid * 2 + 1] = sL[tid];
  }
}

template <int HD>
__global__ void __launch_bounds__(HD)
attn_combine_kernel(AttnArgs A, __nv_bfloat16* out) {
  const int nkv = A.kv.kv_heads;
  const int qb = blockIdx.x, z = blockIdx.y;
  const int s = z / nkv, h = z % nkv;
  const SeqInfo sq = A.seqs[s];
  const int G = A.G;
  const int rows_total = sq.q_len * G;
  const int r0 = qb * kRows;
  if (r0 >= rows_total) return;
  const int rows = min(kRows, rows_total - r0);
  const int ntiles = block_max_key(sq, r0, rows, G) / kKT + 1;
  const int nsplit = (ntiles + kSplitTiles - 1) / kSplitTiles;
  const int d = threadIdx.x;
  for (int r = 0; r < rows; ++r) {
    const int64_t base = ((int64_t)z * A.qblocks + qb) * A.splits;
    float M = -INFINITY;
    for (int sp = 0; sp < nsplit; ++sp) M = fmaxf(M, A.part_ml[((base + sp) * kRows + r) * 2]);
    float den = 0.0f, num = 0.0f;
    for (int sp = 0; sp < nsplit; ++sp) {
      const float m = A.part_ml[((base + sp) * kRows + r) * 2];
      const float w = exp2f(m - M);
      den += w * A.part_ml[((base + sp) * kRows + r) * 2 + 1];
      num += w * A.part_o[((base + sp) * kRows + r) * HD + d];
    }
    const int gr = r0 + r, j = gr / G, g = gr % G;
    out[((int64_t)(sq.q_start + j) * A.nq + h * G + g) * HD + d] = __float2bfloat16_rn(num / den);
  }
}

// fp32 parity attention: one warp per (token, q head), keys in position
// order with an fp32 online softmax (no splits).
__global__ void attn_f32_kernel(const float* __restrict__ q, const SeqInfo* __restrict__ seqs, KvLayout kv,
                                int layer, int nq, int G, float scale, float* __restrict__ out) {
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
  return (size_t)kRows * HD * 2 + 4 * (size_t)kKT * HD * 2 + kRows * 68 * 4 + kRows * 72 * 2 + 3 * kRows * 4;
}

}  // namespace

size_t attention_partial_floats(int num_seqs, int kv_heads, int qblocks, int splits, int hd) {
  return (size_t)num_seqs * kv_heads * qblocks * splits * kRows * (hd + 2);
}

int attention_bf16(const __nv_bfloat16* q, const SeqInfo* seqs, int num_seqs, int max_q_len, int max_key,
                   const KvLayout& kv, int layer, int nq, float* partials, size_t partial_floats,
                   __nv_bfloat16* out, cudaStream_t stream) {
  if (num_seqs == 0) return SR_OK;
  const int hd = kv.head_dim, G = nq / kv.kv_heads;
  SR_REQUIRE(hd == 64 || hd == 128, "bf16 attention supports head_dim 64 or 128");
  SR_REQUIRE(kv.page == kKT, "paged cache page size must be 64 tokens");
  AttnArgs a;
  a.q = q; a.seqs = seqs; a.kv = kv; a.layer = layer; a.nq = nq; a.G = G;
  a.scale_log2 = 1.4426950408889634f / sqrtf((float)hd);
  a.qblocks = ceil_div(max_q_len * G, kRows);
  a.splits = ceil_div(max_key / kKT + 1, kSplitTiles);
  const size_t need = attention_partial_floats(num_seqs, kv.kv_heads, a.qblocks, a.splits, hd);
  SR_REQUIRE(need <= partial_floats, "attention partial workspace too small");
  a.part_o = partials;
  a.part_ml = partials + (size_t)num_seqs * kv.kv_heads * a.qblocks * a.splits * kRows * hd;
  dim3 grid(a.splits, a.qblocks, num_seqs * kv.kv_heads);
  if (hd == 128) {
    static bool set = false;
    if (!set) {
      SR_CHECK_CUDA(cudaFuncSetAttribute(attn_bf16_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)attn_smem<128>()));
      set = true;
    }
    attn_bf16_kernel<128><<<grid, kAttnThreads, attn_smem<128>(), stream>>>(a);
    int rc = check_launch("attn_bf16_kernel<128>");
    if (rc) return rc;
    attn_combine_kernel<128><<<dim3(a.qblocks, num_seqs * kv.kv_heads), 128, 0, stream>>>(a, out);
  } else {
    static bool set = false;
    if (!set) {
      SR_CHECK_CUDA(cudaFuncSetAttribute(attn_bf16_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)attn_smem<64>()));
      set = true;
    }
    attn_bf16_kernel<64><<<grid, kAttnThreads, attn_smem<64>(), stream>>>(a);
    int rc = check_launch("attn_bf16_kernel<64>");
    if (rc) return rc;
    attn_combine_kernel<64><<<dim3(a.qblocks, num_seqs * kv.kv_heads), 64, 0, stream>>>(a, out);
  }
  return check_launch("attn_combine_kernel");
}

int attention_f32(const float* q, const SeqInfo* seqs, int num_seqs, int max_q_len, const KvLayout& kv,
                  int layer, int nq, float* out, cudaStream_t stream) {
  if (num_seqs == 0) return SR_OK;
  SR_REQUIRE(kv.head_dim <= 128, "fp32 attention supports head_dim <= 128");
  const int G = nq / kv.kv_heads;
  dim3 grid(ceil_div(max_q_len * nq, 8), num_seqs);
  attn_f32_kernel<<<grid, 256, 0, stream>>>(q, seqs, kv, layer, nq, G, 1.0f / sqrtf((float)kv.head_dim), out);
  return check_launch("attn_f32_kernel");
}

}  // namespace sr
