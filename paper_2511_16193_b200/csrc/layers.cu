// K6 helpers of the verify forward; see layers.cuh.
#include "common.cuh"
#include "layers.cuh"
#include "sampling.cuh"

namespace sr {

namespace {

template <typename T> __device__ __forceinline__ float to_f(T v);
template <> __device__ __forceinline__ float to_f<float>(float v) { return v; }
template <> __device__ __forceinline__ float to_f<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }
template <typename T> __device__ __forceinline__ T from_f(float v);
template <> __device__ __forceinline__ float from_f<float>(float v) { return v; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }

template <typename T>
__global__ void embed_kernel(const T* __restrict__ table, const int32_t* __restrict__ ids, int H, int vocab,
                             float* __restrict__ x) {
  grid_dep_sync();
  const int row = blockIdx.x;
  // an id outside this model's vocabulary (a drafter whose vocabulary is
  // smaller than the target's padded one, e.g. Qwen2.5-0.5B 151936 vs 7B
  // 152064) embeds as token 0: drafts stay proposals, never out-of-bounds reads
  int id = ids[row];
  if (id < 0 || id >= vocab) id = 0;
  const T* src = table + (int64_t)id * H;
  float* dst = x + (int64_t)row * H;
  for (int i = threadIdx.x; i < H; i += blockDim.x) dst[i] = to_f(src[i]);
}

// One warp per row: float4 loads (all issued before the reduction), xor-
// shuffle tree (fixed order), then scale.  Matches the oracle:
// y = x * rsqrt(mean(x^2) + eps) * w.  H % 4 == 0 takes the vector path.
template <typename T>
__global__ void __launch_bounds__(256)
rmsnorm_kernel(const float* __restrict__ x, const float* __restrict__ w, int M, int H, float eps,
               T* __restrict__ out) {
  grid_dep_sync();
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= M) return;
  const float* xr = x + (int64_t)row * H;
  T* orow = out + (int64_t)row * H;
  float ss = 0.0f;
  if ((H & 3) == 0) {
    const float4* x4 = reinterpret_cast<const float4*>(xr);
    const int n4 = H >> 2;
    float4 buf[12];
#pragma unroll
    for (int i = 0; i < 12; ++i)
      buf[i] = (lane + 32 * i < n4) ? x4[lane + 32 * i] : make_float4(0, 0, 0, 0);
    for (int i = 12 * 32 + lane; i < n4; i += 32) {  // rows wider than 1536
      const float4 v = x4[i];
      ss = fmaf(v.x, v.x, ss); ss = fmaf(v.y, v.y, ss); ss = fmaf(v.z, v.z, ss); ss = fmaf(v.w, v.w, ss);
    }
#pragma unroll
    for (int i = 0; i < 12; ++i) {
      ss = fmaf(buf[i].x, buf[i].x, ss); ss = fmaf(buf[i].y, buf[i].y, ss);
      ss = fmaf(buf[i].z, buf[i].z, ss); ss = fmaf(buf[i].w, buf[i].w, ss);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    const float r = rsqrtf(ss / (float)H + eps);
    const float4* w4 = reinterpret_cast<const float4*>(w);
    auto emit = [&](int i, float4 v) {
      const float4 g = w4[i];
      orow[4 * i + 0] = from_f<T>(v.x * r * g.x);
      orow[4 * i + 1] = from_f<T>(v.y * r * g.y);
      orow[4 * i + 2] = from_f<T>(v.z * r * g.z);
      orow[4 * i + 3] = from_f<T>(v.w * r * g.w);
    };
#pragma unroll
    for (int j = 0; j < 12; ++j)
      if (lane + 32 * j < n4) emit(lane + 32 * j, buf[j]);
    for (int i = 12 * 32 + lane; i < n4; i += 32) emit(i, x4[i]);
    return;
  }
  for (int i = lane; i < H; i += 32) ss = fmaf(xr[i], xr[i], ss);
#pragma unroll
  for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  const float r = rsqrtf(ss / (float)H + eps);
  for (int i = lane; i < H; i += 32) orow[i] = from_f<T>(xr[i] * r * w[i]);
}

template <typename T>
__global__ void rope_scatter_kernel(const T* __restrict__ qkv, const int32_t* __restrict__ positions,
                                    const SeqInfo* __restrict__ seqs, const float* __restrict__ cos_t,
                                    const float* __restrict__ sin_t, int nq, int layer, KvLayout kv,
                                    T* __restrict__ q_out) {
  grid_dep_sync();
  const SeqInfo sq = seqs[blockIdx.y];
  const int j = blockIdx.x;
  if (j >= sq.q_len) return;
  const int tok = sq.q_start + j;
  const int hd = kv.head_dim, half = hd / 2, nkv = kv.kv_heads;
  const int width = (nq + 2 * nkv) * hd;
  const int pos = positions[tok];
  const T* row = qkv + (int64_t)tok * width;
  const float* cr = cos_t + (int64_t)pos * half;
  const float* sr_ = sin_t + (int64_t)pos * half;

  T* kdst;
  T* vdst;
  int64_t head_stride;  // elements between consecutive kv heads at this slot
  int slot_id;          // swizzle key of the destination row
  if (sq.branch < 0) {
    SR_DCHECK(pos >= 0 && pos / kv.page < kv.max_pages);
    const int page = kv.block_table[(int64_t)sq.request * kv.max_pages + pos / kv.page];
    SR_DCHECK(page >= 0 && page < kv.num_pages);
    const int slot = pos % kv.page;
    T* base = reinterpret_cast<T*>(kv.cache) + layer * kv.cache_layer_elems() +
              (int64_t)page * 2 * nkv * kv.page * hd;
    kdst = base + (int64_t)slot * hd;
    vdst = kdst + (int64_t)nkv * kv.page * hd;
    head_stride = (int64_t)kv.page * hd;
    slot_id = slot;
  } else {
    T* base = reinterpret_cast<T*>(kv.window) + layer * kv.window_layer_elems() +
              (int64_t)sq.branch * 2 * nkv * kv.window_max * hd;
    kdst = base + (int64_t)j * hd;
    vdst = kdst + (int64_t)nkv * kv.window_max * hd;
    head_stride = (int64_t)kv.window_max * hd;
    slot_id = j;
  }
  // rotate q heads and k heads (NeoX halves), copy v.  Vector path: a thread
  // owns 8 consecutive dims of the first half and the matching 8 of the
  // second half, so every load/store is one 16-byte chunk (the cache swizzle
  // permutes whole chunks).
  if constexpr (sizeof(T) == 2) {
    if ((half & 7) == 0) {
      const int cph = half / 8;  // chunks per half-head
      for (int e = threadIdx.x; e < (nq + nkv) * cph; e += blockDim.x) {
        const int h = e / cph, c = e % cph, i0 = c * 8;
        const uint4 a = *reinterpret_cast<const uint4*>(row + h * hd + i0);
        const uint4 b = *reinterpret_cast<const uint4*>(row + h * hd + i0 + half);
        const T* pa = reinterpret_cast<const T*>(&a);
        const T* pb = reinterpret_cast<const T*>(&b);
        uint4 ya, yb;
        T* qa = reinterpret_cast<T*>(&ya);
        T* qb = reinterpret_cast<T*>(&yb);
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          const float cc = cr[i0 + t], ss = sr_[i0 + t];
          const float x1 = to_f(pa[t]), x2 = to_f(pb[t]);
          qa[t] = from_f<T>(x1 * cc - x2 * ss);
          qb[t] = from_f<T>(x2 * cc + x1 * ss);
        }
        if (h < nq) {
          T* q = q_out + (int64_t)tok * nq * hd + h * hd;
          *reinterpret_cast<uint4*>(q + i0) = ya;
          *reinterpret_cast<uint4*>(q + i0 + half) = yb;
        } else {
          T* k = kdst + (h - nq) * head_stride;
          *reinterpret_cast<uint4*>(k + kv_phys<T>(slot_id, i0)) = ya;
          *reinterpret_cast<uint4*>(k + kv_phys<T>(slot_id, i0 + half)) = yb;
        }
      }
      for (int e = threadIdx.x; e < nkv * (hd / 8); e += blockDim.x) {
        const int h = e / (hd / 8), d = (e % (hd / 8)) * 8;
        *reinterpret_cast<uint4*>(vdst + h * head_stride + kv_phys<T>(slot_id, d)) =
            *reinterpret_cast<const uint4*>(row + (nq + nkv + h) * hd + d);
      }
      return;
    }
  }
  for (int e = threadIdx.x; e < (nq + nkv) * half; e += blockDim.x) {
    const int h = e / half, i = e % half;
    const float c = cr[i], s = sr_[i];
    const float x1 = to_f(row[h * hd + i]), x2 = to_f(row[h * hd + i + half]);
    const float y1 = x1 * c - x2 * s, y2 = x2 * c + x1 * s;
    if (h < nq) {
      T* q = q_out + (int64_t)tok * nq * hd + h * hd;
      q[i] = from_f<T>(y1);
      q[i + half] = from_f<T>(y2);
    } else {
      T* k = kdst + (h - nq) * head_stride;
      k[kv_phys<T>(slot_id, i)] = from_f<T>(y1);
      k[kv_phys<T>(slot_id, i + half)] = from_f<T>(y2);
    }
  }
  for (int e = threadIdx.x; e < nkv * hd; e += blockDim.x) {
    const int h = e / hd, d = e % hd;
    vdst[h * head_stride + kv_phys<T>(slot_id, d)] = row[(nq + nkv + h) * hd + d];
  }
}

__device__ __forceinline__ bool better(float v, int i, float bv, int bi) {
  return v > bv || (v == bv && i < bi);
}

__global__ void argmax_reduce_kernel(const float* __restrict__ pv, const int32_t* __restrict__ pi,
                                     int M, int tiles, int32_t* __restrict__ ids,
                                     float* __restrict__ vals) {
  grid_dep_sync();
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= M) return;
  float bv = -INFINITY;
  int bi = 0x7fffffff;
  for (int t = lane; t < tiles; t += 32) {
    const float v = pv[(int64_t)row * tiles + t];
    const int i = pi[(int64_t)row * tiles + t];
    if (better(v, i, bv, bi)) { bv = v; bi = i; }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const float v = __shfl_xor_sync(0xffffffffu, bv, o);
    const int i = __shfl_xor_sync(0xffffffffu, bi, o);
    if (better(v, i, bv, bi)) { bv = v; bi = i; }
  }
  if (lane == 0) {
    ids[row] = bi;
    if (vals) vals[row] = bv;
  }
}

__global__ void argmax_rows_kernel(const float* __restrict__ logits, int V, int ld,
                                   int32_t* __restrict__ ids, float* __restrict__ vals) {
  grid_dep_sync();
  const int row = blockIdx.x;
  const float* r = logits + (int64_t)row * ld;
  float bv = -INFINITY;
  int bi = 0x7fffffff;
  for (int i = threadIdx.x; i < V; i += blockDim.x) {
    const float v = r[i];
    if (better(v, i, bv, bi)) { bv = v; bi = i; }
  }
  __shared__ float sv[32];
  __shared__ int si[32];
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const float v = __shfl_xor_sync(0xffffffffu, bv, o);
    const int i = __shfl_xor_sync(0xffffffffu, bi, o);
    if (better(v, i, bv, bi)) { bv = v; bi = i; }
  }
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) { sv[w] = bv; si[w] = bi; }
  __syncthreads();
  if (w == 0) {
    const int nw = blockDim.x >> 5;
    bv = lane < nw ? sv[lane] : -INFINITY;
    bi = lane < nw ? si[lane] : 0x7fffffff;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const float v = __shfl_xor_sync(0xffffffffu, bv, o);
      const int i = __shfl_xor_sync(0xffffffffu, bi, o);
      if (better(v, i, bv, bi)) { bv = v; bi = i; }
    }
    if (lane == 0) {
      ids[row] = bi;
      if (vals) vals[row] = bv;
    }
  }
}

// Keyed Gumbel-max sample of fp32 logit rows (same noise as the fused
// lm_head epilogue): one CTA per row.
__global__ void sample_rows_kernel(const float* __restrict__ logits, int V, int ld,
                                   const int32_t* __restrict__ req, const int32_t* __restrict__ pos,
                                   uint32_t seed, float inv_temp, int32_t* __restrict__ ids,
                                   float* __restrict__ vals) {
  grid_dep_sync();
  const int row = blockIdx.x;
  const float* r = logits + (int64_t)row * ld;
  const int rq = req[row], ps = pos[row];
  float bv = -INFINITY;
  int bi = 0x7fffffff;
  for (int b = threadIdx.x; b * 4 < V; b += blockDim.x) {
    float g[4];
    gumbel4(seed, rq, ps, b, g);
    for (int t = 0; t < 4 && 4 * b + t < V; ++t) {
      const float v = r[4 * b + t] * inv_temp + g[t];
      if (better(v, 4 * b + t, bv, bi)) { bv = v; bi = 4 * b + t; }
    }
  }
  __shared__ float sv[32];
  __shared__ int si[32];
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const float v = __shfl_xor_sync(0xffffffffu, bv, o);
    const int i = __shfl_xor_sync(0xffffffffu, bi, o);
    if (better(v, i, bv, bi)) { bv = v; bi = i; }
  }
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) { sv[w] = bv; si[w] = bi; }
  __syncthreads();
  if (w == 0) {
    const int nw = blockDim.x >> 5;
    bv = lane < nw ? sv[lane] : -INFINITY;
    bi = lane < nw ? si[lane] : 0x7fffffff;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const float v = __shfl_xor_sync(0xffffffffu, bv, o);
      const int i = __shfl_xor_sync(0xffffffffu, bi, o);
      if (better(v, i, bv, bi)) { bv = v; bi = i; }
    }
    if (lane == 0) {
      ids[row] = bi;
      if (vals) vals[row] = bv;
    }
  }
}

// Sampling key of each lm_head row: the request of the sequence holding the
// token row (sequences sorted by q_start) and the position being generated.
__global__ void row_keys_kernel(const SeqInfo* __restrict__ seqs, int S, const int32_t* __restrict__ positions,
                                const int32_t* __restrict__ logit_rows, int R, int32_t* __restrict__ key_req,
                                int32_t* __restrict__ key_pos) {
  grid_dep_sync();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= R) return;
  const int t = logit_rows ? logit_rows[i] : i;
  int lo = 0, hi = S - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (seqs[mid].q_start <= t) lo = mid; else hi = mid - 1;
  }
  key_req[i] = seqs[lo].request;
  key_pos[i] = positions[t] + 1;
}

// Per-row KV destination (same addressing as rope_scatter_kernel).
__global__ void kv_rows_kernel(const SeqInfo* __restrict__ seqs, int S, const int32_t* __restrict__ positions,
                               int M, KvLayout kv, int64_t* __restrict__ dst, int32_t* __restrict__ info) {
  grid_dep_sync();
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= M) return;
  int lo = 0, hi = S - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (seqs[mid].q_start <= t) lo = mid; else hi = mid - 1;
  }
  const SeqInfo sq = seqs[lo];
  const int j = t - sq.q_start;
  if (j < 0 || j >= sq.q_len) {
    info[t] = -1;
    dst[t] = 0;
    return;
  }
  const int hd = kv.head_dim, nkv = kv.kv_heads;
  if (sq.branch < 0) {
    const int pos = positions[t];
    SR_DCHECK(pos >= 0 && pos / kv.page < kv.max_pages);
    const int page = kv.block_table[(int64_t)sq.request * kv.max_pages + pos / kv.page];
    SR_DCHECK(page >= 0 && page < kv.num_pages);
    dst[t] = (int64_t)page * 2 * nkv * kv.page * hd;
    info[t] = pos % kv.page;
  } else {
    dst[t] = (int64_t)sq.branch * 2 * nkv * kv.window_max * hd;
    info[t] = j | (1 << 16);
  }
}

}  // namespace

int kv_rows(const SeqInfo* seqs, int S, const int32_t* positions, int M, const KvLayout& kv, int64_t* dst,
            int32_t* info, cudaStream_t s) {
  if (M == 0) return SR_OK;
  if (S == 0) return config_error("kv_rows: no sequences");
  sr::launch_k(kv_rows_kernel, ceil_div(M, 256), 256, 0, s, seqs, S, positions, M, kv, dst, info);
  return check_launch("kv_rows_kernel");
}

int sample_rows(const float* logits, int M, int V, int ld, const int32_t* req, const int32_t* pos, uint32_t seed,
                float inv_temp, int32_t* ids, float* vals, cudaStream_t s) {
  if (M == 0) return SR_OK;
  sr::launch_k(sample_rows_kernel, M, 512, 0, s, logits, V, ld, req, pos, seed, inv_temp, ids, vals);
  return check_launch("sample_rows_kernel");
}

int row_keys(const SeqInfo* seqs, int S, const int32_t* positions, const int32_t* logit_rows, int R,
             int32_t* key_req, int32_t* key_pos, cudaStream_t s) {
  if (R == 0 || S == 0) return SR_OK;
  sr::launch_k(row_keys_kernel, ceil_div(R, 256), 256, 0, s, seqs, S, positions, logit_rows, R, key_req, key_pos);
  return check_launch("row_keys_kernel");
}

// Producer side of the fused RMSNorm for rows that do not come out of a
// residual GEMM (the embedding): h = bf16(x o w), ssq[row] = {sum x^2, 0, ...}
// over `parts` slots, the layout the consuming GEMM sums (gemm.cuh NormArgs).
__global__ void __launch_bounds__(256)
norm_prep_kernel(const float* __restrict__ x, const float* __restrict__ w, int M, int H, int parts,
                 __nv_bfloat16* __restrict__ h, float* __restrict__ ssq) {
  grid_dep_sync();
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= M) return;
  const float* xr = x + (int64_t)row * H;
  __nv_bfloat16* hr = h + (int64_t)row * H;
  float ss = 0.0f;
  for (int i = lane; i < H; i += 32) {
    const float v = xr[i];
    ss = fmaf(v, v, ss);
    hr[i] = __float2bfloat16_rn(v * w[i]);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  for (int t = lane; t < parts; t += 32) ssq[(int64_t)row * parts + t] = t == 0 ? ss : 0.0f;
}

int norm_prep_rows(const float* x, const float* w, int M, int H, int parts, __nv_bfloat16* h, float* ssq,
                   cudaStream_t s) {
  if (M == 0) return SR_OK;
  sr::launch_k(norm_prep_kernel, ceil_div(M, 8), 256, 0, s, x, w, M, H, parts, h, ssq);
  return check_launch("norm_prep_kernel");
}

template <typename T>
int embed_rows(const T* table, const int32_t* ids, int M, int H, int vocab, float* x, cudaStream_t s) {
  if (M == 0) return SR_OK;
  sr::launch_k(embed_kernel<T>, M, 256, 0, s, table, ids, H, vocab, x);
  return check_launch("embed_kernel");
}

template <typename T>
int rmsnorm_rows(const float* x, const float* w, int M, int H, float eps, T* out, cudaStream_t s) {
  if (M == 0) return SR_OK;
  sr::launch_k(rmsnorm_kernel<T>, ceil_div(M, 8), 256, 0, s, x, w, M, H, eps, out);
  return check_launch("rmsnorm_kernel");
}

template <typename T>
int rope_scatter(const T* qkv, const int32_t* positions, const SeqInfo* seqs, int num_seqs,
                 int max_q_len, const float* cos_t, const float* sin_t, int nq, int layer,
                 const KvLayout& kv, T* q_out, cudaStream_t s) {
  if (num_seqs == 0 || max_q_len == 0) return SR_OK;
  dim3 grid(max_q_len, num_seqs);
  sr::launch_k(rope_scatter_kernel<T>, grid, 128, 0, s, qkv, positions, seqs, cos_t, sin_t, nq, layer, kv, q_out);
  return check_launch("rope_scatter_kernel");
}

int argmax_reduce(const float* pv, const int32_t* pi, int M, int tiles, int32_t* ids, float* vals,
                  cudaStream_t s) {
  if (M == 0) return SR_OK;
  sr::launch_k(argmax_reduce_kernel, ceil_div(M, 8), 256, 0, s, pv, pi, M, tiles, ids, vals);
  return check_launch("argmax_reduce_kernel");
}

int argmax_rows(const float* logits, int M, int V, int ld, int32_t* ids, float* vals, cudaStream_t s) {
  if (M == 0) return SR_OK;
  sr::launch_k(argmax_rows_kernel, M, 512, 0, s, logits, V, ld, ids, vals);
  return check_launch("argmax_rows_kernel");
}

template int embed_rows<float>(const float*, const int32_t*, int, int, int, float*, cudaStream_t);
template int embed_rows<__nv_bfloat16>(const __nv_bfloat16*, const int32_t*, int, int, int, float*, cudaStream_t);
template int rmsnorm_rows<float>(const float*, const float*, int, int, float, float*, cudaStream_t);
template int rmsnorm_rows<__nv_bfloat16>(const float*, const float*, int, int, float, __nv_bfloat16*, cudaStream_t);
template int rope_scatter<float>(const float*, const int32_t*, const SeqInfo*, int, int, const float*,
                                 const float*, int, int, const KvLayout&, float*, cudaStream_t);
template int rope_scatter<__nv_bfloat16>(const __nv_bfloat16*, const int32_t*, const SeqInfo*, int, int,
                                         const float*, const float*, int, int, const KvLayout&,
                                         __nv_bfloat16*, cudaStream_t);

}  // namespace sr
