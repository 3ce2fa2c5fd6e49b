// Small fused ops of the verify forward (K6): embedding gather, RMSNorm,
// RoPE + KV scatter into the paged cache / drafter-branch window buffers,
// vocabulary argmax reduction.  All are HBM-bound elementwise/row kernels;
// each row's arithmetic order is fixed so results are batch invariant.
#pragma once
#include <cuda_bf16.h>
#include <cstdint>

namespace sr {

// Per-sequence descriptor of a verify/prefill/decode batch (device, int32 x 8).
struct SeqInfo {  // same layout as sr_seq_info
  int32_t q_start;   // first token row of this sequence in the batch
  int32_t q_len;     // window positions (k+1 for verify, 1 for decode, P for prefill)
  int32_t request;   // row in block_table / token buffers
  int32_t ctx_len;   // keys already in the paged cache (positions [0, ctx_len))
  int32_t branch;    // -1: window KV goes straight to the paged cache;
                     // >= 0: drafter-branch slot in the window buffer
  int32_t pad0, pad1, pad2;
};

struct KvLayout {
  void* cache;              // [layers, pages, 2, kv_heads, page, head_dim]
  const int32_t* block_table;  // [requests, max_pages]
  int max_pages;
  int page;                 // tokens per page
  int num_pages;
  void* window;             // [layers, branches, 2, kv_heads, window_max, head_dim]
  int window_max;
  int branches;
  int kv_heads, head_dim, layers;

  __host__ __device__ int64_t cache_layer_elems() const {
    return (int64_t)num_pages * 2 * kv_heads * page * head_dim;
  }
  __host__ __device__ int64_t window_layer_elems() const {
    return (int64_t)branches * 2 * kv_heads * window_max * head_dim;
  }
};

// bf16 KV rows (paged cache and branch windows) keep their 16-byte chunks
// XOR-swizzled by (slot & 7): a 64-slot page then streams into shared memory
// with one bulk copy already in the bank-conflict-free layout ldmatrix reads.
// fp32 (parity path) rows stay plain.
template <typename T>
__host__ __device__ __forceinline__ int kv_phys(int slot, int d) {
  if constexpr (sizeof(T) == 2) return ((((d >> 3) ^ (slot & 7))) << 3) | (d & 7);
  else return d;
}

template <typename T>
int embed_rows(const T* table, const int32_t* ids, int M, int H, int vocab, float* x, cudaStream_t s);

int norm_prep_rows(const float* x, const float* w, int M, int H, int parts, __nv_bfloat16* h, float* ssq,
                   cudaStream_t s);
template <typename T>
int rmsnorm_rows(const float* x, const float* w, int M, int H, float eps, T* out, cudaStream_t s);

// qkv [M, (nq + 2 nkv) * hd] -> rotated q [M, nq*hd]; rotated k and v into the
// paged cache (branch < 0) or the branch's window slot.
template <typename T>
int rope_scatter(const T* qkv, const int32_t* positions, const SeqInfo* seqs, int num_seqs,
                 int max_q_len, const float* cos_t, const float* sin_t, int nq, int layer,
                 const KvLayout& kv, T* q_out, cudaStream_t s);

// Reduce argmax partials [M, tiles] (value, index) -> ids [M] (+ max value).
int argmax_reduce(const float* part_val, const int32_t* part_idx, int M, int tiles,
                  int32_t* out_ids, float* out_val, cudaStream_t s);

// Keyed Gumbel-max sample of fp32 logit rows (sampling.cuh); req/pos per row.
int sample_rows(const float* logits, int M, int V, int ld, const int32_t* req, const int32_t* pos, uint32_t seed,
                float inv_temp, int32_t* ids, float* vals, cudaStream_t s);

// (request, generated position) of each lm_head row, from sorted SeqInfo.
int row_keys(const SeqInfo* seqs, int S, const int32_t* positions, const int32_t* logit_rows, int R,
             int32_t* key_req, int32_t* key_pos, cudaStream_t s);

// KV destination of every token row for the fused qkv + RoPE epilogue
// (gemm.cuh RopeArgs): dst[t] = element offset of the row's K block inside a
// layer's cache / window, info[t] = slot | window << 16; rows [0, M) not in a
// sequence get info -1.
int kv_rows(const SeqInfo* seqs, int S, const int32_t* positions, int M, const KvLayout& kv, int64_t* dst,
            int32_t* info, cudaStream_t s);

// Full-row argmax over fp32 logits [M, V] (lowest index on ties).
int argmax_rows(const float* logits, int M, int V, int ld, int32_t* out_ids, float* out_val,
                cudaStream_t s);

}  // namespace sr
