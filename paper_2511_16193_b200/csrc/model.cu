// Verification forward of the target model (K1 + K2 + K6), C++ runtime.
//
// `sr_model_create` takes device pointers to weights, the paged KV cache and
// a caller-owned workspace, builds every GEMM plan (TMA tensor maps) once,
// and `sr_model_forward` enqueues the whole Qwen2-style decoder on one
// stream with no host synchronization and no allocation, so a step can be
// captured in a CUDA graph.  Layer sequence (per layer):
//
//   h   = RMSNorm(x) * ln1                       rmsnorm_rows
//   qkv = h Wqkv^T + b                           tcgen05 GEMM, bias epilogue
//   q,k,v -> RoPE, k/v into paged cache/window   rope_scatter
//   o   = attention(q, cache)                    paged GQA attention
//   x  += o Wo^T                                 GEMM, residual epilogue
//   h   = RMSNorm(x) * ln2
//   a   = silu(h Wg^T) * (h Wu^T)                GEMM, SwiGLU epilogue
//   x  += a Wd^T                                 GEMM, residual epilogue
//
// then the final norm and the lm_head GEMM with a fused vocabulary argmax
// epilogue (logits never reach HBM) or an fp32 logits epilogue.
#include "common.cuh"

#include <cstdlib>
#include "gemm.cuh"
#include "layers.cuh"

#include <cuda_bf16.h>
#include <new>
#include <vector>

namespace sr {

size_t attention_workspace_floats(int max_seqs, int max_tokens, int G, int kv_heads, int max_key, int hd);
int attention_bf16(const __nv_bfloat16* q, const SeqInfo* seqs, int num_seqs, int max_q_len, int max_key,
                   const KvLayout& kv, int layer, int nq, float* partials, size_t partial_floats,
                   __nv_bfloat16* out, cudaStream_t stream, int phase, bool plan);
int attention_f32(const float* q, const SeqInfo* seqs, int num_seqs, int max_q_len, const KvLayout& kv,
                  int layer, int nq, float* out, cudaStream_t stream);

namespace {

constexpr int kLayerPtrs = 7;  // ln1, w_qkv, b_qkv, w_o, ln2, w_gu, w_down
constexpr int kLmBn = 64;  // smallest lm_head tile width: sizes the argmax partials
constexpr int kNarrowRows = 256;  // launches up to this many rows use the narrow plans

__global__ void gather_rows_kernel(const void* __restrict__ src, const int32_t* __restrict__ rows, int H,
                                   int esize, void* __restrict__ dst) {
  grid_dep_sync();
  const int r = blockIdx.x;
  const char* s = reinterpret_cast<const char*>(src) + (int64_t)rows[r] * H * esize;
  char* d = reinterpret_cast<char*>(dst) + (int64_t)r * H * esize;
  for (int i = threadIdx.x * 4; i < H * esize; i += blockDim.x * 4)
    *reinterpret_cast<uint32_t*>(d + i) = *reinterpret_cast<const uint32_t*>(s + i);
}

struct Carve {
  char* base;
  size_t off = 0;
  template <typename T>
  T* take(size_t count) {
    off = (off + 255) & ~size_t(255);
    T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
    off += count * sizeof(T);
    return p;
  }
};

}  // namespace

// Per-category CUDA-event timing of the forward's launches (bench.py's
// roofline evidence): events bracket each launch on the launching stream.
enum ProfCat { kProfQkv, kProfO, kProfGateUp, kProfDown, kProfLmHead, kProfAttn, kProfOther, kProfCombine,
               kProfCats };

struct Profiler {
  bool on = false;
  std::vector<cudaEvent_t> pool;
  std::vector<std::pair<int, int>> marks;  // (category, first event index)
  size_t next = 0;
  cudaEvent_t take() {
    if (next == pool.size()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      pool.push_back(e);
    }
    return pool[next++];
  }
  // Inside stream capture the record must be an *external* event node, or
  // the replayed graph would not time it.
  static void record(cudaEvent_t e, cudaStream_t st) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(st, &cs);
    if (cs == cudaStreamCaptureStatusActive) cudaEventRecordWithFlags(e, st, cudaEventRecordExternal);
    else cudaEventRecord(e, st);
  }
  void begin(int cat, cudaStream_t st) {
    if (!on) return;
    marks.push_back({cat, (int)next});
    record(take(), st);
  }
  void end(cudaStream_t st) {
    if (!on) return;
    record(take(), st);
  }
  ~Profiler() {
    for (auto e : pool) cudaEventDestroy(e);
  }
};

struct Model {
  Profiler prof;
  sr_model_desc d;
  std::vector<const void*> layer_ptrs;
  KvLayout kv;
  int esize;
  int qkv_width;
  int lm_tiles;
  size_t partial_floats;
  // workspace views
  float* x;
  void* h;
  void* qkv;
  void* q;
  void* attn;
  void* act;
  void* h_sel;
  float* logits;       // only when desc.logits_capacity > 0
  float* part_val;
  int32_t* part_idx;
  float* attn_part;
  int32_t* key_req;    // sampling keys of the lm_head rows
  int32_t* key_pos;
  float* ssq;          // fused RMSNorm partial sums of x^2 [T, parts] (bf16 path)
  float* ssq_sel;      // the same for the gathered lm_head rows
  float* swap_ws;      // small-M GEMM mode: fp32 K-range partials
  SwapMaps* swap_maps; // and its tensor maps (device copies, [plan set][layer][qkv, o, gate_up, down])
  int32_t* swap_cnt;   // and its arrival counters (zeroed at create, self-resetting)
  size_t swap_cnt_ints;
  int64_t* kv_dst;     // per token row: KV destination for the fused qkv + RoPE epilogue
  int32_t* kv_info;
  int prep_parts;      // slots the embedding-side norm prep writes (= qkv[0]'s consumer count)
  int lm_parts;        // partial slots behind the lm_head rows (last down's N tiles)
  // plans (bf16); *_sel read the gathered rows (h_sel, ssq_sel)
  std::vector<GemmPlan> p_qkv, p_o, p_gu, p_down;
  // launches of <= kNarrowRows rows (decode, drafter steps) take plans made
  // for that size: narrower tiles over more SMs.  A row's bits do not depend
  // on the tile width (nor on the mode), only on the K ranges, which both
  // plans share.
  bool narrow = false;
  std::vector<GemmPlan> n_qkv, n_o, n_gu, n_down;
  GemmPlan p_lm_argmax, p_lm_logits, p_lm_argmax_sel, p_lm_logits_sel;
};

static size_t carve(const sr_model_desc& d, Model* m, char* base) {
  Carve c{base};
  const int T = d.max_tokens, H = d.hidden;
  const int esize = d.dtype == 1 ? 2 : 4;
  const int qkv_w = (d.q_heads + 2 * d.kv_heads) * d.head_dim;
  const int G = d.q_heads / d.kv_heads;
  const int lm_tiles = (d.vocab + kLmBn - 1) / kLmBn;
  const size_t pf = attention_workspace_floats(d.max_seqs, T, G, d.kv_heads, d.max_key, d.head_dim);
  float* x = c.take<float>((size_t)T * H);
  char* h = c.take<char>((size_t)T * H * esize);
  char* qkv = c.take<char>((size_t)T * qkv_w * esize);
  char* q = c.take<char>((size_t)T * d.q_heads * d.head_dim * esize);
  char* attn = c.take<char>((size_t)T * d.q_heads * d.head_dim * esize);
  char* act = c.take<char>((size_t)T * d.intermediate * esize);
  char* h_sel = c.take<char>((size_t)T * H * esize);
  const int vpad = (d.vocab + 7) / 8 * 8;  // 16-byte aligned logit rows
  float* logits = d.logits_capacity > 0 ? c.take<float>((size_t)d.logits_capacity * vpad) : nullptr;
  float* pv = c.take<float>((size_t)T * lm_tiles);
  int32_t* pi = c.take<int32_t>((size_t)T * lm_tiles);
  float* ap = c.take<float>(d.dtype == 1 ? pf : 0);
  int32_t* kr = c.take<int32_t>((size_t)T);
  int32_t* kp = c.take<int32_t>((size_t)T);
  const int max_parts = (H + kSsqCols - 1) / kSsqCols;  // RMSNorm partials per row
  float* ssq = c.take<float>(d.dtype == 1 ? (size_t)T * max_parts : 0);
  float* ssq_sel = c.take<float>(d.dtype == 1 ? (size_t)T * max_parts : 0);
  int64_t* kv_dst = c.take<int64_t>(d.dtype == 1 ? (size_t)T : 0);
  int32_t* kv_info = c.take<int32_t>(d.dtype == 1 ? (size_t)T : 0);
  // small-M mode partials / counters of the qkv, o and down projections
  size_t swf = 0, swc = 0;
  if (d.dtype == 1) {
    const int nqd = d.q_heads * d.head_dim;
    const int shp[4][3] = {{qkv_w, H, kEpiQkvRope}, {H, nqd, kEpiResidualNorm}, {2 * d.intermediate, H, kEpiSwiGLU},
                           {H, d.intermediate, kEpiResidualNorm}};
    for (auto& g : shp) {
      const int sp = gemm_splits(g[0], g[1], g[2]);
      const size_t f = sp > 1 ? (size_t)sp * kSwapRows * g[0] : 0, cn = (size_t)2 * ((g[0] + 255) / 256);
      swf = f > swf ? f : swf;
      swc = cn > swc ? cn : swc;
    }
  }
  float* sw_ws = c.take<float>(swf);
  int32_t* sw_cnt = c.take<int32_t>(swc);
  // device copies of the qkv / o / down plans' small-M tensor maps (64-byte aligned)
  SwapMaps* sw_maps = d.dtype == 1 ? c.take<SwapMaps>((size_t)8 * d.layers) : nullptr;
  if (m != nullptr) {
    m->swap_ws = sw_ws; m->swap_cnt = sw_cnt; m->swap_cnt_ints = swc; m->swap_maps = sw_maps;
    m->x = x; m->h = h; m->qkv = qkv; m->q = q; m->attn = attn; m->act = act; m->h_sel = h_sel;
    m->logits = logits; m->part_val = pv; m->part_idx = pi; m->attn_part = ap;
    m->key_req = kr; m->key_pos = kp;
    m->ssq = ssq; m->ssq_sel = ssq_sel;
    m->kv_dst = kv_dst; m->kv_info = kv_info;
    m->esize = esize; m->qkv_width = qkv_w; m->lm_tiles = lm_tiles;
    m->partial_floats = d.dtype == 1 ? pf : 0;
  }
  return c.off + 256;
}

static int validate(const sr_model_desc& d) {
  SR_REQUIRE(d.dtype == 0 || d.dtype == 1, "dtype must be 0 (fp32) or 1 (bf16)");
  SR_REQUIRE(d.hidden > 0 && d.intermediate > 0 && d.layers > 0 && d.vocab > 0, "bad model shape");
  SR_REQUIRE(d.q_heads > 0 && d.kv_heads > 0 && d.q_heads % d.kv_heads == 0, "q_heads % kv_heads != 0");
  SR_REQUIRE(d.head_dim % 16 == 0 && d.head_dim <= 128, "head_dim must be a multiple of 16, <= 128");
  SR_REQUIRE(d.dtype == 0 || d.head_dim % 32 == 0, "bf16 models need head_dim % 32 == 0 (fused RoPE)");
  SR_REQUIRE(d.intermediate % 16 == 0, "intermediate must be a multiple of 16");
  SR_REQUIRE(d.page_size == 64, "page_size must be 64");
  SR_REQUIRE(d.max_tokens > 0 && d.max_seqs > 0, "max_tokens / max_seqs must be > 0");
  SR_REQUIRE(d.max_key < d.max_pos, "max_key must be < max_pos (RoPE table)");
  SR_REQUIRE(d.q_heads / d.kv_heads * 1 <= 64, "group size too large");
  return SR_OK;
}

int model_kv_layout(void* handle, KvLayout* kv, int* dtype) {
  SR_REQUIRE(handle && kv && dtype, "null model");
  const Model* m = reinterpret_cast<const Model*>(handle);
  *kv = m->kv;
  *dtype = m->d.dtype;
  return SR_OK;
}

}  // namespace sr

using sr::Model;

extern "C" {

uint64_t sr_model_workspace_bytes(const sr_model_desc* desc) {
  if (desc == nullptr || sr::validate(*desc) != SR_OK) return 0;
  return (uint64_t)sr::carve(*desc, nullptr, nullptr);
}

int sr_model_create(const sr_model_desc* desc, void** handle) {
  SR_REQUIRE(desc && handle, "null pointer");
  int rc = sr::validate(*desc);
  if (rc) return rc;
  const sr_model_desc& d = *desc;
  SR_REQUIRE(d.embed && d.lm_head && d.final_norm && d.layer_weights && d.rope_cos && d.rope_sin &&
                 d.kv_cache && d.block_table && d.workspace,
             "null model pointer");
  const size_t need = sr::carve(d, nullptr, nullptr);
  SR_REQUIRE(d.workspace_bytes >= need, "workspace too small (see sr_model_workspace_bytes)");
  Model* m = new (std::nothrow) Model();
  if (m == nullptr) return sr::config_error("out of host memory");
  m->d = d;
  m->layer_ptrs.assign(d.layer_weights, d.layer_weights + (size_t)d.layers * sr::kLayerPtrs);
  m->d.layer_weights = m->layer_ptrs.data();
  sr::carve(d, m, reinterpret_cast<char*>(d.workspace));
  sr::KvLayout& kv = m->kv;
  kv.cache = d.kv_cache;
  kv.block_table = d.block_table;
  kv.max_pages = d.max_pages_per_req;
  kv.page = d.page_size;
  kv.num_pages = d.num_pages;
  kv.window = d.window_kv;
  kv.window_max = d.window_max;
  kv.branches = d.max_branches;
  kv.kv_heads = d.kv_heads;
  kv.head_dim = d.head_dim;
  kv.layers = d.layers;
  if (d.dtype == 1) {
    using bf = __nv_bfloat16;
    const int T = d.max_tokens, H = d.hidden, I = d.intermediate;
    const int nqd = d.q_heads * d.head_dim;
    m->p_qkv.resize(d.layers);
    m->p_o.resize(d.layers);
    m->p_gu.resize(d.layers);
    m->p_down.resize(d.layers);
    for (int l = 0; l < d.layers; ++l) {
      const void* const* w = m->layer_ptrs.data() + (size_t)l * sr::kLayerPtrs;
      // SR_QKV_BN (measurement knob): explicit pair tile width of the qkv plan
      static const int qkv_bn = [] {
        const char* v = getenv("SR_QKV_BN");
        return v ? -atoi(v) : 0;
      }();
      rc = sr::gemm_bf16_plan(&m->p_qkv[l], T, m->qkv_width, H, (const bf*)m->h, H, (const bf*)w[1], H,
                              m->qkv, m->qkv_width, sr::kEpiQkvRope, (const float*)w[2], qkv_bn);
      if (!rc) {
        sr::RopeArgs& ra = m->p_qkv[l].rope;
        ra.kv_dst = m->kv_dst;
        ra.kv_info = m->kv_info;
        ra.cos = d.rope_cos;
        ra.sin = d.rope_sin;
        ra.q_out = (bf*)m->q;
        ra.cache = (bf*)d.kv_cache + l * kv.cache_layer_elems();
        ra.window = d.window_kv ? (bf*)d.window_kv + l * kv.window_layer_elems() : nullptr;
        ra.nq = d.q_heads;
        ra.nkv = d.kv_heads;
        ra.hd = d.head_dim;
        ra.page = d.page_size;
        ra.window_max = d.window_max;
      }
      if (!rc) rc = sr::gemm_bf16_plan(&m->p_o[l], T, H, nqd, (const bf*)m->attn, nqd, (const bf*)w[3], nqd,
                                       m->x, H, sr::kEpiResidualNorm, nullptr, 0);
      if (!rc) rc = sr::gemm_bf16_plan(&m->p_gu[l], T, 2 * I, H, (const bf*)m->h, H, (const bf*)w[5], H,
                                       m->act, I, sr::kEpiSwiGLU, nullptr, 0);
      if (!rc) rc = sr::gemm_bf16_plan(&m->p_down[l], T, H, I, (const bf*)m->act, I, (const bf*)w[6], I,
                                       m->x, H, sr::kEpiResidualNorm, nullptr, 0);
      if (rc) { delete m; return rc; }
      int j = 0;
      for (sr::GemmPlan* gp : {&m->p_qkv[l], &m->p_o[l], &m->p_gu[l], &m->p_down[l]}) {
        gp->sw.ws = m->swap_ws;
        gp->sw.cnt = m->swap_cnt;
        if (sr::gemm_swap_ws_floats(*gp) > 0 && m->swap_ws == nullptr) rc = sr::config_error("swap workspace");
        if (gp->sw.max_m > 0) {
          sr::SwapMaps* dst = m->swap_maps + 4 * l + j;
          if (cudaMemcpy(dst, &gp->sw_maps, sizeof(sr::SwapMaps), cudaMemcpyHostToDevice) != cudaSuccess)
            rc = sr::config_error("cannot upload the GEMM tensor maps");
          gp->sw.maps = dst;
        }
        ++j;
      }
      if (rc) { delete m; return rc; }
    }
    if (m->swap_cnt_ints > 0 && cudaMemset(m->swap_cnt, 0, m->swap_cnt_ints * sizeof(int32_t)) != cudaSuccess) {
      delete m;
      return sr::config_error("cannot zero the GEMM counters");
    }
    for (int sel = 0; sel < 2 && !rc; ++sel) {
      const bf* a_in = (const bf*)(sel ? m->h_sel : m->h);
      rc = sr::gemm_bf16_plan(sel ? &m->p_lm_argmax_sel : &m->p_lm_argmax, T, d.vocab, H, a_in, H,
                              (const bf*)d.lm_head, H, m->part_val, m->lm_tiles, sr::kEpiArgmax, nullptr, 0,
                              m->part_idx);
      if (!rc && m->logits)
        rc = sr::gemm_bf16_plan(sel ? &m->p_lm_logits_sel : &m->p_lm_logits, T, d.vocab, H, a_in, H,
                                (const bf*)d.lm_head, H, m->logits, (d.vocab + 7) / 8 * 8, sr::kEpiStoreF32,
                                nullptr, 0);
    }
    // the logits lm_head (parity / rejection-sampling output) keeps the
    // large-M mode: a vocabulary-wide N already spreads over every SM
    m->p_lm_logits.sw.max_m = 0;
    m->p_lm_logits_sel.sw.max_m = 0;
    if (!rc) m->lm_tiles = sr::gemm_num_n_tiles(d.vocab, m->p_lm_argmax.bn);
    if (rc) { delete m; return rc; }
    // Fused RMSNorm wiring: o / down write bf16(x o w_next) + partials; qkv /
    // gate_up / lm_head scale rows by r from the producer's partials.
    auto producer = [&](sr::GemmPlan& p, const float* wn) {
      p.norm.h_out = (bf*)m->h;
      p.norm.w = wn;
      p.norm.ssq_out = m->ssq;
      p.norm.ld_h = H;
      return (H + sr::kSsqCols - 1) / sr::kSsqCols;
    };
    auto consumer = [&](sr::GemmPlan& p, const float* ssq, int parts) {
      p.norm.ssq_in = ssq;
      p.norm.parts_in = parts;
      p.norm.hdim = (float)H;
      p.norm.eps = d.rms_eps;
    };
    int parts = m->prep_parts = (H + sr::kSsqCols - 1) / sr::kSsqCols;
    for (int l = 0; l < d.layers; ++l) {
      const void* const* w = m->layer_ptrs.data() + (size_t)l * sr::kLayerPtrs;
      const void* const* wn = l + 1 < d.layers ? w + sr::kLayerPtrs : nullptr;
      consumer(m->p_qkv[l], m->ssq, parts);
      const int po = producer(m->p_o[l], (const float*)w[4]);
      consumer(m->p_gu[l], m->ssq, po);
      parts = producer(m->p_down[l], wn ? (const float*)wn[0] : d.final_norm);
    }
    consumer(m->p_lm_argmax, m->ssq, parts);
    consumer(m->p_lm_logits, m->ssq, parts);
    consumer(m->p_lm_argmax_sel, m->ssq_sel, parts);
    consumer(m->p_lm_logits_sel, m->ssq_sel, parts);
    m->lm_parts = parts;
    // narrow plans (same operands, epilogue wiring and K ranges; tiles for <= kNarrowRows rows)
    m->narrow = T > sr::kNarrowRows;
    if (m->narrow) {
      m->n_qkv = m->p_qkv; m->n_o = m->p_o; m->n_gu = m->p_gu; m->n_down = m->p_down;
      for (int l = 0; l < d.layers && !rc; ++l) {
        const void* const* w = m->layer_ptrs.data() + (size_t)l * sr::kLayerPtrs;
        struct { sr::GemmPlan* big; sr::GemmPlan* nar; int N, K; const void* A; int lda; const void* W; int epi; } g[4] = {
            {&m->p_qkv[l], &m->n_qkv[l], m->qkv_width, H, m->h, H, w[1], sr::kEpiQkvRope},
            {&m->p_o[l], &m->n_o[l], H, nqd, m->attn, nqd, w[3], sr::kEpiResidualNorm},
            {&m->p_gu[l], &m->n_gu[l], 2 * I, H, m->h, H, w[5], sr::kEpiSwiGLU},
            {&m->p_down[l], &m->n_down[l], H, I, m->act, I, w[6], sr::kEpiResidualNorm}};
        for (int j = 0; j < 4 && !rc; ++j) {
          sr::GemmPlan np;
          rc = sr::gemm_bf16_plan(&np, sr::kNarrowRows, g[j].N, g[j].K, (const bf*)g[j].A, g[j].lda, (const bf*)g[j].W,
                                  g[j].K, g[j].big->c, g[j].big->ldc, g[j].epi, g[j].big->bias, 0, g[j].big->aux);
          if (rc) break;
          if (np.sw.splits != g[j].big->sw.splits) { rc = sr::config_error("narrow plan K ranges differ"); break; }
          np.norm = g[j].big->norm;
          np.rope = g[j].big->rope;
          np.sw.ws = g[j].big->sw.ws;
          np.sw.cnt = g[j].big->sw.cnt;
          if (np.sw.max_m > 0) {
            sr::SwapMaps* dst = m->swap_maps + 4 * (d.layers + l) + j;
            if (cudaMemcpy(dst, &np.sw_maps, sizeof(sr::SwapMaps), cudaMemcpyHostToDevice) != cudaSuccess)
              rc = sr::config_error("cannot upload the GEMM tensor maps");
            np.sw.maps = dst;
          }
          *g[j].nar = np;
        }
      }
      if (rc) { delete m; return rc; }
    }
  }
  *handle = m;
  return SR_OK;
}

int sr_model_destroy(void* handle) {
  delete reinterpret_cast<Model*>(handle);
  return SR_OK;
}

int sr_model_forward(void* handle, const sr_forward_args* a, sr_stream_t stream_) {
  SR_REQUIRE(handle && a, "null pointer");
  Model* m = reinterpret_cast<Model*>(handle);
  const sr_model_desc& d = m->d;
  cudaStream_t st = (cudaStream_t)stream_;
  const int M = a->num_tokens, S = a->num_seqs;
  SR_REQUIRE(M >= 0 && M <= d.max_tokens, "num_tokens exceeds max_tokens");
  SR_REQUIRE(S >= 0 && S <= d.max_seqs, "num_seqs exceeds max_seqs");
  SR_REQUIRE(a->max_key >= 0 && a->max_key <= d.max_key, "max_key exceeds the model's max_key");
  SR_REQUIRE(a->token_ids && a->positions && a->seqs && a->out, "null forward pointer");
  const int R = a->logit_rows ? a->num_logit_rows : M;
  SR_REQUIRE(R >= 0 && R <= d.max_tokens, "bad logit row count");
  SR_REQUIRE(a->output == 0 || (a->output == 1 && m->logits != nullptr && R <= d.logits_capacity) ||
                 a->output == 2,
             "logits output needs logits_capacity >= rows");
  SR_REQUIRE(a->output != 2 || a->temperature > 0.0f, "sampling needs temperature > 0");

  if (M == 0) return SR_OK;
  const auto* seqs = reinterpret_cast<const sr::SeqInfo*>(a->seqs);
  const sr::SampleArgs sample{m->key_req, m->key_pos, a->seed,
                              a->output == 2 ? 1.0f / a->temperature : 0.0f};
  const int H = d.hidden, I = d.intermediate, nqd = d.q_heads * d.head_dim;
  int rc;
#define SR_TRY(x) do { rc = (x); if (rc) return rc; } while (0)
  if (a->output == 2) SR_TRY(sr::row_keys(seqs, S, a->positions, a->logit_rows, R, m->key_req, m->key_pos, st));
  if (d.dtype == 1) {
    using bf = __nv_bfloat16;
    SR_TRY(sr::embed_rows<bf>((const bf*)d.embed, a->token_ids, M, H, d.vocab, m->x, st));
    // input norm of layer 0; every later norm is fused into the o / down GEMMs
    SR_TRY(sr::norm_prep_rows(m->x, (const float*)m->layer_ptrs[0], M, H, m->prep_parts, (bf*)m->h, m->ssq, st));
    // KV destination of every row, shared by all layers' qkv + RoPE epilogues
    SR_TRY(sr::kv_rows(seqs, S, a->positions, M, m->kv, m->kv_dst, m->kv_info, st));
    for (int l = 0; l < d.layers; ++l) {
      auto& P = m->prof;
      P.begin(sr::kProfQkv, st);
      const bool nar = m->narrow && M <= sr::kNarrowRows;
      sr::GemmPlan& pq = nar ? m->n_qkv[l] : m->p_qkv[l];
      sr::GemmPlan& po = nar ? m->n_o[l] : m->p_o[l];
      sr::GemmPlan& pg = nar ? m->n_gu[l] : m->p_gu[l];
      sr::GemmPlan& pd = nar ? m->n_down[l] : m->p_down[l];
      pq.rope.pos = a->positions;
      pq.m_live = a->live_rows;
      SR_TRY(sr::gemm_bf16_launch(pq, st, M));
      P.end(st);
      P.begin(sr::kProfAttn, st);
      SR_TRY(sr::attention_bf16((const bf*)m->q, seqs, S, a->max_q_len, a->max_key, m->kv, l, d.q_heads,
                                m->attn_part, m->partial_floats, (bf*)m->attn, st, 0, l == 0));
      P.end(st);
      P.begin(sr::kProfCombine, st);
      SR_TRY(sr::attention_bf16((const bf*)m->q, seqs, S, a->max_q_len, a->max_key, m->kv, l, d.q_heads,
                                m->attn_part, m->partial_floats, (bf*)m->attn, st, 1, false));
      P.end(st);
      P.begin(sr::kProfO, st);
      po.m_live = a->live_rows;
      SR_TRY(sr::gemm_bf16_launch(po, st, M));
      P.end(st);
      P.begin(sr::kProfGateUp, st);
      pg.m_live = a->live_rows;
      SR_TRY(sr::gemm_bf16_launch(pg, st, M));
      P.end(st);
      P.begin(sr::kProfDown, st);
      pd.m_live = a->live_rows;
      SR_TRY(sr::gemm_bf16_launch(pd, st, M));
      P.end(st);
    }
    // the last down GEMM left bf16(x o final_norm) in h and its partials in ssq
    const bool sel = a->logit_rows != nullptr;
    if (sel) {
      sr::launch_k(sr::gather_rows_kernel, R, 256, 0, st, m->h, a->logit_rows, H, 2, m->h_sel);
      SR_TRY(sr::check_launch("gather_rows_kernel"));
      sr::launch_k(sr::gather_rows_kernel, R, 256, 0, st, (const void*)m->ssq, a->logit_rows, m->lm_parts, 4,
                   (void*)m->ssq_sel);
      SR_TRY(sr::check_launch("gather_rows_kernel"));
    }
    if (a->output == 1) {
      sr::GemmPlan& lmp = sel ? m->p_lm_logits_sel : m->p_lm_logits;
      lmp.m_live = sel ? nullptr : a->live_rows;
      SR_TRY(sr::gemm_bf16_launch(lmp, st, R));
      const size_t vpad = (size_t)(d.vocab + 7) / 8 * 8;
      SR_CHECK_CUDA(cudaMemcpy2DAsync(a->out, (size_t)d.vocab * 4, m->logits, vpad * 4, (size_t)d.vocab * 4, R,
                                      cudaMemcpyDeviceToDevice, st));
    } else {
      m->prof.begin(sr::kProfLmHead, st);
      sr::GemmPlan& lm = sel ? m->p_lm_argmax_sel : m->p_lm_argmax;
      lm.sample = sample;
      lm.m_live = sel ? nullptr : a->live_rows;
      SR_TRY(sr::gemm_bf16_launch(lm, st, R));
      m->prof.end(st);
      m->prof.begin(sr::kProfOther, st);
      SR_TRY(sr::argmax_reduce(m->part_val, m->part_idx, R, m->lm_tiles, (int32_t*)a->out, a->out_val, st));
      m->prof.end(st);
    }
  } else {
    SR_TRY(sr::embed_rows<float>((const float*)d.embed, a->token_ids, M, H, d.vocab, m->x, st));
    for (int l = 0; l < d.layers; ++l) {
      const void* const* w = m->layer_ptrs.data() + (size_t)l * sr::kLayerPtrs;
      float* h = (float*)m->h;
      SR_TRY(sr::rmsnorm_rows<float>(m->x, (const float*)w[0], M, H, d.rms_eps, h, st));
      SR_TRY(sr::gemm_f32(M, m->qkv_width, H, h, H, (const float*)w[1], H, m->qkv, m->qkv_width,
                          sr::kEpiStoreF32, (const float*)w[2], st));
      SR_TRY(sr::rope_scatter<float>((const float*)m->qkv, a->positions, seqs, S, a->max_q_len, d.rope_cos,
                                     d.rope_sin, d.q_heads, l, m->kv, (float*)m->q, st));
      SR_TRY(sr::attention_f32((const float*)m->q, seqs, S, a->max_q_len, m->kv, l, d.q_heads,
                               (float*)m->attn, st));
      SR_TRY(sr::gemm_f32(M, H, nqd, (const float*)m->attn, nqd, (const float*)w[3], nqd, m->x, H,
                          sr::kEpiResidualF32, nullptr, st));
      SR_TRY(sr::rmsnorm_rows<float>(m->x, (const float*)w[4], M, H, d.rms_eps, h, st));
      SR_TRY(sr::gemm_f32(M, 2 * I, H, h, H, (const float*)w[5], H, m->act, I, sr::kEpiSwiGLU, nullptr, st));
      SR_TRY(sr::gemm_f32(M, H, I, (const float*)m->act, I, (const float*)w[6], I, m->x, H,
                          sr::kEpiResidualF32, nullptr, st));
    }
    SR_TRY(sr::rmsnorm_rows<float>(m->x, d.final_norm, M, H, d.rms_eps, (float*)m->h, st));
    if (a->logit_rows) {
      sr::launch_k(sr::gather_rows_kernel, R, 256, 0, st, m->h, a->logit_rows, H, 4, m->h_sel);
      SR_TRY(sr::check_launch("gather_rows_kernel"));
    } else {
      SR_CHECK_CUDA(cudaMemcpyAsync(m->h_sel, m->h, (size_t)M * H * 4, cudaMemcpyDeviceToDevice, st));
    }
    float* logits = a->output == 1 ? (float*)a->out : m->logits;
    SR_REQUIRE(logits != nullptr && R <= (a->output == 1 ? d.max_tokens : d.logits_capacity),
               "fp32 path needs logits_capacity >= rows for argmax");
    SR_TRY(sr::gemm_f32(R, d.vocab, H, (const float*)m->h_sel, H, (const float*)d.lm_head, H, logits, d.vocab,
                        sr::kEpiStoreF32, nullptr, st));
    if (a->output == 0) SR_TRY(sr::argmax_rows(logits, R, d.vocab, d.vocab, (int32_t*)a->out, a->out_val, st));
    if (a->output == 2)
      SR_TRY(sr::sample_rows(logits, R, d.vocab, d.vocab, m->key_req, m->key_pos, a->seed, sample.inv_temp,
                             (int32_t*)a->out, a->out_val, st));
  }
#undef SR_TRY
  return SR_OK;
}

int sr_model_profile(void* handle, int enable, float* ms_out, int32_t* count_out) {
  SR_REQUIRE(handle, "null model");
  Model* m = reinterpret_cast<Model*>(handle);
  auto& P = m->prof;
  if (ms_out || count_out) {
    for (int c = 0; c < sr::kProfCats; ++c) {
      if (ms_out) ms_out[c] = 0.0f;
      if (count_out) count_out[c] = 0;
    }
    if (!P.marks.empty()) SR_CHECK_CUDA(cudaEventSynchronize(P.pool[P.next - 1]));
    for (auto& mk : P.marks) {
      float ms = 0.0f;
      SR_CHECK_CUDA(cudaEventElapsedTime(&ms, P.pool[mk.second], P.pool[mk.second + 1]));
      if (ms_out) ms_out[mk.first] += ms;
      if (count_out) count_out[mk.first] += 1;
    }
  }
  P.marks.clear();
  P.next = 0;
  P.on = enable != 0;
  return SR_OK;
}

int sr_sample_rows(const float* logits, int rows, int vocab, int ld, const int32_t* req, const int32_t* pos,
                   uint32_t seed, float temperature, int32_t* ids, sr_stream_t stream) {
  SR_REQUIRE(rows >= 0 && vocab > 0 && ld >= vocab, "bad logits shape");
  SR_REQUIRE(temperature > 0.0f, "temperature must be > 0");
  if (rows == 0) return SR_OK;
  SR_REQUIRE(logits && req && pos && ids, "null pointer");
  return sr::sample_rows(logits, rows, vocab, ld, req, pos, seed, 1.0f / temperature, ids, nullptr,
                         (cudaStream_t)stream);
}

}  // extern "C"
