// K1 host side: GEMM plans (tensor maps, tile / K-range / mode choice),
// launches, the single-CTA kernel instantiations, the fp32 parity GEMM and
// the C-ABI entry points.  Device code: gemm_dev.cuh; the CTA-pair kernel
// is instantiated per tile width in gemm_pair_bn*.cu (parallel builds).
#include "gemm_dev.cuh"

namespace sr {

namespace {

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

}  // namespace

int num_sms() {
  if (g_num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  return g_num_sms;
}

namespace {

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


int launch_pair(const GemmPlan& p, int M, cudaStream_t stream) {
  switch (p.bn) {
    case 64: return launch_pair_bn64(p, M, stream);
    case 96: return launch_pair_bn96(p, M, stream);
    case 112: return launch_pair_bn112(p, M, stream);
    case 128: return launch_pair_bn128(p, M, stream);
    case 160: return launch_pair_bn160(p, M, stream);
    case 192: return launch_pair_bn192(p, M, stream);
    case 224: return launch_pair_bn224(p, M, stream);
    case 256: return launch_pair_bn256(p, M, stream);
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

void choose_pair_tile(int M, int N, int K, int epi, int bn_max, int* bn_out, int* mc_out) {
  static const int cands[] = {256, 224, 192, 160, 128, 96, 64};
  const int num_m = (M + 255) / 256;
  const int kb = (K + 63) / 64;
  const int pairs = num_sms() / 2;
  if (bn_max > g_pair_bn_max) bn_max = g_pair_bn_max;
  int best = 64;
  double best_t = 1e30;
  for (int bn : cands) {
    if (bn > bn_max) continue;
    if ((epi == kEpiSwiGLU || epi == kEpiQkvRope) && bn % 32 != 0) continue;
    if (epi == kEpiResidualNorm && bn % kSsqCols != 0) continue;  // norm groups within a tile
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
// small-M mode threshold override (live rows; 0 disables the mode)
int g_swap_max_m = [] {
  const char* v = getenv("SR_SWAP_MAX_M");
  const int m = v ? atoi(v) : -1;
  return m < 0 ? -1 : (m > kSwapRows ? kSwapRows : m);
}();

// Live rows up to which the small-M mode beats the pair mode (B200,
// scripts/small_m_gemm_probe.py): the pair mode costs about the same for any
// M <= 256, the small-M mode grows ~1.5-3 us per 32 rows (epilogue and
// K-range reduction per token group) but streams the weights on more SMs,
// so the crossover moves up with the weight bytes: 1.5B qkv / o (5-6 MB)
// ~40 rows, 0.5B down (9 MB) ~90, 1.5B down and every 7B / 32B projection
// (>= 25 MB) past 128.
// measurement knobs: cap on K ranges, weight staging before the wait
int g_splits_max = [] {
  const char* v = getenv("SR_GEMM_SPLITS_MAX");
  const int m = v ? atoi(v) : 4;
  return m < 1 ? 1 : (m > 4 ? 4 : m);
}();
int g_preissue = [] {
  const char* v = getenv("SR_GEMM_PREISSUE");
  return v ? atoi(v) : 1;
}();

int swap_max_m(int N, int K) {
  if (g_swap_max_m >= 0) return g_swap_max_m;
  const double wmb = 2.0 * N * K / 1e6;
  return wmb >= 16.0 ? 128 : wmb >= 8.0 ? 64 : 0;
}

bool swap_epi(int epi) {
  return epi == kEpiStoreBf16 || epi == kEpiStoreF32 || epi == kEpiResidualF32 || epi == kEpiResidualNorm ||
         epi == kEpiQkvRope || epi == kEpiSwiGLU;
}

// sr_gemm's own partials / counters (the model carves its own)
float* g_swap_ws = nullptr;
unsigned long long* g_trace_dev = nullptr;  // SR_GEMM_TRACE builds
SwapMaps* g_swap_maps = nullptr;
int32_t* g_swap_cnt = nullptr;
size_t g_swap_ws_floats = 0, g_swap_cnt_ints = 0;
}  // namespace

// K ranges for a (N, K) projection, from the shape alone (never from the
// batch): enough (256-row weight tile, range) units to stream the weights on
// most SMs at small M, ranges of >= 8 chunks of 64, at most 4 (the pair
// mode keeps one TMEM accumulator per range).  Cost model in 64-k chunks of
// one CTA: waves x (chunks per range + ~15 fill/drain) + ~7 for the partial
// round trip.
int gemm_splits(int N, int K, int epi) {
  if (!swap_epi(epi) || K % kBK != 0) return 1;
  // projections below 8 MB of weights keep the pair mode at every M (see
  // swap_max_m): one accumulator, no extra TMEM reads in its epilogue
  if (2.0 * N * K < 8e6) return 1;
  const int chunks = K / kBK;
  const int tiles = (N + 255) / 256;
  const int pairs = num_sms() / 2;
  int best = 1;
  double best_t = 1e30;
  // below 64 MB the pair mode's extra accumulator reads (large batches)
  // outweigh more than two ranges for the small-M mode (1.5B down: the
  // bench step +1.5% at 4 ranges)
  const int smax = 2.0 * N * K < 64e6 && g_splits_max > 2 ? 2 : g_splits_max;
  for (int s = 1; s <= smax; ++s) {
    if (chunks % s != 0 || (s > 1 && chunks / s < 8)) continue;
    const int waves = (tiles * s + pairs - 1) / pairs;
    const double t = waves * (chunks / s + 15.0) + (s > 1 ? 7.0 : 0.0);
    if (t < best_t * 0.999) { best_t = t; best = s; }
  }
  return best;
}

size_t gemm_swap_ws_floats(const GemmPlan& p) {
  return p.sw.max_m > 0 && p.sw.splits > 1 ? (size_t)p.sw.splits * kSwapRows * p.N : 0;  // [range][n][token]
}
size_t gemm_swap_cnt_ints(const GemmPlan& p) { return p.sw.max_m > 0 ? (size_t)2 * ((p.N + 255) / 256) : 0; }

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

// bf16 paged KV cache [blocks][64 slots][128 head dims] (blocks = layers x
// pages x K/V x kv heads; rows already XOR-swizzled by slot in HBM) viewed as
// (64 dims, slot in group, head-dim half, 8-slot group, block): one box
// (64, 8, 2, 8, 1) is a whole page landing as [group][half][8 slots][128 B]
// -- 1 KB SWIZZLE_128B atoms, K chunk (half) stride 1 KB, 8-row group stride
// 2 KB -- so the copy itself must not swizzle again.
int make_tmap_kv_pages(CUtensorMap* map, const void* cache, uint64_t blocks) {
  auto enc = tmap_encoder();
  if (enc == nullptr) {
    set_error("cuTensorMapEncodeTiled unavailable (driver too old?)");
    return SR_ERR_RUNTIME;
  }
  cuuint64_t dims[5] = {64, 8, 2, 8, blocks};
  cuuint64_t strides[4] = {256, 128, 8 * 256, 64 * 256};
  cuuint32_t box[5] = {64, 8, 2, 8, 1};
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, const_cast<void*>(cache), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled (kv pages) failed (%d): blocks=%llu", (int)r, (unsigned long long)blocks);
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
  // swap-capable projections (qkv, o, down) always take the pair kernel, so
  // one launch serves both modes; their K ranges come from the shape alone
  const bool swappable = swap_epi(epi) && K % kBK == 0 && g_pair_kc == 2;
  int splits = swappable ? gemm_splits(N, K, epi) : 1;
  if (bn == 0) {
    pair = M >= 256 || swappable;
    // gate_up at M = 256j + (<= 128) rows (e.g. 64 prompts x 5 = 320): the
    // last 256-row pair block would be mostly padding; 128-row single-CTA
    // tiles waste less (7B 99 -> 90 us, 32B 200 -> 190 us at M = 320)
    if (pair && epi == kEpiSwiGLU && M % 256 != 0 && M % 256 <= 128) pair = false;
    if (pair) choose_pair_tile(M, N, K, epi, 512 / splits, &bn, &mc);
    else bn = N >= 4096 ? 256 : 128;
  } else if (bn < 0) {
    pair = true;
    bn = -bn;
    if (bn > 1024) { mc = 2; bn -= 1024; }
    // an explicit tile: as many K ranges as its accumulators fit (probes only)
    while (splits > 1 && (splits * bn > 512 || (K / kBK) % splits != 0)) --splits;
  } else {
    pair = false;
    splits = 1;
    SR_REQUIRE(bn == 128 || bn == 256, "single-CTA bn must be 128 or 256");
  }
  SR_REQUIRE(epi != kEpiResidualNorm || bn % kSsqCols == 0, "residual+norm epilogue needs bn 128 or 256");
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
  p->sw.splits = pair ? splits : 1;
  p->sw.max_m = (pair && p->kc == 2 && swappable) ? swap_max_m(N, K) : 0;
  p->sw.flags = g_preissue ? 1 : 0;
  // plans for more than 256 rows: the small-M mode only as a dual launch
  // (pair + small-M kernel, the device picks by live rows), and only for
  // weights >= 64 MB where small live batches (compacted verify tails,
  // 7B / 32B targets) gain far more than the ~1-2 us of the second launch;
  // smaller projections run their small batches through narrow plans
  if (p->sw.max_m > 0 && M > 256) {
    if (2.0 * N * K >= 64e6 || g_swap_max_m > 0) p->sw.flags |= 2;
    else p->sw.max_m = 0;
  }
  p->sw.ws = nullptr;
  p->sw.cnt = nullptr;
  p->sw.maps = nullptr;
#ifdef SR_GEMM_TRACE
  if (g_trace_dev == nullptr) {
    cudaMalloc(&g_trace_dev, 1024 * 8 * sizeof(unsigned long long));
    cudaMemset(g_trace_dev, 0, 1024 * 8 * sizeof(unsigned long long));
  }
  p->sw.trace = g_trace_dev;
#endif
  if (p->sw.max_m > 0) {
    int rc = make_tmap_bf16_3d(&p->sw_maps.w, W, (uint64_t)K, (uint64_t)N, (uint64_t)ldw * 2, 128, 2);
    for (int g = 0; g < 4 && rc == 0; ++g)
      rc = make_tmap_bf16_3d(&p->sw_maps.x[g], A, (uint64_t)K, (uint64_t)mrows, (uint64_t)lda * 2, 16 * (g + 1), 2);
    if (rc) return rc;
  }
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
  SR_REQUIRE(p.sw.max_m == 0 || (p.sw.maps != nullptr && p.sw.cnt != nullptr && (p.sw.splits == 1 || p.sw.ws != nullptr)),
             "small-M mode needs its device tensor maps, partials workspace and counters (SwapArgs)");
  if (p.pair && p.sw.max_m > 0) {
    // the launch's row count bounds the live rows: small-M mode alone
    if (M <= p.sw.max_m) return launch_swap(p, M, stream);
    // only the device knows the live rows: both kernels, each exits if not its case
    if (p.sw.flags & 2) {
      const int rc = launch_swap(p, M, stream);
      if (rc) return rc;
    }
  }
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
    // small-M mode: a process-wide partials buffer (grown outside any capture)
    const size_t wf = sr::gemm_swap_ws_floats(plan), wc = sr::gemm_swap_cnt_ints(plan);
    if (wf > sr::g_swap_ws_floats) {
      if (sr::g_swap_ws) cudaFree(sr::g_swap_ws);
      SR_CHECK_CUDA(cudaMalloc(&sr::g_swap_ws, wf * sizeof(float)));
      sr::g_swap_ws_floats = wf;
    }
    if (wc > sr::g_swap_cnt_ints) {
      if (sr::g_swap_cnt) cudaFree(sr::g_swap_cnt);
      SR_CHECK_CUDA(cudaMalloc(&sr::g_swap_cnt, wc * sizeof(int32_t)));
      SR_CHECK_CUDA(cudaMemset(sr::g_swap_cnt, 0, wc * sizeof(int32_t)));
      sr::g_swap_cnt_ints = wc;
    }
    plan.sw.ws = sr::g_swap_ws;
    plan.sw.cnt = sr::g_swap_cnt;
    if (plan.sw.max_m > 0) {  // stream-ordered upload of this call's maps (graph-capturable)
      if (sr::g_swap_maps == nullptr) SR_CHECK_CUDA(cudaMalloc(&sr::g_swap_maps, sizeof(sr::SwapMaps)));
      SR_CHECK_CUDA(cudaMemcpyAsync(sr::g_swap_maps, &plan.sw_maps, sizeof(sr::SwapMaps), cudaMemcpyHostToDevice,
                                    (cudaStream_t)stream));
      plan.sw.maps = sr::g_swap_maps;
    }
    return sr::gemm_bf16_launch(plan, (cudaStream_t)stream);
  }
  SR_REQUIRE(dtype == 0, "dtype must be 0 (f32) or 1 (bf16)");
  SR_REQUIRE(epilogue != sr::kEpiArgmax, "argmax epilogue is bf16-only; use sr_argmax_rows");
  return sr::gemm_f32(M, N, K, reinterpret_cast<const float*>(A), lda,
                      reinterpret_cast<const float*>(W), ldw, C, ldc, epilogue, bias,
                      (cudaStream_t)stream);
}

extern "C" int sr_gemm_splits(int N, int K, int epilogue) {
  if (N <= 0 || K <= 0) return sr::config_error("bad GEMM shape");
  return sr::gemm_splits(N, K, epilogue);
}

// Measurement builds only: copy the per-CTA stamps of the last traced launch.
extern "C" int sr_debug_gemm_trace(unsigned long long* out, int n) {
#ifdef SR_GEMM_TRACE
  if (n > 1024 * 8) n = 1024 * 8;
  if (sr::g_trace_dev == nullptr) return sr::config_error("no traced GEMM plan yet");
  if (out) SR_CHECK_CUDA(cudaMemcpy(out, sr::g_trace_dev, (size_t)n * 8, cudaMemcpyDeviceToHost));
  SR_CHECK_CUDA(cudaMemset(sr::g_trace_dev, 0, 1024 * 8 * sizeof(unsigned long long)));  // cleared for the next launch
  return SR_OK;
#else
  (void)out;
  (void)n;
  return sr::config_error("not a trace build (-DSR_GEMM_TRACE)");
#endif
}

// Small-M mode threshold for plans made afterwards: -1 = per shape
// (swap_max_m), 0 = off, 1..128 = live rows (tests / tuning).
extern "C" int sr_set_gemm_swap_max_m(int max_m) {
  if (max_m < -1 || max_m > sr::kSwapRows) return sr::config_error("swap max_m must be in [-1, 128]");
  sr::g_swap_max_m = max_m;
  return SR_OK;
}
