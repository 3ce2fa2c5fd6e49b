// a1/a2 keyed draws on device: one thread = one (seed, keys...) stream chunk.
//
// Replaces the per-position Python calls `_Sim.true_token` (sim.py:313-320)
// and `_Sim.accept_draw` (sim.py:322-336), which materialize 256-draw chunks
// of numpy streams.  The whole truth/uniform table of a rollout is generated
// once, in parallel, and stays resident in HBM for the verify kernels.
// Output goes through shared memory so the global stores of a block are
// coalesced (each thread produces 256 consecutive values).
#include "common.cuh"
#include "keyed_stream.cuh"

namespace sr {

constexpr int kMaxWords = 16;
constexpr int kStreamsPerBlock = 32;

template <typename T, bool kUniform>
__global__ void __launch_bounds__(kStreamsPerBlock)
keyed_fill_kernel(int num_streams, const uint32_t* __restrict__ words,
                  const int32_t* __restrict__ num_words, int max_words,
                  uint32_t rng, int per_stream, T* __restrict__ out) {
  grid_dep_sync();
  const int s = blockIdx.x * kStreamsPerBlock + threadIdx.x;
  Pcg64 g;
  if (s < num_streams) {
    uint32_t ent[kMaxWords];
    int n = num_words[s];
    n = n > max_words ? max_words : n;
    for (int i = 0; i < n; ++i) ent[i] = words[(int64_t)s * max_words + i];
    g = pcg_from_entropy(ent, n);
  }
  // Stage 32 values per stream per pass in smem, then store row-contiguous.
  __shared__ T tile[kStreamsPerBlock][33];
  const int first = blockIdx.x * kStreamsPerBlock;
  const int rows = min(kStreamsPerBlock, num_streams - first);
  for (int base = 0; base < per_stream; base += 32) {
    const int cnt = min(32, per_stream - base);
    if (s < num_streams) {
      for (int i = 0; i < cnt; ++i) {
        if constexpr (kUniform) tile[threadIdx.x][i] = (T)pcg_next_double(g);
        else tile[threadIdx.x][i] = (T)pcg_bounded(g, rng);
      }
    }
    __syncthreads();
    for (int r = 0; r < rows; ++r)
      if ((int)threadIdx.x < cnt)
        out[(int64_t)(first + r) * per_stream + base + threadIdx.x] = tile[r][threadIdx.x];
    __syncthreads();
  }
}

}  // namespace sr

extern "C" {

int sr_keyed_tokens(int num_streams, const uint32_t* words, const int32_t* num_words,
                    int max_words, int64_t high, int per_stream, int32_t* out,
                    sr_stream_t stream) {
  SR_REQUIRE(num_streams >= 0 && per_stream >= 0, "negative sizes");
  SR_REQUIRE(max_words >= 1 && max_words <= sr::kMaxWords, "max_words out of [1,16]");
  SR_REQUIRE(high >= 1 && high <= 0x7FFFFFFFll, "high out of [1, 2^31)");
  if (num_streams == 0 || per_stream == 0) return SR_OK;
  SR_REQUIRE(words && num_words && out, "null pointer");
  dim3 grid(sr::ceil_div(num_streams, sr::kStreamsPerBlock));
  sr::launch_k(sr::keyed_fill_kernel<int32_t, false>, grid, sr::kStreamsPerBlock, 0, (cudaStream_t)stream, 
      num_streams, words, num_words, max_words, (uint32_t)(high - 1), per_stream, out);
  return sr::check_launch("keyed_fill_kernel<tokens>");
}

int sr_keyed_uniforms(int num_streams, const uint32_t* words, const int32_t* num_words,
                      int max_words, int per_stream, double* out, sr_stream_t stream) {
  SR_REQUIRE(num_streams >= 0 && per_stream >= 0, "negative sizes");
  SR_REQUIRE(max_words >= 1 && max_words <= sr::kMaxWords, "max_words out of [1,16]");
  if (num_streams == 0 || per_stream == 0) return SR_OK;
  SR_REQUIRE(words && num_words && out, "null pointer");
  dim3 grid(sr::ceil_div(num_streams, sr::kStreamsPerBlock));
  sr::launch_k(sr::keyed_fill_kernel<double, true>, grid, sr::kStreamsPerBlock, 0, (cudaStream_t)stream, 
      num_streams, words, num_words, max_words, 0u, per_stream, out);
  return sr::check_launch("keyed_fill_kernel<uniforms>");
}

}  // extern "C"
