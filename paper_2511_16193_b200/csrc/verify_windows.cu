// a3/a4/a5: verify a batch of speculation windows in reference ("truth") mode.
//
// One warp per window.  The reference walks a window token by token
// (`_verify_prefix`, sim.py:977-981: accept while u[pos] < p), then commits
// the accepted prefix plus the corrected / bonus token (`_apply_outcome`,
// sim.py:983-1042) and advances the committed-high watermark (`commit`,
// sim.py:340-353).  Here lane i tests position start+i, a ballot yields the
// first rejection, lanes write the committed tokens, and a ballot scan
// advances the watermark.  A conflicting commit (the invariant asserted at
// sim.py:344-347) is reported as high = -1.
#include "common.cuh"

namespace sr {

__global__ void __launch_bounds__(256)
verify_windows_kernel(int W, const int32_t* __restrict__ win, int method, int M, int stride,
                      const int32_t* __restrict__ truth, const double* __restrict__ uni,
                      const double* __restrict__ accept_p, const int32_t* __restrict__ true_len,
                      int bonus, int32_t* __restrict__ seq, int32_t* __restrict__ high,
                      int32_t* __restrict__ out) {
  grid_dep_sync();
  const int lane = threadIdx.x & 31;
  const int w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (w >= W) return;
  const int row = win[w], start = win[W + w], n = win[2 * W + w], extra = win[3 * W + w];
  const int L = true_len[row];
  const int64_t rbase = (int64_t)row * stride;

  // accepted prefix: first index whose uniform fails u < p (sim.py:977-981)
  int a = 0;
  if (n > 0) {
    const double p = accept_p[(int64_t)row * M + method];
    const double* u = uni + ((int64_t)row * M + method) * stride + start;
    a = n;
    for (int base = 0; base < n; base += 32) {
      const int i = base + lane;
      const bool ok = i < n ? (u[i] < p) : true;
      const unsigned rej = __ballot_sync(0xffffffffu, !ok);
      if (rej) {
        a = base + __ffs(rej) - 1;
        break;
      }
    }
  }
  int committed, wasted;
  if (n == 0) {  // plain decode step (sim.py:966-975)
    committed = 1;
    wasted = 0;
  } else if (a == n) {  // full accept (+ optional bonus token)
    committed = n + ((bonus && start + n < L) ? 1 : 0);
    wasted = 0;
  } else {  // accepted prefix + corrected token; rest (+ depth-2 successor) wasted
    committed = a + 1;
    wasted = max(n - a - 1, 0) + extra;
  }

  // commit target tokens (sim.py:340-347)
  bool conflict = false;
  for (int j = lane; j < committed; j += 32) {
    const int64_t at = rbase + start + j;
    const int32_t tok = truth[at];
    const int32_t prev = seq[at];
    if (prev < 0) seq[at] = tok;
    else if (prev != tok) conflict = true;
  }
  conflict = __any_sync(0xffffffffu, conflict);
  __syncwarp();

  // committed-high watermark scan (sim.py:348-353)
  int h = high[row];
  while (h < L) {
    const int pos = h + lane;
    const bool filled = pos < L && seq[rbase + pos] >= 0;
    const unsigned holes = __ballot_sync(0xffffffffu, !filled);
    if (holes) {
      h += __ffs(holes) - 1;
      break;
    }
    h += 32;
  }
  h = min(h, L);
  if (lane == 0) {
    high[row] = h;
    out[w] = a;
    out[W + w] = committed;
    out[2 * W + w] = wasted;
    out[3 * W + w] = conflict ? -1 : h;
  }
}

}  // namespace sr

extern "C" int sr_verify_windows(int num_windows, const int32_t* win, int method,
                                 int num_methods, int row_stride, const int32_t* truth,
                                 const double* uniforms, const double* accept_p,
                                 const int32_t* true_len, int bonus_token, int32_t* seq,
                                 int32_t* high, int32_t* out, sr_stream_t stream) {
  SR_REQUIRE(num_windows >= 0, "negative window count");
  if (num_windows == 0) return SR_OK;
  SR_REQUIRE(num_methods >= 1 && method >= 0 && method < num_methods, "method out of range");
  SR_REQUIRE(row_stride >= 1, "row_stride must be >= 1");
  SR_REQUIRE(win && truth && uniforms && accept_p && true_len && seq && high && out,
             "null pointer");
  const int warps_per_block = 8;
  dim3 grid(sr::ceil_div(num_windows, warps_per_block));
  sr::launch_k(sr::verify_windows_kernel, grid, warps_per_block * 32, 0, (cudaStream_t)stream, 
      num_windows, win, method, num_methods, row_stride, truth, uniforms, accept_p, true_len,
      bonus_token, seq, high, out);
  return sr::check_launch("verify_windows_kernel");
}
