// k_tdaeq.cu -- the float per-symbol 4x4 RDE comparator on the GPU.
//
// Reference: fntdsp/aeq.py:193-249 (_td_rde_kernel, td_aeq_float): for every
// symbol m >= L-1, y[s2][m] = sum over (s1, k) of w[s2][s1][k] x[s1][m-k] summed
// sequentially (s1 major, k minor, starting from 0.0), then per polarization the
// radius-directed error e = R^2 - (yI^2 + yQ^2) (nearest ring, first minimum) and
// w[s2] += (mu e y[s2]) x for both outputs of the polarization when that factor
// is non-zero. Not on the FNT path (the paper's float comparator); float64 with
// every product and sum rounded separately (--fmad=false), so the outputs equal
// the reference's numba kernel bit for bit.
//
// One warp per stream, lane = 8 s2 + 2 s1 + h: the lane owns w[s2][s1][8h..8h+7]
// and the matching window x[s1][m - 8h - j]; it forms its 8 products, the warp
// stages them in shared memory, and lane 8 s2 runs output s2's sequential sum.
#include <cmath>

#include "internal.h"

namespace fntgpu {

namespace {
constexpr int TD_L = 16;
constexpr int TD_WARPS = 4;

struct TdScratch {
  double prod[4][4 * TD_L];  // products of the symbol, [s2][s1 * 16 + k]
  double y[4];
  double g[4];
};

__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
}  // namespace

__global__ void __launch_bounds__(TD_WARPS * 32) k_td_aeq(fntgpu_td_aeq_io io) {
  __shared__ TdScratch scratch[TD_WARPS];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t S_idx = (int64_t)blockIdx.x * TD_WARPS + warp;
  if (S_idx >= io.n_streams) return;
  TdScratch& S = scratch[warp];
  const int s2 = lane >> 3, s1 = (lane >> 1) & 3, h = lane & 1;
  const double* xs = io.x + S_idx * io.x_stream_stride + s1 * io.x_row_stride;
  double* wl = io.w + S_idx * 4 * 4 * TD_L + (s2 * 4 + s1) * TD_L + 8 * h;
  double* yo = io.y + S_idx * io.y_stream_stride;
  double w[8], xw[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) w[j] = wl[j];
  const int64_t n = io.n;
  // outputs before the first full window are zero (aeq.py:196)
  for (int64_t m = lane; m < (n < TD_L - 1 ? n : TD_L - 1); m += 32)
    for (int r = 0; r < 4; ++r) yo[r * io.y_row_stride + m] = 0.0;
  // window for m = L-1: xw[j] = x[s1][m - 8h - j]
#pragma unroll
  for (int j = 0; j < 8; ++j) xw[j] = (TD_L - 1 - 8 * h - j >= 0 && TD_L - 1 < n) ? xs[TD_L - 1 - 8 * h - j] : 0.0;
  for (int64_t m = TD_L - 1; m < n; ++m) {
#pragma unroll
    for (int j = 0; j < 8; ++j) S.prod[s2][s1 * TD_L + 8 * h + j] = dmul(w[j], xw[j]);
    __syncwarp();
    if ((lane & 7) == 0) {
      double acc = 0.0;
#pragma unroll 16
      for (int i = 0; i < 4 * TD_L; ++i) acc = dadd(acc, S.prod[s2][i]);
      S.y[s2] = acc;
      yo[s2 * io.y_row_stride + m] = acc;
    }
    __syncwarp();
    if (lane < 2) {
      const double yi = S.y[2 * lane], yq = S.y[2 * lane + 1];
      const double r2 = dadd(dmul(yi, yi), dmul(yq, yq));
      const double r = __dsqrt_rn(r2);
      double best = io.radii[0];
      for (int ri = 1; ri < io.n_radii; ++ri)
        if (fabs(dsub(io.radii[ri], r)) < fabs(dsub(best, r))) best = io.radii[ri];
      const double e = dsub(dmul(best, best), r2);
      const double me = dmul(io.mu[m], e);
      S.g[2 * lane] = dmul(me, yi);
      S.g[2 * lane + 1] = dmul(me, yq);
    }
    __syncwarp();
    const double g = S.g[s2];
    if (g != 0.0) {
#pragma unroll
      for (int j = 0; j < 8; ++j) w[j] = dadd(w[j], dmul(g, xw[j]));
    }
    // slide the window to m + 1
#pragma unroll
    for (int j = 7; j > 0; --j) xw[j] = xw[j - 1];
    if (m + 1 < n) xw[0] = xs[m + 1 - 8 * h];
    __syncwarp();
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) wl[j] = w[j];
}

cudaError_t launch_td_aeq(const fntgpu_td_aeq_io& io, cudaStream_t s) {
  if (io.n_streams <= 0) return cudaSuccess;
  const unsigned grid = (unsigned)((io.n_streams + TD_WARPS - 1) / TD_WARPS);
  k_td_aeq<<<grid, TD_WARPS * 32, 0, s>>>(io);
  return cudaGetLastError();
}

}  // namespace fntgpu
