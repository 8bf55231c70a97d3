// k_transform.cu -- batched FNT / IFNT and fused cyclic convolutions.
//
// Reference: fntdsp/fnt.py:86-161 (_butterflies, fnt, ifnt, cyclic_convolve_real,
// cyclic_convolve_complex) and fermat.py:124-133 (encode/decode arrays).
//
// Fast path (aeq32: alpha = 2, N = 32; cdc64: alpha = sqrt2 = 4080, N = 64):
//   a CTA stages a tile of 64 vectors through shared memory with coalesced int64
//   loads/stores; one thread owns one length-N vector in registers; the DIT network is fully
//   unrolled with compile-time twiddles that are rotates in Z/(2^32-1) (fermat.cuh),
//   so no general multiplication appears inside a transform (the reference's
//   "shift-add" claim, fnt.py:1-8) and the only general products are the
//   pointwise ones of the convolutions.
// Generic path (any plan make_plan accepts, e.g. mod17): a CTA transforms a tile
//   of vectors in shared memory with per-stage twiddle tables and 64-bit products.
#include "fermat.cuh"
#include "internal.h"

namespace fntgpu {

// ---------------------------------------------------------------------------
// fast path

// Coalesced staging of a CTA's tile of T consecutive length-N int64 vectors: the
// CTA reads the tile's contiguous int64 words (T threads, stride T), encodes them
// into Z/M words and parks them in a padded [T][N + 1] shared array; each thread
// then takes its own row (conflict-free), and results go back the same way.
constexpr int TILE = 64;  // vectors (= threads) per CTA of the fast kernels

template <int N>
__device__ __forceinline__ void stage_tile_in(uint32_t (*s)[N + 1], const int64_t* __restrict__ x,
                                              int64_t b0, int64_t batch) {
  const int64_t* src = x + b0 * N;
  if (batch - b0 >= TILE) {
    // full tile: batches of 16 independent loads per thread in flight
    constexpr int PER = N, B = 16;
#pragma unroll
    for (int j0 = 0; j0 < PER; j0 += B) {
      int64_t v[B];
#pragma unroll
      for (int j = 0; j < B; ++j) v[j] = __ldg(src + (j0 + j) * TILE + threadIdx.x);
#pragma unroll
      for (int j = 0; j < B; ++j) {
        const int e = (j0 + j) * TILE + threadIdx.x;
        s[e / N][e % N] = f4_enc64(v[j]);
      }
    }
    return;
  }
  const int64_t words = (batch - b0) * N;
  for (int64_t e = threadIdx.x; e < words; e += TILE) s[e / N][e % N] = f4_enc64(src[e]);
}

template <int N>
__device__ __forceinline__ void stage_tile_out(const uint32_t (*s)[N + 1], int64_t* __restrict__ y,
                                               int64_t b0, int64_t batch, int flags) {
  const int64_t rows = batch - b0 < TILE ? batch - b0 : TILE;
  const int64_t words = rows * N;
  int64_t* dst = y + b0 * N;
  for (int64_t e = threadIdx.x; e < words; e += TILE) {
    const uint32_t v = s[e / N][e % N];
    dst[e] = (flags & FNTGPU_DECODE_SIGNED) ? (int64_t)f4_signed(v) : (int64_t)f4_canon(v);
  }
}

template <int N>
__device__ __forceinline__ void row_bitrev(uint32_t (&a)[N], const uint32_t* row) {
  constexpr int LG = ilog2(N);
#pragma unroll
  for (int i = 0; i < N; ++i) a[bitrev(i, LG)] = row[i];
}

// One transform of a shared-memory row in place (read in bit-reversed order,
// written in natural order; the inverse also applies the rotation `rot`). Kept
// out of line: the complex convolution runs it 6 times per vector and fully
// unrolled copies of the 64-point network overflow the instruction cache (2.6x
// slower inline; the real convolution's 3 inline copies are 5% faster than calls).
template <int N, int KIND, bool INV>
__device__ __noinline__ void fnt_row(uint32_t* row, int rot) {
  uint32_t a[N];
  row_bitrev<N>(a, row);
  fnt_dit<N, KIND, INV>(a);
#pragma unroll
  for (int i = 0; i < N; ++i) row[i] = INV ? m_rot(a[i], rot) : a[i];
}

template <int N, int KIND>
__global__ void __launch_bounds__(TILE) k_fnt_fast(const int64_t* x, int64_t* y, int64_t batch,
                                                   int inverse, int flags) {
  constexpr int LG = ilog2(N);
  __shared__ uint32_t sA[TILE][N + 1];
  const int64_t b0 = (int64_t)blockIdx.x * TILE;
  stage_tile_in<N>(sA, x, b0, batch);
  __syncthreads();
  uint32_t a[N];
  row_bitrev<N>(a, sA[threadIdx.x]);
  if (inverse) {
    fnt_dit<N, KIND, true>(a);
#pragma unroll
    for (int i = 0; i < N; ++i) a[i] = m_rot(a[i], 32 - LG);  // * N^-1 = 2^-LG = 2^(32-LG)
  } else {
    fnt_dit<N, KIND, false>(a);
  }
#pragma unroll
  for (int i = 0; i < N; ++i) sA[threadIdx.x][i] = a[i];  // own row only: no barrier needed before
  __syncthreads();
  stage_tile_out<N>(sA, y, b0, batch, flags);
}

template <int N, int KIND>
__global__ void __launch_bounds__(TILE) k_conv_real_fast(const int64_t* x, const int64_t* h,
                                                         int64_t h_stride, int64_t* z,
                                                         int64_t batch, int flags) {
  constexpr int LG = ilog2(N);
  __shared__ uint32_t sX[TILE][N + 1];
  __shared__ uint32_t sH[TILE][N + 1];
  const int64_t b0 = (int64_t)blockIdx.x * TILE;
  stage_tile_in<N>(sX, x, b0, batch);
  if (h_stride != 0) {
    stage_tile_in<N>(sH, h, b0, batch);
  } else {
    for (int i = threadIdx.x; i < N; i += TILE) sH[0][i] = f4_enc64(h[i]);  // shared taps
  }
  __syncthreads();
  // Tap spectra first, parked back in shared memory (each thread its own row, or
  // thread 0 the CTA's one shared row), so only one spectrum is register-resident.
  const int hr = h_stride != 0 ? threadIdx.x : 0;
  if (h_stride != 0 || threadIdx.x == 0) {
    uint32_t H[N];
    row_bitrev<N>(H, sH[hr]);
    fnt_dit<N, KIND, false>(H);
#pragma unroll
    for (int i = 0; i < N; ++i) sH[hr][i] = H[i];
  }
  if (h_stride == 0) __syncthreads();  // uniform over the CTA
  uint32_t X[N];
  row_bitrev<N>(X, sX[threadIdx.x]);
  fnt_dit<N, KIND, false>(X);
#pragma unroll
  for (int i = 0; i < N; ++i) X[i] = m_mul(X[i], sH[hr][i]);  // the N general products (fnt.py:123)
  to_bitrev<N>(X);
  fnt_dit<N, KIND, true>(X);
#pragma unroll
  for (int i = 0; i < N; ++i) sX[threadIdx.x][i] = m_rot(X[i], 32 - LG);
  __syncthreads();
  stage_tile_out<N>(sX, z, b0, batch, flags);
}

// Per-vector taps (config 1: h_stride == N), two threads per vector: a CTA of two
// warps owns PAIR_TILE consecutive vectors; warp 0 stages and transforms the signal
// rows, warp 1 the tap rows (its spectra go back to shared memory), then warp 0
// forms the N products and the inverse. Each warp stages its tile with batches of 32
// independent loads per lane in flight (twice the memory-level parallelism and twice
// the warps per SM of the one-thread-per-vector kernel, whose 512 warps over 148 SMs
// left both the loads and the transforms latency-bound).
constexpr int PAIR_TILE = 32;

template <int N>
__device__ __forceinline__ void stage_warp_in(uint32_t (*s)[N + 1], const int64_t* __restrict__ src,
                                              int64_t rows, int lane) {
  if (rows == PAIR_TILE) {
    constexpr int PER = N, B = 32;  // N * PAIR_TILE words over 32 lanes
#pragma unroll
    for (int j0 = 0; j0 < PER; j0 += B) {
      int64_t v[B];
#pragma unroll
      for (int j = 0; j < B; ++j) v[j] = __ldg(src + (j0 + j) * 32 + lane);
#pragma unroll
      for (int j = 0; j < B; ++j) {
        const int e = (j0 + j) * 32 + lane;
        s[e / N][e % N] = f4_enc64(v[j]);
      }
    }
    return;
  }
  const int64_t words = rows * N;
  for (int64_t e = lane; e < words; e += 32) s[e / N][e % N] = f4_enc64(src[e]);
}

template <int N, int KIND>
__global__ void __launch_bounds__(2 * PAIR_TILE) k_conv_real_pair(const int64_t* x, const int64_t* h,
                                                                   int64_t* z, int64_t batch, int flags) {
  constexpr int LG = ilog2(N);
  __shared__ uint32_t sX[PAIR_TILE][N + 1];
  __shared__ uint32_t sH[PAIR_TILE][N + 1];
  const int64_t b0 = (int64_t)blockIdx.x * PAIR_TILE;
  const int64_t rows = batch - b0 < PAIR_TILE ? batch - b0 : PAIR_TILE;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t (*own)[N + 1] = warp == 0 ? sX : sH;
  stage_warp_in<N>(own, (warp == 0 ? x : h) + b0 * N, rows, lane);
  __syncwarp();
  uint32_t A[N];
  row_bitrev<N>(A, own[lane]);
  fnt_dit<N, KIND, false>(A);
  if (warp == 1) {
#pragma unroll
    for (int i = 0; i < N; ++i) sH[lane][i] = A[i];  // tap spectrum of vector `lane`
  }
  __syncthreads();
  // The inverse, split over the two warps by its first decimation-in-frequency stage:
  // with beta = alpha^-1 and beta^(N/2) = -1, the even outputs are the half-length
  // inverse of u[k] = P[k] + P[k + N/2] and the odd ones that of
  // v[k] = (P[k] - P[k + N/2]) beta^k (root beta^2 = alpha^-2 for both halves).
  constexpr int H = N / 2;
  constexpr int HKIND = KIND == SQRT2 ? RADIX2 : RADIX4;  // alpha^2: sqrt2^2 = 2, 2^2 = 4
  if (warp == 0) {
#pragma unroll
    for (int i = 0; i < N; ++i) A[i] = m_mul(A[i], sH[lane][i]);  // the N general products (fnt.py:123)
#pragma unroll
    for (int k = 0; k < H; ++k) {
      sX[lane][k] = m_add(A[k], A[k + H]);
      const Tw t = twiddle<KIND>(m_sub(A[k], A[k + H]), (N - k) % N);
      sH[lane][k] = t.neg ? ~t.v : t.v;  // -v = ~v in Z/(2^32 - 1)
    }
  }
  __syncthreads();
  {
    uint32_t B[H];
    row_bitrev<H>(B, warp == 0 ? sX[lane] : sH[lane]);
    __syncthreads();  // every u row is read before either warp's outputs overwrite sX
    fnt_dit<H, HKIND, true>(B);
#pragma unroll
    for (int m = 0; m < H; ++m) sX[lane][2 * m + warp] = m_rot(B[m], 32 - LG);  // * N^-1
  }
  __syncthreads();
  const int64_t words = rows * N;
  int64_t* dst = z + b0 * N;
  for (int64_t e = threadIdx.x; e < words; e += 2 * PAIR_TILE) {
    const uint32_t v = sX[e / N][e % N];
    dst[e] = (flags & FNTGPU_DECODE_SIGNED) ? (int64_t)f4_signed(v) : (int64_t)f4_canon(v);
  }
}

// Staging of a complex tile in the combined form of Eqs. (7)-(8): P = re + 2^8 im,
// M = re - 2^8 im (linearity lets the combination happen in the time domain).
template <int N>
__device__ __forceinline__ void stage_pair_in(uint32_t (*sP)[N + 1], uint32_t (*sM)[N + 1],
                                              const int64_t* __restrict__ re,
                                              const int64_t* __restrict__ im, int64_t rows) {
  if (rows >= TILE) {
    constexpr int B = 8;
#pragma unroll
    for (int j0 = 0; j0 < N; j0 += B) {
      int64_t vr[B], vi[B];
#pragma unroll
      for (int j = 0; j < B; ++j) {
        vr[j] = __ldg(re + (j0 + j) * TILE + threadIdx.x);
        vi[j] = __ldg(im + (j0 + j) * TILE + threadIdx.x);
      }
#pragma unroll
      for (int j = 0; j < B; ++j) {
        const int e = (j0 + j) * TILE + threadIdx.x;
        const uint32_t r = f4_enc64(vr[j]), i8 = m_rot(f4_enc64(vi[j]), 8);
        sP[e / N][e % N] = m_add(r, i8);
        sM[e / N][e % N] = m_sub(r, i8);
      }
    }
    return;
  }
  const int64_t words = rows * N;
  for (int64_t e = threadIdx.x; e < words; e += TILE) {
    const uint32_t r = f4_enc64(re[e]), i8 = m_rot(f4_enc64(im[e]), 8);
    sP[e / N][e % N] = m_add(r, i8);
    sM[e / N][e % N] = m_sub(r, i8);
  }
}

// Eqs. (7)-(8): a+- = X_r +- 2^8 X_i, b+- likewise, u+- = a+- * b+-,
// z_re = 2^-1 IFNT(u+ + u-), z_im = 2^-9 IFNT(u+ - u-). Tiles are staged
// coalesced; each thread keeps one N-word array in registers and parks the
// others in its own shared-memory rows (the tap spectra b+- in the CTA's one
// shared row when the taps are common to the batch).
template <int N, int KIND>
__global__ void __launch_bounds__(TILE) k_conv_complex_fast(const int64_t* xr, const int64_t* xi,
                                                            const int64_t* yr, const int64_t* yi,
                                                            int64_t y_stride, int64_t* zr,
                                                            int64_t* zi, int64_t batch, int flags) {
  constexpr int LG = ilog2(N);
  extern __shared__ uint32_t smem_c[];
  typedef uint32_t Row[N + 1];
  Row* sAp = reinterpret_cast<Row*>(smem_c);
  Row* sAm = sAp + TILE;
  Row* sBp = sAm + TILE;
  Row* sBm = sBp + (y_stride != 0 ? TILE : 1);
  const int64_t b0 = (int64_t)blockIdx.x * TILE;
  const int64_t rows = batch - b0 < TILE ? batch - b0 : TILE;
  const int t = threadIdx.x;
  stage_pair_in<N>(sAp, sAm, xr + b0 * N, xi + b0 * N, rows);
  if (y_stride != 0) stage_pair_in<N>(sBp, sBm, yr + b0 * N, yi + b0 * N, rows);
  else stage_pair_in<N>(sBp, sBm, yr, yi, 1);
  __syncthreads();
  const int hr = y_stride != 0 ? t : 0;
  if (y_stride != 0 || t == 0) {  // b+- spectra, in place
    fnt_row<N, KIND, false>(sBp[hr], 0);
    fnt_row<N, KIND, false>(sBm[hr], 0);
  }
  if (y_stride == 0) __syncthreads();  // uniform over the CTA
  uint32_t *ap = sAp[t], *am = sAm[t];
  fnt_row<N, KIND, false>(ap, 0);
  fnt_row<N, KIND, false>(am, 0);
#pragma unroll
  for (int i = 0; i < N; ++i) {  // u+- = a+- * b+-; s = u+ + u- -> am, d = u+ - u- -> ap
    const uint32_t up = m_mul(ap[i], sBp[hr][i]), um = m_mul(am[i], sBm[hr][i]);
    am[i] = m_add(up, um);
    ap[i] = m_sub(up, um);
  }
  // c_re * N^-1 = 2^-1 * 2^-LG ; c_im * N^-1 = 2^-9 * 2^-LG (fnt.py:155-158)
  fnt_row<N, KIND, true>(am, (64 - 1 - LG) & 31);
  fnt_row<N, KIND, true>(ap, (64 - 9 - LG) & 31);
  __syncthreads();
  stage_tile_out<N>(sAm, zr, b0, batch, flags);
  stage_tile_out<N>(sAp, zi, b0, batch, flags);
}

// ---------------------------------------------------------------------------
// generic path (shared memory, canonical residues, 64-bit products)

__device__ __forceinline__ uint32_t g_mul(uint32_t a, uint32_t b, uint32_t F) {
  return (uint32_t)(((uint64_t)a * b) % F);
}
__device__ __forceinline__ uint32_t g_enc(int64_t v, uint32_t F) {
  int64_t r = v % (int64_t)F;
  return (uint32_t)(r < 0 ? r + F : r);
}
__device__ __forceinline__ int64_t g_out(uint32_t r, uint32_t F, int flags) {
  if ((flags & FNTGPU_DECODE_SIGNED) && r > (F - 1) / 2) return (int64_t)r - (int64_t)F;
  return (int64_t)r;
}

// cnt vectors of length n at s[v*n + .], bit-reversed order in, natural order out.
__device__ void smem_fnt(uint32_t* s, int cnt, const DevPlan& p, bool inverse) {
  const int n = p.n;
  const uint32_t F = p.F;
  const uint32_t* tw = inverse ? p.tw_inv : p.tw_fwd;
  const int nb = cnt * (n >> 1);
  for (int st = 0; st < p.lg; ++st) {
    const int half = 1 << st;
    for (int q = threadIdx.x; q < nb; q += blockDim.x) {
      const int v = q / (n >> 1);
      const int j2 = q - v * (n >> 1);
      const int grp = j2 >> st;
      const int j = j2 & (half - 1);
      const int i0 = v * n + grp * 2 * half + j;
      const uint32_t u = s[i0];
      const uint32_t w = g_mul(s[i0 + half], __ldg(tw + half - 1 + j), F);
      const uint32_t a = u + w;
      s[i0] = a >= F ? a - F : a;
      s[i0 + half] = u >= w ? u - w : u + F - w;
    }
    __syncthreads();
  }
  if (inverse) {
    for (int i = threadIdx.x; i < cnt * n; i += blockDim.x) s[i] = g_mul(s[i], p.n_inv, F);
    __syncthreads();
  }
}

__device__ __forceinline__ int brev_idx(int k, int lg) { return lg == 0 ? 0 : (int)(__brev((unsigned)k) >> (32 - lg)); }

__global__ void k_fnt_generic(DevPlan p, int inverse, const int64_t* x, int64_t* y, int64_t batch,
                              int per, int flags) {
  extern __shared__ uint32_t sm[];
  const int n = p.n;
  for (int64_t base = (int64_t)blockIdx.x * per; base < batch; base += (int64_t)gridDim.x * per) {
    const int cnt = (int)((batch - base) < (int64_t)per ? (batch - base) : (int64_t)per);
    for (int i = threadIdx.x; i < cnt * n; i += blockDim.x) {
      const int v = i / n, k = i - v * n;
      sm[v * n + brev_idx(k, p.lg)] = g_enc(x[(base + v) * n + k], p.F);
    }
    __syncthreads();
    smem_fnt(sm, cnt, p, inverse != 0);
    for (int i = threadIdx.x; i < cnt * n; i += blockDim.x) y[base * n + i] = g_out(sm[i], p.F, flags);
    __syncthreads();
  }
}

__global__ void k_conv_real_generic(DevPlan p, const int64_t* x, const int64_t* h, int64_t h_stride,
                                    int64_t* z, int64_t batch, int per, int flags) {
  extern __shared__ uint32_t sm[];
  const int n = p.n;
  uint32_t* sx = sm;
  uint32_t* sh = sm + per * n;
  for (int64_t base = (int64_t)blockIdx.x * per; base < batch; base += (int64_t)gridDim.x * per) {
    const int cnt = (int)((batch - base) < (int64_t)per ? (batch - base) : (int64_t)per);
    for (int i = threadIdx.x; i < cnt * n; i += blockDim.x) {
      const int v = i / n, k = i - v * n;
      sx[v * n + brev_idx(k, p.lg)] = g_enc(x[(base + v) * n + k], p.F);
      sh[v * n + brev_idx(k, p.lg)] = g_enc(h[(base + v) * h_stride + k], p.F);
    }
    __syncthreads();
    smem_fnt(sx, cnt, p, false);
    smem_fnt(sh, cnt, p, false);
    for (int i = threadIdx.x; i < cnt * n; i += blockDim.x) sx[i] = g_mul(sx[i], sh[i], p.F);
    __syncthreads();
    for (int i = threadIdx.x; i < cnt * n; i += blockDim.x) {
      const int v = i / n, k = i - v * n;
      sh[v * n + brev_idx(k, p.lg)] = sx[i];
    }
    __syncthreads();
    smem_fnt(sh, cnt, p, true);
    for (int i = threadIdx.x; i < cnt * n; i += blockDim.x) z[base * n + i] = g_out(sh[i], p.F, flags);
    __syncthreads();
  }
}

__global__ void k_conv_complex_generic(DevPlan p, const int64_t* xr, const int64_t* xi,
                                       const int64_t* yr, const int64_t* yi, int64_t y_stride,
                                       int64_t* zr, int64_t* zi, int64_t batch, int per, int flags) {
  extern __shared__ uint32_t sm[];
  const int n = p.n;
  const uint32_t F = p.F;
  const int q = 1 << p.t;
  const uint32_t j = (uint32_t)(1u << (q / 2)) % F;
  uint32_t* s0 = sm;
  uint32_t* s1 = sm + per * n;
  uint32_t* s2 = sm + 2 * per * n;
  uint32_t* s3 = sm + 3 * per * n;
  // c_re = -2^(q-1), c_im = -2^(q/2-1) (fnt.py:157-158)
  const uint32_t c_re = (F - (uint32_t)((1ull << (q - 1)) % F)) % F;
  const uint32_t c_im = (F - (uint32_t)((1ull << (q / 2 - 1)) % F)) % F;
  for (int64_t base = (int64_t)blockIdx.x * per; base < batch; base += (int64_t)gridDim.x * per) {
    const int cnt = (int)((batch - base) < (int64_t)per ? (batch - base) : (int64_t)per);
    for (int i = threadIdx.x; i < cnt * n; i += blockDim.x) {
      const int v = i / n, k = i - v * n;
      const int d = v * n + brev_idx(k, p.lg);
      s0[d] = g_enc(xr[(base + v) * n + k], F);
      s1[d] = g_enc(xi[(base + v) * n + k], F);
      s2[d] = g_enc(yr[(base + v) * y_stride + k], F);
      s3[d] = g_enc(yi[(base + v) * y_stride + k], F);
    }
    __syncthreads();
    smem_fnt(s0, cnt, p, false);
    smem_fnt(s1, cnt, p, false);
    smem_fnt(s2, cnt, p, false);
    smem_fnt(s3, cnt, p, false);
    for (int i = threadIdx.x; i < cnt * n; i += blockDim.x) {
      const uint32_t jx = g_mul(j, s1[i], F), jy = g_mul(j, s3[i], F);
      const uint32_t ap = (s0[i] + jx) % F, am = (s0[i] + F - jx) % F;
      const uint32_t bp = (s2[i] + jy) % F, bm = (s2[i] + F - jy) % F;
      const uint32_t up = g_mul(ap, bp, F), um = g_mul(am, bm, F);
      s2[i] = (up + um) % F;
      s3[i] = (up + F - um) % F;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < cnt * n; i += blockDim.x) {
      const int v = i / n, k = i - v * n;
      s0[v * n + brev_idx(k, p.lg)] = s2[i];
      s1[v * n + brev_idx(k, p.lg)] = s3[i];
    }
    __syncthreads();
    smem_fnt(s0, cnt, p, true);
    smem_fnt(s1, cnt, p, true);
    for (int i = threadIdx.x; i < cnt * n; i += blockDim.x) {
      zr[base * n + i] = g_out(g_mul(s0[i], c_re, F), F, flags);
      zi[base * n + i] = g_out(g_mul(s1[i], c_im, F), F, flags);
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// launchers

static int g_num_sms() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

static int generic_per(int n, int arrays) {
  int per = 1024 / n;
  if (per < 1) per = 1;
  (void)arrays;
  return per;
}

static unsigned grid_for(int64_t items, int per_cta) {
  int64_t g = (items + per_cta - 1) / per_cta;
  int64_t cap = (int64_t)g_num_sms() * 16;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (unsigned)g;
}

static cudaError_t smem_cfg(const void* fn, size_t bytes) {
  if (bytes > 48 * 1024)
    return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  return cudaSuccess;
}

cudaError_t launch_fnt(const DevPlan& p, int inverse, const int64_t* x, int64_t* y, int64_t batch,
                       int flags, cudaStream_t st) {
  if (batch <= 0) return cudaSuccess;
  if (p.kind == KIND_SQRT2_64) {
    k_fnt_fast<64, SQRT2><<<(unsigned)((batch + TILE - 1) / TILE), TILE, 0, st>>>(x, y, batch, inverse, flags);
  } else if (p.kind == KIND_RADIX2_32) {
    k_fnt_fast<32, RADIX2><<<(unsigned)((batch + TILE - 1) / TILE), TILE, 0, st>>>(x, y, batch, inverse, flags);
  } else {
    const int per = generic_per(p.n, 1);
    const size_t sm = (size_t)per * p.n * sizeof(uint32_t);
    cudaError_t e = smem_cfg((const void*)k_fnt_generic, sm);
    if (e != cudaSuccess) return e;
    k_fnt_generic<<<grid_for(batch, per), 256, sm, st>>>(p, inverse, x, y, batch, per, flags);
  }
  return cudaGetLastError();
}

cudaError_t launch_conv_real(const DevPlan& p, const int64_t* x, const int64_t* h, int64_t h_stride,
                             int64_t* z, int64_t batch, int flags, cudaStream_t st) {
  if (batch <= 0) return cudaSuccess;
  if (p.kind == KIND_SQRT2_64 && h_stride != 0) {
    k_conv_real_pair<64, SQRT2><<<(unsigned)((batch + PAIR_TILE - 1) / PAIR_TILE), 2 * PAIR_TILE, 0, st>>>(
        x, h, z, batch, flags);
  } else if (p.kind == KIND_SQRT2_64) {
    k_conv_real_fast<64, SQRT2><<<(unsigned)((batch + TILE - 1) / TILE), TILE, 0, st>>>(x, h, h_stride, z, batch, flags);
  } else if (p.kind == KIND_RADIX2_32) {
    k_conv_real_fast<32, RADIX2><<<(unsigned)((batch + TILE - 1) / TILE), TILE, 0, st>>>(x, h, h_stride, z, batch, flags);
  } else {
    const int per = generic_per(p.n, 2);
    const size_t sm = 2 * (size_t)per * p.n * sizeof(uint32_t);
    cudaError_t e = smem_cfg((const void*)k_conv_real_generic, sm);
    if (e != cudaSuccess) return e;
    k_conv_real_generic<<<grid_for(batch, per), 256, sm, st>>>(p, x, h, h_stride, z, batch, per, flags);
  }
  return cudaGetLastError();
}

cudaError_t launch_conv_complex(const DevPlan& p, const int64_t* xr, const int64_t* xi,
                                const int64_t* yr, const int64_t* yi, int64_t y_stride,
                                int64_t* zr, int64_t* zi, int64_t batch, int flags,
                                cudaStream_t st) {
  if (batch <= 0) return cudaSuccess;
  if (p.kind == KIND_SQRT2_64) {
    const size_t sm = (2 * TILE + 2 * (y_stride != 0 ? TILE : 1)) * (64 + 1) * sizeof(uint32_t);
    cudaError_t e = smem_cfg((const void*)k_conv_complex_fast<64, SQRT2>, sm);
    if (e != cudaSuccess) return e;
    k_conv_complex_fast<64, SQRT2><<<(unsigned)((batch + TILE - 1) / TILE), TILE, sm, st>>>(
        xr, xi, yr, yi, y_stride, zr, zi, batch, flags);
  } else if (p.kind == KIND_RADIX2_32) {
    const size_t sm = (2 * TILE + 2 * (y_stride != 0 ? TILE : 1)) * (32 + 1) * sizeof(uint32_t);
    k_conv_complex_fast<32, RADIX2><<<(unsigned)((batch + TILE - 1) / TILE), TILE, sm, st>>>(
        xr, xi, yr, yi, y_stride, zr, zi, batch, flags);
  } else {
    const int per = generic_per(p.n, 4);
    const size_t sm = 4 * (size_t)per * p.n * sizeof(uint32_t);
    cudaError_t e = smem_cfg((const void*)k_conv_complex_generic, sm);
    if (e != cudaSuccess) return e;
    k_conv_complex_generic<<<grid_for(batch, per), 256, sm, st>>>(p, xr, xi, yr, yi, y_stride, zr,
                                                                  zi, batch, per, flags);
  }
  return cudaGetLastError();
}

}  // namespace fntgpu
