// k_transform.cu -- batched FNT / IFNT and fused cyclic convolutions.
//
// Reference: fntdsp/fnt.py:86-161 (_butterflies, fnt, ifnt, cyclic_convolve_real,
// cyclic_convolve_complex) and fermat.py:124-133 (encode/decode arrays).
//
// Fast path (aeq32: alpha = 2, N = 32; cdc64: alpha = sqrt2 = 4080, N = 64):
//   one thread owns one length-N vector in registers; the DIT network is fully
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

template <int N>
__device__ __forceinline__ void store_vec(int64_t* __restrict__ y, const uint32_t (&a)[N], int flags) {
#pragma unroll
  for (int i = 0; i < N; ++i) {
    y[i] = (flags & FNTGPU_DECODE_SIGNED) ? (int64_t)f4_signed(a[i]) : (int64_t)f4_canon(a[i]);
  }
}

template <int N>
__device__ __forceinline__ void load_bitrev(uint32_t (&a)[N], const int64_t* __restrict__ x) {
  constexpr int LG = ilog2(N);
#pragma unroll
  for (int i = 0; i < N; ++i) a[bitrev(i, LG)] = f4_enc64(x[i]);
}

template <int N, int KIND>
__global__ void __launch_bounds__(128) k_fnt_fast(const int64_t* x, int64_t* y, int64_t batch,
                                                  int inverse, int flags) {
  constexpr int LG = ilog2(N);
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= batch) return;
  uint32_t a[N];
  load_bitrev<N>(a, x + b * N);
  if (inverse) {
    fnt_dit<N, KIND, true>(a);
#pragma unroll
    for (int i = 0; i < N; ++i) a[i] = m_rot(a[i], 32 - LG);  // * N^-1 = 2^-LG = 2^(32-LG)
  } else {
    fnt_dit<N, KIND, false>(a);
  }
  store_vec<N>(y + b * N, a, flags);
}

template <int N, int KIND>
__global__ void __launch_bounds__(128) k_conv_real_fast(const int64_t* x, const int64_t* h,
                                                        int64_t h_stride, int64_t* z,
                                                        int64_t batch, int flags) {
  constexpr int LG = ilog2(N);
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= batch) return;
  uint32_t X[N], H[N];
  load_bitrev<N>(X, x + b * N);
  load_bitrev<N>(H, h + b * h_stride);
  fnt_dit<N, KIND, false>(X);
  fnt_dit<N, KIND, false>(H);
#pragma unroll
  for (int i = 0; i < N; ++i) X[i] = m_mul(X[i], H[i]);  // the N general products (fnt.py:123)
  to_bitrev<N>(X);
  fnt_dit<N, KIND, true>(X);
#pragma unroll
  for (int i = 0; i < N; ++i) X[i] = m_rot(X[i], 32 - LG);
  store_vec<N>(z + b * N, X, flags);
}

// Eqs. (7)-(8): a+- = X_r +- 2^8 X_i, b+- likewise (linearity lets us form them in
// the time domain), u+- = a+- * b+-, z_re = 2^-1 IFNT(u+ + u-), z_im = 2^-9 IFNT(u+ - u-).
template <int N, int KIND>
__global__ void __launch_bounds__(64) k_conv_complex_fast(const int64_t* xr, const int64_t* xi,
                                                           const int64_t* yr, const int64_t* yi,
                                                           int64_t y_stride, int64_t* zr,
                                                           int64_t* zi, int64_t batch, int flags) {
  constexpr int LG = ilog2(N);
  const int64_t b0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool live = b0 < batch;
  const int64_t b = live ? b0 : batch - 1;  // idle lanes recompute the last vector, store nothing
  // u+ is parked in shared memory (padded rows) while u- is formed: three live
  // N-word arrays would not fit the register file for N = 64.
  __shared__ uint32_t sU[64][N + 1];
  uint32_t* U = sU[threadIdx.x];
  uint32_t A[N], B[N];
  // u+ = FNT(x_r + j x_i) * FNT(y_r + j y_i)
#pragma unroll
  for (int i = 0; i < N; ++i) {
    const int p = bitrev(i, LG);
    A[p] = m_add(f4_enc64(xr[b * N + i]), m_rot(f4_enc64(xi[b * N + i]), 8));
    B[p] = m_add(f4_enc64(yr[b * y_stride + i]), m_rot(f4_enc64(yi[b * y_stride + i]), 8));
  }
  fnt_dit<N, KIND, false>(A);
  fnt_dit<N, KIND, false>(B);
#pragma unroll
  for (int i = 0; i < N; ++i) U[i] = m_mul(A[i], B[i]);
  __syncwarp();  // scheduling fence: keeps the u- loads from being hoisted above (register pressure)
  // u- = FNT(x_r - j x_i) * FNT(y_r - j y_i)
#pragma unroll
  for (int i = 0; i < N; ++i) {
    const int p = bitrev(i, LG);
    A[p] = m_sub(f4_enc64(xr[b * N + i]), m_rot(f4_enc64(xi[b * N + i]), 8));
    B[p] = m_sub(f4_enc64(yr[b * y_stride + i]), m_rot(f4_enc64(yi[b * y_stride + i]), 8));
  }
  fnt_dit<N, KIND, false>(A);
  fnt_dit<N, KIND, false>(B);
#pragma unroll
  for (int i = 0; i < N; ++i) {
    const uint32_t um = m_mul(A[i], B[i]);
    const uint32_t up = U[i];
    A[i] = m_add(up, um);  // s = u+ + u-
    B[i] = m_sub(up, um);  // d = u+ - u-
  }
  to_bitrev<N>(A);
  to_bitrev<N>(B);
  fnt_dit<N, KIND, true>(A);
  fnt_dit<N, KIND, true>(B);
  // c_re * N^-1 = 2^-1 * 2^-LG ; c_im * N^-1 = 2^-9 * 2^-LG (fnt.py:155-158)
#pragma unroll
  for (int i = 0; i < N; ++i) {
    A[i] = m_rot(A[i], (64 - 1 - LG) & 31);
    B[i] = m_rot(B[i], (64 - 9 - LG) & 31);
  }
  if (live) {
    store_vec<N>(zr + b * N, A, flags);
    store_vec<N>(zi + b * N, B, flags);
  }
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
    k_fnt_fast<64, SQRT2><<<(unsigned)((batch + 63) / 64), 64, 0, st>>>(x, y, batch, inverse, flags);
  } else if (p.kind == KIND_RADIX2_32) {
    k_fnt_fast<32, RADIX2><<<(unsigned)((batch + 63) / 64), 64, 0, st>>>(x, y, batch, inverse, flags);
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
  if (p.kind == KIND_SQRT2_64) {
    k_conv_real_fast<64, SQRT2><<<(unsigned)((batch + 63) / 64), 64, 0, st>>>(x, h, h_stride, z, batch, flags);
  } else if (p.kind == KIND_RADIX2_32) {
    k_conv_real_fast<32, RADIX2><<<(unsigned)((batch + 63) / 64), 64, 0, st>>>(x, h, h_stride, z, batch, flags);
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
    k_conv_complex_fast<64, SQRT2><<<(unsigned)((batch + 63) / 64), 64, 0, st>>>(
        xr, xi, yr, yi, y_stride, zr, zi, batch, flags);
  } else if (p.kind == KIND_RADIX2_32) {
    k_conv_complex_fast<32, RADIX2><<<(unsigned)((batch + 63) / 64), 64, 0, st>>>(
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
