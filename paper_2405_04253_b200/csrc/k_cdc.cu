// k_cdc.cu -- fused FNT-CDC overlap-save kernel (cdc64 plan).
//
// Reference: fntdsp/cdc.py:89-95 (_overlap_save_blocks), 124-135 (tap spectra),
// 141-156 (_convolve_blocks), 165-180 (process_int / process) and the CDC->AEQ glue
// of linksim.py:283-308, 399-404 (float rescale, requantization, decimation metric).
//
// A CTA owns CDC_BLK = 64 consecutive 64-sample overlap-save blocks (hop 32) of one
// stream. Each block is split over two threads in different warps (warp-uniform
// sign, so the two halves of Eqs. (7)-(8) are branch-free):
//   sign +: a+ = x_r + 2^8 x_i  ->  FNT-64  ->  * b+'  ->  IFNT-64 (outputs 32..63)
//   sign -: a- = x_r - 2^8 x_i  ->  FNT-64  ->  * b-'  ->  IFNT-64 (outputs 32..63)
// (b+- pre-scaled by c_re * N^-1 = 2^25; radix-sqrt2 DIT with rotate-only twiddles
// in Z/(2^32-1), fermat.cuh). The epilogue combines z_re = u+ + u-,
// z_im = 2^24 (u+ - u-), folds mod F4 and decodes, then streams the contiguous
// output range of the CTA (and the fused requantization / decimation
// statistics) with coalesced stores. One HBM read per input sample (the 32-sample
// halo between neighbouring blocks is re-read from shared memory) and one HBM
// write per output.
#include <type_traits>

#include "fermat.cuh"
#include "internal.h"

namespace fntgpu {

constexpr int CDC_CTA = 128;                    // threads
constexpr int CDC_BLK = 64;                     // overlap-save blocks per CTA
constexpr int CDC_N = 64;
constexpr int CDC_HOP = 32;
constexpr int WIN = CDC_HOP * (CDC_BLK + 1);    // input samples staged per plane
constexpr int UP = 33;                          // padded pitch of the u staging rows

struct CdcArgs {
  uint32_t bp[CDC_N];  // b+ * 2^25 mod F4
  uint32_t bm[CDC_N];  // b- * 2^25 mod F4
  fntgpu_cdc_io io;
  int64_t blk_begin;   // first overlap-save block index of this launch
  int64_t blk_count;   // blocks per stream
  int32_t c;           // n_taps // 2
};

__device__ __forceinline__ int32_t sext8(uint32_t w, int k) {
  return (int32_t)(w << (24 - 8 * k)) >> 24;
}

// Stage the CTA's input window [g0, g0 + WIN) of one plane into shared memory,
// zero outside the stream [0, L). int8 planes move in 16-byte vectors.
template <typename TIN, typename TS>
__device__ __forceinline__ void stage_plane(TS* dst, const TIN* src, int64_t g0,
                                            const fntgpu_cdc_io& io) {
  const int64_t lo = io.x_first > 0 ? io.x_first : 0;
  const int64_t hi_avail = io.x_first + io.x_count;
  const int64_t hi = hi_avail < io.length ? hi_avail : io.length;
  if (sizeof(TIN) == 1) {
    constexpr int CH = WIN / 16;
    for (int ch = threadIdx.x; ch < CH; ch += blockDim.x) {
      const int64_t g = g0 + 16 * ch;
      const TIN* p = src + (g - io.x_first);
      uint4 v;
      if (g >= lo && g + 16 <= hi && ((reinterpret_cast<uintptr_t>(p) & 15) == 0)) {
        v = __ldg(reinterpret_cast<const uint4*>(p));
      } else {
        uint32_t w[4] = {0u, 0u, 0u, 0u};
        for (int k = 0; k < 16; ++k) {
          const int64_t gk = g + k;
          if (gk >= lo && gk < hi) w[k >> 2] |= ((uint32_t)(uint8_t)src[gk - io.x_first]) << (8 * (k & 3));
        }
        v = make_uint4(w[0], w[1], w[2], w[3]);
      }
      reinterpret_cast<uint4*>(dst)[ch] = v;
    }
  } else {
    for (int i = threadIdx.x; i < WIN; i += blockDim.x) {
      const int64_t g = g0 + i;
      dst[i] = (g >= lo && g < hi) ? (TS)src[g - io.x_first] : (TS)0;
    }
  }
}

template <typename TIN>
__global__ void __launch_bounds__(CDC_CTA) k_cdc64(const __grid_constant__ CdcArgs A) {
  using TS = typename std::conditional<sizeof(TIN) == 1, int8_t, int32_t>::type;
  constexpr int IN_BYTES = 2 * WIN * (int)sizeof(TS);
  constexpr int U_BYTES = 2 * CDC_BLK * UP * 4;
  // the input window and the u staging rows are never live at the same time
  __shared__ __align__(16) unsigned char smem[IN_BYTES > U_BYTES ? IN_BYTES : U_BYTES];
  TS* s_xr = reinterpret_cast<TS*>(smem);
  TS* s_xi = s_xr + WIN;
  uint32_t* s_u = reinterpret_cast<uint32_t*>(smem);  // [sign][block][UP]

  const fntgpu_cdc_io& io = A.io;
  const int s = blockIdx.y;
  const int64_t cta_blk0 = A.blk_begin + (int64_t)blockIdx.x * CDC_BLK;
  const int64_t g0 = cta_blk0 * CDC_HOP - CDC_HOP;  // first input sample of block cta_blk0

  const TIN* xr_s = reinterpret_cast<const TIN*>(io.xr) + (size_t)s * io.x_stride;
  const TIN* xi_s = reinterpret_cast<const TIN*>(io.xi) + (size_t)s * io.x_stride;
  stage_plane<TIN, TS>(s_xr, xr_s, g0, io);
  stage_plane<TIN, TS>(s_xi, xi_s, g0, io);
  __syncthreads();

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int sgn = warp & 1;                   // 0: a+ / b+, 1: a- / b-
  const int bl = (warp >> 1) * 32 + lane;     // block within the CTA
  const int32_t m256 = sgn ? -256 : 256;
  uint32_t a[CDC_N];
  {
    const TS* wr = s_xr + bl * CDC_HOP;
    const TS* wi = s_xi + bl * CDC_HOP;
    if (sizeof(TS) == 1) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint4 r4 = reinterpret_cast<const uint4*>(wr)[q];
        const uint4 i4 = reinterpret_cast<const uint4*>(wi)[q];
        const uint32_t rw[4] = {r4.x, r4.y, r4.z, r4.w};
        const uint32_t iw[4] = {i4.x, i4.y, i4.z, i4.w};
#pragma unroll
        for (int w = 0; w < 4; ++w)
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int i = q * 16 + w * 4 + k;
            // x_r +- 2^8 x_i + bias (bias = 256 F4 keeps the word non-negative)
            a[bitrev(i, 6)] = (uint32_t)(sext8(rw[w], k) + (int32_t)F4_BIAS + m256 * sext8(iw[w], k));
          }
      }
    } else {
#pragma unroll
      for (int i = 0; i < CDC_N; ++i)
        a[bitrev(i, 6)] = (uint32_t)((int32_t)wr[i] + (int32_t)F4_BIAS + m256 * (int32_t)wi[i]);
    }
  }
  fnt_dit<CDC_N, SQRT2, false>(a);
  const uint32_t* B = sgn ? A.bm : A.bp;
#pragma unroll
  for (int k = 0; k < CDC_N; ++k) a[k] = m_mul(a[k], B[k]);  // the 64 general products
  to_bitrev<CDC_N>(a);
  fnt_dit<CDC_N, SQRT2, true, false, true>(a);             // outputs 32..63 only
  __syncthreads();  // every thread has consumed the input window
  {
    uint32_t* row = s_u + (sgn * CDC_BLK + bl) * UP;
#pragma unroll
    for (int j = 0; j < CDC_HOP; ++j) row[j] = a[CDC_HOP + j];
  }
  __syncthreads();

  // ---- epilogue: outputs of this CTA are global indices [32*cta_blk0 - c, ... + 32*CDC_BLK)
  const int64_t n0 = cta_blk0 * CDC_HOP - A.c;
  int64_t lo = n0, hi = n0 + (int64_t)CDC_BLK * CDC_HOP;
  const int64_t o_lo = io.out_first, o_hi = io.out_first + io.out_count;
  lo = lo < o_lo ? o_lo : lo;
  hi = hi > o_hi ? o_hi : hi;
  // n advances by CDC_CTA (even): each thread only ever sees one sampling phase
  const int my_ph = (int)((lo + tid) & 1);
  unsigned long long s2 = 0, s4lo = 0, s4hi = 0;
  for (int64_t n = lo + tid; n < hi; n += CDC_CTA) {
    const int idx = (int)(n - n0);
    const int r = (idx >> 5) * UP + (idx & 31);
    const uint32_t up = s_u[r], um = s_u[CDC_BLK * UP + r];
    const int32_t zr = f4_signed(m_add(up, um));
    const int32_t zi = f4_signed(m_rot(m_sub(up, um), 24));
    const int64_t o = n - io.out_first;
    switch (io.out_dtype) {
      case FNTGPU_I16:
        reinterpret_cast<int16_t*>(io.yr)[s * io.y_stride + o] = (int16_t)zr;
        reinterpret_cast<int16_t*>(io.yi)[s * io.y_stride + o] = (int16_t)zi;
        break;
      case FNTGPU_I32:
        reinterpret_cast<int32_t*>(io.yr)[s * io.y_stride + o] = zr;
        reinterpret_cast<int32_t*>(io.yi)[s * io.y_stride + o] = zi;
        break;
      case FNTGPU_I64:
        reinterpret_cast<int64_t*>(io.yr)[s * io.y_stride + o] = zr;
        reinterpret_cast<int64_t*>(io.yi)[s * io.y_stride + o] = zi;
        break;
      case FNTGPU_C128: {
        double2 v;
        v.x = __dmul_rn((double)zr, io.inv_scale);  // numpy complex / real == * (1/scale) (cdc.py:180)
        v.y = __dmul_rn((double)zi, io.inv_scale);
        reinterpret_cast<double2*>(io.yr)[s * io.y_stride + o] = v;
        break;
      }
      default:
        break;
    }
    if (io.qr) {
      // quantize_real(s, spec) on s = y_int * (1/output_scale)  (linksim.py:404)
      const double vr = __dmul_rn(__dmul_rn((double)zr, io.inv_scale), io.q_scale);
      const double vi = __dmul_rn(__dmul_rn((double)zi, io.inv_scale), io.q_scale);
      double ar = floor(__dadd_rn(fabs(vr), 0.5)), ai = floor(__dadd_rn(fabs(vi), 0.5));
      const double qm = (double)io.q_max;
      ar = ar > qm ? qm : ar;
      ai = ai > qm ? qm : ai;
      io.qr[s * io.q_stride + o] = (int8_t)(vr < 0 ? -(int)ar : (int)ar);
      io.qi[s * io.q_stride + o] = (int8_t)(vi < 0 ? -(int)ai : (int)ai);
    }
    if (io.decim_acc) {
      const unsigned long long m2 =
          (unsigned long long)((int64_t)zr * zr) + (unsigned long long)((int64_t)zi * zi);
      const unsigned long long m4 = m2 * m2;  // |y|^4 < 2^62
      s2 += m2;
      s4lo += m4;
      s4hi += (s4lo < m4);
    }
  }
  if (io.decim_acc) {
    // exact integer statistics: warp-reduce 32-bit limbs per phase, one atomic per value
    const unsigned long long v[4] = {s2, s4lo & 0xffffffffull, s4lo >> 32, s4hi};
#pragma unroll
    for (int ph = 0; ph < 2; ++ph) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        unsigned long long x = my_ph == ph ? v[k] : 0ull;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) x += __shfl_xor_sync(0xffffffffu, x, off);
        if ((tid & 31) == 0 && x) atomicAdd(io.decim_acc + ((int64_t)s * 2 + ph) * 4 + k, x);
      }
    }
  }
}

// Reduce the fused statistics to the decimation phase (linksim.py:249-260):
// metric(ph) = sum_pols mean(|d|^4) / mean(|d|^2)^2 ; scale-free, so the integer
// outputs stand in for d = y_int / output_scale.
__global__ void k_decim_phase(const fntgpu_decim_io io) {
  const int l = blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= io.n_links) return;
  double m[2] = {0.0, 0.0};
  for (int ph = 0; ph < 2; ++ph) {
    const double cnt = (double)((io.length - ph + 1) / 2);
    for (int pol = 0; pol < 2; ++pol) {
      const unsigned long long* a = io.acc + (((int64_t)(2 * l + pol)) * 2 + ph) * 4;
      const double S2 = (double)a[0];
      const double S4 = (double)a[3] * 18446744073709551616.0 + (double)a[2] * 4294967296.0 + (double)a[1];
      const double p2 = S2 / cnt;
      m[ph] += (S4 / cnt) / (p2 * p2);
    }
  }
  io.phase[l] = m[1] < m[0] ? 1 : 0;  // first minimum wins (strict <, linksim.py:258)
  if (io.gap) {
    const double mx = m[0] > m[1] ? m[0] : m[1];
    io.gap[l] = mx > 0 ? fabs(m[0] - m[1]) / mx : 0.0;
  }
}

static inline void scale_taps(const uint32_t* src, uint32_t* dst) {
  for (int k = 0; k < CDC_N; ++k) dst[k] = (uint32_t)(((uint64_t)src[k] % F4) * (1ull << 25) % F4);
}

cudaError_t launch_cdc64(const fntgpu_cdc_taps& taps, const fntgpu_cdc_io& io, cudaStream_t st) {
  if (io.out_count <= 0 || io.n_streams <= 0) return cudaSuccess;
  CdcArgs A;
  scale_taps(taps.b_plus, A.bp);
  scale_taps(taps.b_minus, A.bm);
  A.io = io;
  A.c = taps.n_taps / 2;
  // blocks B needed for outputs n in [out_first, out_first+out_count): B = (n + c) / 32
  const int64_t b_lo = (io.out_first + A.c) / CDC_HOP;
  const int64_t b_hi = (io.out_first + io.out_count - 1 + A.c) / CDC_HOP;
  A.blk_begin = b_lo;
  A.blk_count = b_hi - b_lo + 1;
  dim3 grid((unsigned)((A.blk_count + CDC_BLK - 1) / CDC_BLK), (unsigned)io.n_streams);
  switch (io.in_dtype) {
    case FNTGPU_I8: k_cdc64<int8_t><<<grid, CDC_CTA, 0, st>>>(A); break;
    case FNTGPU_I32: k_cdc64<int32_t><<<grid, CDC_CTA, 0, st>>>(A); break;
    case FNTGPU_I64: k_cdc64<int64_t><<<grid, CDC_CTA, 0, st>>>(A); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_decim_phase(const fntgpu_decim_io& io, cudaStream_t s) {
  if (io.n_links <= 0) return cudaSuccess;
  k_decim_phase<<<(io.n_links + 127) / 128, 128, 0, s>>>(io);
  return cudaGetLastError();
}

}  // namespace fntgpu
