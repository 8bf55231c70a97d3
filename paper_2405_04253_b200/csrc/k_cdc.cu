// k_cdc.cu -- fused FNT-CDC overlap-save kernel (cdc64 plan).
//
// Reference: fntdsp/cdc.py:89-95 (_overlap_save_blocks), 124-135 (tap spectra),
// 141-156 (_convolve_blocks), 165-180 (process_int / process) and the CDC->AEQ glue
// of linksim.py:283-308, 399-404 (float rescale, requantization, decimation metric).
//
// One thread owns one 64-sample overlap-save block (hop 32) and produces its 32
// valid outputs; a CTA owns CDC_CTA consecutive blocks. Per thread:
//   a+- = x_r +- 2^8 x_i (time domain, linearity of the FNT)         64 x 3 ops
//   FNT-64(a+), FNT-64(a-)  radix-sqrt2 DIT, rotates in Z/(2^32-1)   2 x 192 butterflies
//   u+- = a+- * b+-'   (b+- pre-scaled by c_re * N^-1 = 2^25)         128 products
//   IFNT-64(u+), IFNT-64(u-) with the last stage pruned to outputs 32..63
//   z_re = u+ + u-,  z_im = 2^24 (u+ - u-)   -> fold mod F4, signed decode
// so the whole block is one HBM read of the input and one write of the output.
// Inputs are staged into shared memory once per CTA (the 32-sample halo between
// neighbouring blocks is read from shared memory, not re-fetched from HBM), and
// outputs are staged so the global stores are contiguous across the CTA.
#include <type_traits>

#include "fermat.cuh"
#include "internal.h"

namespace fntgpu {

constexpr int CDC_CTA = 128;
constexpr int CDC_N = 64;
constexpr int CDC_HOP = 32;
constexpr int OUT_PITCH = 33;  // padded row pitch of the output staging tile (bank-conflict free)

struct CdcArgs {
  uint32_t bp[CDC_N];  // b+ * 2^25 mod F4
  uint32_t bm[CDC_N];  // b- * 2^25 mod F4
  fntgpu_cdc_io io;
  int64_t blk_begin;   // first overlap-save block index of this launch
  int64_t blk_count;   // blocks per stream
  int32_t c;           // n_taps // 2
};

template <typename T>
__device__ __forceinline__ int32_t ld_in(const void* base, int64_t idx) {
  return (int32_t)reinterpret_cast<const T*>(base)[idx];
}

__device__ __forceinline__ int32_t sext8(uint32_t w, int k) {
  return (int32_t)(w << (24 - 8 * k)) >> 24;
}

// Stage the CTA's input window [g0, g0 + n) of one plane into shared memory (zero
// outside the stream [0, L)). TIN = int8 uses byte smem, wider inputs int32 smem.
template <typename TIN, typename TS>
__device__ __forceinline__ void stage_plane(TS* dst, const void* src, int64_t g0, int n,
                                            const fntgpu_cdc_io& io) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int64_t g = g0 + i;
    int32_t v = 0;
    if (g >= 0 && g < io.length) v = ld_in<TIN>(src, g - io.x_first);
    dst[i] = (TS)v;
  }
}

template <typename TIN>
__global__ void __launch_bounds__(CDC_CTA) k_cdc64(const __grid_constant__ CdcArgs A) {
  using TS = typename std::conditional<sizeof(TIN) == 1, int8_t, int32_t>::type;
  constexpr int WIN = CDC_HOP * (CDC_CTA + 1);
  constexpr int IN_BYTES = 2 * WIN * (int)sizeof(TS);
  constexpr int OUT_BYTES = 2 * CDC_CTA * OUT_PITCH * 4;
  // input staging and output staging are never live at the same time: one buffer
  __shared__ __align__(16) unsigned char smem[IN_BYTES > OUT_BYTES ? IN_BYTES : OUT_BYTES];
  TS* s_xr = reinterpret_cast<TS*>(smem);
  TS* s_xi = s_xr + WIN;
  int32_t* s_or = reinterpret_cast<int32_t*>(smem);
  int32_t* s_oi = s_or + CDC_CTA * OUT_PITCH;

  const fntgpu_cdc_io& io = A.io;
  const int s = blockIdx.y;
  const int64_t cta_blk0 = A.blk_begin + (int64_t)blockIdx.x * CDC_CTA;
  const int64_t g0 = cta_blk0 * CDC_HOP - CDC_HOP;  // first input sample of block cta_blk0

  const int es = sizeof(TIN);
  const char* xr_s = reinterpret_cast<const char*>(io.xr) + (size_t)s * io.x_stride * es;
  const char* xi_s = reinterpret_cast<const char*>(io.xi) + (size_t)s * io.x_stride * es;
  stage_plane<TIN, TS>(s_xr, xr_s, g0, WIN, io);
  stage_plane<TIN, TS>(s_xi, xi_s, g0, WIN, io);
  __syncthreads();

  const int tid = threadIdx.x;
  const bool active = cta_blk0 + tid < A.blk_begin + A.blk_count;
  uint32_t ap[CDC_N], am[CDC_N];
  {
    const TS* wr = s_xr + tid * CDC_HOP;
    const TS* wi = s_xi + tid * CDC_HOP;
    if (sizeof(TS) == 1) {
      const uint4* vr = reinterpret_cast<const uint4*>(wr);
      const uint4* vi = reinterpret_cast<const uint4*>(wi);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint4 r4 = vr[q], i4 = vi[q];
        const uint32_t rw[4] = {r4.x, r4.y, r4.z, r4.w};
        const uint32_t iw[4] = {i4.x, i4.y, i4.z, i4.w};
#pragma unroll
        for (int w = 0; w < 4; ++w)
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int i = q * 16 + w * 4 + k;
            const int32_t xr = sext8(rw[w], k), xi = sext8(iw[w], k);
            const int32_t t = xr + (int32_t)F4_BIAS;
            const uint32_t p = (uint32_t)(t + xi * 256);
            ap[bitrev(i, 6)] = p;
            am[bitrev(i, 6)] = (uint32_t)(2 * t) - p;  // x_r - 2^8 x_i + bias
          }
      }
    } else {
#pragma unroll
      for (int i = 0; i < CDC_N; ++i) {
        const int32_t xr = (int32_t)wr[i], xi = (int32_t)wi[i];
        const int32_t t = xr + (int32_t)F4_BIAS;
        const uint32_t p = (uint32_t)(t + xi * 256);
        ap[bitrev(i, 6)] = p;
        am[bitrev(i, 6)] = (uint32_t)(2 * t) - p;
      }
    }
  }
  __syncthreads();  // the input window is dead; smem is reused for the outputs
  if (active) {
    fnt_dit<CDC_N, SQRT2, false>(ap);
    fnt_dit<CDC_N, SQRT2, false>(am);
#pragma unroll
    for (int k = 0; k < CDC_N; ++k) {
      ap[k] = m_mul(ap[k], A.bp[k]);
      am[k] = m_mul(am[k], A.bm[k]);
    }
    to_bitrev<CDC_N>(ap);
    to_bitrev<CDC_N>(am);
    fnt_dit<CDC_N, SQRT2, true, false, true>(ap);
    fnt_dit<CDC_N, SQRT2, true, false, true>(am);
    int32_t* orow = s_or + tid * OUT_PITCH;
    int32_t* irow = s_oi + tid * OUT_PITCH;
#pragma unroll
    for (int j = 0; j < CDC_HOP; ++j) {
      const uint32_t up = ap[CDC_HOP + j], um = am[CDC_HOP + j];
      orow[j] = f4_signed(m_add(up, um));
      irow[j] = f4_signed(m_rot(m_sub(up, um), 24));
    }
  }
  __syncthreads();

  // ---- epilogue: outputs of this CTA are global indices [32*cta_blk0 - c, ... + 32*CDC_CTA)
  const int64_t n0 = cta_blk0 * CDC_HOP - A.c;
  int64_t lo = n0, hi = n0 + (int64_t)CDC_CTA * CDC_HOP;
  const int64_t o_lo = io.out_first, o_hi = io.out_first + io.out_count;
  lo = lo < o_lo ? o_lo : lo;
  hi = hi > o_hi ? o_hi : hi;
  // n advances by CDC_CTA (even): each thread only ever sees one sampling phase
  const int my_ph = (int)((lo + tid) & 1);
  unsigned long long s2 = 0, s4lo = 0, s4hi = 0;
  for (int64_t n = lo + tid; n < hi; n += CDC_CTA) {
    const int idx = (int)(n - n0);
    const int32_t zr = s_or[(idx >> 5) * OUT_PITCH + (idx & 31)];
    const int32_t zi = s_oi[(idx >> 5) * OUT_PITCH + (idx & 31)];
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
  dim3 grid((unsigned)((A.blk_count + CDC_CTA - 1) / CDC_CTA), (unsigned)io.n_streams);
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
