// k_cdc.cu -- fused FNT-CDC overlap-save kernel (cdc64 plan).
//
// Reference: fntdsp/cdc.py:89-95 (_overlap_save_blocks), 124-135 (tap spectra),
// 141-156 (_convolve_blocks), 165-180 (process_int / process) and the CDC->AEQ glue
// of linksim.py:283-308, 399-404 (float rescale, requantization, decimation metric).
//
// A CTA owns CDC_BLK = 128 consecutive 64-sample overlap-save blocks (hop 32) of one
// stream. Each block is split over two threads in different warps (warp-uniform
// sign, so the two halves of Eqs. (7)-(8) are branch-free):
//   sign +: a+ = x_r + 2^8 x_i  ->  FNT-64  ->  * b+'  ->  IFNT-64 (outputs 32..63)
//   sign -: a- = x_r - 2^8 x_i  ->  FNT-64  ->  * b-'  ->  IFNT-64 (outputs 32..63)
// (b+- pre-scaled by c_re * N^-1 = 2^25; radix-sqrt2 DIT with rotate-only twiddles
// in Z/(2^32-1), fermat.cuh; on int8 planes the first two stages run carry-free in
// plain int32). The epilogue combines z_re = u+ + u-, z_im = 2^24 (u+ - u-), reduces
// mod F4 (multiply-high) and decodes, then streams the contiguous output range of
// the CTA (and the fused requantization / decimation statistics) with coalesced
// stores. The CTA's input window arrives by two TMA bulk copies (interior windows
// of int8 planes) or 16-byte vector loads; one HBM read per input sample (the
// 32-sample halo between neighbouring blocks is re-read from shared memory) and
// one HBM write per output.
#include <type_traits>

#include "fermat.cuh"
#include "internal.h"

namespace fntgpu {

#ifndef CDC_MIN_CTAS
#define CDC_MIN_CTAS 3  // 3 x 256 threads per SM: caps registers at 80
#endif
#ifndef CDC_FWD_CM
#define CDC_FWD_CM FNT_CARRY_MODE  // carry form of the forward transform's modular stages
#endif
#ifndef CDC_INV_CM
#define CDC_INV_CM FNT_CARRY_MODE  // carry form of the inverse transform
#endif
#ifndef CDC_TMA
#define CDC_TMA 1  // interior input windows staged by cp.async.bulk (TMA) + mbarrier
#endif
#ifndef CDC_PROBE
#define CDC_PROBE 0  // timing probes only: 1 / 2 drop the fused requantization / statistics
#endif
#ifndef CDC_THREADS
#define CDC_THREADS 256  // 8 warps, 3 CTAs / SM: fewer independent instruction streams per SM
#endif                   // than 6 x 128 (the kernel is ~60 KB of straight-line code):
                         // 40.4 -> 37.7 ms at config 5, 133 -> 140 Gsamples/s at config 4
constexpr int CDC_CTA = CDC_THREADS;            // threads
constexpr int CDC_BLK = CDC_CTA / 2;            // overlap-save blocks per CTA (2 threads each)
constexpr int CDC_N = 64;
constexpr int CDC_HOP = 32;
constexpr int WIN = CDC_HOP * (CDC_BLK + 1);    // input samples staged per plane
#ifndef CDC_UP
#define CDC_UP 36
#endif
constexpr int UP = CDC_UP;                      // pitch of the u staging rows: 36 words keeps
                                                // rows 16-byte aligned (vector stores / loads)
                                                // with conflict-free 128-bit wavefronts

struct CdcArgs {
  uint32_t bp[CDC_N];  // b+ * 2^25 mod F4
  uint32_t bm[CDC_N];  // b- * 2^25 mod F4
  fntgpu_cdc_io io;
  int64_t blk_begin;   // first overlap-save block index of this launch
  int64_t blk_count;   // blocks per stream
  int32_t c;           // n_taps // 2
  int32_t s_base;      // first stream of this launch (grid.y is limited to 65535)
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

// Exact integer form of the AEQ-input requantization q = quantize_real(y * inv, q_scale)
// when inv * q_scale == 2^-k up to rounding: the float64 product is within 3 ulp of
// y / 2^k, so round-half-away agrees with the exact rounding except at exact ties
// |y| = 2^(k-1) + j 2^k, whose float64 outcome the host precomputed (io.q_tie).
__device__ __forceinline__ int32_t requant_int(int32_t y, int k, const int8_t* tie, int qmax) {
  const int32_t a = abs(y);
  const int32_t base = a >> k;
  const int32_t rem = a & ((1 << k) - 1);
  const int32_t half = 1 << (k - 1);
  int32_t q = base + (rem > half ? 1 : 0);
  if (rem == half) q = tie[base < qmax ? base : qmax];
  q = q < qmax ? q : qmax;
  return y < 0 ? -q : q;
}

// Chain epilogue: 4 consecutive outputs per thread, 32-bit indices, packed int8 /
// int16 stores, 32-bit |y|^2 and IMAD.WIDE |y|^4 statistics. Preconditions checked
// on the host (launch_cdc64): out_dtype in {NONE, I16}, q_shift >= 1 when
// requantizing, (c + out_first) % 4 == 0 and 4-byte aligned planes and strides.
__device__ __forceinline__ void cdc_epilogue_fast(const CdcArgs& A, const uint32_t* s_u, int s,
                                                  int64_t n0, int lo, int hi) {
  const fntgpu_cdc_io& io = A.io;
  const int tid = threadIdx.x;
  const int64_t base_o = n0 - io.out_first;  // output index of local index 0
  int8_t* qr = io.qr ? io.qr + s * io.q_stride + base_o : nullptr;
  int8_t* qi = io.qr ? io.qi + s * io.q_stride + base_o : nullptr;
  int16_t* yr = io.out_dtype == FNTGPU_I16 ? reinterpret_cast<int16_t*>(io.yr) + s * io.y_stride + base_o : nullptr;
  int16_t* yi = io.out_dtype == FNTGPU_I16 ? reinterpret_cast<int16_t*>(io.yi) + s * io.y_stride + base_o : nullptr;
  const bool stats = io.decim_acc != nullptr;
  const int k = io.q_shift, qmax = io.q_max;
  const int8_t* tie = io.q_tie;
  // accumulators for even (A) and odd (B) local indices
  unsigned long long a2 = 0, b2 = 0, a4 = 0, b4 = 0;
  uint32_t a4h = 0, b4h = 0;
  for (int v = 4 * tid; v < CDC_BLK * CDC_HOP; v += 4 * CDC_CTA) {
    if (v + 4 <= lo || v >= hi) continue;
    const bool full = v >= lo && v + 4 <= hi;
    const int rb = (v >> 5) * UP + (v & 31);
    int32_t zr[4], zi[4];
    uint32_t upv[4], umv[4];
    if (UP % 4 == 0) {
      const uint4 p4 = *reinterpret_cast<const uint4*>(s_u + rb);
      const uint4 m4 = *reinterpret_cast<const uint4*>(s_u + CDC_BLK * UP + rb);
      upv[0] = p4.x; upv[1] = p4.y; upv[2] = p4.z; upv[3] = p4.w;
      umv[0] = m4.x; umv[1] = m4.y; umv[2] = m4.z; umv[3] = m4.w;
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e) { upv[e] = s_u[rb + e]; umv[e] = s_u[CDC_BLK * UP + rb + e]; }
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const uint32_t up = upv[e], um = umv[e];
      zr[e] = (int32_t)f4_mod(m_add(up, um)) - 32768;
      zi[e] = (int32_t)f4_mod(m_rot(m_sub(up, um), 24)) - 32768;
    }
    if (CDC_PROBE != 1 && qr) {
      uint32_t pr = 0, pi = 0;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        pr |= ((uint32_t)requant_int(zr[e], k, tie, qmax) & 0xffu) << (8 * e);
        pi |= ((uint32_t)requant_int(zi[e], k, tie, qmax) & 0xffu) << (8 * e);
      }
      if (full) {
        *reinterpret_cast<uint32_t*>(qr + v) = pr;
        *reinterpret_cast<uint32_t*>(qi + v) = pi;
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (v + e >= lo && v + e < hi) {
            qr[v + e] = (int8_t)(pr >> (8 * e));
            qi[v + e] = (int8_t)(pi >> (8 * e));
          }
      }
    }
    if (yr) {
      if (full) {
        *reinterpret_cast<uint2*>(yr + v) = make_uint2(((uint32_t)zr[0] & 0xffffu) | ((uint32_t)zr[1] << 16),
                                                       ((uint32_t)zr[2] & 0xffffu) | ((uint32_t)zr[3] << 16));
        *reinterpret_cast<uint2*>(yi + v) = make_uint2(((uint32_t)zi[0] & 0xffffu) | ((uint32_t)zi[1] << 16),
                                                       ((uint32_t)zi[2] & 0xffffu) | ((uint32_t)zi[3] << 16));
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (v + e >= lo && v + e < hi) {
            yr[v + e] = (int16_t)zr[e];
            yi[v + e] = (int16_t)zi[e];
          }
      }
    }
    if (CDC_PROBE != 2 && stats) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const bool ok = full || (v + e >= lo && v + e < hi);
        const uint32_t m2 = ok ? (uint32_t)(zr[e] * zr[e]) + (uint32_t)(zi[e] * zi[e]) : 0u;  // <= 2^31
        const unsigned long long m4 = (unsigned long long)m2 * m2;                          // < 2^62
        if (e & 1) {
          b2 += m2;
          b4 += m4;
          b4h += (b4 < m4);
        } else {
          a2 += m2;
          a4 += m4;
          a4h += (a4 < m4);
        }
      }
    }
  }
  if (stats) {
    // even local indices carry phase (n0 & 1), odd ones the other phase
    const int pa = (int)(n0 & 1);
    const unsigned long long va[4] = {a2, a4 & 0xffffffffull, a4 >> 32, a4h};
    const unsigned long long vb[4] = {b2, b4 & 0xffffffffull, b4 >> 32, b4h};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      unsigned long long x = va[q], y = vb[q];
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        x += __shfl_xor_sync(0xffffffffu, x, off);
        y += __shfl_xor_sync(0xffffffffu, y, off);
      }
      if ((tid & 31) == 0) {
        if (x) atomicAdd(io.decim_acc + ((int64_t)s * 2 + pa) * 4 + q, x);
        if (y) atomicAdd(io.decim_acc + ((int64_t)s * 2 + (pa ^ 1)) * 4 + q, y);
      }
    }
  }
}

// sign-extended byte k of w: PRMT with the selector's sign-replication bit
__device__ __forceinline__ int32_t sx8(uint32_t w, int k) {
  int32_t r;
  const uint32_t sel = (uint32_t)k | ((uint32_t)(k | 8) << 4) | ((uint32_t)(k | 8) << 8) | ((uint32_t)(k | 8) << 12);
  asm("prmt.b32 %0, %1, 0, %2;" : "=r"(r) : "r"(w), "r"(sel));
  return r;
}

template <typename TIN, bool FAST>
__global__ void __launch_bounds__(CDC_CTA, CDC_MIN_CTAS) k_cdc64(const __grid_constant__ CdcArgs A) {
  using TS = typename std::conditional<sizeof(TIN) == 1, int8_t, int32_t>::type;
  // the input window and the u staging rows are never live at the same time
  extern __shared__ __align__(16) unsigned char smem[];
  TS* s_xr = reinterpret_cast<TS*>(smem);
  TS* s_xi = s_xr + WIN;
  uint32_t* s_u = reinterpret_cast<uint32_t*>(smem);  // [sign][block][UP]

  const fntgpu_cdc_io& io = A.io;
  const int s = A.s_base + (int)blockIdx.y;
  const int64_t cta_blk0 = A.blk_begin + (int64_t)blockIdx.x * CDC_BLK;
  const int64_t g0 = cta_blk0 * CDC_HOP - CDC_HOP;  // first input sample of block cta_blk0

  const TIN* xr_s = reinterpret_cast<const TIN*>(io.xr) + (size_t)s * io.x_stride;
  const TIN* xi_s = reinterpret_cast<const TIN*>(io.xi) + (size_t)s * io.x_stride;
  bool bulk = false;
  if (sizeof(TIN) == 1 && CDC_TMA) {
    // interior windows of int8 planes: two 1-D bulk copies (TMA engine) straight into
    // shared memory, completion counted on an mbarrier; edges and unaligned views
    // take the vectorised load path
    const int64_t lo = io.x_first > 0 ? io.x_first : 0;
    const int64_t hi_avail = io.x_first + io.x_count;
    const int64_t hi = hi_avail < io.length ? hi_avail : io.length;
    const TIN* pr = xr_s + (g0 - io.x_first);
    const TIN* pi = xi_s + (g0 - io.x_first);
    bulk = g0 >= lo && g0 + WIN <= hi && ((reinterpret_cast<uintptr_t>(pr) | reinterpret_cast<uintptr_t>(pi)) & 15) == 0;
    if (bulk) {
      __shared__ __align__(8) uint64_t mbar;
      const uint32_t mb = (uint32_t)__cvta_generic_to_shared(&mbar);
      if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(mb) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(mb), "r"(2 * WIN) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     :: "r"((uint32_t)__cvta_generic_to_shared(s_xr)), "l"(pr), "r"(WIN), "r"(mb) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     :: "r"((uint32_t)__cvta_generic_to_shared(s_xi)), "l"(pi), "r"(WIN), "r"(mb) : "memory");
      }
      __syncthreads();  // barrier initialised before anyone polls it
      uint32_t done = 0;
      while (!done) {
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\t"
                     "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(done) : "r"(mb) : "memory");
      }
    }
  }
  if (!bulk) {
    stage_plane<TIN, TS>(s_xr, xr_s, g0, io);
    stage_plane<TIN, TS>(s_xi, xi_s, g0, io);
  }
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
            // x_r +- 2^8 x_i as a plain signed integer (|a| <= 32896 < 2^16)
            a[bitrev(i, 6)] = (uint32_t)(sx8(rw[w], k) + m256 * sx8(iw[w], k));
          }
      }
    } else {
#pragma unroll
      for (int i = 0; i < CDC_N; ++i)
        a[bitrev(i, 6)] = (uint32_t)((int32_t)wr[i] + (int32_t)F4_BIAS + m256 * (int32_t)wi[i]);
    }
  }
  if (sizeof(TS) == 1) {
    // int8 planes: stages 0-1 (twiddles 1, 2^8) keep |values| < 2^26 in plain int32
    // arithmetic (no carries); a multiple of F4 above 2^26 then makes them
    // non-negative words of Z/M for stages 2-5
    fnt_stage_plain<CDC_N, SQRT2, 0, 2>(a);
#pragma unroll
    for (int k = 0; k < CDC_N; ++k) a[k] += F4 * 1024u;
    fnt_stage<CDC_N, SQRT2, false, false, false, 2, -1, CDC_FWD_CM>(a);
  } else {
    fnt_dit<CDC_N, SQRT2, false>(a);
  }
  const uint32_t* B = sgn ? A.bm : A.bp;
#pragma unroll
  for (int k = 0; k < CDC_N; ++k) a[k] = m_mul(a[k], B[k]);  // the 64 general products
  // decode offsets: +K on the DC bin adds K to every output of the (unscaled) inverse.
  // K+ = 16320, K- = 16448 put +32768 on both z_re = u+ + u- and z_im = 2^24 (u+ - u-)
  // (2^24 * -128 = -2^31 == 2^15 mod F4), so the epilogue decodes each value as
  // f4_mod(.) - 32768 (fermat.cuh) instead of a two-sided range fold.
  a[0] = m_add(a[0], sgn ? 16448u : 16320u);
  to_bitrev<CDC_N>(a);
  fnt_dit<CDC_N, SQRT2, true, false, true, CDC_INV_CM>(a);  // outputs 32..63 only
  __syncthreads();  // every thread has consumed the input window
  {
    uint32_t* row = s_u + (sgn * CDC_BLK + bl) * UP;
    if (UP % 4 == 0) {
#pragma unroll
      for (int j = 0; j < CDC_HOP; j += 4)
        *reinterpret_cast<uint4*>(row + j) = make_uint4(a[CDC_HOP + j], a[CDC_HOP + j + 1],
                                                        a[CDC_HOP + j + 2], a[CDC_HOP + j + 3]);
    } else {
#pragma unroll
      for (int j = 0; j < CDC_HOP; ++j) row[j] = a[CDC_HOP + j];
    }
  }
  __syncthreads();

  // ---- epilogue: outputs of this CTA are global indices [32*cta_blk0 - c, ... + 32*CDC_BLK)
  const int64_t n0 = cta_blk0 * CDC_HOP - A.c;
  int64_t lo = n0, hi = n0 + (int64_t)CDC_BLK * CDC_HOP;
  const int64_t o_lo = io.out_first, o_hi = io.out_first + io.out_count;
  lo = lo < o_lo ? o_lo : lo;
  hi = hi > o_hi ? o_hi : hi;
  if (FAST) {
    cdc_epilogue_fast(A, s_u, s, n0, (int)(lo - n0), (int)(hi - n0));
    return;
  }
  // n advances by CDC_CTA (even): each thread only ever sees one sampling phase
  const int my_ph = (int)((lo + tid) & 1);
  unsigned long long s2 = 0, s4lo = 0, s4hi = 0;
  for (int64_t n = lo + tid; n < hi; n += CDC_CTA) {
    const int idx = (int)(n - n0);
    const int r = (idx >> 5) * UP + (idx & 31);
    const uint32_t up = s_u[r], um = s_u[CDC_BLK * UP + r];
    const int32_t zr = (int32_t)f4_mod(m_add(up, um)) - 32768;
    const int32_t zi = (int32_t)f4_mod(m_rot(m_sub(up, um), 24)) - 32768;
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

template <typename TIN, bool FAST>
static cudaError_t launch_k(const CdcArgs& A, dim3 grid, cudaStream_t st) {
  using TS = typename std::conditional<sizeof(TIN) == 1, int8_t, int32_t>::type;
  constexpr int IN_BYTES = 2 * WIN * (int)sizeof(TS);
  constexpr int U_BYTES = 2 * CDC_BLK * UP * 4;
  constexpr int SMEM = IN_BYTES > U_BYTES ? IN_BYTES : U_BYTES;
  auto* k = k_cdc64<TIN, FAST>;
  if (SMEM > 48 * 1024) {
    const cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    if (e != cudaSuccess) return e;
  }
  k<<<grid, CDC_CTA, SMEM, st>>>(A);
  return cudaGetLastError();
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
  dim3 grid((unsigned)((A.blk_count + CDC_BLK - 1) / CDC_BLK), 1u);
  // vectorised epilogue preconditions (see cdc_epilogue_fast)
  auto al4 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 3) == 0; };
  bool fast = (io.out_dtype == FNTGPU_NONE || io.out_dtype == FNTGPU_I16) &&
              ((A.c + io.out_first) % 4 == 0);
  if (io.qr) fast = fast && io.q_shift >= 1 && io.q_shift < 31 && al4(io.qr) && al4(io.qi) &&
                    io.q_stride % 4 == 0 && io.q_max <= 127;
  if (io.out_dtype == FNTGPU_I16)
    fast = fast && (reinterpret_cast<uintptr_t>(io.yr) & 7) == 0 &&
           (reinterpret_cast<uintptr_t>(io.yi) & 7) == 0 && io.y_stride % 4 == 0;
  if (io.in_dtype != FNTGPU_I8 && io.in_dtype != FNTGPU_I32 && io.in_dtype != FNTGPU_I64)
    return cudaErrorInvalidValue;
  for (int64_t s0 = 0; s0 < io.n_streams; s0 += 65535) {
    A.s_base = (int32_t)s0;
    grid.y = (unsigned)(io.n_streams - s0 < 65535 ? io.n_streams - s0 : 65535);
    cudaError_t e;
    switch (io.in_dtype) {
      case FNTGPU_I8:
        e = fast ? launch_k<int8_t, true>(A, grid, st) : launch_k<int8_t, false>(A, grid, st);
        break;
      case FNTGPU_I32: e = launch_k<int32_t, false>(A, grid, st); break;
      default: e = launch_k<int64_t, false>(A, grid, st); break;
    }
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t launch_decim_phase(const fntgpu_decim_io& io, cudaStream_t s) {
  if (io.n_links <= 0) return cudaSuccess;
  k_decim_phase<<<(io.n_links + 127) / 128, 128, 0, s>>>(io);
  return cudaGetLastError();
}

}  // namespace fntgpu
