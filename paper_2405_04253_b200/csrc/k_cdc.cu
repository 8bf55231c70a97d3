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
#include <atomic>
#include <cstdio>
#include <cstdlib>
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
  uint32_t rbp[CDC_N]; // b+ mod F4 (tensor-core form: unscaled, cdc.py:124-135)
  uint32_t rbm[CDC_N]; // b- mod F4
  fntgpu_cdc_io io;
  int64_t blk_begin;   // first overlap-save block index of this launch
  int64_t blk_count;   // blocks per stream
  int32_t c;           // n_taps // 2
  int32_t s_base;      // first stream of this launch (grid.y is limited to 65535)
  int32_t q_away;      // every tie of the exact requantization rounds away from zero
                       // (io.q_tie[j] == min(j + 1, q_max)): q = min((|y| + 2^(k-1)) >> k, q_max)
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

// Float64 front-end samples quantized on load (in_dtype FNTGPU_F64): quantize_real
// (fixedpoint.py:51-60) with in_scale / in_max, v = x * scale, q = sign(v) floor(|v| +
// 0.5), clipped when |q| > in_max, then clipped to +-in_max -- the float64 steps of
// k_quant.cu (identical bits), fused into the staging of the CDC input window, so the
// float samples cross HBM once and the int8 planes never exist in global memory.
// Returns the clip count over the window positions [own_lo, own_hi) (global indices).
// floor(|v| + 0.5) straight to an integer (cvt.rmi: the float64 add is rounded
// first, as numpy's is); a NaN converts to 0 and an out-of-range value saturates,
// so |q| > max_int flags exactly the clipped samples (k_quant.cu semantics).
__device__ __forceinline__ int8_t quant_in(double x, double scale, int32_t mx, uint32_t& clip) {
  const double v = __dmul_rn(x, scale);
  const int32_t a = __double2int_rd(__dadd_rn(fabs(v), 0.5));
  clip = a > mx;
  const int32_t c = min(a, mx);
  return (int8_t)(v < 0 ? -c : c);
}

__device__ __forceinline__ uint32_t stage_plane_f64(int8_t* dst, const double* src, int64_t g0,
                                                    const fntgpu_cdc_io& io, int64_t own_lo,
                                                    int64_t own_hi) {
  const int64_t lo = io.x_first > 0 ? io.x_first : 0;
  const int64_t hi_avail = io.x_first + io.x_count;
  const int64_t hi = hi_avail < io.length ? hi_avail : io.length;
  const int32_t mx = io.in_max;
  uint32_t clips = 0;
  constexpr int CH = WIN / 16;
  for (int ch = threadIdx.x; ch < CH; ch += blockDim.x) {
    const int64_t g = g0 + 16 * ch;
    const double* p = src + (g - io.x_first);
    uint32_t w[4] = {0u, 0u, 0u, 0u};
    if (g >= lo && g + 16 <= hi && ((reinterpret_cast<uintptr_t>(p) & 15) == 0)) {
      const bool own = g >= own_lo && g + 16 <= own_hi;
#pragma unroll
      for (int k2 = 0; k2 < 8; ++k2) {
        const double2 v = __ldg(reinterpret_cast<const double2*>(p) + k2);
        uint32_t c0, c1;
        const int8_t q0 = quant_in(v.x, io.in_scale, mx, c0), q1 = quant_in(v.y, io.in_scale, mx, c1);
        const int k = 2 * k2;
        w[k >> 2] |= (((uint32_t)(uint8_t)q0) | ((uint32_t)(uint8_t)q1 << 8)) << (8 * (k & 3));
        if (own) clips += c0 + c1;
        else clips += (c0 & (g + k >= own_lo && g + k < own_hi)) + (c1 & (g + k + 1 >= own_lo && g + k + 1 < own_hi));
      }
    } else {
      for (int k = 0; k < 16; ++k) {
        const int64_t gk = g + k;
        if (gk >= lo && gk < hi) {
          uint32_t c;
          const int8_t q = quant_in(src[gk - io.x_first], io.in_scale, mx, c);
          w[k >> 2] |= ((uint32_t)(uint8_t)q) << (8 * (k & 3));
          clips += c & (gk >= own_lo && gk < own_hi);
        }
      }
    }
    reinterpret_cast<uint4*>(dst)[ch] = make_uint4(w[0], w[1], w[2], w[3]);
  }
  return clips;
}

// Exact integer form of the AEQ-input requantization q = quantize_real(y * inv, q_scale)
// when inv * q_scale == 2^-k up to rounding: the float64 product is within 3 ulp of
// y / 2^k, so round-half-away agrees with the exact rounding except at exact ties
// |y| = 2^(k-1) + j 2^k, whose float64 outcome the host precomputed (io.q_tie).
// requant_int when the host found every tie rounding away (CdcArgs.q_away): no tie
// table lookup, no comparisons beyond the clamp
// Signed form: for y < 0, (y + 2^(k-1) - 1) >> k (arithmetic) = -floor((|y| + 2^(k-1)) / 2^k).
__device__ __forceinline__ int32_t requant_away(int32_t y, int k, int qmax) {
  const int32_t q = (y + (1 << (k - 1)) + (y >> 31)) >> k;
  return max(min(q, qmax), -qmax);
}

// low bytes of four words packed into one (byte e = low byte of q[e])
__device__ __forceinline__ uint32_t pack_bytes4(uint32_t q0, uint32_t q1, uint32_t q2, uint32_t q3) {
  uint32_t lo, hi, r;
  asm("prmt.b32 %0, %1, %2, 0x0040;" : "=r"(lo) : "r"(q0), "r"(q1));
  asm("prmt.b32 %0, %1, %2, 0x0040;" : "=r"(hi) : "r"(q2), "r"(q3));
  asm("prmt.b32 %0, %1, %2, 0x5410;" : "=r"(r) : "r"(lo), "r"(hi));
  return r;
}

// Per-thread decimation statistics of one output parity: S2 = sum |y|^2 (< 2^34 for
// the <= 8 outputs a thread of the fast epilogue owns per parity) and
// S4 = sum |y|^4 as 96 bits (h:hi:lo). |y|^2 <= 2^31, so a pair of |y|^4 terms
// fits 64 bits and one carry chain per pair suffices.
struct DecimAcc {
  unsigned long long s2 = 0;
  uint32_t lo = 0, hi = 0, h = 0;
  __device__ __forceinline__ void add_pair(uint32_t m0, uint32_t m1) {
    s2 += (unsigned long long)m0 + m1;
    const unsigned long long t = (unsigned long long)m0 * m0 + (unsigned long long)m1 * m1;  // < 2^63
    asm("add.cc.u32 %0, %0, %3;\n\taddc.cc.u32 %1, %1, %4;\n\taddc.u32 %2, %2, 0;"
        : "+r"(lo), "+r"(hi), "+r"(h)
        : "r"((uint32_t)t), "r"((uint32_t)(t >> 32)));
  }
  // Warp sums as 27-bit limbs (S2 = A0 + A1 2^27, S4 = L0 + L1 2^27 + L2 2^54), so
  // each warp-wide redux.add of 32 limbs is exact in 32 bits: S2 < 2^35 and
  // S4 < 2^66 per thread (h <= 1).
  __device__ __forceinline__ void warp_limbs(uint32_t (&l)[5]) const {
    constexpr uint32_t M27 = (1u << 27) - 1;
    l[0] = __reduce_add_sync(0xffffffffu, (uint32_t)s2 & M27);
    l[1] = __reduce_add_sync(0xffffffffu, (uint32_t)(s2 >> 27));
    l[2] = __reduce_add_sync(0xffffffffu, lo & M27);
    l[3] = __reduce_add_sync(0xffffffffu, __funnelshift_r(lo, hi, 27) & M27);
    l[4] = __reduce_add_sync(0xffffffffu, (hi >> 22) | (h << 10));
  }
};

// Limb sums of a CTA (each < 2^35) into the (S2, S4 = w3 2^64 + w2 2^32 + w1) words at
// acc, S4 regrouped on the 2^32 word boundaries
__device__ __forceinline__ void decim_flush(unsigned long long* acc, const unsigned long long (&l)[5]) {
  const unsigned long long w[4] = {l[0] + (l[1] << 27), l[2] + ((l[3] & 31u) << 27),
                                   (l[3] >> 5) + ((l[4] & 1023u) << 22), l[4] >> 10};
#pragma unroll
  for (int q = 0; q < 4; ++q)
    if (w[q]) atomicAdd(acc + q, w[q]);
}

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
// PRE: s_u holds the decoded outputs + 32768 (tensor-core form) instead of the u+-
// words of the two inverse transforms.
template <bool PRE = false>
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
  DecimAcc sa, sb;
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
      if (PRE) {
        zr[e] = (int32_t)up - 32768;
        zi[e] = (int32_t)um - 32768;
      } else {
        zr[e] = (int32_t)f4_mod(m_add(up, um)) - 32768;
        zi[e] = (int32_t)f4_mod(m_rot(m_sub(up, um), 24)) - 32768;
      }
    }
    if (CDC_PROBE != 1 && qr) {
      uint32_t pr = 0, pi = 0;
      if (A.q_away) {
        pr = pack_bytes4(requant_away(zr[0], k, qmax), requant_away(zr[1], k, qmax),
                         requant_away(zr[2], k, qmax), requant_away(zr[3], k, qmax));
        pi = pack_bytes4(requant_away(zi[0], k, qmax), requant_away(zi[1], k, qmax),
                         requant_away(zi[2], k, qmax), requant_away(zi[3], k, qmax));
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          pr |= ((uint32_t)requant_int(zr[e], k, tie, qmax) & 0xffu) << (8 * e);
          pi |= ((uint32_t)requant_int(zi[e], k, tie, qmax) & 0xffu) << (8 * e);
        }
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
      uint32_t m2[4];  // |y|^2 <= 2^31
#pragma unroll
      for (int e = 0; e < 4; ++e) m2[e] = (uint32_t)(zr[e] * zr[e]) + (uint32_t)(zi[e] * zi[e]);
      if (!full) {
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (v + e < lo || v + e >= hi) m2[e] = 0u;
      }
      sa.add_pair(m2[0], m2[2]);
      sb.add_pair(m2[1], m2[3]);
    }
  }
  static_assert(CDC_BLK * CDC_HOP / (4 * CDC_CTA) * 2 <= 8, "DecimAcc per-thread bounds");
  if (stats) {
    // warp limb sums -> shared memory -> one thread per (parity, limb) sums the CTA's
    // warps -> one set of atomics per CTA and parity
    constexpr int NW = CDC_CTA / 32;
    __shared__ uint32_t red[10][NW];
    uint32_t la[5], lb[5];
    sa.warp_limbs(la);
    sb.warp_limbs(lb);
    if ((tid & 31) == 0) {
#pragma unroll
      for (int i = 0; i < 5; ++i) {
        red[i][tid >> 5] = la[i];
        red[5 + i][tid >> 5] = lb[i];
      }
    }
    __syncthreads();
    if (tid < 32) {
      unsigned long long v = 0;
      if (tid < 10) {
#pragma unroll
        for (int w = 0; w < NW; ++w) v += red[tid][w];
      }
      unsigned long long l[5];
#pragma unroll
      for (int i = 0; i < 5; ++i) l[i] = __shfl_sync(0xffffffffu, v, (tid < 5 ? 0 : 5) + i);
      // even local indices carry phase (n0 & 1), odd ones the other phase
      const int pa = (int)(n0 & 1);
      if (tid == 0) decim_flush(io.decim_acc + ((int64_t)s * 2 + pa) * 4, l);
      if (tid == 5) decim_flush(io.decim_acc + ((int64_t)s * 2 + (pa ^ 1)) * 4, l);
    }
  }
}

// Any-dtype epilogue (process_int int16/32/64, process complex128, float64
// requantization): one output per thread per step.
template <bool PRE = false>
__device__ __forceinline__ void cdc_epilogue_generic(const CdcArgs& A, const uint32_t* s_u, int s,
                                                     int64_t n0, int64_t lo, int64_t hi) {
  const fntgpu_cdc_io& io = A.io;
  const int tid = threadIdx.x;
  // n advances by CDC_CTA (even): each thread only ever sees one sampling phase
  const int my_ph = (int)((lo + tid) & 1);
  unsigned long long s2 = 0, s4lo = 0, s4hi = 0;
  for (int64_t n = lo + tid; n < hi; n += CDC_CTA) {
    const int idx = (int)(n - n0);
    const int r = (idx >> 5) * UP + (idx & 31);
    const uint32_t up = s_u[r], um = s_u[CDC_BLK * UP + r];
    const int32_t zr = PRE ? (int32_t)up - 32768 : (int32_t)f4_mod(m_add(up, um)) - 32768;
    const int32_t zi = PRE ? (int32_t)um - 32768 : (int32_t)f4_mod(m_rot(m_sub(up, um), 24)) - 32768;
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

// sign-extended byte k of w: PRMT with the selector's sign-replication bit
__device__ __forceinline__ int32_t sx8(uint32_t w, int k) {
  int32_t r;
  const uint32_t sel = (uint32_t)k | ((uint32_t)(k | 8) << 4) | ((uint32_t)(k | 8) << 8) | ((uint32_t)(k | 8) << 12);
  asm("prmt.b32 %0, %1, 0, %2;" : "=r"(r) : "r"(w), "r"(sel));
  return r;
}

// One CTA item after its input window is staged in shared memory (s_xr, s_xi):
// forward FNT-64 of this thread's block and sign, tap products, pruned inverse, then
// the epilogue over the CTA's output range (s_u aliases the window).
// `where(s, cta_blk0)` yields the item's stream and first block when the epilogue
// needs them (recomputed from blockIdx, or re-read from shared memory by the persistent
// kernels, so they are not held in registers across the transforms).
template <typename TS, bool FAST, typename Where>
__device__ __forceinline__ void cdc_item(const CdcArgs& A, Where where, const TS* s_xr,
                                         const TS* s_xi, uint32_t* s_u) {
  const fntgpu_cdc_io& io = A.io;
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
    fnt_stage_plain<CDC_N, SQRT2, 0, 2, F4 * 1024u>(a);
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
  int s;
  int64_t cta_blk0;
  where(s, cta_blk0);
  const int64_t n0 = cta_blk0 * CDC_HOP - A.c;
  int64_t lo = n0, hi = n0 + (int64_t)CDC_BLK * CDC_HOP;
  const int64_t o_lo = io.out_first, o_hi = io.out_first + io.out_count;
  lo = lo < o_lo ? o_lo : lo;
  hi = hi > o_hi ? o_hi : hi;
  if (FAST) {
    cdc_epilogue_fast(A, s_u, s, n0, (int)(lo - n0), (int)(hi - n0));
    return;
  }
  cdc_epilogue_generic(A, s_u, s, n0, lo, hi);
}

template <typename TIN, bool FAST>
__global__ void __launch_bounds__(CDC_CTA, CDC_MIN_CTAS) k_cdc64(const __grid_constant__ CdcArgs A) {
  constexpr bool F64IN = std::is_same<TIN, double>::value;  // quantized on load to int8
  using TS = typename std::conditional<sizeof(TIN) == 1 || F64IN, int8_t, int32_t>::type;
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
  if constexpr (F64IN) {
    // this CTA's own samples (second halves of its launched blocks): each sample of
    // the launch is counted once
    const int64_t own_lo = cta_blk0 * CDC_HOP;
    const int64_t blk_end = A.blk_begin + A.blk_count;
    const int64_t own_hi = (cta_blk0 + CDC_BLK < blk_end ? cta_blk0 + CDC_BLK : blk_end) * CDC_HOP;
    uint32_t clips = stage_plane_f64(reinterpret_cast<int8_t*>(s_xr), reinterpret_cast<const double*>(xr_s),
                                     g0, io, own_lo, own_hi);
    clips += stage_plane_f64(reinterpret_cast<int8_t*>(s_xi), reinterpret_cast<const double*>(xi_s), g0,
                             io, own_lo, own_hi);
    if (io.in_clipped) {
      clips = __reduce_add_sync(0xffffffffu, clips);
      if ((threadIdx.x & 31) == 0 && clips) atomicAdd(io.in_clipped, (unsigned long long)clips);
    }
  } else if (!bulk) {
    stage_plane<TIN, TS>(s_xr, xr_s, g0, io);
    stage_plane<TIN, TS>(s_xi, xi_s, g0, io);
  }
  __syncthreads();
  cdc_item<TS, FAST>(A, [&](int& s_, int64_t& b_) {
    s_ = A.s_base + (int)blockIdx.y;
    b_ = A.blk_begin + (int64_t)blockIdx.x * CDC_BLK;
  }, s_xr, s_xi, s_u);
}

// ---------------------------------------------------------------------------------
// Float64 inputs quantized on load, persistent form (CDC_F64P). A CTA's float64 window
// is 8x the int8 one (66 KB for both planes), so in the one-item-per-CTA kernel every
// CTA spent a quarter of its life waiting for it. Here each CTA walks items
// it, it + gridDim.x, ...: the next item's raw window arrives by two TMA bulk copies
// into a shared-memory buffer while the current item's FNTs run, and is quantized from
// shared memory (quant_in, the k_quant.cu / fixedpoint.py:51-60 float64 steps) into the
// int8 window the shift-add path reads. Stream edges and unaligned views take the
// synchronous global-load staging. Two CTAs per SM (raw buffer + window / u rows).
#ifndef CDC_F64P
#define CDC_F64P 1
#endif
constexpr int F64P_WORK = (2 * WIN > 2 * CDC_BLK * UP * 4) ? 2 * WIN : 2 * CDC_BLK * UP * 4;

// quantize a landed raw window (samples g0 .. g0 + WIN of one plane, all inside the
// stream) into int8, two samples per thread per step (conflict-free 16-byte reads);
// returns the clips among this CTA's own samples [own_lo, own_hi)
__device__ __forceinline__ uint32_t quant_window_smem(int8_t* dst, const double* raw, int64_t g0,
                                                      const fntgpu_cdc_io& io, int64_t own_lo,
                                                      int64_t own_hi) {
  uint32_t clips = 0;
  const int32_t mx = io.in_max;
  for (int j = threadIdx.x; j < WIN / 2; j += blockDim.x) {
    const double2 v = reinterpret_cast<const double2*>(raw)[j];
    uint32_t c0, c1;
    const int8_t q0 = quant_in(v.x, io.in_scale, mx, c0), q1 = quant_in(v.y, io.in_scale, mx, c1);
    reinterpret_cast<uint16_t*>(dst)[j] = (uint16_t)((uint32_t)(uint8_t)q0 | ((uint32_t)(uint8_t)q1 << 8));
    const int64_t g = g0 + 2 * j;
    clips += (c0 & (g >= own_lo && g < own_hi)) + (c1 & (g + 1 >= own_lo && g + 1 < own_hi));
  }
  return clips;
}

#ifndef CDC_F64P_PLANES
// raw float64 planes prefetched per item: 2 (both, 103 KB per CTA, 2 CTAs per SM) or
// 1 (the real plane prefetched, the imaginary one loaded at the item's start into the
// same buffer: 70 KB per CTA, 3 CTAs per SM and the int8 kernel's register budget).
// Measured at 2^27 samples: 2 planes 116 Gsamples/s, 1 plane 107 (the exposed load of
// the second plane costs more than the third CTA gains).
#define CDC_F64P_PLANES 2
#endif
constexpr int F64P_RAWB = CDC_F64P_PLANES * WIN * (int)sizeof(double);

template <bool FAST>
__global__ void __launch_bounds__(CDC_CTA, CDC_F64P_PLANES == 2 ? 2 : CDC_MIN_CTAS)
k_cdc64_f64p(const __grid_constant__ CdcArgs A) {
  constexpr int NP = CDC_F64P_PLANES;
  extern __shared__ __align__(16) unsigned char smem[];
  double* raw = reinterpret_cast<double*>(smem);  // [NP][WIN]
  unsigned char* work = smem + F64P_RAWB;
  int8_t* s_xr = reinterpret_cast<int8_t*>(work);
  int8_t* s_xi = s_xr + WIN;
  uint32_t* s_u = reinterpret_cast<uint32_t*>(work);
  __shared__ __align__(8) uint64_t mbar;
  // loop state in shared memory, launch constants recomputed per item: nothing extra
  // stays live in registers across the transforms (the int8 kernel's 80 registers)
  __shared__ int64_t sh_it, sh_blk0;
  __shared__ int sh_s;
  __shared__ uint32_t sh_phase;
  const int tid = threadIdx.x;
  if (tid == 0) {
    const uint32_t mb = (uint32_t)__cvta_generic_to_shared(&mbar);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(mb) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    sh_it = -1;
    sh_phase = 0;
  }
  __syncthreads();
  for (;;) {
    const fntgpu_cdc_io& io = A.io;
    const int64_t chunks = (A.blk_count + CDC_BLK - 1) / CDC_BLK;
    const int64_t items = chunks * io.n_streams;
    const int64_t lo = io.x_first > 0 ? io.x_first : 0;
    const int64_t hi_avail = io.x_first + io.x_count;
    const int64_t hi = hi_avail < io.length ? hi_avail : io.length;
    const double* xr0 = reinterpret_cast<const double*>(io.xr);
    const double* xi0 = reinterpret_cast<const double*>(io.xi);
    const uint32_t mb = (uint32_t)__cvta_generic_to_shared(&mbar);
    auto where = [&](int64_t it, int& s, int64_t& blk0) {
      s = (int)(it / chunks);
      blk0 = A.blk_begin + (it - (int64_t)s * chunks) * CDC_BLK;
    };
    auto src = [&](const double* base, int s, int64_t g0) {
      return base + (size_t)s * io.x_stride + (g0 - io.x_first);
    };
    auto bulk_ok = [&](int64_t it) {
      int s;
      int64_t blk0;
      where(it, s, blk0);
      const int64_t g0 = blk0 * CDC_HOP - CDC_HOP;
      return g0 >= lo && g0 + WIN <= hi &&
             ((reinterpret_cast<uintptr_t>(src(xr0, s, g0)) | reinterpret_cast<uintptr_t>(src(xi0, s, g0))) & 15) == 0;
    };
    // thread 0: planes [p0, p0 + n) of item `it` into raw[0 .. n)
    auto issue = [&](int64_t it, int p0, int n) {
      int s;
      int64_t blk0;
      where(it, s, blk0);
      const int64_t g0 = blk0 * CDC_HOP - CDC_HOP;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(mb), "r"(n * WIN * 8) : "memory");
      for (int q = 0; q < n; ++q)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     :: "r"((uint32_t)__cvta_generic_to_shared(raw + q * WIN)),
                        "l"(src(p0 + q ? xi0 : xr0, s, g0)), "r"(WIN * 8), "r"(mb) : "memory");
    };
    auto wait = [&](uint32_t& phase) {
      uint32_t done = 0;
      while (!done) {
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                     "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(done) : "r"(mb), "r"(phase) : "memory");
      }
      phase ^= 1u;
    };
    int64_t it = sh_it;
    if (it < 0) {  // first pass
      it = blockIdx.x;
      if (tid == 0 && it < items && bulk_ok(it)) issue(it, 0, NP);
    }
    if (it >= items) break;
    uint32_t phase = sh_phase;
    int s;
    int64_t cta_blk0;
    where(it, s, cta_blk0);
    const int64_t g0 = cta_blk0 * CDC_HOP - CDC_HOP;
    const int64_t own_lo = cta_blk0 * CDC_HOP;
    const int64_t blk_end = A.blk_begin + A.blk_count;
    const int64_t own_hi = (cta_blk0 + CDC_BLK < blk_end ? cta_blk0 + CDC_BLK : blk_end) * CDC_HOP;
    uint32_t clips;
    if (bulk_ok(it)) {
      wait(phase);
      clips = quant_window_smem(s_xr, raw, g0, io, own_lo, own_hi);
      if (NP == 2) {
        clips += quant_window_smem(s_xi, raw + WIN, g0, io, own_lo, own_hi);
      } else {
        __syncthreads();  // the real plane is converted: its buffer takes the imaginary one
        if (tid == 0) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          issue(it, 1, 1);
        }
        wait(phase);
        clips += quant_window_smem(s_xi, raw, g0, io, own_lo, own_hi);
      }
    } else {
      clips = stage_plane_f64(s_xr, src(xr0, s, io.x_first), g0, io, own_lo, own_hi);
      clips += stage_plane_f64(s_xi, src(xi0, s, io.x_first), g0, io, own_lo, own_hi);
    }
    if (io.in_clipped) {
      clips = __reduce_add_sync(0xffffffffu, clips);
      if ((tid & 31) == 0 && clips) atomicAdd(io.in_clipped, (unsigned long long)clips);
    }
    __syncthreads();  // int8 window complete; every thread is done with the raw buffer and the loop state
    if (tid == 0) {
      sh_s = s;  // read back by the epilogue (ordered by cdc_item's barriers)
      sh_blk0 = cta_blk0;
      sh_it = it + gridDim.x;
      sh_phase = phase;
      const int64_t nx = it + gridDim.x;
      if (nx < items && bulk_ok(nx)) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue(nx, 0, NP);  // lands while this item's transforms run
      }
    }
    cdc_item<int8_t, FAST>(A, [&](int& s_, int64_t& b_) {
      s_ = *(volatile int*)&sh_s;
      b_ = *(volatile int64_t*)&sh_blk0;
    }, s_xr, s_xi, s_u);
    __syncthreads();  // the epilogue's reads of s_u are done before the next window
  }
}

// ---------------------------------------------------------------------------------
// Tensor-core form: the same overlap-save blocks with the 64-point forward FNT and
// the pruned inverse as split-integer matrix products on the int8 tensor cores
// (mma.sync m16n8k32, SASS IMMA.16832, exact int32 accumulation), the pointwise tap
// products and mod-F4 reductions on the CUDA cores. Every transform matrix entry is a
// 64th root of unity alpha^e (alpha = sqrt(2) = 4080), stored as two 8-bit limbs
// t = 256 t1 + t0 with t1 in [0, 255] (u8) and t0 in [-128, 127] (s8), a split that
// holds every root (tests/test_tc_math.py restates the whole algorithm in numpy).
// One warp owns an M-tile of 16 consecutive blocks (rows); lane = 4 g + tig.
//   forward  X_r = T x_r, X_i = T x_i        (K = 64 samples, N = 64 bins x 2 limbs)
//            X = 256 P1 + P0 == FNT(x) mod F4
//   products s = A+ b+ + A- b- = X_r beta1 + X_i beta2, d = X_r beta3 + X_i beta4
//            (A+- = X_r +- 2^8 X_i, cdc.py:148-149; two IMAD.WIDE each), then
//            w = (s + 32896) mod F4 in [0, 65536]: the signed limbs of s are the bytes
//            of w ^ 0x80 (w = 65536 does not fit and is corrected after the MMAs)
//   inverse  z_re = M_re s, z_im = M_im d      (K = 64 bins, N = 32 kept outputs, 2 x 2
//            limb products: z == 256 Qmid + Q00 - Q11 since 2^16 == -1 mod F4)
// The accumulator fragments of the forward products are laid out so that each
// thread's values are exactly the A-fragment bytes of the inverse MMA (the inverse
// matrix rows are permuted to match), so nothing moves between lanes.
#ifndef CDC_TC_MIN_CTAS
#define CDC_TC_MIN_CTAS 3
#endif
constexpr int TC_E_RE = 50;  // c_re * N^-1 = 2^25 = alpha^50 (cdc.py:152)
constexpr int TC_E_IM = 34;  // c_im * N^-1 = 2^17 = alpha^34 (cdc.py:153)

struct TcTables {
  uint4 fwd[8][2][32];   // [bin n-tile][k-step][lane]: (t1 b0, t1 b1, t0 b0, t0 b1) of T[k][n]
  uint4 inv[2][8][32];   // [k-step][out n-tile: re 0-3, im 4-7][lane]
  uint4 beta[CDC_N];     // per bin: beta1..beta4 (canonical residues)
  uint32_t root[CDC_N];  // alpha^e mod F4
  uint32_t flags[CDC_CTA / 32][16][2][2];  // rare path: (row, s|d, bin) with w == 65536
  uint4 afr[CDC_CTA / 32][2][2][2][32];    // inverse A quads [warp][s|d][k-step][lo|hi limb][lane]
  int8_t x[2][2][WIN];                     // input windows [buffer][re|im] (TMA double buffer)
};

// D (+)= A B on the int8 tensor cores. Not volatile: no side effects, so the compiler
// may interleave the MMAs with the CUDA-core epilogue of the previous chunk. The _z
// forms start a chain from zero (C = RZ, no register initialisation).
#define FNT_MMA(NAME, TA, TB)                                                                    \
  __device__ __forceinline__ void NAME(int (&d)[4], const uint32_t (&a)[4], uint32_t b0,          \
                                       uint32_t b1) {                                            \
    asm("mma.sync.aligned.m16n8k32.row.col.s32." TA "." TB ".s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, " \
        "{%8,%9}, {%0,%1,%2,%3};"                                                                \
        : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])                                         \
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));                        \
  }                                                                                              \
  __device__ __forceinline__ void NAME##_z(int (&d)[4], const uint32_t (&a)[4], uint32_t b0,      \
                                           uint32_t b1) {                                        \
    asm("mma.sync.aligned.m16n8k32.row.col.s32." TA "." TB ".s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, " \
        "{%8,%9}, {%10,%10,%10,%10};"                                                            \
        : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3])                                         \
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1), "r"(0));                 \
  }
FNT_MMA(mma_s8u8, "s8", "u8")
FNT_MMA(mma_s8s8, "s8", "s8")
#undef FNT_MMA

// (u8, s8) limb bytes of a root: t1 in byte 0 of .x, t0 in byte 0 of .y
__device__ __forceinline__ uint2 tc_limbs(uint32_t t) {
  const int32_t v = t > 65407u ? (int32_t)t - (int32_t)F4 : (int32_t)t;
  const int32_t t0 = ((v + 128) & 255) - 128;
  const int32_t t1 = (v - t0) >> 8;
  return make_uint2((uint32_t)t1 & 255u, (uint32_t)t0 & 255u);
}

// Fragment tables, built by every CTA once (the kernel is persistent).
__device__ void tc_build_tables(TcTables& T, const CdcArgs& A) {
  const int tid = threadIdx.x;
  if (tid < CDC_N) {
    const int h = tid >> 1;
    uint32_t p2 = h < 16 ? (1u << h) : F4 - (1u << (h - 16));  // 2^h mod F4
    T.root[tid] = (tid & 1) ? (uint32_t)(((uint64_t)p2 * 4080u) % F4) : p2;
    const uint64_t bp = A.rbp[tid] % F4, bm = A.rbm[tid] % F4;
    const uint64_t sum = (bp + bm) % F4, dif = (bp + F4 - bm) % F4;
    T.beta[tid] = make_uint4((uint32_t)sum, (uint32_t)(256 * dif % F4), (uint32_t)dif,
                             (uint32_t)(256 * sum % F4));
  }
  for (int i = tid; i < CDC_CTA / 32 * 64; i += CDC_CTA) (&T.flags[0][0][0][0])[i] = 0u;
  __syncthreads();
  // word w of a table = one of (t1 b0, t1 b1, t0 b0, t0 b1) of one lane of one fragment
  for (int i = tid; i < 2 * 8 * 2 * 32 * 4; i += CDC_CTA) {
    const int q = i & 3, lane = (i >> 2) & 31, g = lane >> 2, tig = lane & 3;
    const int half = q & 1;  // b0 (K 0-15) or b1 (K 16-31)
    const bool lo_limb = q >= 2;
    uint32_t word = 0;
    if (i < 8 * 2 * 32 * 4) {
      // forward: [nt][ks][lane]; column g <-> bin 8 nt + g, K byte j <-> window sample
      // n = 32 ks + 16 half + 4 tig + j (natural order: the A quads come from ldmatrix)
      const int ks = (i >> 7) & 1, nt = i >> 8;
      const int k = 8 * nt + g;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int n = 32 * ks + 16 * half + 4 * tig + j;
        const uint2 l = tc_limbs(T.root[(n * k) & 63]);
        word |= (lo_limb ? l.y : l.x) << (8 * j);
      }
      (&T.fwd[0][0][0].x)[i] = word;
    } else {
      // inverse: [ks][ot][lane]; column g <-> output m = 32 + 8 (ot & 3) + g; K byte j of
      // half h <-> bin 32 ks + 16 h + 8 (j >> 1) + 2 tig + (j & 1) (forward C layout)
      const int ii = i - 8 * 2 * 32 * 4;
      const int ot = (ii >> 7) & 7, ks = ii >> 10;
      const int m = 32 + 8 * (ot & 3) + g;
      const int E = ot < 4 ? TC_E_RE : TC_E_IM;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int k = 32 * ks + 16 * half + 8 * (j >> 1) + 2 * tig + (j & 1);
        const uint2 l = tc_limbs(T.root[(E - m * k) & 63]);
        word |= (lo_limb ? l.y : l.x) << (8 * j);
      }
      (&T.inv[0][0][0].x)[ii] = word;
    }
  }
  __syncthreads();
}

// (X_r b1 + X_i b2 + 32896) mod F4 in [0, 65536]: 64-bit products (|X| < 2^30, b <= 2^16)
// folded with 2^32 == 1; the high word is small, so one end-around carry suffices.
__device__ __forceinline__ uint32_t tc_w(int32_t xr, int32_t xi, uint32_t b1, uint32_t b2) {
  const long long p = (long long)xr * (int32_t)b1 + (long long)xi * (int32_t)b2;
  const uint32_t lo = (uint32_t)p;
  const uint32_t t = (uint32_t)((int32_t)(p >> 32) + (int32_t)(F4 + 32896u));
  return f4_mod(m_add(lo, t));
}

// signed limbs of the 4 values of one A-fragment register (bytes j = 0..3 in K order)
__device__ __forceinline__ void tc_pack(uint32_t w0, uint32_t w1, uint32_t w2, uint32_t w3,
                                        uint32_t& lo, uint32_t& hi) {
  const uint32_t ab = __byte_perm(w0, w1, 0x5140), cd = __byte_perm(w2, w3, 0x5140);
  lo = __byte_perm(ab, cd, 0x5410) ^ 0x80808080u;
  hi = __byte_perm(ab, cd, 0x7632) ^ 0x80808080u;
}

// four 8x16-byte shared-memory matrices -> one IMMA A-operand quad (ldmatrix.x4)
__device__ __forceinline__ void ldsm_x4(uint32_t (&a)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(a[0]), "=r"(a[1]), "=r"(a[2]), "=r"(a[3])
               : "r"((uint32_t)__cvta_generic_to_shared(p)));
}

// Window staging of one item: interior windows by two TMA bulk copies completing on
// the buffer's mbarrier, others by vector loads (CTA-synchronous).
__device__ __forceinline__ bool tc_bulk_ok(const CdcArgs& A, int64_t chunks, int64_t it,
                                           int64_t in_lo, int64_t in_hi) {
  const fntgpu_cdc_io& io = A.io;
  const int s = (int)(it / chunks);
  const int64_t g0 = (A.blk_begin + (it - (int64_t)s * chunks) * CDC_BLK) * CDC_HOP - CDC_HOP;
  const uintptr_t pr = reinterpret_cast<uintptr_t>(reinterpret_cast<const int8_t*>(io.xr) +
                                                   (size_t)s * io.x_stride + (g0 - io.x_first));
  const uintptr_t pi = reinterpret_cast<uintptr_t>(reinterpret_cast<const int8_t*>(io.xi) +
                                                   (size_t)s * io.x_stride + (g0 - io.x_first));
  return CDC_TMA && g0 >= in_lo && g0 + WIN <= in_hi && ((pr | pi) & 15) == 0;
}

__device__ __forceinline__ void tc_issue_bulk(const CdcArgs& A, int64_t chunks, int64_t it,
                                              int8_t* dst_r, int8_t* dst_i, uint32_t mb) {
  const fntgpu_cdc_io& io = A.io;
  const int s = (int)(it / chunks);
  const int64_t g0 = (A.blk_begin + (it - (int64_t)s * chunks) * CDC_BLK) * CDC_HOP - CDC_HOP;
  const int8_t* pr = reinterpret_cast<const int8_t*>(io.xr) + (size_t)s * io.x_stride + (g0 - io.x_first);
  const int8_t* pi = reinterpret_cast<const int8_t*>(io.xi) + (size_t)s * io.x_stride + (g0 - io.x_first);
  // the buffer was last read through the generic proxy (two items ago)
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(mb), "r"(2 * WIN) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"((uint32_t)__cvta_generic_to_shared(dst_r)), "l"(pr), "r"(WIN), "r"(mb) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"((uint32_t)__cvta_generic_to_shared(dst_i)), "l"(pi), "r"(WIN), "r"(mb) : "memory");
}

// Fast-path outputs straight from the inverse fragments (FAST preconditions of
// cdc_epilogue_fast): this thread's outputs are local indices
// idx = 32 bl + 8 j + 2 tig + e2 (bl = block row), as (re, im) pairs over e2.
struct TcStats {
  unsigned long long a2 = 0, b2 = 0, a4 = 0, b4 = 0;  // even (a) / odd (b) local indices
  uint32_t a4h = 0, b4h = 0;
};

__device__ __forceinline__ void tc_store_pair(const CdcArgs& A, int s, int64_t base_o, int idx,
                                              int lo, int hi, const int32_t (&zr)[2],
                                              const int32_t (&zi)[2], TcStats& st) {
  const fntgpu_cdc_io& io = A.io;
  const bool v0 = idx >= lo && idx < hi, v1 = idx + 1 >= lo && idx + 1 < hi;
  if (!(v0 | v1)) return;
  const int64_t o = s * io.y_stride + base_o + idx;
  if (io.out_dtype == FNTGPU_I16) {
    int16_t* yr = reinterpret_cast<int16_t*>(io.yr) + o;
    int16_t* yi = reinterpret_cast<int16_t*>(io.yi) + o;
    if (v0 & v1) {
      *reinterpret_cast<uint32_t*>(yr) = ((uint32_t)zr[0] & 0xffffu) | ((uint32_t)zr[1] << 16);
      *reinterpret_cast<uint32_t*>(yi) = ((uint32_t)zi[0] & 0xffffu) | ((uint32_t)zi[1] << 16);
    } else {
      const int e = v0 ? 0 : 1;
      yr[e] = (int16_t)zr[e];
      yi[e] = (int16_t)zi[e];
    }
  }
  if (CDC_PROBE != 1 && io.qr) {
    const int k = io.q_shift, qmax = io.q_max;
    const uint32_t qr0 = (uint32_t)requant_int(zr[0], k, io.q_tie, qmax) & 0xffu;
    const uint32_t qr1 = (uint32_t)requant_int(zr[1], k, io.q_tie, qmax) & 0xffu;
    const uint32_t qi0 = (uint32_t)requant_int(zi[0], k, io.q_tie, qmax) & 0xffu;
    const uint32_t qi1 = (uint32_t)requant_int(zi[1], k, io.q_tie, qmax) & 0xffu;
    int8_t* qr = io.qr + s * io.q_stride + base_o + idx;
    int8_t* qi = io.qi + s * io.q_stride + base_o + idx;
    if (v0 & v1) {
      *reinterpret_cast<uint16_t*>(qr) = (uint16_t)(qr0 | (qr1 << 8));
      *reinterpret_cast<uint16_t*>(qi) = (uint16_t)(qi0 | (qi1 << 8));
    } else if (v0) {
      qr[0] = (int8_t)qr0;
      qi[0] = (int8_t)qi0;
    } else {
      qr[1] = (int8_t)qr1;
      qi[1] = (int8_t)qi1;
    }
  }
  if (CDC_PROBE != 2 && io.decim_acc) {
    const uint32_t m0 = v0 ? (uint32_t)(zr[0] * zr[0]) + (uint32_t)(zi[0] * zi[0]) : 0u;  // <= 2^31
    const uint32_t m1 = v1 ? (uint32_t)(zr[1] * zr[1]) + (uint32_t)(zi[1] * zi[1]) : 0u;
    const unsigned long long q0 = (unsigned long long)m0 * m0, q1 = (unsigned long long)m1 * m1;
    st.a2 += m0;
    st.a4 += q0;
    st.a4h += (st.a4 < q0);
    st.b2 += m1;
    st.b4 += q1;
    st.b4h += (st.b4 < q1);
  }
}

// Output pointers / parameters of the fast epilogue, read from param space once.
struct TcOut {
  int16_t* yr;
  int16_t* yi;
  int8_t* qr;
  int8_t* qi;
  unsigned long long* acc;
  int64_t y_stride, q_stride;
  int k, qmax;
  bool i16, away;
  __device__ explicit TcOut(const CdcArgs& A)
      : yr(reinterpret_cast<int16_t*>(A.io.yr)), yi(reinterpret_cast<int16_t*>(A.io.yi)), qr(A.io.qr),
        qi(A.io.qi), acc(A.io.decim_acc), y_stride(A.io.y_stride), q_stride(A.io.q_stride),
        k(A.io.q_shift), qmax(A.io.q_max), i16(A.io.out_dtype == FNTGPU_I16), away(A.q_away != 0) {}
};

// 8 consecutive outputs idx .. idx + 7 of stream s (idx multiple of 8)
__device__ __forceinline__ void tc_store8(const TcOut& O, const int8_t* tie, int s, int64_t base_o, int idx,
                                          int lo, int hi, const int32_t (&zr)[8], const int32_t (&zi)[8],
                                          TcStats& st) {
  if (idx + 8 <= lo || idx >= hi) return;
  const bool full = idx >= lo && idx + 8 <= hi;
  if (O.i16) {
    int16_t* yr = O.yr + s * O.y_stride + base_o + idx;
    int16_t* yi = O.yi + s * O.y_stride + base_o + idx;
    if (full) {
      uint32_t pr[4], pi[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        pr[e] = ((uint32_t)zr[2 * e] & 0xffffu) | ((uint32_t)zr[2 * e + 1] << 16);
        pi[e] = ((uint32_t)zi[2 * e] & 0xffffu) | ((uint32_t)zi[2 * e + 1] << 16);
      }
      // base_o + idx is a multiple of 4 (launch precondition): 8-byte aligned pairs
      reinterpret_cast<uint2*>(yr)[0] = make_uint2(pr[0], pr[1]);
      reinterpret_cast<uint2*>(yr)[1] = make_uint2(pr[2], pr[3]);
      reinterpret_cast<uint2*>(yi)[0] = make_uint2(pi[0], pi[1]);
      reinterpret_cast<uint2*>(yi)[1] = make_uint2(pi[2], pi[3]);
    } else {
#pragma unroll
      for (int e = 0; e < 8; ++e)
        if (idx + e >= lo && idx + e < hi) {
          yr[e] = (int16_t)zr[e];
          yi[e] = (int16_t)zi[e];
        }
    }
  }
  if (CDC_PROBE != 1 && O.qr) {
    uint32_t qr[2] = {0u, 0u}, qi[2] = {0u, 0u};
    if (O.away) {
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        qr[e >> 2] |= ((uint32_t)requant_away(zr[e], O.k, O.qmax) & 0xffu) << (8 * (e & 3));
        qi[e >> 2] |= ((uint32_t)requant_away(zi[e], O.k, O.qmax) & 0xffu) << (8 * (e & 3));
      }
    } else {
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        qr[e >> 2] |= ((uint32_t)requant_int(zr[e], O.k, tie, O.qmax) & 0xffu) << (8 * (e & 3));
        qi[e >> 2] |= ((uint32_t)requant_int(zi[e], O.k, tie, O.qmax) & 0xffu) << (8 * (e & 3));
      }
    }
    int8_t* pq = O.qr + s * O.q_stride + base_o + idx;
    int8_t* pqi = O.qi + s * O.q_stride + base_o + idx;
    if (full) {
      *reinterpret_cast<uint32_t*>(pq) = qr[0];
      *reinterpret_cast<uint32_t*>(pq + 4) = qr[1];
      *reinterpret_cast<uint32_t*>(pqi) = qi[0];
      *reinterpret_cast<uint32_t*>(pqi + 4) = qi[1];
    } else {
#pragma unroll
      for (int e = 0; e < 8; ++e)
        if (idx + e >= lo && idx + e < hi) {
          pq[e] = (int8_t)(qr[e >> 2] >> (8 * (e & 3)));
          pqi[e] = (int8_t)(qi[e >> 2] >> (8 * (e & 3)));
        }
    }
  }
  if (CDC_PROBE != 2 && O.acc) {
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const bool ok = full || (idx + e >= lo && idx + e < hi);
      const uint32_t m2 = ok ? (uint32_t)(zr[e] * zr[e]) + (uint32_t)(zi[e] * zi[e]) : 0u;  // <= 2^31
      const unsigned long long m4 = (unsigned long long)m2 * m2;
      if (e & 1) {
        st.b2 += m2;
        st.b4 += m4;
        st.b4h += (st.b4 < m4);
      } else {
        st.a2 += m2;
        st.a4 += m4;
        st.a4h += (st.a4 < m4);
      }
    }
  }
}

template <bool FAST>
__global__ void __launch_bounds__(CDC_CTA, CDC_TC_MIN_CTAS) k_cdc64_tc(const __grid_constant__ CdcArgs A) {
  extern __shared__ __align__(16) unsigned char smem[];
  TcTables& T = *reinterpret_cast<TcTables*>(smem);
  uint32_t* s_u = reinterpret_cast<uint32_t*>(smem + sizeof(TcTables));  // generic epilogue only
  __shared__ __align__(8) uint64_t mbar[2];
  const uint32_t mb0 = (uint32_t)__cvta_generic_to_shared(&mbar[0]);

  const fntgpu_cdc_io& io = A.io;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, tig = lane & 3;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(mb0) : "memory");
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(mb0 + 8) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tc_build_tables(T, A);  // ends with __syncthreads

  const int64_t chunks = (A.blk_count + CDC_BLK - 1) / CDC_BLK;
  const int64_t items = chunks * io.n_streams;
  const int64_t in_lo = io.x_first > 0 ? io.x_first : 0;
  const int64_t in_hi = io.x_first + io.x_count < io.length ? io.x_first + io.x_count : io.length;
  uint32_t phase = 0;  // parity bit per buffer
  int64_t it = blockIdx.x;
  if (tid == 0 && it < items && tc_bulk_ok(A, chunks, it, in_lo, in_hi))
    tc_issue_bulk(A, chunks, it, T.x[0][0], T.x[0][1], mb0);
  for (int buf = 0; it < items; it += gridDim.x, buf ^= 1) {
    const int s = (int)(it / chunks);
    const int64_t cta_blk0 = A.blk_begin + (it - (int64_t)s * chunks) * CDC_BLK;
    int8_t* s_xr = T.x[buf][0];
    int8_t* s_xi = T.x[buf][1];
    if (tc_bulk_ok(A, chunks, it, in_lo, in_hi)) {
      uint32_t done = 0;
      const uint32_t par = (phase >> buf) & 1u;
      while (!done) {
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                     "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(done) : "r"(mb0 + 8 * buf), "r"(par) : "memory");
      }
      phase ^= 1u << buf;
    } else {
      const int64_t g0 = cta_blk0 * CDC_HOP - CDC_HOP;
      stage_plane<int8_t, int8_t>(s_xr, reinterpret_cast<const int8_t*>(io.xr) + (size_t)s * io.x_stride, g0, io);
      stage_plane<int8_t, int8_t>(s_xi, reinterpret_cast<const int8_t*>(io.xi) + (size_t)s * io.x_stride, g0, io);
    }
    __syncthreads();  // window visible; every warp is done with the other buffer (and s_u)
    {
      const int64_t nx = it + gridDim.x;
      if (tid == 0 && nx < items && tc_bulk_ok(A, chunks, nx, in_lo, in_hi))
        tc_issue_bulk(A, chunks, nx, T.x[buf ^ 1][0], T.x[buf ^ 1][1], mb0 + 8 * (buf ^ 1));
    }

    // ---- forward: X_r, X_i of the warp's 16 blocks, 16 bins at a time
    bool flagged = false;
#pragma unroll 1
    for (int c = 0; c < 4; ++c) {
      int p1r[2][4], p0r[2][4], p1i[2][4], p0i[2][4];
      {
        uint32_t ax[2][4];
        // ldmatrix.x4: lanes 8q..8q+7 address the 16-byte rows of matrix q = (rows 0-7 |
        // 8-15) x (K 0-15 | 16-31) of the M-tile; the result is the A quad in place
        const int off = 32 * (16 * warp + (lane & 15)) + 16 * (lane >> 4);
        ldsm_x4(ax[0], s_xr + off);
        ldsm_x4(ax[1], s_xr + off + 32);
#pragma unroll
        for (int jj = 0; jj < 2; ++jj) {
          const uint4 B0 = T.fwd[2 * c + jj][0][lane], B1 = T.fwd[2 * c + jj][1][lane];
          mma_s8u8_z(p1r[jj], ax[0], B0.x, B0.y);
          mma_s8s8_z(p0r[jj], ax[0], B0.z, B0.w);
          mma_s8u8(p1r[jj], ax[1], B1.x, B1.y);
          mma_s8s8(p0r[jj], ax[1], B1.z, B1.w);
        }
        ldsm_x4(ax[0], s_xi + off);
        ldsm_x4(ax[1], s_xi + off + 32);
#pragma unroll
        for (int jj = 0; jj < 2; ++jj) {
          const uint4 B0 = T.fwd[2 * c + jj][0][lane], B1 = T.fwd[2 * c + jj][1][lane];
          mma_s8u8_z(p1i[jj], ax[0], B0.x, B0.y);
          mma_s8s8_z(p0i[jj], ax[0], B0.z, B0.w);
          mma_s8u8(p1i[jj], ax[1], B1.x, B1.y);
          mma_s8s8(p0i[jj], ax[1], B1.z, B1.w);
        }
      }
      // C fragment: e = 0, 1 row g, cols 2 tig, 2 tig + 1; e = 2, 3 row g + 8
      uint32_t ws[2][4], wd[2][4];
      uint32_t any = 0;
#pragma unroll
      for (int jj = 0; jj < 2; ++jj) {
#pragma unroll
        for (int e2 = 0; e2 < 2; ++e2) {
          const uint4 be = T.beta[16 * c + 8 * jj + 2 * tig + e2];
#pragma unroll
          for (int r = 0; r < 2; ++r) {
            const int e = 2 * r + e2;
            const int32_t xr = p1r[jj][e] * 256 + p0r[jj][e];
            const int32_t xi = p1i[jj][e] * 256 + p0i[jj][e];
            ws[jj][e] = tc_w(xr, xi, be.x, be.y);
            wd[jj][e] = tc_w(xr, xi, be.z, be.w);
            any |= ws[jj][e] | wd[jj][e];
          }
        }
      }
      // A-fragment registers of inverse k-step c >> 1: K half c & 1 -> quad positions
      // (0, 1) or (2, 3); stored for the inverse (shared memory keeps registers free)
      {
        uint32_t sl0, sh0, sl1, sh1, dl0, dh0, dl1, dh1;
        tc_pack(ws[0][0], ws[0][1], ws[1][0], ws[1][1], sl0, sh0);
        tc_pack(ws[0][2], ws[0][3], ws[1][2], ws[1][3], sl1, sh1);
        tc_pack(wd[0][0], wd[0][1], wd[1][0], wd[1][1], dl0, dh0);
        tc_pack(wd[0][2], wd[0][3], wd[1][2], wd[1][3], dl1, dh1);
        const int ks = c >> 1, h = c & 1;
        reinterpret_cast<uint2*>(&T.afr[warp][0][ks][0][lane])[h] = make_uint2(sl0, sl1);
        reinterpret_cast<uint2*>(&T.afr[warp][0][ks][1][lane])[h] = make_uint2(sh0, sh1);
        reinterpret_cast<uint2*>(&T.afr[warp][1][ks][0][lane])[h] = make_uint2(dl0, dl1);
        reinterpret_cast<uint2*>(&T.afr[warp][1][ks][1][lane])[h] = make_uint2(dh0, dh1);
      }
      if (__any_sync(0xffffffffu, any & 0x10000u)) {
        // rare (p ~ 2^-16 per value): record the bins whose value the bytes cannot hold
        flagged = true;
#pragma unroll
        for (int jj = 0; jj < 2; ++jj)
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int k = 16 * c + 8 * jj + 2 * tig + (e & 1), row = g + 8 * (e >> 1);
            if (ws[jj][e] >> 16) atomicOr(&T.flags[warp][row][0][k >> 5], 1u << (k & 31));
            if (wd[jj][e] >> 16) atomicOr(&T.flags[warp][row][1][k >> 5], 1u << (k & 31));
          }
      }
    }
    __syncwarp();  // afr (and flags) written by every lane
    // ---- inverse, one output n-tile j at a time for z_re (from s) and z_im (from d)
    const int64_t n0 = cta_blk0 * CDC_HOP - A.c;
    int64_t lo64 = n0, hi64 = n0 + (int64_t)CDC_BLK * CDC_HOP;
    const int64_t o_lo = io.out_first, o_hi = io.out_first + io.out_count;
    lo64 = lo64 < o_lo ? o_lo : lo64;
    hi64 = hi64 > o_hi ? o_hi : hi64;
    const int lo = (int)(lo64 - n0), hi = (int)(hi64 - n0);
    TcStats st;
#pragma unroll 1
    for (int j = 0; j < 4; ++j) {
      int32_t zv[2][4];  // decoded z + 32768: [re | im][fragment element]
#pragma unroll
      for (int sd = 0; sd < 2; ++sd) {
        int q11[4], qm[4], q00[4];
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
          const uint4 l4 = T.afr[warp][sd][ks][0][lane], h4 = T.afr[warp][sd][ks][1][lane];
          const uint32_t aL[4] = {l4.x, l4.y, l4.z, l4.w}, aH[4] = {h4.x, h4.y, h4.z, h4.w};
          const uint4 B = T.inv[ks][4 * sd + j][lane];
          if (ks == 0) {
            mma_s8u8_z(q11, aH, B.x, B.y);
            mma_s8s8_z(qm, aH, B.z, B.w);
            mma_s8s8_z(q00, aL, B.z, B.w);
          } else {
            mma_s8u8(q11, aH, B.x, B.y);
            mma_s8s8(qm, aH, B.z, B.w);
            mma_s8s8(q00, aL, B.z, B.w);
          }
          mma_s8u8(qm, aL, B.x, B.y);
        }
        if (flagged) {
          // a flagged bin k carried value + 1: subtract its matrix column
          const int E = sd ? TC_E_IM : TC_E_RE;
#pragma unroll
          for (int r = 0; r < 2; ++r) {
            const int row = g + 8 * r;
            for (int wd2 = 0; wd2 < 2; ++wd2) {
              uint32_t bits = T.flags[warp][row][sd][wd2];
              while (bits) {
                const int k = 32 * wd2 + __ffs(bits) - 1;
                bits &= bits - 1;
#pragma unroll
                for (int e2 = 0; e2 < 2; ++e2) {
                  const int m = 32 + 8 * j + 2 * tig + e2;
                  q00[2 * r + e2] -= (int32_t)T.root[(E - m * k) & 63];
                }
              }
            }
          }
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          // z == 256 Qmid + Q00 - Q11 (|z| < 2^30): canonical residue + 32768, decoded
          // by subtracting 32768 (fermat.py:131-133)
          const int32_t z = qm[e] * 256 + q00[e] - q11[e];
          zv[sd][e] = (int32_t)f4_mod((uint32_t)(z + (int32_t)(F4 * 16384u)) + 32768u);
        }
      }
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int bl = 16 * warp + g + 8 * r;
        if (FAST) {
          const int32_t zr2[2] = {zv[0][2 * r] - 32768, zv[0][2 * r + 1] - 32768};
          const int32_t zi2[2] = {zv[1][2 * r] - 32768, zv[1][2 * r + 1] - 32768};
          tc_store_pair(A, s, n0 - io.out_first, 32 * bl + 8 * j + 2 * tig, lo, hi, zr2, zi2, st);
        } else {
          uint32_t* u = s_u + bl * UP + 8 * j + 2 * tig;
          *reinterpret_cast<uint2*>(u) = make_uint2((uint32_t)zv[0][2 * r], (uint32_t)zv[0][2 * r + 1]);
          *reinterpret_cast<uint2*>(u + CDC_BLK * UP) = make_uint2((uint32_t)zv[1][2 * r], (uint32_t)zv[1][2 * r + 1]);
        }
      }
    }
    if (flagged) {
      __syncwarp();
      for (int i = lane; i < 64; i += 32) (&T.flags[warp][0][0][0])[i] = 0u;
    }
    if (FAST) {
      if (io.decim_acc) {
        // exact integer statistics per phase: warp-reduce 32-bit limbs, one atomic per value
        const int pa = (int)(n0 & 1);  // even local indices carry phase n0 & 1
        const unsigned long long va[4] = {st.a2, st.a4 & 0xffffffffull, st.a4 >> 32, st.a4h};
        const unsigned long long vb[4] = {st.b2, st.b4 & 0xffffffffull, st.b4 >> 32, st.b4h};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          unsigned long long x = va[q], y = vb[q];
#pragma unroll
          for (int off = 16; off > 0; off >>= 1) {
            x += __shfl_xor_sync(0xffffffffu, x, off);
            y += __shfl_xor_sync(0xffffffffu, y, off);
          }
          if (lane == 0) {
            if (x) atomicAdd(io.decim_acc + ((int64_t)s * 2 + pa) * 4 + q, x);
            if (y) atomicAdd(io.decim_acc + ((int64_t)s * 2 + (pa ^ 1)) * 4 + q, y);
          }
        }
      }
    } else {
      __syncthreads();
      cdc_epilogue_generic<true>(A, s_u, s, n0, lo64, hi64);
    }
  }
}

// ---------------------------------------------------------------------------------
// tcgen05 form of the split-integer matrix FNT-CDC (the same algorithm as
// k_cdc64_tc, tests/test_tc_math.py): the MMAs run asynchronously on the 5th-generation
// tensor cores (tcgen05.mma kind::i8, M = 128 blocks per CTA tile, operands in shared
// memory, int32 accumulators in tensor memory) issued by one thread; all 8 warps run
// the CUDA-core stages in between and read the accumulators back with tcgen05.ld (a
// warp sees the 32 TMEM lanes = 32 blocks of its lane quarter; warps w and w + 4 split
// the columns). Per 128-block item:
//   relayout  window -> x_r, x_i as K-major canonical operands (8-row x 16-byte core
//             matrices; overlapping windows cannot be addressed by a descriptor)
//   MMA 1     P1r, P0r, P1i, P0i = x_{r,i} [T1 | T0]          (8 x N=64, TMEM cols 0-255)
//   stage 1   X = 256 P1 + P0, s/d products with the tap spectra, limb bytes -> smem
//   MMA 2     Q11, Qmid, Q00 of z_re (from s) and z_im (from d) (16 x N=32, cols 0-191)
//   stage 2   z = 256 Qmid + Q00 - Q11 mod F4, decode, outputs / requantization / stats
#ifndef CDC_UMMA_MIN_CTAS
#define CDC_UMMA_MIN_CTAS 2
#endif
constexpr int UM_ROWS = CDC_BLK;  // 128 blocks = MMA M
constexpr uint32_t UM_TMEM_COLS = 256;

struct UmmaSmem {
  uint8_t ax[2][UM_ROWS * 64];       // x_r, x_i windows, canonical K-major [128 x 64 B]
  uint8_t ai[4][UM_ROWS * 64];       // inverse A: s lo, s hi, d lo, d hi limbs [128 x 64 B]
  uint8_t bf[2][CDC_N * 64];         // forward B: T1 (u8), T0 (s8) [64 bins x 64 samples]
  uint8_t bi[4][32 * 64];            // inverse B: M_re t1, M_re t0, M_im t1, M_im t0 [32 x 64 bins]
  uint4 beta[CDC_N];
  uint32_t root[CDC_N];
  uint32_t flags[UM_ROWS][2][2];     // [row][s|d][bin half]: w == 65536 bits (rare path)
  int8_t x[2][2][WIN];               // input windows [buffer][re|im] (TMA double buffer)
  uint64_t mbar_x[2];
  uint64_t mbar_mma;
  uint32_t tmem_base;
};

// canonical K-major, no swizzle: 8-row x 16-byte core matrices; LBO = 128 B between the
// two K-adjacent core matrices of one MMA (K = 32 bytes), SBO = 512 B between row groups
__host__ __device__ constexpr int um_off(int row, int kb) {
  return (row >> 3) * 512 + (kb >> 4) * 128 + (row & 7) * 16 + (kb & 15);
}
__device__ __forceinline__ uint64_t um_desc(const void* p) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(p);
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(512 >> 4) << 32) |
         (1ull << 46);  // version 1 (sm_100), base offset 0, layout SWIZZLE_NONE
}
// instruction descriptor: kind::i8, S32 accumulate, K-major A and B, M = 128
__host__ __device__ constexpr uint32_t um_idesc(int n, bool a_signed, bool b_signed) {
  return (2u << 4) | ((a_signed ? 1u : 0u) << 7) | ((b_signed ? 1u : 0u) << 10) |
         ((uint32_t)(n >> 3) << 17) | ((uint32_t)(UM_ROWS >> 4) << 24);
}
__device__ __forceinline__ void um_mma(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, bool acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}"
               :: "r"(d_tmem), "l"(a), "l"(b), "r"(idesc), "r"((uint32_t)acc));
}
__device__ __forceinline__ void um_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
               :: "r"((uint32_t)__cvta_generic_to_shared(bar)) : "memory");
}
__device__ __forceinline__ void um_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t mb = (uint32_t)__cvta_generic_to_shared(bar);
  uint32_t done = 0;
  while (!done) {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                 "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(done) : "r"(mb), "r"(parity) : "memory");
  }
}
__device__ __forceinline__ void um_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void um_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
// 8 consecutive TMEM columns of this thread's lane
__device__ __forceinline__ void um_ld8(uint32_t addr, int32_t (&v)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(addr));
}
__device__ __forceinline__ void um_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
// Registers written by tcgen05.ld are defined only after tcgen05.wait::ld: this empty
// volatile asm (after the wait) "redefines" them, so no use can be scheduled earlier.
__device__ __forceinline__ void um_ld_fence(int32_t (&v)[8]) {
  asm volatile("" : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]), "+r"(v[6]), "+r"(v[7]));
}

__device__ void um_build_tables(UmmaSmem& S, const CdcArgs& A) {
  const int tid = threadIdx.x;
  if (tid < CDC_N) {
    const int h = tid >> 1;
    const uint32_t p2 = h < 16 ? (1u << h) : F4 - (1u << (h - 16));
    S.root[tid] = (tid & 1) ? (uint32_t)(((uint64_t)p2 * 4080u) % F4) : p2;
    const uint64_t bp = A.rbp[tid] % F4, bm = A.rbm[tid] % F4;
    const uint64_t sum = (bp + bm) % F4, dif = (bp + F4 - bm) % F4;
    S.beta[tid] = make_uint4((uint32_t)sum, (uint32_t)(256 * dif % F4), (uint32_t)dif, (uint32_t)(256 * sum % F4));
  }
  __syncthreads();
  // forward B: row = bin k, K byte = window sample n, entry alpha^(nk)
  for (int i = tid; i < CDC_N * 64; i += blockDim.x) {
    const int k = i >> 6, n = i & 63;
    const uint2 l = tc_limbs(S.root[(n * k) & 63]);
    S.bf[0][um_off(k, n)] = (uint8_t)l.x;
    S.bf[1][um_off(k, n)] = (uint8_t)l.y;
  }
  // inverse B: row = kept output m - 32, K byte = bin k; c_re N^-1 alpha^(-mk), c_im N^-1 alpha^(-mk)
  for (int i = tid; i < 32 * 64; i += blockDim.x) {
    const int mo = i >> 6, k = i & 63, m = 32 + mo;
    const uint2 lr = tc_limbs(S.root[(TC_E_RE - m * k) & 63]);
    const uint2 li = tc_limbs(S.root[(TC_E_IM - m * k) & 63]);
    S.bi[0][um_off(mo, k)] = (uint8_t)lr.x;
    S.bi[1][um_off(mo, k)] = (uint8_t)lr.y;
    S.bi[2][um_off(mo, k)] = (uint8_t)li.x;
    S.bi[3][um_off(mo, k)] = (uint8_t)li.y;
  }
}

template <bool FAST>
__global__ void __launch_bounds__(CDC_CTA, CDC_UMMA_MIN_CTAS) k_cdc64_umma(const __grid_constant__ CdcArgs A) {
  extern __shared__ __align__(16) unsigned char smem[];
  UmmaSmem& S = *reinterpret_cast<UmmaSmem*>(smem);
  uint32_t* s_u = reinterpret_cast<uint32_t*>(smem + sizeof(UmmaSmem));  // generic epilogue only
  const fntgpu_cdc_io& io = A.io;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int row = 32 * (warp & 3) + lane;  // TMEM lane = block row of the item
  const int half = warp >> 2;              // column half this warp reads
  const uint32_t mbx = (uint32_t)__cvta_generic_to_shared(&S.mbar_x[0]);

  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(mbx) : "memory");
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(mbx + 8) : "memory");
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"((uint32_t)__cvta_generic_to_shared(&S.mbar_mma)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 :: "r"((uint32_t)__cvta_generic_to_shared(&S.tmem_base)), "n"(UM_TMEM_COLS) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  um_build_tables(S, A);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // tables are MMA operands
  um_fence_before();
  __syncthreads();
  um_fence_after();
  const uint32_t tmem = S.tmem_base;
  const uint32_t tlane = tmem + ((uint32_t)(32 * (warp & 3)) << 16);
  const TcOut O(A);

  const int64_t chunks = (A.blk_count + CDC_BLK - 1) / CDC_BLK;
  const int64_t items = chunks * io.n_streams;
  const int64_t in_lo = io.x_first > 0 ? io.x_first : 0;
  const int64_t in_hi = io.x_first + io.x_count < io.length ? io.x_first + io.x_count : io.length;
  uint32_t xphase = 0, mphase = 0;
  int64_t it = blockIdx.x;
  if (tid == 0 && it < items && tc_bulk_ok(A, chunks, it, in_lo, in_hi))
    tc_issue_bulk(A, chunks, it, S.x[0][0], S.x[0][1], mbx);
  for (int buf = 0; it < items; it += gridDim.x, buf ^= 1) {
    const int s = (int)(it / chunks);
    const int64_t cta_blk0 = A.blk_begin + (it - (int64_t)s * chunks) * CDC_BLK;
    int8_t* s_xr = S.x[buf][0];
    int8_t* s_xi = S.x[buf][1];
    if (tc_bulk_ok(A, chunks, it, in_lo, in_hi)) {
      um_wait(&S.mbar_x[buf], (xphase >> buf) & 1u);  // every thread acquires the TMA bytes
      xphase ^= 1u << buf;
    } else {
      const int64_t g0 = cta_blk0 * CDC_HOP - CDC_HOP;
      stage_plane<int8_t, int8_t>(s_xr, reinterpret_cast<const int8_t*>(io.xr) + (size_t)s * io.x_stride, g0, io);
      stage_plane<int8_t, int8_t>(s_xi, reinterpret_cast<const int8_t*>(io.xi) + (size_t)s * io.x_stride, g0, io);
      __syncthreads();  // vector-staged window visible (stream edges only)
    }
    // the other buffer was last read by the previous item's relayout, which every thread
    // finished before that item's operand barrier: the next window can land there now
    {
      const int64_t nx = it + gridDim.x;
      if (tid == 0 && nx < items && tc_bulk_ok(A, chunks, nx, in_lo, in_hi))
        tc_issue_bulk(A, chunks, nx, S.x[buf ^ 1][0], S.x[buf ^ 1][1], mbx + 8 * (buf ^ 1));
    }
    // ---- relayout: row b, 16-byte chunk q of plane p <- window bytes [32 b + 16 q, + 16)
#pragma unroll
    for (int i = tid; i < 2 * UM_ROWS * 4; i += CDC_CTA) {
      const int p = i >> 9, b = (i >> 2) & 127, q = i & 3;
      const uint4 v = *reinterpret_cast<const uint4*>((p ? s_xi : s_xr) + 32 * b + 16 * q);
      *reinterpret_cast<uint4*>(&S.ax[p][um_off(b, 16 * q)]) = v;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    um_fence_before();
    __syncthreads();  // operands written; previous item's TMEM reads complete
    um_fence_after();
    if (tid == 0) {
      // MMA 1: cols 64 (2 p + l) + bin, l = 0: T1 (u8), 1: T0 (s8)
#pragma unroll
      for (int p = 0; p < 2; ++p)
#pragma unroll
        for (int l = 0; l < 2; ++l)
#pragma unroll
          for (int ks = 0; ks < 2; ++ks)
            um_mma(tmem + 64 * (2 * p + l), um_desc(&S.ax[p][256 * ks]), um_desc(&S.bf[l][256 * ks]),
                   um_idesc(64, true, l == 1), ks > 0);
      um_commit(&S.mbar_mma);
    }
    um_wait(&S.mbar_mma, mphase);
    mphase ^= 1u;
    um_fence_after();
    // ---- stage 1: this thread's row, bins [32 half, 32 half + 32), 8 at a time; the
    // TMEM loads of the next 8 bins are in flight while these are computed
    uint32_t fl_s = 0, fl_d = 0;  // w == 65536 bits per bin (rare)
    int32_t acc[2][4][8];
#pragma unroll
    for (int gq = 0; gq < 4; ++gq) um_ld8(tlane + 64 * gq + 32 * half, acc[0][gq]);
    um_ld_wait();
#pragma unroll
    for (int c8 = 0; c8 < 4; ++c8) {
      int32_t (&cur)[4][8] = acc[c8 & 1];
#pragma unroll
      for (int gq = 0; gq < 4; ++gq) um_ld_fence(cur[gq]);
      if (c8 < 3) {
#pragma unroll
        for (int gq = 0; gq < 4; ++gq) um_ld8(tlane + 64 * gq + 32 * half + 8 * (c8 + 1), acc[(c8 + 1) & 1][gq]);
      }
      const int k0 = 32 * half + 8 * c8;
      uint32_t ws[8], wd[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const uint4 be = S.beta[k0 + e];
        const int32_t xr = cur[0][e] * 256 + cur[1][e];
        const int32_t xi = cur[2][e] * 256 + cur[3][e];
        ws[e] = tc_w(xr, xi, be.x, be.y);
        wd[e] = tc_w(xr, xi, be.z, be.w);
        fl_s |= (ws[e] >> 16) << (8 * c8 + e);
        fl_d |= (wd[e] >> 16) << (8 * c8 + e);
      }
      // limb bytes (w ^ 0x80 per byte): 8 bins = 8 contiguous bytes of the K-major row
      uint32_t sl[2], sh[2], dl[2], dh[2];
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        tc_pack(ws[4 * q], ws[4 * q + 1], ws[4 * q + 2], ws[4 * q + 3], sl[q], sh[q]);
        tc_pack(wd[4 * q], wd[4 * q + 1], wd[4 * q + 2], wd[4 * q + 3], dl[q], dh[q]);
      }
      const int o = um_off(row, k0);
      *reinterpret_cast<uint2*>(&S.ai[0][o]) = make_uint2(sl[0], sl[1]);
      *reinterpret_cast<uint2*>(&S.ai[1][o]) = make_uint2(sh[0], sh[1]);
      *reinterpret_cast<uint2*>(&S.ai[2][o]) = make_uint2(dl[0], dl[1]);
      *reinterpret_cast<uint2*>(&S.ai[3][o]) = make_uint2(dh[0], dh[1]);
      if (c8 < 3) um_ld_wait();
    }
    S.flags[row][0][half] = fl_s;
    S.flags[row][1][half] = fl_d;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    um_fence_before();
    __syncthreads();  // inverse operands written; MMA-1 accumulators consumed
    um_fence_after();
    if (tid == 0) {
      // MMA 2: z_re from s (A = ai 0/1, B = bi 0/1), z_im from d (ai 2/3, bi 2/3);
      // cols 96 sd + {0: Q11, 32: Qmid, 64: Q00} + output
#pragma unroll
      for (int sd = 0; sd < 2; ++sd) {
        const uint32_t d0 = tmem + 96 * sd;
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
          const uint64_t aL = um_desc(&S.ai[2 * sd][256 * ks]), aH = um_desc(&S.ai[2 * sd + 1][256 * ks]);
          const uint64_t b1 = um_desc(&S.bi[2 * sd][256 * ks]), b0 = um_desc(&S.bi[2 * sd + 1][256 * ks]);
          um_mma(d0 + 0, aH, b1, um_idesc(32, true, false), ks > 0);   // Q11 += hi x t1
          um_mma(d0 + 32, aH, b0, um_idesc(32, true, true), ks > 0);   // Qmid += hi x t0
          um_mma(d0 + 32, aL, b1, um_idesc(32, true, false), true);    //       + lo x t1
          um_mma(d0 + 64, aL, b0, um_idesc(32, true, true), ks > 0);   // Q00 += lo x t0
        }
      }
      um_commit(&S.mbar_mma);
    }
    um_wait(&S.mbar_mma, mphase);
    mphase ^= 1u;
    um_fence_after();
    // ---- stage 2: outputs m' in [16 half, 16 half + 16) of this thread's block row
    const int64_t n0 = cta_blk0 * CDC_HOP - A.c;
    int64_t lo64 = n0, hi64 = n0 + (int64_t)CDC_BLK * CDC_HOP;
    const int64_t o_lo = io.out_first, o_hi = io.out_first + io.out_count;
    lo64 = lo64 < o_lo ? o_lo : lo64;
    hi64 = hi64 > o_hi ? o_hi : hi64;
    const int lo = (int)(lo64 - n0), hi = (int)(hi64 - n0);
    const uint32_t fl[2][2] = {{S.flags[row][0][0], S.flags[row][0][1]}, {S.flags[row][1][0], S.flags[row][1][1]}};
    TcStats st;
#pragma unroll 1
    for (int c8 = 0; c8 < 2; ++c8) {
      const int m0 = 16 * half + 8 * c8;  // kept-output index m - 32
      int32_t z[2][8];
#pragma unroll
      for (int sd = 0; sd < 2; ++sd) {
        int32_t q11[8], qm[8], q00[8];
        um_ld8(tlane + 96 * sd + 0 + m0, q11);
        um_ld8(tlane + 96 * sd + 32 + m0, qm);
        um_ld8(tlane + 96 * sd + 64 + m0, q00);
        um_ld_wait();
        um_ld_fence(q11);
        um_ld_fence(qm);
        um_ld_fence(q00);
        if ((fl[sd][0] | fl[sd][1]) != 0u) {
          // a flagged bin k carried value + 1: subtract its matrix column
          const int E = sd ? TC_E_IM : TC_E_RE;
          for (int w2 = 0; w2 < 2; ++w2) {
            uint32_t bits = fl[sd][w2];
            while (bits) {
              const int k = 32 * w2 + __ffs(bits) - 1;
              bits &= bits - 1;
#pragma unroll
              for (int e = 0; e < 8; ++e) q00[e] -= (int32_t)S.root[(E - (32 + m0 + e) * k) & 63];
            }
          }
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const int32_t zz = qm[e] * 256 + q00[e] - q11[e];
          z[sd][e] = (int32_t)f4_mod((uint32_t)(zz + (int32_t)(F4 * 16384u)) + 32768u);
        }
      }
      const int idx = 32 * row + m0;  // local output index of z[.][0]
      if (FAST) {
        int32_t zr8[8], zi8[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          zr8[e] = z[0][e] - 32768;
          zi8[e] = z[1][e] - 32768;
        }
        tc_store8(O, io.q_tie, s, n0 - io.out_first, idx, lo, hi, zr8, zi8, st);
      } else {
        uint32_t* u = s_u + row * UP + m0;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          u[e] = (uint32_t)z[0][e];
          u[CDC_BLK * UP + e] = (uint32_t)z[1][e];
        }
      }
    }
    um_fence_before();  // TMEM reads of this item precede the next item's MMA 1
    if (FAST) {
      if (O.acc) {
        const int pa = (int)(n0 & 1);  // even local indices carry phase n0 & 1
        const unsigned long long va[4] = {st.a2, st.a4 & 0xffffffffull, st.a4 >> 32, st.a4h};
        const unsigned long long vb[4] = {st.b2, st.b4 & 0xffffffffull, st.b4 >> 32, st.b4h};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          unsigned long long x = va[q], y = vb[q];
#pragma unroll
          for (int off = 16; off > 0; off >>= 1) {
            x += __shfl_xor_sync(0xffffffffu, x, off);
            y += __shfl_xor_sync(0xffffffffu, y, off);
          }
          if (lane == 0) {
            if (x) atomicAdd(io.decim_acc + ((int64_t)s * 2 + pa) * 4 + q, x);
            if (y) atomicAdd(io.decim_acc + ((int64_t)s * 2 + (pa ^ 1)) * 4 + q, y);
          }
        }
      }
    } else {
      __syncthreads();
      cdc_epilogue_generic<true>(A, s_u, s, n0, lo64, hi64);
    }
  }
  __syncthreads();
  um_fence_after();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem), "n"(UM_TMEM_COLS) : "memory");
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
  using TS = typename std::conditional<sizeof(TIN) == 1 || std::is_same<TIN, double>::value,
                                       int8_t, int32_t>::type;
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

// Persistent-grid launch configuration of a tensor-core CDC kernel on the current
// device: the dynamic shared-memory attribute is per device, so it is set (and the
// resident CTAs per SM measured) once per device ordinal.
struct TcLaunchCfg {
  std::atomic<int> per_sm{0};
  std::atomic<int> sms{0};
};
template <typename K>
static cudaError_t tc_launch_cfg(TcLaunchCfg (&cfgs)[64], K* k, int smem, int cap, int& per_sm, int& sms) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  TcLaunchCfg& c = cfgs[dev];
  if (c.per_sm.load(std::memory_order_acquire) == 0) {
    e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e == cudaSuccess)  // all of L1 as shared memory: the kernels stream, they do not cache
      e = cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    int n = 0, m = 0, smem_sm = 0, reserved = 0;
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&m, cudaDevAttrMultiProcessorCount, dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&reserved, cudaDevAttrReservedSharedMemoryPerBlock, dev);
    if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, CDC_CTA, smem);
    if (e != cudaSuccess) return e;
    // cap < 0: up to -cap CTAs (the occupancy API under-reports for the 85 KB tcgen05
    // variant, where ncu shows two resident CTAs; TMEM allows at most two), bounded by
    // what the SM's shared memory actually holds, so a smaller carve-out (another
    // driver's reservation, MIG, green contexts) shrinks the persistent grid instead
    // of running half of it as a serialized tail wave
    int v;
    if (cap < 0) {
      const int by_smem = smem_sm / (smem + reserved);
      v = by_smem < -cap ? by_smem : -cap;
      if (v < 1) v = 1;
      if (getenv("FNTGPU_DEBUG") && by_smem < -cap)
        fprintf(stderr, "tensor-core CDC kernel: shared memory holds %d CTAs per SM (wanted %d)\n",
                by_smem, -cap);
    } else {
      v = n > cap ? cap : (n > 0 ? n : 1);
    }
    c.sms.store(m, std::memory_order_relaxed);
    c.per_sm.store(v, std::memory_order_release);
    if (getenv("FNTGPU_DEBUG"))
      fprintf(stderr, "tensor-core CDC kernel on device %d: smem %d B, %d CTAs/SM by occupancy, grid %d x %d SMs\n",
              dev, smem, n, v, m);
  }
  per_sm = c.per_sm.load(std::memory_order_acquire);
  sms = c.sms.load(std::memory_order_relaxed);
  return cudaSuccess;
}

template <bool FAST>
static cudaError_t launch_tc(const CdcArgs& A, cudaStream_t st) {
  constexpr int SMEM = (int)sizeof(TcTables) + (FAST ? 0 : 2 * CDC_BLK * UP * 4);
  static TcLaunchCfg cfgs[64];
  int per_sm = 0, sms = 0;
  const cudaError_t e = tc_launch_cfg(cfgs, k_cdc64_tc<FAST>, SMEM, 3, per_sm, sms);
  if (e != cudaSuccess) return e;
  const int64_t items = (A.blk_count + CDC_BLK - 1) / CDC_BLK * A.io.n_streams;
  const int64_t full = (int64_t)per_sm * sms;
  const unsigned grid = (unsigned)(items < full ? items : full);
  k_cdc64_tc<FAST><<<grid, CDC_CTA, SMEM, st>>>(A);
  return cudaGetLastError();
}

template <bool FAST>
static cudaError_t launch_f64p(const CdcArgs& A, cudaStream_t st) {
  constexpr int SMEM = F64P_RAWB + F64P_WORK;
  static TcLaunchCfg cfgs[64];
  int per_sm = 0, sms = 0;
  const cudaError_t e = tc_launch_cfg(cfgs, k_cdc64_f64p<FAST>, SMEM, CDC_F64P_PLANES == 2 ? 2 : CDC_MIN_CTAS,
                                      per_sm, sms);
  if (e != cudaSuccess) return e;
  const int64_t items = (A.blk_count + CDC_BLK - 1) / CDC_BLK * A.io.n_streams;
  const int64_t full = (int64_t)per_sm * sms;
  const unsigned grid = (unsigned)(items < full ? items : full);
  k_cdc64_f64p<FAST><<<grid, CDC_CTA, SMEM, st>>>(A);
  return cudaGetLastError();
}

template <bool FAST>
static cudaError_t launch_umma(const CdcArgs& A, cudaStream_t st) {
  constexpr int SMEM = (int)sizeof(UmmaSmem) + (FAST ? 0 : 2 * CDC_BLK * UP * 4);
  static TcLaunchCfg cfgs[64];
  int per_sm = 0, sms = 0;
  // 256 TMEM columns per CTA: two resident CTAs hold all 512 columns of an SM
  const cudaError_t e = tc_launch_cfg(cfgs, k_cdc64_umma<FAST>, SMEM, FAST ? -2 : 2, per_sm, sms);
  if (e != cudaSuccess) return e;
  const int64_t items = (A.blk_count + CDC_BLK - 1) / CDC_BLK * A.io.n_streams;
  const int64_t full = (int64_t)per_sm * sms;
  const unsigned grid = (unsigned)(items < full ? items : full);
  k_cdc64_umma<FAST><<<grid, CDC_CTA, SMEM, st>>>(A);
  return cudaGetLastError();
}

cudaError_t launch_cdc64(const fntgpu_cdc_taps& taps, const fntgpu_cdc_io& io, cudaStream_t st) {
  if (io.out_count <= 0 || io.n_streams <= 0) return cudaSuccess;
  CdcArgs A;
  scale_taps(taps.b_plus, A.bp);
  scale_taps(taps.b_minus, A.bm);
  for (int k = 0; k < CDC_N; ++k) {
    A.rbp[k] = taps.b_plus[k] % F4;
    A.rbm[k] = taps.b_minus[k] % F4;
  }
  A.io = io;
  A.c = taps.n_taps / 2;
  A.q_away = 0;
  if (io.qr && io.q_shift >= 1 && io.q_max >= 0 && io.q_max < 128) {
    A.q_away = 1;
    for (int j = 0; j <= io.q_max; ++j)
      if (io.q_tie[j] != (j + 1 < io.q_max ? j + 1 : io.q_max)) A.q_away = 0;
  }
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
  if (io.in_dtype != FNTGPU_I8 && io.in_dtype != FNTGPU_I32 && io.in_dtype != FNTGPU_I64 &&
      io.in_dtype != FNTGPU_F64)
    return cudaErrorInvalidValue;
  // Tensor-core forms for int8 planes (their samples are the int8 MMA operands), on
  // request only. Auto runs the shift-add butterflies: the tcgen05 form measured
  // 1.07x at config 4 and 1.01x in the config-5 chain (profiles/cdc_tc_r01.json), below
  // the 1.15x that would justify its TMEM / residency assumptions as the default
  // (DESIGN.md section 3); mma.sync measured 0.87-0.90x.
  int kern = taps.kernel;
  if (kern == FNTGPU_CDC_KERNEL_AUTO) kern = FNTGPU_CDC_KERNEL_SHIFT;
  if (io.in_dtype == FNTGPU_I8 && kern == FNTGPU_CDC_KERNEL_TC) {
    A.s_base = 0;
    return fast ? launch_tc<true>(A, st) : launch_tc<false>(A, st);
  }
  if (io.in_dtype == FNTGPU_I8 && kern == FNTGPU_CDC_KERNEL_UMMA) {
    A.s_base = 0;
    return fast ? launch_umma<true>(A, st) : launch_umma<false>(A, st);
  }
  if (io.in_dtype == FNTGPU_F64 && CDC_F64P) {
    A.s_base = 0;
    return fast ? launch_f64p<true>(A, st) : launch_f64p<false>(A, st);
  }
  for (int64_t s0 = 0; s0 < io.n_streams; s0 += 65535) {
    A.s_base = (int32_t)s0;
    grid.y = (unsigned)(io.n_streams - s0 < 65535 ? io.n_streams - s0 : 65535);
    cudaError_t e;
    switch (io.in_dtype) {
      case FNTGPU_I8:
        e = fast ? launch_k<int8_t, true>(A, grid, st) : launch_k<int8_t, false>(A, grid, st);
        break;
      case FNTGPU_I32: e = launch_k<int32_t, false>(A, grid, st); break;
      case FNTGPU_F64:
        e = fast ? launch_k<double, true>(A, grid, st) : launch_k<double, false>(A, grid, st);
        break;
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
