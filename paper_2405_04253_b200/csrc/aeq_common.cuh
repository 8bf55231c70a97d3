// aeq_common.cuh -- FNT-AEQ pieces shared by the one-warp-per-stream kernel
// (k_aeq.cu) and the polarization-split kernel (k_aeq_pol.cu): the launch
// argument block, the float64 update primitives in numpy's rounding, the exact
// y_int / D division, the ring decision and the packed 14-bit tap formats.
//
// Reference: fntdsp/aeq.py:53-58 (rde_error), 118-170 (equalize_block,
// update_taps), fntdsp/fixedpoint.py:111-143 (split_taps / recombine).
#pragma once
#include <cmath>
#include <cstring>

#ifndef FNT_CARRY_MODE
#define FNT_CARRY_MODE 0
#endif
#include "fermat.cuh"
#include "internal.h"

namespace fntgpu {

constexpr int AEQ_L = 16;            // taps per filter = hop (aeq.py:45)
constexpr int AEQ_N = 32;            // block length
constexpr int AEQ_TAP_MAX = 16383;   // TAP_MAG_MAX (aeq.py:26)
constexpr int XF_LUT = 128;          // x / sig_scale table for |x| <= 128 (int8 includes -128)

struct AeqArgs {
  fntgpu_aeq_params prm;
  fntgpu_aeq_io io;
  double R2[8];               // radii[i] * radii[i] (nearest ** 2, aeq.py:58)
  double T[8];                // ring decision thresholds on r2 (rde fast path, see rde_thresholds)
  double D;                   // sig_scale * tap_scale (aeq.py:142)
  double Dinv;                // RN(1 / D): y = y_int / D by one Markstein correction step
  int32_t fast_rde;           // 1: ring chosen by comparing r2 with T[] (no sqrt)
  int32_t fast_div;           // 1: D in [2^-500, 2^500] (div_D's correction step is exact)
};

__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }

// sign-extended byte k (0..3, may be a runtime value) of w
__device__ __forceinline__ int32_t sbyte(uint32_t w, uint32_t k) {
  return (int32_t)(w << (24u - 8u * k)) >> 24;
}

// split_taps (fixedpoint.py:111-121): sign * (|w| >> 7) or sign * (|w| & 127)
// (|w| < 2^14 always: taps are clipped to +-16383 and split_taps rejects larger)
__device__ __forceinline__ int32_t tap_group(int32_t w, int g) {
  const int32_t m = abs(w);
  const int32_t v = (m >> (g ? 0 : 7)) & 127;
  return w < 0 ? -v : v;
}

// rde_error (aeq.py:53-58) for one output pair (y_I, y_Q). The 3-ring case
// (16QAM, qam16_radii) is unrolled; other ring counts loop.
template <bool QUICK = false>
__device__ __forceinline__ double rde(double yi, double yq, const AeqArgs& A) {
  const double r2 = dadd(dmul(yi, yi), dmul(yq, yq));
  double best_r2;
  if (QUICK) {  // launch-time checked: fast_rde && n_radii == 3
    best_r2 = r2 >= A.T[2] ? A.R2[2] : (r2 >= A.T[1] ? A.R2[1] : A.R2[0]);
    return dsub(best_r2, r2);
  }
  if (A.fast_rde) {
    // argmin_i |sqrt(r2) - R_i| is a step function of r2 over the reachable range;
    // the host located its steps exactly (rde_thresholds), so no sqrt is needed.
    if (A.prm.n_radii == 3) {
      best_r2 = r2 >= A.T[2] ? A.R2[2] : (r2 >= A.T[1] ? A.R2[1] : A.R2[0]);
    } else {
      int sel = 0;
      for (int i = 1; i < A.prm.n_radii; ++i) sel += r2 >= A.T[i];
      best_r2 = A.R2[sel];
    }
    return dsub(best_r2, r2);
  }
  const double r = __dsqrt_rn(r2);
  if (A.prm.n_radii == 3) {
    const double d0 = fabs(dsub(r, A.prm.radii[0]));
    const double d1 = fabs(dsub(r, A.prm.radii[1]));
    const double d2 = fabs(dsub(r, A.prm.radii[2]));
    // np.argmin: first minimum
    const bool take1 = d1 < d0;
    const double dm = take1 ? d1 : d0;
    best_r2 = d2 < dm ? A.R2[2] : (take1 ? A.R2[1] : A.R2[0]);
  } else {
    int best = 0;
    double bd = fabs(dsub(r, A.prm.radii[0]));
    for (int i = 1; i < A.prm.n_radii; ++i) {
      const double d = fabs(dsub(r, A.prm.radii[i]));
      if (d < bd) { bd = d; best = i; }
    }
    best_r2 = A.R2[best];
  }
  return dsub(best_r2, r2);
}

// np.rint(w * tap_scale).astype(int64), then |.| > 16383 -> count and clip
// (aeq.py:165-168). Values whose rint is not a representable int64 (|r| >= 2^63,
// NaN) become INT64_MIN in numpy on x86-64: not counted, clipped to -16383.
// cvt.rni.s32.f64 rounds half-to-even like np.rint and saturates, so |rint| > 16383
// is read off the int32; |p| >= 2^63 exactly when |rint(p)| >= 2^63 (doubles there
// are integers).
__device__ __forceinline__ int32_t requantize_tap(double w, double tap_scale, uint32_t& sat) {
  const double p = dmul(w, tap_scale);
  const int32_t i = __double2int_rn(p);
  const bool huge = !(fabs(p) < 9.2233720368547758e18);
  const int32_t c = min(max(i, -AEQ_TAP_MAX), AEQ_TAP_MAX);
  sat += (c != i) & !huge;  // clipped exactly when |rint| > 16383
  return huge ? -AEQ_TAP_MAX : c;
}

// y_int / D correctly rounded: q0 = RN(y_int * RN(1/D)) is within 1 ulp of the
// quotient, the residual y_int - q0 D is exact in one FMA, and one more FMA rounds
// the corrected quotient (Markstein's theorem; no over/underflow for |y_int| < 2^32
// and the D range the host admits). fntgpu_aeq_selfcheck (tests/test_gpu_parity.py)
// checks it against IEEE division over every int32 numerator for the configured D.
template <bool QUICK = false>
__device__ __forceinline__ double div_D(int32_t yi, const AeqArgs& A) {
  const double a = (double)yi;
  if (!QUICK && !A.fast_div) return __ddiv_rn(a, A.D);
  const double q0 = dmul(a, A.Dinv);
  const double r = __fma_rn(-q0, A.D, a);
  return __fma_rn(r, A.Dinv, q0);
}

// Both 7-bit groups of a tap in one word: p = sign * (hi + lo * 2^16) with
// hi = |w| >> 7, lo = |w| & 127 (fixedpoint.py:111-121). Since w = sign (128 hi + lo),
// p = w * 2^16 - (w / 128) * (2^23 - 1) (C division truncates like sign * (|w| >> 7)).
// Unpack: hi group = low 16 bits sign-extended (|hi| < 2^15); lo group =
// (p + 2^15) >> 16 (the low half's sign borrow is cancelled by the rounding).
__device__ __forceinline__ uint32_t pack_groups(int32_t w) {
  return (uint32_t)(w * 65536 - (w / 128) * 8388607);
}
__device__ __forceinline__ int32_t unpack_group(uint32_t p, int g) {
  return g ? ((int32_t)(p + 0x8000u) >> 16) : ((int32_t)(p << 16) >> 16);
}

// FNT forward with the transform-domain sum over input streams (AEQ_FUSE_T): taps
// are kept as balanced base-64 digits instead, w = 64 a + b with b in [-32, 31] and
// |a| <= 256.
// The balanced digits are packed as two 16-bit halves, p = (a mod 2^16) | b << 16,
// and read back with PRMT's sign-replicating selectors: one instruction per digit,
// and the byte select can take the half from either of two words (own / partner).
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
  return r;
}
constexpr uint32_t DIG_A = 0x9910u;    // sign-extended low half of the first word: digit a
constexpr uint32_t DIG_B = 0xBB32u;    // sign-extended high half of the first word: digit b
constexpr uint32_t DIG_A2 = 0xDD54u;   // digit a of the second word
constexpr uint32_t DIG_B2 = 0xFF76u;   // digit b of the second word
template <bool BAL>
__device__ __forceinline__ uint32_t pack_taps(int32_t w) {
  if (!BAL) return pack_groups(w);
  const int32_t a = (w + 32) >> 6;                      // w = 64 a + b, b in [-32, 31]
  return prmt((uint32_t)a, (uint32_t)(w - 64 * a), 0x5410u);
}
template <bool BAL>
__device__ __forceinline__ int32_t unpack_tap(uint32_t p) {
  if (!BAL) return 128 * unpack_group(p, 0) + unpack_group(p, 1);
  return 64 * (int32_t)prmt(p, 0u, DIG_A) + (int32_t)prmt(p, 0u, DIG_B);
}
// the reference's split_taps group g of a packed tap (fixedpoint.py:111-121)
template <bool BAL>
__device__ __forceinline__ int32_t ref_group(uint32_t p, int g) {
  if (!BAL) return unpack_group(p, g);
  return tap_group(unpack_tap<true>(p), g);
}

// x / sig_scale exactly as numpy's true_divide (IEEE) from a table of the int8 range
// (all of it, -128 included); wider inputs fall back to the division.
template <bool NARROW>
__device__ __forceinline__ double xf_of(int32_t x, const double* lut, double sig) {
  if (NARROW) return lut[x + XF_LUT];
  return (x >= -XF_LUT && x <= XF_LUT) ? lut[x + XF_LUT] : __ddiv_rn((double)x, sig);
}

// polarization-split form of k_aeq_process (k_aeq_pol.cu): two warps per stream
cudaError_t launch_aeq_pol(fntgpu_aeq_state* st, const AeqArgs& A, cudaStream_t s);

}  // namespace fntgpu
