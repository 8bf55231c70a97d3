// fermat.cuh -- Fermat-ring arithmetic for the sm_100a FNT kernels.
//
// Reference semantics: fntdsp/fermat.py:56-117 (reduce, mul_pow2, sqrt2) and the
// vectorised residue arithmetic of fntdsp/fnt.py:86-161.
//
// B200 design: F4 = 2^16 + 1 divides M = 2^32 - 1 = (2^16 - 1)(2^16 + 1). Every
// transform / product / sum is therefore computed in the ring Z/M on full 32-bit
// words and reduced mod F4 once, at the end. In Z/M:
//   * a + b  = 32-bit add + end-around carry          (IADD3 + IMAD.X)
//   * a - b  = a + ~b                                  (IMAD + IADD3 + IMAD.X)
//   * a * 2^j = 32-bit rotate left by j               (one SHF.L.W)
//   * -a     = ~a                                      (free inside LOP3 / swaps)
// so a radix-2 butterfly with a power-of-two twiddle is 6 integer instructions
// split evenly over the ALU and FMA pipes, with no data-dependent reduction, and the sqrt(2) twiddles of the 64-point plan
// (sqrt2 = 2^12 - 2^4, fermat.py:111-117) are two rotates and one subtraction.
// The final fold x mod F4 = lo16 - hi16 (fermat.py:56-66) is one SHF + one IMAD.
#pragma once
#include <cstdint>

namespace fntgpu {

constexpr uint32_t F4 = 65537u;
constexpr int32_t F4_HALF = 32768;

// Pipe balance. On sm_100 the ALU pipe (IADD3 with carry-out, IADD3.X, SHF, LOP3)
// and the FMA pipe (IMAD*, incl. IMAD.X) each accept one warp instruction every
// other cycle per SM sub-partition. A carry-propagating add must start on the ALU
// (IADD3 writes the carry predicate) but its end-around carry can finish on the
// FMA pipe (madc -> IMAD.X), and a - b = a + ~b in Z/M with ~b computed as
// b * (-1) + (-1) (IMAD). A rotate-twiddled butterfly is then 3 ALU + 3 FMA
// instructions (6 issue cycles) instead of 4 ALU + 1 FMA (8 cycles on the ALU pipe):
// tools/bfly_bench.cu measures 5.76 vs 4.59 T butterflies/s on B200.
// FNT_CARRY_MODE 0 keeps the plain addc / subc forms for A/B comparison.
#ifndef FNT_CARRY_MODE
#define FNT_CARRY_MODE 2
#endif
// -1 that ptxas cannot constant-fold (a literal -1 multiplier becomes an ALU IADD3)
static __constant__ uint32_t c_fnt_minus1 = 0xFFFFFFFFu;

// a + b (mod 2^32 - 1); CM selects the carry form per call site (default: the
// translation unit's FNT_CARRY_MODE)
template <int CM = FNT_CARRY_MODE>
__device__ __forceinline__ uint32_t m_add(uint32_t a, uint32_t b) {
  uint32_t r;
  if (CM == 2) {
    asm("{\n\t.reg .u32 t;\n\tadd.cc.u32 t, %1, %2;\n\tmadc.lo.u32 %0, t, 1, 0;\n\t}"
        : "=r"(r) : "r"(a), "r"(b));
  } else {
    asm("{\n\t.reg .u32 t;\n\tadd.cc.u32 t, %1, %2;\n\taddc.u32 %0, t, 0;\n\t}"
        : "=r"(r) : "r"(a), "r"(b));
  }
  return r;
}

// a - b (mod 2^32 - 1)
template <int CM = FNT_CARRY_MODE>
__device__ __forceinline__ uint32_t m_sub(uint32_t a, uint32_t b) {
  uint32_t r;
  if (CM == 2) {
    const uint32_t m1 = c_fnt_minus1;
    asm("{\n\t.reg .u32 t, nb;\n\tmad.lo.u32 nb, %2, %3, %3;\n\tadd.cc.u32 t, %1, nb;\n\t"
        "madc.lo.u32 %0, t, 1, 0;\n\t}"
        : "=r"(r) : "r"(a), "r"(b), "r"(m1));
  } else {
    asm("{\n\t.reg .u32 t;\n\tsub.cc.u32 t, %1, %2;\n\tsubc.u32 %0, t, 0;\n\t}"
        : "=r"(r) : "r"(a), "r"(b));
  }
  return r;
}

// a * 2^j (mod 2^32 - 1), j in [0, 32). FNT_ROT_MODE 0: one funnel shift (ALU
// pipe); 1: one 32x32->64 IMAD.WIDE (FMA pipe) + disjoint-bit add, to balance pipes.
#ifndef FNT_ROT_MODE
#define FNT_ROT_MODE 0
#endif
__device__ __forceinline__ uint32_t m_rot(uint32_t a, int j) {
  if (j == 0) return a;
#if FNT_ROT_MODE == 1
  uint32_t lo, hi;
  asm("{\n\t.reg .u64 p;\n\tmul.wide.u32 p, %2, %3;\n\tmov.b64 {%0, %1}, p;\n\t}"
      : "=r"(lo), "=r"(hi) : "r"(a), "r"(1u << j));
  return lo + hi;
#else
  return __funnelshift_l(a, a, j);
#endif
}

// a * b (mod 2^32 - 1): 64-bit product folded with 2^32 == 1. FNT_MUL_MODE 1 (default)
// forms the product with one IMAD.WIDE instead of IMAD + IMAD.HI (measured: CDC
// 35.9 -> 35.3 ms at config 5, 147 -> 154 Gsamples/s at config 4; AEQ 138.0 -> 136.6 ms).
#ifndef FNT_MUL_MODE
#define FNT_MUL_MODE 1
#endif
__device__ __forceinline__ uint32_t m_mul(uint32_t a, uint32_t b) {
#if FNT_MUL_MODE == 1
  uint32_t lo, hi;
  asm("{\n\t.reg .u64 p;\n\tmul.wide.u32 p, %2, %3;\n\tmov.b64 {%0, %1}, p;\n\t}"
      : "=r"(lo), "=r"(hi) : "r"(a), "r"(b));
  return m_add(lo, hi);
#else
  return m_add(a * b, __umulhi(a, b));
#endif
}

// Canonical residue in [0, F4) of a word of Z/M.
__device__ __forceinline__ uint32_t f4_canon(uint32_t x) {
  int32_t r = (int32_t)(x - (x >> 16) * F4);  // lo16 - hi16 in [-65535, 65535]
  return (uint32_t)(r < 0 ? r + (int32_t)F4 : r);
}

// Signed residue in [-32768, 32768]: decode_signed(canon(x)) (fermat.py:117-118, 131-133).
__device__ __forceinline__ int32_t f4_signed(uint32_t x) {
  int32_t r = (int32_t)(x - (x >> 16) * F4);
  r = r > F4_HALF ? r - (int32_t)F4 : r;
  r = r < -F4_HALF ? r + (int32_t)F4 : r;
  return r;
}

// Canonical residue x mod F4 in [0, F4) of any 32-bit word: floor(x / 65537) =
// umulhi(x, 0xFFFF0001) >> 16 exactly for every x < 2^32 (checked exhaustively), so
// this is IMAD.HI + SHF + IMAD with no data-dependent correction. The signed decode
// (fermat.py:131-133) of a residue r is (r + 32768) mod F4 - 32768: callers add the
// 32768 before the transform or sum and subtract it after their reduction.
__device__ __forceinline__ uint32_t f4_mod(uint32_t x) {
  const uint32_t q = __umulhi(x, 0xFFFF0001u) >> 16;
  return x - q * F4;
}

// Encode a signed integer |v| < 2^31 - F4*256 into Z/M with the right residue mod F4.
// Adding a multiple of F4 keeps the residue (the mod-M class does not matter:
// only the final mod-F4 reduction is observed).
constexpr uint32_t F4_BIAS = 65537u * 256u;  // > 32768 * 257, keeps v + bias >= 0
__device__ __forceinline__ uint32_t f4_enc_small(int32_t v) { return (uint32_t)(v + (int32_t)F4_BIAS); }

// Encode an arbitrary int64 into Z/M (fnt.py accepts any int64 and reduces it,
// probe t17): v = hi * 2^32 + lo == hi + lo (mod 2^32 - 1), with a negative hi
// represented as M + hi. No 64-bit division.
__device__ __forceinline__ uint32_t f4_enc64(int64_t v) {
  const uint32_t lo = (uint32_t)(uint64_t)v;
  const int32_t hi = (int32_t)((uint64_t)v >> 32);
  const uint32_t h = (uint32_t)hi - (hi < 0 ? 1u : 0u);
  return m_add(lo, h);
}

// ---------------------------------------------------------------------------
// Twiddles of the two shift-add plans, as compile-time-resolved operations.
//   kind RADIX2 : alpha = 2, N <= 32         alpha^e = 2^e
//   kind SQRT2  : alpha = 2^12 - 2^4 (4080), N = 64
//                 alpha^(2h) = 2^h, alpha^(2h+1) = 2^h * (2^12 - 2^4)
//   kind RADIX4 : alpha = 2^2, N <= 16          alpha^e = 2^(2e)  (sub-transforms of
//   kind RADIX16: alpha = 2^4, N <= 8           alpha^e = 2^(4e)   a 32-point one)
//   kind RADIX256: alpha = 2^8, N <= 4          alpha^e = 2^(8e)
// The result is returned as (value, negate) where negate means the caller must
// use -value (absorbed by swapping the butterfly's add and subtract): a rotate
// by r >= 16 equals -(rotate by r - 16) modulo F4.
enum TwKind { RADIX2 = 0, SQRT2 = 1, RADIX16 = 2, RADIX4 = 3, RADIX256 = 4 };

struct Tw {
  uint32_t v;
  bool neg;
};

template <int KIND, int CM = FNT_CARRY_MODE>
__device__ __forceinline__ Tw twiddle(uint32_t a, int e /* exponent of alpha, >= 0 */) {
  if (KIND != SQRT2) {
    int r = (KIND == RADIX256 ? 8 * e : KIND == RADIX16 ? 4 * e : KIND == RADIX4 ? 2 * e : e) & 31;
    if (r >= 16) return {m_rot(a, r - 16), true};
    return {m_rot(a, r), false};
  } else {
    e &= 63;
    if ((e & 1) == 0) {
      int r = (e >> 1) & 31;
      if (r >= 16) return {m_rot(a, r - 16), true};
      return {m_rot(a, r), false};
    }
    int h = e >> 1;
    int r1 = (h + 12) & 31, r2 = (h + 4) & 31;
    bool neg = false;
    // 2^r1 - 2^r2; fold rotates >= 16 into signs, preferring one overall negate.
    if (r1 >= 16 && r2 >= 16) { r1 -= 16; r2 -= 16; neg = true; }
    if (r1 >= 16) {  // -(2^(r1-16)) - 2^r2 = -(2^(r1-16) + 2^r2)
      return {m_add<CM>(m_rot(a, r1 - 16), m_rot(a, r2)), !neg};
    }
    if (r2 >= 16) {  // 2^r1 + 2^(r2-16)
      return {m_add<CM>(m_rot(a, r1), m_rot(a, r2 - 16)), neg};
    }
    return {m_sub<CM>(m_rot(a, r1), m_rot(a, r2)), neg};
  }
}

// Radix-2 DIT butterfly (fnt.py:94-102): (u, v) -> (u + tw*v, u - tw*v).
template <int KIND, int CM = FNT_CARRY_MODE>
__device__ __forceinline__ void bfly(uint32_t& u, uint32_t& v, int e) {
  Tw t = twiddle<KIND, CM>(v, e);
  uint32_t s = t.neg ? m_sub<CM>(u, t.v) : m_add<CM>(u, t.v);
  uint32_t d = t.neg ? m_add<CM>(u, t.v) : m_sub<CM>(u, t.v);
  u = s;
  v = d;
}

// Only the difference output u - tw*v (pruned last stage of an inverse transform).
template <int KIND, int CM = FNT_CARRY_MODE>
__device__ __forceinline__ uint32_t bfly_hi(uint32_t u, uint32_t v, int e) {
  Tw t = twiddle<KIND, CM>(v, e);
  return t.neg ? m_add<CM>(u, t.v) : m_sub<CM>(u, t.v);
}

__host__ __device__ constexpr int ilog2(int n) { return n <= 1 ? 0 : 1 + ilog2(n >> 1); }

__host__ __device__ constexpr int bitrev(int i, int lg) {
  int r = 0;
  for (int b = 0; b < lg; ++b) { r = (r << 1) | ((i >> b) & 1); }
  return r;
}

// natural order -> bit-reversed order (register renaming only; free after unrolling)
template <int N>
__device__ __forceinline__ void to_bitrev(uint32_t (&a)[N]) {
  constexpr int LG = ilog2(N);
  uint32_t t[N];
#pragma unroll
  for (int i = 0; i < N; ++i) t[bitrev(i, LG)] = a[i];
#pragma unroll
  for (int i = 0; i < N; ++i) a[i] = t[i];
}

// In-register radix-2 DIT transform over a[N] held in BIT-REVERSED order on entry,
// natural order on exit (fnt.py:86-103). INV selects alpha^-1 twiddles (the N^-1
// scale is left to the caller, who folds it into a rotate). ZERO_TOP declares that
// inputs with natural index >= N/2 are zero (first stage becomes a copy).
// PRUNE_LO skips the low-half outputs of the last stage (only a[N/2..N) valid).
// Stages are expanded by template recursion so every register index is a
// compile-time constant (no local-memory arrays).
// Stages [S, S_END) are run (S_END = -1: to the end).
template <int N, int KIND, bool INV, bool ZERO_TOP, bool PRUNE_LO, int S, int S_END = -1,
          int CM = FNT_CARRY_MODE>
__device__ __forceinline__ void fnt_stage(uint32_t (&a)[N]) {
  constexpr int LG = ilog2(N);
  constexpr int END = S_END < 0 ? LG : S_END;
  constexpr int half = 1 << S;
  constexpr int step = N >> (S + 1);
#pragma unroll
  for (int q = 0; q < N / 2; ++q) {
    const int g = (q / half) * 2 * half;
    const int j = q % half;
    int e = j * step;
    if (INV) e = (N - e) % N;
    if (ZERO_TOP && S == 0) {
      a[g + j + half] = a[g + j];
    } else if (PRUNE_LO && S == LG - 1) {
      a[g + j + half] = bfly_hi<KIND, CM>(a[g + j], a[g + j + half], e);
    } else {
      bfly<KIND, CM>(a[g + j], a[g + j + half], e);
    }
  }
  if constexpr (S + 1 < END) fnt_stage<N, KIND, INV, ZERO_TOP, PRUNE_LO, S + 1, S_END, CM>(a);
}

template <int N, int KIND, bool INV, bool ZERO_TOP = false, bool PRUNE_LO = false,
          int CM = FNT_CARRY_MODE>
__device__ __forceinline__ void fnt_dit(uint32_t (&a)[N]) {
  fnt_stage<N, KIND, INV, ZERO_TOP, PRUNE_LO, 0, -1, CM>(a);
}

// Stages [S, S_END) of a forward RADIX2 DIT transform on small signed integers in
// plain two's-complement arithmetic: while |values| * 2^e stays below 2^31 no
// modular reduction is needed, so a butterfly is one shift and two adds (no
// carries). Callers bound the magnitudes and move to Z/M with a bias add after.
// BIAS (a multiple of F4 above the magnitude bound) is added to every output of the
// last stage inside its 3-input adds, making the words non-negative residues of Z/M
// for the modular stages that follow at no extra instruction.
template <int N, int KIND, int S, int S_END, uint32_t BIAS = 0>
__device__ __forceinline__ void fnt_stage_plain(uint32_t (&a)[N]) {
  constexpr int half = 1 << S;
  constexpr int step = N >> (S + 1);
  constexpr uint32_t B = S + 1 == S_END ? BIAS : 0u;
#pragma unroll
  for (int q = 0; q < N / 2; ++q) {
    const int g = (q / half) * 2 * half;
    const int j = q % half;
    // alpha^(j step): RADIX2 2^(j step); SQRT2 (even exponents only in these
    // early stages) 2^(j step / 2)
    const int e = KIND == RADIX2 ? j * step : KIND == RADIX4 ? 2 * j * step : (j * step) / 2;
    static_assert(KIND != SQRT2 || ((N >> (S + 1)) % 2 == 0), "odd sqrt2 power in a plain stage");
    const uint32_t u = a[g + j], w = a[g + j + half] << e;
    a[g + j] = u + w + B;
    a[g + j + half] = u - w + B;
  }
  if constexpr (S + 1 < S_END) fnt_stage_plain<N, KIND, S + 1, S_END, BIAS>(a);
}

}  // namespace fntgpu
