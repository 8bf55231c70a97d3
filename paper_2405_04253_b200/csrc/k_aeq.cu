// k_aeq.cu -- FNT-AEQ: 4x4 real-valued MIMO radius-directed block equalizer.
//
// Reference: fntdsp/aeq.py:53-58 (rde_error), 61-81 (RvMimoTaps, split_taps),
// 84-190 (FntAeq: __init__, _spectra, equalize_block, update_taps, process).
//
// One warp owns one stream for the whole call (the block recursion through the
// taps is strictly sequential, aeq.py:182-189). Lane = 8 s + 2 t + g with
//   s = output stream, t = input stream, g = tap group (hi/lo) in the forward
//   path and tap half (k in [8g, 8g+8)) in the update.
// Taps (float w and 14-bit w_int) live in registers across all blocks. Inputs
// arrive two samples per lane per block (lane L loads samples 2(L&7), 2(L&7)+1 of
// input stream L>>3, one block ahead) into per-warp shared rings of the block's
// integers and of x / sig_scale, so no lane ever indexes registers dynamically.
//
// Forward path, FNTGPU_AEQ_FWD_FNT (aeq.py:118-144): the four 32-point input
//   transforms are computed by 8 lanes each in registers + shuffles (four-step
//   form); lane (s,t,g) transforms its 16-tap group padded to 32 in registers
//   (first DIT stage free, the next two carry-free), multiplies pointwise (the 32
//   general products of that filter group), runs the inverse pruned to outputs
//   16..31 and decodes -- the reference's residue convolution per (group, s, t);
//   recombine 128*hi + lo and sum over t, g. All transforms: alpha = 2, rotates
//   in Z/(2^32-1) (fermat.cuh).
// Forward path, FNTGPU_AEQ_FWD_DIRECT: the same integer per-group sums computed
//   as a time-domain FIR (each group sum reduced mod F4 and decoded exactly as the
//   residue path, so the bits are identical for every input the reference accepts).
// Update (aeq.py:148-170): float64 with explicit __dmul_rn/__dadd_rn (never
//   contracted into FMA), correctly rounded division and ring decisions, numpy's einsum reduction order
//   over m (two lanes of even/odd m, unrolled by 4) and numpy's
//   pairwise order for the err_trace mean.
// Pipe balance for this kernel (fermat.cuh): the AEQ's FMA pipe already carries the
// residue products and the FP64 update's partner work, so the plain addc / subc
// forms measure faster here (tools/ab_run.sh: 161 vs 165 ms at config 5).
#ifndef FNT_CARRY_MODE
#define FNT_CARRY_MODE 0
#endif
#include "aeq_common.cuh"

namespace fntgpu {

#ifndef AEQ_WARPS
#define AEQ_WARPS 1                  // streams (warps) per CTA: one-warp CTAs schedule best
#endif                               // (FNT 124.4 -> 121.7 ms, direct 83.6 -> 75.0 ms vs 4)
#ifndef AEQ_LOCKSTEP
// With several warps per CTA, they meet every AEQ_LOCKSTEP blocks (power of two; 0 =
// never) so they walk the ~29 KB loop body together and share its instruction-cache
// lines (4-warp CTAs: 161 -> 156 ms at config 5). One-warp CTAs do not need it.
#define AEQ_LOCKSTEP (AEQ_WARPS > 1 ? 1 : 0)
#endif
#ifndef AEQ_IFNT_CM
#define AEQ_IFNT_CM FNT_CARRY_MODE   // carry form of the inverse transform (fermat.cuh)
#endif
#ifndef AEQ_TAP_CM
#define AEQ_TAP_CM FNT_CARRY_MODE    // carry form of the tap transform's modular stages
#endif
#ifndef AEQ_DP4A
#define AEQ_DP4A 1                   // DIRECT forward on int8 inputs by DP4A int8 dot products
#endif
#ifndef AEQ_PROBE
#define AEQ_PROBE 0                  // timing probes only: 1-4 drop one phase (wrong results)
#endif
#ifndef AEQ_FUSE_T
#define AEQ_FUSE_T 1                 // FNT forward: sum over t before the inverse when exact
#endif
#ifndef AEQ_MAC_T
#define AEQ_MAC_T 1                  // stream sum as 64-bit multiply-accumulates (fused_inverse_mac)
#endif
#ifndef AEQ_MIN_CTAS
// Register target of the launch bounds. 13 lets ptxas schedule with up to 157
// registers; every instance still lands at <= 128 (cuobjdump -res-usage), so 16
// one-warp CTAs stay resident per SM (shared memory allows 16), and the code is
// better scheduled than under a hard 128 cap (16): C5 AEQ 108.9 -> 105.0 ms.
#define AEQ_MIN_CTAS (13 / AEQ_WARPS)
#endif

struct __align__(16) AeqScratch {
  double wf[8][32];           // float taps (aeq.py:99), lane-contiguous: wf[kk][lane] = w[s][t][8g+kk]
  int32_t part[32][34];       // per-lane partial sums (direct: 16 hi + 16 lo; fnt: 16); the even
                              // pitch lets lanes write pairs and the readers (s, m0) load pairs
                              // with no bank conflicts
  double ey[4][AEQ_L];        // e * y per output stream
  double xf[4][66];           // x / sig_scale ring of 32, stored twice: [t][1 + 16 * parity + j (+ 32)];
                              // the +1 makes the gradient's x pairs 16-byte aligned, and the
                              // 66-double row stride keeps its 8 distinct LDS.128 conflict-free
                              // so every window is contiguous (odd t-stride: no bank conflicts)
  int32_t xi[4][2 * AEQ_L + 8]; // input integer ring: [t][16 * block parity + j]; the 40-word
                                // pitch keeps the input transform's loads conflict-free
  uint32_t X[4][AEQ_N + 8];   // cooperative input spectra (FNT path), 16-B aligned padded rows;
                              // AEQ_MAC_T: canonical residues at [t][8 (k mod 4) + k / 4]
  double err[32];             // |e| values for the err_trace mean
  uint8_t xq[4][64];          // DIRECT, int8 inputs: x_block[t] reversed as bytes, ring of 32
                              // stored twice: block b's samples j at 16 * parity + 15 - j (+ 32)
};


// S.part row pairs: 64-bit stores of (v[m], v[m+1]) and loads of columns (m0, m0 + 1)
__device__ __forceinline__ void part_store16(int32_t* row, const int32_t (&v)[AEQ_L]) {
#pragma unroll
  for (int m = 0; m < AEQ_L; m += 2) *reinterpret_cast<int2*>(row + m) = make_int2(v[m], v[m + 1]);
}
__device__ __forceinline__ int2 part_pair(const int32_t* row, int m0) {
  return *reinterpret_cast<const int2*>(row + m0);
}


// einsum("sm,tmk->stk") inner reduction over m in numpy's SSE2 order.
__device__ __forceinline__ double einsum_m(const double (&P)[AEQ_L]) {
  double c0 = P[6], c1 = P[7];
  c0 = dadd(P[4], c0);  c1 = dadd(P[5], c1);
  c0 = dadd(P[2], c0);  c1 = dadd(P[3], c1);
  c0 = dadd(P[0], c0);  c1 = dadd(P[1], c1);
  c0 = dadd(P[14], c0); c1 = dadd(P[15], c1);
  c0 = dadd(P[12], c0); c1 = dadd(P[13], c1);
  c0 = dadd(P[10], c0); c1 = dadd(P[11], c1);
  c0 = dadd(P[8], c0);  c1 = dadd(P[9], c1);
  return dadd(c0, c1);
}


// This lane's 8 taps k = 8g .. 8g+7 of filter (s, t): the 14-bit values in
// registers, the float values in the warp's shared scratch (S.wf, lane-contiguous).
struct LaneTaps {
  uint32_t gp[8];  // packed taps: 7-bit groups of w_int (pack_groups), or balanced
                   // base-64 digits (pack_taps<true>)
  uint32_t sat;    // saturations counted by this lane (flushed to 64 bits every 2^24 blocks)
  uint32_t asum;   // balanced digits: sum of |a| over this lane's 8 taps
};

template <bool BAL>
__device__ __forceinline__ void set_tap(LaneTaps& T, int kk, int32_t w) {
  T.gp[kk] = pack_taps<BAL>(w);
  if (BAL) T.asum += (uint32_t)abs((w + 32) >> 6);
}

// Exchange the e values, compute the err_trace mean (lane 0 writes *err_out when
// non-null) and, when mu != 0, the float update of this lane's 8 taps.
template <bool QUICK = false, bool BAL = false>
__device__ __forceinline__ void lane_update(const AeqArgs& A, AeqScratch& S, int lane, int m0,
                                            double y0, double y1, int cur, double mu,
                                            LaneTaps& T, double* err_out) {
  const int s = lane >> 3, t = (lane >> 1) & 3, g = lane & 1;
  // rde: the I lane (s even) takes m0, the Q lane (s odd) takes m0 + 1
  const double send = (s & 1) ? y0 : y1;
  const double recv = __shfl_xor_sync(0xffffffffu, send, 8);
  // one (branch-free) rde per lane: (y_I, y_Q) = (recv, y1) on odd s, (y0, recv) on even s
  const double yI = (s & 1) ? recv : y0, yQ = (s & 1) ? y1 : recv;
  double e_mine = rde<QUICK>(yI, yQ, A);
  const double e_other = __shfl_xor_sync(0xffffffffu, e_mine, 8);
  const double e0 = (s & 1) ? e_other : e_mine;  // e[p][m0]
  const double e1 = (s & 1) ? e_mine : e_other;  // e[p][m0 + 1]
  if ((s & 1) == 0) {
    const int p = s >> 1;
    S.err[p * 16 + m0] = fabs(e0);
    S.err[p * 16 + m0 + 1] = fabs(e1);
  }
  *reinterpret_cast<double2*>(&S.ey[s][m0]) = make_double2(dmul(e0, y0), dmul(e1, y1));
  __syncwarp();
  if (QUICK || err_out != nullptr) {
    // np.mean(|e|) over (2 pols x 16): numpy pairwise order r[j] = a[j]+a[j+8]+a[j+16]+a[j+24]
    double r = 0.0;
    if (lane < 8) {
      r = dadd(dadd(dadd(S.err[lane], S.err[lane + 8]), S.err[lane + 16]), S.err[lane + 24]);
    }
    r = dadd(r, __shfl_xor_sync(0xffffffffu, r, 1));
    r = dadd(r, __shfl_xor_sync(0xffffffffu, r, 2));
    r = dadd(r, __shfl_xor_sync(0xffffffffu, r, 4));
    if (lane == 0) *err_out = dmul(r, 1.0 / 32.0);
  }
  if (mu != 0.0) {
    // gradient for taps k in [8g, 8g+8): sum_m ey[s][m] * xf[t][16 + m - k]
    // x_block[t][j] sits at ring position 16 * prev + j (duplicated ring: no wrap);
    // tap kk (k = 8g + kk) uses x_block[t][16 + m - 8g - kk] = xs[7 - kk + m].
    const double* xs = S.xf[t] + 1 + AEQ_L * (cur ^ 1) + 9 - 8 * g;
    // all 8 taps advance together through numpy's m order (two chains per tap,
    // even m: 6,4,2,0,14,12,10,8 and odd m: 7,5,...,9): 16 independent FP64 chains
    // hide the DADD latency, and only one m pair of e*y and 9 x values are live.
    const double2* eyv = reinterpret_cast<const double2*>(S.ey[s]);
    double c0[8], c1[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int me = (i < 4 ? 6 : 22) - 2 * i;   // 6, 4, 2, 0, 14, 12, 10, 8
      const double2 e2 = eyv[me / 2];             // ey[me], ey[me + 1]
      double xv[9];  // xs + me is 16-byte aligned (me even, ring offset +1): 4 LDS.128 + 1 LDS.64
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const double2 v = reinterpret_cast<const double2*>(xs + me)[q];
        xv[2 * q] = v.x;
        xv[2 * q + 1] = v.y;
      }
      xv[8] = xs[me + 8];
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const double pe = dmul(e2.x, xv[7 - kk]), po = dmul(e2.y, xv[8 - kk]);
        c0[kk] = i == 0 ? pe : dadd(pe, c0[kk]);
        c1[kk] = i == 0 ? po : dadd(po, c1[kk]);
      }
    }
    T.asum = 0;
    uint32_t smask = 0;  // taps whose rint left [-16383, 16383] (or the int32 range)
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      const double gr = dadd(c0[kk], c1[kk]);
      const double w = dadd(S.wf[kk][lane], dmul(mu, gr));
      S.wf[kk][lane] = w;
      // requantize_tap without its per-tap |p| >= 2^63 test: such a p saturates the
      // int32 conversion, so it is among the clipped taps settled below; a NaN p
      // converts to 0 (cvt.rni.s32.f64), so it is flagged explicitly
      const double p = dmul(w, A.prm.tap_scale);
      const int32_t i = __double2int_rn(p);
      const int32_t c = min(max(i, -AEQ_TAP_MAX), AEQ_TAP_MAX);
      // clipped exactly when |p| >= 16383.5 (rint rounds half to even: 16383.5 -> 16384);
      // the negated compare also flags NaN
      smask |= (uint32_t)!(fabs(p) < 16383.5) << kk;
      set_tap<BAL>(T, kk, c);
    }
    T.sat += __popc(smask);
    if (__any_sync(0xffffffffu, smask != 0u)) {
      // rare: a clipped tap whose rint is not an int64 (numpy: INT64_MIN) becomes
      // -16383 and is not counted (requantize_tap, aeq.py:165-168)
      bool redo = false;
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        if ((smask >> kk) & 1u) {
          const double p = dmul(S.wf[kk][lane], A.prm.tap_scale);
          if (!(fabs(p) < 9.2233720368547758e18)) {
            T.sat -= 1;
            T.gp[kk] = pack_taps<BAL>(-AEQ_TAP_MAX);
            redo = true;
          }
        }
      }
      if (BAL && redo) {
        T.asum = 0;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) T.asum += (uint32_t)abs((unpack_tap<BAL>(T.gp[kk]) + 32) >> 6);
      }
    }
  }
  __syncwarp();
}

// 32-point forward transforms of the four input streams' blocks
// x_block[t] = [ring prev | ring cur] into S.X[t][k] (natural order).
__device__ __forceinline__ void warp_input_fnt(AeqScratch& S, int lane, int cur) {
  const int prev = cur ^ 1;
  // Four-step form, 8 lanes per stream (n = n1 + 8 n2, k = k2 + 4 k1, n1 = lane & 7):
  //   A[k2] = sum_n2 x[n1 + 8 n2] 2^(8 n2 k2)     4-point transform in registers
  //   B[k2] = A[k2] 2^(n1 k2)                     twiddles (2^16 == -1: complement)
  //   X[k2 + 4 k1] = sum_n1 B[k2] 2^(4 n1 k1)     8-point DIF across the 8 lanes
  // (3 shuffle stages; lane n1 ends with k1 = bitrev3(n1)). No shared-memory round
  // trips or warp barriers inside; N^-1 = 2^-5 of the inverse is folded in.
  {
    const int tq = lane >> 3, n1 = lane & 7;
    // x[n1], x[n1 + 8] from the previous block's ring half, x[n1 + 16], x[n1 + 24] from this one
    const int32_t* xr = S.xi[tq];
    uint32_t a0 = f4_enc_small(xr[AEQ_L * prev + n1]), a1 = f4_enc_small(xr[AEQ_L * prev + n1 + 8]);
    uint32_t a2 = f4_enc_small(xr[AEQ_L * cur + n1]), a3 = f4_enc_small(xr[AEQ_L * cur + n1 + 8]);
    const uint32_t s02 = m_add(a0, a2), d02 = m_sub(a0, a2);
    const uint32_t s13 = m_add(a1, a3), d13 = m_rot(m_sub(a1, a3), 8);
    uint32_t v[4] = {m_add(s02, s13), m_add(d02, d13), m_sub(s02, s13), m_sub(d02, d13)};
#pragma unroll
    for (int k2 = 1; k2 < 4; ++k2) {
      const int e = n1 * k2;                       // <= 21
      const uint32_t r = __funnelshift_l(v[k2], v[k2], e & 15);
      v[k2] = (e & 16) ? ~r : r;
    }
#pragma unroll
    for (int st = 2; st >= 0; --st) {              // spans 4, 2, 1
      const int h = 1 << st;
      const bool upper = (n1 & h) != 0;
      const uint32_t mask = upper ? 0xffffffffu : 0u;
      const int e = upper ? (n1 & (h - 1)) * (16 >> st) : 0;  // bottom twiddle (2^(16/2^st))^j
#pragma unroll
      for (int k2 = 0; k2 < 4; ++k2) {
        const uint32_t o = __shfl_xor_sync(0xffffffffu, v[k2], h);
        const uint32_t t = m_add(v[k2] ^ mask, o);  // lower: v + o; upper: o - v
        v[k2] = st > 0 ? __funnelshift_l(t, t, e) : t;
      }
    }
    const int k1 = (int)(__brev((unsigned)n1) >> 29);
    uint4 out = make_uint4(m_rot(v[0], 27), m_rot(v[1], 27), m_rot(v[2], 27), m_rot(v[3], 27));
#if AEQ_MAC_T
    // canonical residues (< 2^17: the 64-bit multiply-accumulate of fused_inverse_mac
    // cannot overflow), bins k = k2 + 4 k1 at 8 k2 + k1
    S.X[tq][k1] = f4_mod(out.x);
    S.X[tq][8 + k1] = f4_mod(out.y);
    S.X[tq][16 + k1] = f4_mod(out.z);
    S.X[tq][24 + k1] = f4_mod(out.w);
#else
    reinterpret_cast<uint4*>(S.X[tq])[k1] = out;
#endif
  }
  __syncwarp();
}

// Forward path for one block: returns y_int[s][m0], y_int[s][m0+1] in yi0, yi1.
// DIRECT form on int8 inputs: the per-group sums of 8 taps as two 4-way int8 dot
// products (DP4A) per output, from the reversed byte ring (x_block[16 + m - k] for
// k = 8g + q is byte 15 - m + q of the lane's window, and 19 - m + q for k + 4).
__device__ __forceinline__ void direct_dp4a(const AeqScratch& S, int t, int g, int cur,
                                            const LaneTaps& T, int32_t (&hi)[AEQ_L],
                                            int32_t (&lo)[AEQ_L]) {
  const uint2* qb = reinterpret_cast<const uint2*>(S.xq[t] + AEQ_L * cur + 8 * g);
  uint32_t R[6];
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    const uint2 v = qb[q];
    R[2 * q] = v.x;
    R[2 * q + 1] = v.y;
  }
  // tap groups as int8 quadruples: hi group = byte 0 of p, lo group = byte 2 of
  // p + 2^15 (pack_groups: p = sign (hi + lo 2^16), |hi|, |lo| <= 127)
  uint32_t th[2], tl[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const uint32_t p0 = T.gp[4 * h], p1 = T.gp[4 * h + 1], p2 = T.gp[4 * h + 2], p3 = T.gp[4 * h + 3];
    th[h] = __byte_perm(__byte_perm(p0, p1, 0x0040), __byte_perm(p2, p3, 0x0040), 0x5410);
    const uint32_t q0 = p0 + 0x8000u, q1 = p1 + 0x8000u, q2 = p2 + 0x8000u, q3 = p3 + 0x8000u;
    tl[h] = __byte_perm(__byte_perm(q0, q1, 0x0062), __byte_perm(q2, q3, 0x0062), 0x5410);
  }
#pragma unroll
  for (int m = 0; m < AEQ_L; ++m) {
    const int oa = 15 - m, ob = 19 - m;
    const uint32_t xa = (oa & 3) ? __funnelshift_r(R[oa >> 2], R[(oa >> 2) + 1], 8 * (oa & 3)) : R[oa >> 2];
    const uint32_t xb = (ob & 3) ? __funnelshift_r(R[ob >> 2], R[(ob >> 2) + 1], 8 * (ob & 3)) : R[ob >> 2];
    hi[m] = __dp4a((int)th[0], (int)xa, __dp4a((int)th[1], (int)xb, 0));
    lo[m] = __dp4a((int)tl[0], (int)xa, __dp4a((int)tl[1], (int)xb, 0));
  }
}

// Exact test for summing the four input streams in the transform domain (balanced
// digits, AEQ_FUSE_T). With A = max |x| over the block window (all four streams):
//  (1) A <= 16: each of the reference's per-(s,t,g) group convolutions is then
//      within [-32768, 32768] (|group| <= 127, 16 taps), so its decoded sum
//      (aeq.py:139-143) is the exact integer FIR sum_t,k w x;
//  (2) A * sum_{s,t,k} |a_stk| <= 32768, and (from (1) and |b| <= 32)
//      A * sum_{t,k} |b_stk| <= 32768: the digit convolutions summed over t are in
//      range for every s, so their decoded residues are exact too.
// Then 64 dec(sum_t conv a) + dec(sum_t conv b) is the same exact FIR. amax is the
// warp's A (uniform), so the result is warp-uniform.
__device__ __forceinline__ bool fused_ok(const LaneTaps& T, uint32_t amax) {
  const uint32_t asum = __reduce_add_sync(0xffffffffu, T.asum);  // <= 256 * 256
  return amax <= 16u && asum * amax <= 32768u;
}

// Forward outputs of one block with the products P_t = X_t W_stg of this lane
// (s, t, g) summed over groups of F input streams before the inverse: ONE inverse
// per (s, g, group), split over the group's F lanes by k = k1 + F k2 (k1 = t mod F):
//   y[n] = sum_k1 2^(-n k1) Q_k1[n mod 32/F],  Q_k1[j] = sum_k2 P[k1 + F k2] 2^(-F j k2)
// Products go through S.part as [32][32] words, row = lane, logical column
// k1 * (32/F) + k2, rotated by 4 f(lane & 7) words (conflict-free both ways).
template <int F, int BASE>
__device__ __forceinline__ void fused_inverse(AeqScratch& S, int lane, const uint32_t (&X)[AEQ_N],
                                              int m0, int32_t& yi0, int32_t& yi1) {
  constexpr int NB = AEQ_N / F;  // bins per lane = inverse length
  const int s = lane >> 3, t = (lane >> 1) & 3, g = lane & 1;
  const int k1 = t & (F - 1), t0 = t & ~(F - 1);
  auto swz = [](int r) { const int x = r & 7; return 4 * (x ^ ((x & 4) >> 1)); };
  uint32_t* prod = reinterpret_cast<uint32_t*>(S.part);
  const int rot = swz(lane);
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int c1 = (4 * q) / NB, c2 = (4 * q) % NB;  // logical column 4q = c1 * NB + c2
    const uint4 v = make_uint4(X[c1 + F * c2], X[c1 + F * (c2 + 1)], X[c1 + F * (c2 + 2)],
                               X[c1 + F * (c2 + 3)]);
    reinterpret_cast<uint4*>(prod + 32 * lane)[((4 * q + rot) & 31) >> 2] = v;
  }
  __syncwarp();
  uint32_t Q[NB];
#pragma unroll
  for (int i = 0; i < F; ++i) {
    const int r = 8 * s + 2 * (t0 + i) + g;
    const int rr = swz(r);
#pragma unroll
    for (int h = 0; h < NB / 4; ++h) {
      const uint4 v = reinterpret_cast<const uint4*>(prod + 32 * r)[((NB * k1 + 4 * h + rr) & 31) >> 2];
      if (i == 0) {
        Q[4 * h] = v.x; Q[4 * h + 1] = v.y; Q[4 * h + 2] = v.z; Q[4 * h + 3] = v.w;
      } else {
        Q[4 * h] = m_add(Q[4 * h], v.x); Q[4 * h + 1] = m_add(Q[4 * h + 1], v.y);
        Q[4 * h + 2] = m_add(Q[4 * h + 2], v.z); Q[4 * h + 3] = m_add(Q[4 * h + 3], v.w);
      }
    }
  }
  // +32768 on the group's DC bin (lane k1 = 0, k2 = 0): +32768 on every output
  Q[0] = m_add(Q[0], k1 == 0 ? 32768u : 0u);
  to_bitrev<NB>(Q);
  fnt_dit<NB, F == 4 ? RADIX16 : RADIX4, true, false, false, AEQ_IFNT_CM>(Q);
  __syncwarp();  // every lane has read its products before S.part is reused
  {
    int32_t c[AEQ_L];
#pragma unroll
    for (int m = 0; m < AEQ_L; ++m) {
      const uint32_t q = Q[m % NB];
      c[m] = (int32_t)__funnelshift_l(q, q, ((16 - m) * k1) & 31);  // 2^(-(16+m) k1)
    }
    part_store16(S.part[lane], c);
  }
  __syncwarp();
  // y_int = sum over groups of BASE dec(digit 0) + dec(digit 1), each summed over F lanes
  int32_t a0 = -(4 / F) * (BASE + 1) * 32768, a1 = a0;
#pragma unroll
  for (int grp = 0; grp < 4 / F; ++grp) {
    uint32_t h0 = 0, h1 = 0, l0 = 0, l1 = 0;
#pragma unroll
    for (int i = 0; i < F; ++i) {
      const int r = 8 * s + 2 * (F * grp + i);
      const int2 hv = part_pair(S.part[r], m0), lv = part_pair(S.part[r + 1], m0);
      h0 = m_add(h0, (uint32_t)hv.x);
      h1 = m_add(h1, (uint32_t)hv.y);
      l0 = m_add(l0, (uint32_t)lv.x);
      l1 = m_add(l1, (uint32_t)lv.y);
    }
    a0 += BASE * (int32_t)f4_mod(h0) + (int32_t)f4_mod(l0);
    a1 += BASE * (int32_t)f4_mod(h1) + (int32_t)f4_mod(l1);
  }
  yi0 = a0;
  yi1 = a1;
  __syncwarp();
}

// fused_inverse<4, 64> with the transform-domain stream sum as 64-bit multiply-
// accumulates (AEQ_MAC_T): each lane publishes its tap spectrum W_stg (not its
// products), and the inverse lane (s, k1 = t, g) forms
//   Q[k2] = sum_t'' X_t''[k1 + 4 k2] * W_st''g[k1 + 4 k2]
// with IMAD.WIDE.U32 into 64-bit accumulators (X canonical < 2^17, W < 2^32: the four
// terms stay below 2^51), folded once per bin (2^32 == 1 mod 2^32 - 1): 32 MACs + 8
// folds instead of 32 products (3 instructions each) + 24 modular adds.
__device__ __forceinline__ void fused_inverse_mac(AeqScratch& S, int lane, const uint32_t (&W)[AEQ_N],
                                                  int m0, int32_t& yi0, int32_t& yi1) {
  constexpr int F = 4, NB = AEQ_N / F;
  const int s = lane >> 3, t = (lane >> 1) & 3, g = lane & 1;
  const int k1 = t;
  auto swz = [](int r) { const int x = r & 7; return 4 * (x ^ ((x & 4) >> 1)); };
  uint32_t* prod = reinterpret_cast<uint32_t*>(S.part);
  const int rot = swz(lane);
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int c1 = (4 * q) / NB, c2 = (4 * q) % NB;  // logical column 4q = c1 * NB + c2
    const uint4 v = make_uint4(W[c1 + F * c2], W[c1 + F * (c2 + 1)], W[c1 + F * (c2 + 2)],
                               W[c1 + F * (c2 + 3)]);
    reinterpret_cast<uint4*>(prod + 32 * lane)[((4 * q + rot) & 31) >> 2] = v;
  }
  __syncwarp();
  uint64_t acc[NB];
#pragma unroll
  for (int i = 0; i < F; ++i) {
    const int r = 8 * s + 2 * i + g;
    const int rr = swz(r);
    const uint4* xq = reinterpret_cast<const uint4*>(&S.X[i][8 * k1]);
#pragma unroll
    for (int h = 0; h < NB / 4; ++h) {
      const uint4 w = reinterpret_cast<const uint4*>(prod + 32 * r)[((NB * k1 + 4 * h + rr) & 31) >> 2];
      const uint4 x = xq[h];
      const uint32_t wv[4] = {w.x, w.y, w.z, w.w}, xv[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const uint64_t p = (uint64_t)xv[e] * wv[e];
        acc[4 * h + e] = i == 0 ? p : acc[4 * h + e] + p;
      }
    }
  }
  uint32_t Q[NB];
#pragma unroll
  for (int c2 = 0; c2 < NB; ++c2) Q[c2] = m_add((uint32_t)acc[c2], (uint32_t)(acc[c2] >> 32));
  // +32768 on the group's DC bin (lane k1 = 0, k2 = 0): +32768 on every output
  Q[0] = m_add(Q[0], k1 == 0 ? 32768u : 0u);
  to_bitrev<NB>(Q);
  fnt_dit<NB, RADIX16, true, false, false, AEQ_IFNT_CM>(Q);
  __syncwarp();  // every lane has read its spectra before S.part is reused
  {
    int32_t c[AEQ_L];
#pragma unroll
    for (int m = 0; m < AEQ_L; ++m) {
      const uint32_t q = Q[m % NB];
      c[m] = (int32_t)__funnelshift_l(q, q, ((16 - m) * k1) & 31);  // 2^(-(16+m) k1)
    }
    part_store16(S.part[lane], c);
  }
  __syncwarp();
  int32_t a0 = -65 * 32768, a1 = a0;
  {
    uint32_t h0 = 0, h1 = 0, l0 = 0, l1 = 0;
#pragma unroll
    for (int i = 0; i < F; ++i) {
      const int r = 8 * s + 2 * i;
      const int2 hv = part_pair(S.part[r], m0), lv = part_pair(S.part[r + 1], m0);
      h0 = m_add(h0, (uint32_t)hv.x);
      h1 = m_add(h1, (uint32_t)hv.y);
      l0 = m_add(l0, (uint32_t)lv.x);
      l1 = m_add(l1, (uint32_t)lv.y);
    }
    a0 += 64 * (int32_t)f4_mod(h0) + (int32_t)f4_mod(l0);
    a1 += 64 * (int32_t)f4_mod(h1) + (int32_t)f4_mod(l1);
  }
  yi0 = a0;
  yi1 = a1;
  __syncwarp();
}

template <int FWD, bool NARROW = false>
__device__ __forceinline__ void lane_forward(AeqScratch& S, int lane, int cur, const LaneTaps& T,
                                             int m0, int32_t& yi0, int32_t& yi1,
                                             bool use_dp4a = false, uint32_t amax = 0xffffffffu) {
  const int s = lane >> 3, t = (lane >> 1) & 3, g = lane & 1;
  if (FWD == FNTGPU_AEQ_FWD_FNT) {
    constexpr bool BAL = AEQ_FUSE_T != 0;
#if AEQ_PROBE != 1
    warp_input_fnt(S, lane, cur);
#endif
    const bool fused = BAL && fused_ok(T, amax);
    // all 16 taps of filter (s, t), own 8 + partner's 8 (lane ^ 1 holds the other
    // half): digit g (fused) or the reference's group g (split_taps,
    // fixedpoint.py:111-121)
    uint32_t W[AEQ_N];
    if (fused) {
      // digit g of tap kk (owned by lane g' = 0) and of tap 8 + kk (lane g' = 1): one
      // PRMT each, from this lane's word or its partner's
      const uint32_t sel_lo = g ? DIG_B2 : DIG_A, sel_hi = g ? DIG_B : DIG_A2;
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint32_t other = __shfl_xor_sync(0xffffffffu, T.gp[kk], 1);
        W[bitrev(kk, 5)] = prmt(T.gp[kk], other, sel_lo);      // tap kk
        W[bitrev(8 + kk, 5)] = prmt(T.gp[kk], other, sel_hi);  // tap 8 + kk
      }
    } else {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint32_t other = __shfl_xor_sync(0xffffffffu, T.gp[kk], 1);
        W[bitrev(kk, 5)] = (uint32_t)ref_group<BAL>(g == 0 ? T.gp[kk] : other, g);
        W[bitrev(8 + kk, 5)] = (uint32_t)ref_group<BAL>(g == 0 ? other : T.gp[kk], g);
      }
    }
#pragma unroll
    for (int k = AEQ_L; k < AEQ_N; ++k) W[bitrev(k, 5)] = 0u;
    // taps zero-padded: stage 0 is a copy; |group| <= 256 keeps stages 1-2 (twiddles
    // 2^0..2^12) below 2^29 in plain int32, then a multiple of F4 makes the words
    // non-negative residues of Z/M for stages 3-4
    fnt_stage<AEQ_N, RADIX2, false, true, false, 0, 1>(W);
#if AEQ_PROBE != 2
    // + F4 * 8192 = 536 879 104 > 256 * 257 * 4097 on every output of stage 2
    fnt_stage_plain<AEQ_N, RADIX2, 1, 3, F4 * 8192u>(W);
#endif
#if AEQ_PROBE != 2
    fnt_stage<AEQ_N, RADIX2, false, false, false, 3, -1, AEQ_TAP_CM>(W);
#endif
#if AEQ_FUSE_T && AEQ_MAC_T
    if (fused) { fused_inverse_mac(S, lane, W, m0, yi0, yi1); return; }
#endif
    uint32_t X[AEQ_N];
#pragma unroll
    for (int q = 0; q < AEQ_N / 4; ++q) {
      const uint4 v = reinterpret_cast<const uint4*>(S.X[t])[q];
#if AEQ_MAC_T
      // permuted layout: word 4q + e holds bin k with 8 (k mod 4) + k / 4 = 4q + e
      const uint32_t ve[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int idx = 4 * q + e;
        X[(idx >> 3) + 4 * (idx & 7)] = ve[e];
      }
#else
      X[4 * q] = v.x; X[4 * q + 1] = v.y; X[4 * q + 2] = v.z; X[4 * q + 3] = v.w;
#endif
    }
#pragma unroll
    for (int k = 0; k < AEQ_N; ++k) X[k] = m_mul(X[k], W[k]);  // 32 general products
#if AEQ_FUSE_T
    if (fused) { fused_inverse<4, 64>(S, lane, X, m0, yi0, yi1); return; }
#endif
    // +32768 on every output of the inverse = +32768 on its DC bin (X carries N^-1),
    // so each output decodes as f4_mod(.) - 32768 (fermat.cuh: f4_mod)
    X[0] = m_add(X[0], 32768u);
    to_bitrev<AEQ_N>(X);
#if AEQ_PROBE != 3
    fnt_dit<AEQ_N, RADIX2, true, false, true, AEQ_IFNT_CM>(X);  // outputs 16..31 only
#endif
    const int sh = g == 0 ? 7 : 0;                 // recombine 128 hi + lo (fixedpoint.py:139-143)
    {
      int32_t c[AEQ_L];
#pragma unroll
      for (int m = 0; m < AEQ_L; ++m) c[m] = (int32_t)(f4_mod(X[AEQ_L + m]) << sh);
      part_store16(S.part[lane], c);
    }
    __syncwarp();
    // sum over (t, g) of 128^[g=0] (c - 32768): the offsets total 4 * 129 * 32768
    int32_t a0 = -4 * 129 * 32768, a1 = -4 * 129 * 32768;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int2 v = part_pair(S.part[s * 8 + q], m0);
      a0 += v.x;
      a1 += v.y;
    }
    yi0 = a0;
    yi1 = a1;
  } else if (NARROW && AEQ_DP4A && use_dp4a) {
    int32_t hi[AEQ_L], lo[AEQ_L];
    direct_dp4a(S, t, g, cur, T, hi, lo);
    part_store16(S.part[lane], hi);
    part_store16(S.part[lane] + AEQ_L, lo);
    __syncwarp();
    int32_t a0, a1;
    if (amax <= 16u) {
      // every group sum is within +-16 * 127 * 16 = +-32512: its decode is the identity
      // (fused_ok (1)), so y_int is the plain sum
      a0 = 0;
      a1 = 0;
#pragma unroll
      for (int tt = 0; tt < 4; ++tt) {
        const int l0 = s * 8 + tt * 2;
        const int2 h0 = part_pair(S.part[l0], m0), h1 = part_pair(S.part[l0 + 1], m0);
        const int2 l0v = part_pair(S.part[l0], AEQ_L + m0), l1v = part_pair(S.part[l0 + 1], AEQ_L + m0);
        a0 += 128 * (h0.x + h1.x) + (l0v.x + l1v.x);
        a1 += 128 * (h0.y + h1.y) + (l0v.y + l1v.y);
      }
    } else {
      a0 = -4 * 129 * 32768;
      a1 = -4 * 129 * 32768;
#pragma unroll
      for (int tt = 0; tt < 4; ++tt) {
        const int l0 = s * 8 + tt * 2;
        const int32_t B = (int32_t)(F4 * 1024u) + 32768;
        const int2 h0 = part_pair(S.part[l0], m0), h1 = part_pair(S.part[l0 + 1], m0);
        const int2 l0v = part_pair(S.part[l0], AEQ_L + m0), l1v = part_pair(S.part[l0 + 1], AEQ_L + m0);
        a0 += 128 * (int32_t)f4_mod((uint32_t)(h0.x + h1.x + B)) + (int32_t)f4_mod((uint32_t)(l0v.x + l1v.x + B));
        a1 += 128 * (int32_t)f4_mod((uint32_t)(h0.y + h1.y + B)) + (int32_t)f4_mod((uint32_t)(l0v.y + l1v.y + B));
      }
    }
    yi0 = a0;
    yi1 = a1;
  } else {
    int32_t xb[AEQ_N];
    const int prev = cur ^ 1;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int4 a = reinterpret_cast<const int4*>(S.xi[t] + AEQ_L * prev)[q];
      const int4 b = reinterpret_cast<const int4*>(S.xi[t] + AEQ_L * cur)[q];
      xb[4 * q] = a.x; xb[4 * q + 1] = a.y; xb[4 * q + 2] = a.z; xb[4 * q + 3] = a.w;
      xb[16 + 4 * q] = b.x; xb[16 + 4 * q + 1] = b.y; xb[16 + 4 * q + 2] = b.z; xb[16 + 4 * q + 3] = b.w;
    }
    // time-domain per-group partial sums over this lane's 8 taps k = 8g + kk
    int32_t hi[AEQ_L], lo[AEQ_L];
#pragma unroll
    for (int m = 0; m < AEQ_L; ++m) { hi[m] = 0; lo[m] = 0; }
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      const int32_t th = unpack_group(T.gp[kk], 0), tl = unpack_group(T.gp[kk], 1);
#pragma unroll
      for (int m = 0; m < AEQ_L; ++m) {
        // x index 16 + m - k, k = 8g + kk  (runtime g: select between two windows)
        const int32_t xv = g == 0 ? xb[AEQ_L + m - kk] : xb[AEQ_L + m - 8 - kk];
        hi[m] += th * xv;
        lo[m] += tl * xv;
      }
    }
    part_store16(S.part[lane], hi);
    part_store16(S.part[lane] + AEQ_L, lo);
    __syncwarp();
    int32_t a0 = -4 * 129 * 32768, a1 = -4 * 129 * 32768;
#pragma unroll
    for (int tt = 0; tt < 4; ++tt) {
      const int l0 = s * 8 + tt * 2;
      const int2 h0 = part_pair(S.part[l0], m0), h1 = part_pair(S.part[l0 + 1], m0);
      const int2 l0v = part_pair(S.part[l0], AEQ_L + m0), l1v = part_pair(S.part[l0 + 1], AEQ_L + m0);
      // each group convolution is a residue mod F4, decoded (aeq.py:139-140) as
      // f4_mod(v + 32768) - 32768; the -32768 offsets are summed into the start value
      const int32_t B = (int32_t)(F4 * 1024u) + 32768;
      a0 += 128 * (int32_t)f4_mod((uint32_t)(h0.x + h1.x + B)) + (int32_t)f4_mod((uint32_t)(l0v.x + l1v.x + B));
      a1 += 128 * (int32_t)f4_mod((uint32_t)(h0.y + h1.y + B)) + (int32_t)f4_mod((uint32_t)(l0v.y + l1v.y + B));
    }
    yi0 = a0;
    yi1 = a1;
  }
  __syncwarp();
}

// -------------------------------------------------------------------------------------
// process (aeq.py:172-190) for one stream per warp

// QUICK: the launch verified fast_rde && n_radii == 3 && fast_div (the 16QAM rings
// with an ordinary scale) and an adapting call with per-block mu and an err_trace
// output (the receiver chain), so those paths are resolved at compile time.
template <int FWD, int IN_MODE, typename TIN, bool QUICK>
__global__ void __launch_bounds__(AEQ_WARPS * 32, AEQ_MIN_CTAS) k_aeq_process(fntgpu_aeq_state* __restrict__ st,
                                                                 const __grid_constant__ AeqArgs A) {
  constexpr bool NARROW = sizeof(TIN) == 1;
  extern __shared__ __align__(16) unsigned char aeq_dyn_smem[];
  AeqScratch* scratch = reinterpret_cast<AeqScratch*>(aeq_dyn_smem);
  __shared__ double lut[2 * XF_LUT + 1];
  for (int i = threadIdx.x; i < 2 * XF_LUT + 1; i += blockDim.x)
    lut[i] = __ddiv_rn((double)(i - XF_LUT), A.prm.sig_scale);
  __syncthreads();

  const fntgpu_aeq_io& io = A.io;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t S_idx = (int64_t)blockIdx.x * AEQ_WARPS + warp;
  if (S_idx >= io.n_streams) return;
  AeqScratch& S = scratch[warp];
  fntgpu_aeq_state& state = st[S_idx];
#if AEQ_LOCKSTEP
  const int64_t n_act = io.n_streams - (int64_t)blockIdx.x * AEQ_WARPS;
  const int bar_threads = 32 * (int)(n_act < AEQ_WARPS ? n_act : AEQ_WARPS);
#endif

  const int s = lane >> 3, t = (lane >> 1) & 3, g = lane & 1;
  const int j8 = lane & 7;  // m0 = 8*b0 + 4*b1 + 2*b2 with (b2 b1 b0) = lane bits 2,1,0
  const int m0 = 8 * (j8 & 1) + 4 * ((j8 >> 1) & 1) + 2 * ((j8 >> 2) & 1);
  // input-loader role: samples iq, iq + 1 of input stream tq
  const int tq = lane >> 3, iq = 2 * (lane & 7);

  constexpr bool BAL = FWD == FNTGPU_AEQ_FWD_FNT && AEQ_FUSE_T;
  LaneTaps T;
  T.asum = 0;
#pragma unroll
  for (int kk = 0; kk < 8; ++kk) {
    S.wf[kk][lane] = state.w[s][t][8 * g + kk];
    set_tap<BAL>(T, kk, state.w_int[s][t][8 * g + kk]);
  }
  T.sat = 0;
  // history -> ring slot 1 (the slot block 0 treats as "previous")
  {
    const int32_t h0 = state.hist[tq][iq], h1 = state.hist[tq][iq + 1];
    *reinterpret_cast<int2*>(S.xi[tq] + AEQ_L + iq) = make_int2(h0, h1);
    const double f0 = xf_of<false>(h0, lut, A.prm.sig_scale), f1 = xf_of<false>(h1, lut, A.prm.sig_scale);
    S.xf[tq][1 + AEQ_L + iq] = f0;
    S.xf[tq][1 + AEQ_L + iq + 1] = f1;
    S.xf[tq][1 + AEQ_L + iq + 32] = f0;
    S.xf[tq][1 + AEQ_L + iq + 33] = f1;
    if (FWD == FNTGPU_AEQ_FWD_DIRECT && NARROW && AEQ_DP4A) {
      // reversed byte ring, slot 1: samples iq + 1, iq at 16 + 14 - iq (+ 32); only
      // used when the whole history fits int8 (use_dp4a)
      const uint16_t pr = (uint16_t)(((uint32_t)h1 & 0xffu) | (((uint32_t)h0 & 0xffu) << 8));
      *reinterpret_cast<uint16_t*>(&S.xq[tq][AEQ_L + 14 - iq]) = pr;
      *reinterpret_cast<uint16_t*>(&S.xq[tq][AEQ_L + 14 - iq + 32]) = pr;
    }
  }

  // DP4A direct form: int8 inputs and an int8-range history (a history set through
  // the API or left by a wide-input call takes the 32-bit multiply path)
  const bool use_dp4a = FWD == FNTGPU_AEQ_FWD_DIRECT && NARROW && AEQ_DP4A &&
                        __all_sync(0xffffffffu, state.hist[tq][iq] >= -128 && state.hist[tq][iq] <= 127 &&
                                                    state.hist[tq][iq + 1] >= -128 && state.hist[tq][iq + 1] <= 127);
  // this lane's input row (stream tq) and a one-block-ahead prefetch of its 2 samples
  const char* row;
  uint32_t sel0 = 0, sel1 = 1;
  if (IN_MODE == FNTGPU_AEQ_IN_PLANAR) {
    row = reinterpret_cast<const char*>(reinterpret_cast<const TIN*>(io.x) + S_idx * io.x_stream_stride +
                                        tq * io.x_row_stride);
  } else {
    const int8_t* plane = (tq & 1) ? io.qi : io.qr;
    row = reinterpret_cast<const char*>(plane + (2 * S_idx + (tq >> 1)) * io.q_stride);
    const uint32_t ph = (uint32_t)io.phase[S_idx];
    sel0 = ph;       // byte of symbol iq within the 4-byte word (2 iq .. 2 iq + 3)
    sel1 = 2 + ph;   // byte of symbol iq + 1
  }
  // per-block input advance in bytes
  constexpr int64_t IN_STEP = IN_MODE == FNTGPU_AEQ_IN_DECIM ? 2 * AEQ_L : (int64_t)sizeof(TIN) * AEQ_L;
  row += IN_MODE == FNTGPU_AEQ_IN_DECIM ? 2 * iq : (int64_t)sizeof(TIN) * iq;
  auto fetch = [&](const char* p) -> uint2 {
    if (IN_MODE == FNTGPU_AEQ_IN_DECIM) {
      return make_uint2(__ldg(reinterpret_cast<const uint32_t*>(p)), 0u);
    } else if (NARROW) {
      return make_uint2(__ldg(reinterpret_cast<const uint16_t*>(p)), 0u);
    } else {
      const int2 v = __ldg(reinterpret_cast<const int2*>(p));
      return make_uint2((uint32_t)v.x, (uint32_t)v.y);
    }
  };
  auto decode = [&](uint2 raw, int32_t& v0, int32_t& v1) {
    if (IN_MODE == FNTGPU_AEQ_IN_DECIM) {
      v0 = sbyte(raw.x, sel0);
      v1 = sbyte(raw.x, sel1);
    } else if (NARROW) {
      v0 = sbyte(raw.x, 0);
      v1 = sbyte(raw.x, 1);
    } else {
      v0 = (int32_t)raw.x;
      v1 = (int32_t)raw.y;
    }
  };

  long long sat64 = 0;
  int32_t v0 = 0, v1 = 0;
  // max |x| of this lane's two samples in the previous block (window = prev + cur)
  auto mag = [](int32_t v) -> uint32_t { return v < 0 ? 0u - (uint32_t)v : (uint32_t)v; };
  uint32_t amax_prev = max(mag(state.hist[tq][iq]), mag(state.hist[tq][iq + 1]));
  const int64_t nb = io.n_blocks;
  uint2 raw = make_uint2(0u, 0u);
  if (nb > 0) raw = fetch(row);
  double2* yrow = reinterpret_cast<double2*>(io.y + S_idx * io.y_stream_stride + s * io.y_row_stride + m0);
  const double* mu_p = io.mu_blocks;
  double mu_next = mu_p && nb > 0 ? mu_p[0] : A.prm.mu;
  double* err_out = io.err ? io.err + S_idx * io.err_stream_stride : nullptr;
  // blocks in chunks of 2^24 so the 32-bit per-lane saturation counter (<= 8 per
  // block) is flushed outside the hot loop
  for (int64_t b0 = 0; b0 < nb; b0 += (int64_t)1 << 24) {
    const int64_t b1 = nb - b0 < ((int64_t)1 << 24) ? nb : b0 + ((int64_t)1 << 24);
    for (int64_t b = b0; b < b1; ++b) {
      const int cur = (int)(b & 1);
      decode(raw, v0, v1);
      const double mu = mu_next;
      if (QUICK) {
        // branch-free one-block-ahead prefetch (the last block re-reads its own input)
        const bool more = b + 1 < nb;
        row += more ? IN_STEP : 0;
        raw = fetch(row);
        mu_next = mu_p[more ? b + 1 : b];
      } else if (b + 1 < nb) {
        row += IN_STEP;
        raw = fetch(row);
        if (mu_p) mu_next = mu_p[b + 1];
      }
      *reinterpret_cast<int2*>(S.xi[tq] + AEQ_L * cur + iq) = make_int2(v0, v1);
      if (FWD == FNTGPU_AEQ_FWD_DIRECT && NARROW && AEQ_DP4A) {
        const uint16_t pr = (uint16_t)(((uint32_t)v1 & 0xffu) | (((uint32_t)v0 & 0xffu) << 8));
        *reinterpret_cast<uint16_t*>(&S.xq[tq][AEQ_L * cur + 14 - iq]) = pr;
        *reinterpret_cast<uint16_t*>(&S.xq[tq][AEQ_L * cur + 14 - iq + 32]) = pr;
      }
      if (QUICK || io.adapt) {
        const double f0 = xf_of<NARROW>(v0, lut, A.prm.sig_scale), f1 = xf_of<NARROW>(v1, lut, A.prm.sig_scale);
        double* xr = &S.xf[tq][1 + AEQ_L * cur + iq];
        xr[0] = f0;
        xr[1] = f1;
        xr[32] = f0;
        xr[33] = f1;
      }
#if AEQ_LOCKSTEP
      if ((b & (AEQ_LOCKSTEP - 1)) == 0) asm volatile("bar.sync 1, %0;" :: "r"(bar_threads) : "memory");
#endif
      uint32_t amax = 0xffffffffu;  // max |x| over the block window (4 x 32 samples)
      if (FWD != FNTGPU_AEQ_FWD_FNT || AEQ_FUSE_T) {
        const uint32_t a_cur = max(mag(v0), mag(v1));
        amax = __reduce_max_sync(0xffffffffu, max(a_cur, amax_prev));
        amax_prev = a_cur;
      }
      __syncwarp();
      int32_t yi0, yi1;
      lane_forward<FWD, NARROW>(S, lane, cur, T, m0, yi0, yi1, use_dp4a, amax);
      const double y0 = div_D<QUICK>(yi0, A);  // y_int / (sig_scale * tap_scale)
      const double y1 = div_D<QUICK>(yi1, A);
      *yrow = make_double2(y0, y1);
      yrow += AEQ_L / 2;
      if (QUICK || io.adapt) {
#if AEQ_PROBE != 4
        lane_update<QUICK, BAL>(A, S, lane, m0, y0, y1, cur, mu, T, err_out);
#endif
        if (QUICK || err_out) ++err_out;
      }
    }
    sat64 += T.sat;
    T.sat = 0;
  }

  // write back the stream state
  __syncwarp();
#pragma unroll
  for (int kk = 0; kk < 8; ++kk) {
    state.w[s][t][8 * g + kk] = S.wf[kk][lane];
    state.w_int[s][t][8 * g + kk] = unpack_tap<BAL>(T.gp[kk]);
  }
  if (io.n_blocks > 0) {
    state.hist[tq][iq] = v0;
    state.hist[tq][iq + 1] = v1;
  }
  long long sat = sat64 + T.sat;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) sat += __shfl_xor_sync(0xffffffffu, sat, off);
  if (lane == 0) {
    state.saturations += sat;
    state.symbols += io.n_blocks * AEQ_L;
    if (io.adapt) state.n_err += io.n_blocks;
  }
}

// update_taps with caller-given x_block (4, 32) and y (4, 16) (aeq.py:148-170)
__global__ void k_aeq_update_once(fntgpu_aeq_state* st, const __grid_constant__ AeqArgs A,
                                  const int64_t* xblk, const double* y, double mu, double* err) {
  __shared__ AeqScratch S;
  const int lane = threadIdx.x & 31;
  const int s = lane >> 3, t = (lane >> 1) & 3, g = lane & 1;
  const int j8 = lane & 7;
  const int m0 = 8 * (j8 & 1) + 4 * ((j8 >> 1) & 1) + 2 * ((j8 >> 2) & 1);
  LaneTaps T;
  T.asum = 0;
#pragma unroll
  for (int kk = 0; kk < 8; ++kk) {
    S.wf[kk][lane] = st->w[s][t][8 * g + kk];
    T.gp[kk] = pack_groups(st->w_int[s][t][8 * g + kk]);
  }
  T.sat = 0;
  if (s == 0 && g == 0) {
    for (int i = 0; i < AEQ_L; ++i) {
      // x_block may hold any int64 the reference accepted; divide exactly
      // block parity cur = 0: x_block[t][j] at ring position 16 + j (and + 32)
      const double a = __ddiv_rn((double)xblk[t * AEQ_N + i], A.prm.sig_scale);
      const double b = __ddiv_rn((double)xblk[t * AEQ_N + AEQ_L + i], A.prm.sig_scale);
      S.xf[t][1 + AEQ_L + i] = a;
      S.xf[t][1 + AEQ_L + i + 32] = a;
      S.xf[t][1 + i] = b;
      S.xf[t][1 + i + 32] = b;
    }
  }
  __syncwarp();
  const double y0 = y[s * AEQ_L + m0], y1 = y[s * AEQ_L + m0 + 1];
  lane_update(A, S, lane, m0, y0, y1, 0, mu, T, err);
#pragma unroll
  for (int kk = 0; kk < 8; ++kk) {
    st->w[s][t][8 * g + kk] = S.wf[kk][lane];
    st->w_int[s][t][8 * g + kk] = 128 * unpack_group(T.gp[kk], 0) + unpack_group(T.gp[kk], 1);
  }
  long long sat = T.sat;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) sat += __shfl_xor_sync(0xffffffffu, sat, off);
  if (lane == 0) { st->saturations += sat; st->n_err += 1; }
}

__global__ void k_aeq_init(fntgpu_aeq_state* st, int n_streams, double tap_scale, int32_t spike) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t total = (int64_t)n_streams * 256;
  if (i >= total) return;
  fntgpu_aeq_state& S = st[i / 256];
  const int r = (int)(i % 256);
  const int s = r >> 6, t = (r >> 4) & 3, k = r & 15;
  const bool on = (s == t) && (k == AEQ_L / 2);
  S.w_int[s][t][k] = on ? spike : 0;
  S.w[s][t][k] = on ? __ddiv_rn((double)spike, tap_scale) : 0.0;  // w_int / tap_scale (aeq.py:99)
  if (r < 64) S.hist[r >> 4][r & 15] = 0;
  if (r == 0) { S.saturations = 0; S.symbols = 0; S.n_err = 0; S.reserved = 0; }
}

// Ring index rde_error picks for a squared radius r2 (aeq.py:56-58): r = sqrt(r2)
// (IEEE, correctly rounded), first argmin of |r - R_i| -- the device slow path.
static int ring_of(double r2, const fntgpu_aeq_params& prm) {
  const double r = std::sqrt(r2);
  int best = 0;
  double bd = std::fabs(r - prm.radii[0]);
  for (int i = 1; i < prm.n_radii; ++i) {
    const double d = std::fabs(r - prm.radii[i]);
    if (d < bd) { bd = d; best = i; }
  }
  return best;
}

// rde fast path: for sorted radii the chosen ring is a non-decreasing step function
// of r2 (r = RN(sqrt r2) is monotone, and between neighbouring radii one distance
// grows while the other shrinks; the radii are >= 2^-30 apart relative, far above an
// ulp of the reachable r). T[k] = the least double r2 with ring_of(r2) >= k, found by
// bisection over the ordered bit patterns, so r2 >= T[k] reproduces the decision
// exactly. Enabled only when |y| <= 2^25 / D keeps r2 in the range the argument
// covers; otherwise the kernel computes the square root.
static void rde_thresholds(AeqArgs& A) {
  const fntgpu_aeq_params& prm = A.prm;
  A.fast_rde = 0;
  for (int i = 0; i < 8; ++i) A.T[i] = INFINITY;
  if (prm.n_radii < 1 || prm.n_radii > 8) return;
  for (int i = 0; i < prm.n_radii; ++i) {
    if (!std::isfinite(prm.radii[i]) || prm.radii[i] < 0.0) return;
    if (i > 0 && !(prm.radii[i] - prm.radii[i - 1] > std::ldexp(prm.radii[i], -30))) return;
  }
  if (!(A.D >= 1.0 / 1024.0) || !std::isfinite(A.D)) return;
  // |y_int| <= 4 * 129 * 32768 < 2^25 (every group residue is decoded to [-2^15, 2^15])
  const double ymax = std::ldexp(1.0, 25) / A.D;
  const double r2max = 4.0 * ymax * ymax;
  if (!(r2max < std::ldexp(1.0, 90))) return;
  auto bits = [](double v) { uint64_t u; std::memcpy(&u, &v, 8); return u; };
  auto val = [](uint64_t u) { double v; std::memcpy(&v, &u, 8); return v; };
  const uint64_t hi_bits = bits(r2max);
  for (int k = 1; k < prm.n_radii; ++k) {
    if (ring_of(r2max, prm) < k) continue;  // unreachable: stays +inf
    uint64_t lo = 0, hi = hi_bits;         // ring_of(val(hi)) >= k
    if (ring_of(0.0, prm) >= k) { A.T[k] = 0.0; continue; }
    while (hi - lo > 1) {
      const uint64_t mid = lo + (hi - lo) / 2;
      if (ring_of(val(mid), prm) >= k) hi = mid; else lo = mid;
    }
    A.T[k] = val(hi);
  }
  A.fast_rde = 1;
}

static AeqArgs make_args(const fntgpu_aeq_params& prm, const fntgpu_aeq_io* io) {
  AeqArgs A;
  std::memset(&A, 0, sizeof(A));
  A.prm = prm;
  if (io) A.io = *io;
  for (int i = 0; i < 8; ++i) A.R2[i] = prm.radii[i] * prm.radii[i];
  A.D = prm.sig_scale * prm.tap_scale;
  A.Dinv = 1.0 / A.D;
  const double aD = std::fabs(A.D);
  A.fast_div = aD >= std::ldexp(1.0, -500) && aD <= std::ldexp(1.0, 500);
  rde_thresholds(A);
  return A;
}

cudaError_t launch_aeq_init(fntgpu_aeq_state* st, int n_streams, const fntgpu_aeq_params& prm,
                            cudaStream_t s) {
  if (n_streams <= 0) return cudaSuccess;
  // int(round(tap_scale)) with Python's round-half-even (aeq.py:97)
  const int32_t spike = (int32_t)nearbyint(prm.tap_scale);
  const int64_t total = (int64_t)n_streams * 256;
  k_aeq_init<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(st, n_streams, prm.tap_scale, spike);
  return cudaGetLastError();
}

template <int FWD, int IN_MODE, typename TIN, bool QUICK>
static cudaError_t launch_one(fntgpu_aeq_state* st, const AeqArgs& A, cudaStream_t s) {
  const unsigned grid = (unsigned)((A.io.n_streams + AEQ_WARPS - 1) / AEQ_WARPS);
#ifndef AEQ_SMEM_PAD
#define AEQ_SMEM_PAD 0  // experiments only: extra dynamic smem to cap resident CTAs
#endif
  constexpr size_t smem = sizeof(AeqScratch) * AEQ_WARPS + AEQ_SMEM_PAD;
  auto* k = k_aeq_process<FWD, IN_MODE, TIN, QUICK>;
  if (smem > 48 * 1024) {
    const cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  k<<<grid, AEQ_WARPS * 32, smem, s>>>(st, A);
  return cudaGetLastError();
}

template <int FWD, bool QUICK>
static cudaError_t launch_fwd_q(fntgpu_aeq_state* st, const AeqArgs& A, cudaStream_t s) {
  if (A.io.in_mode == FNTGPU_AEQ_IN_DECIM) return launch_one<FWD, FNTGPU_AEQ_IN_DECIM, int8_t, QUICK>(st, A, s);
  if (A.io.in_dtype == FNTGPU_I8) return launch_one<FWD, FNTGPU_AEQ_IN_PLANAR, int8_t, QUICK>(st, A, s);
  if (A.io.in_dtype == FNTGPU_I32) return launch_one<FWD, FNTGPU_AEQ_IN_PLANAR, int32_t, QUICK>(st, A, s);
  return cudaErrorInvalidValue;
}

template <int FWD>
static cudaError_t launch_fwd(fntgpu_aeq_state* st, const AeqArgs& A, cudaStream_t s) {
  const bool quick = A.fast_rde && A.prm.n_radii == 3 && A.fast_div && A.io.adapt &&
                     A.io.err != nullptr && A.io.mu_blocks != nullptr;
  return quick ? launch_fwd_q<FWD, true>(st, A, s) : launch_fwd_q<FWD, false>(st, A, s);
}

// Streams per SM below which AUTO runs the polarization-split kernel: one warp per
// stream needs >= 12 warps per SM to saturate the issue slots.
#ifndef AEQ_POL_AUTO_PER_SM
#define AEQ_POL_AUTO_PER_SM 4
#endif

static bool use_pol_kernel(const fntgpu_aeq_params& prm, int64_t n_streams) {
  if (prm.forward != FNTGPU_AEQ_FWD_FNT) return false;
  if (prm.kernel == FNTGPU_AEQ_KERNEL_POL) return true;
  if (prm.kernel == FNTGPU_AEQ_KERNEL_WARP) return false;
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return n_streams < (int64_t)AEQ_POL_AUTO_PER_SM * sms;
}

cudaError_t launch_aeq_process(fntgpu_aeq_state* st, const fntgpu_aeq_params& prm,
                               const fntgpu_aeq_io& io, cudaStream_t s) {
  if (io.n_streams <= 0) return cudaSuccess;
  const AeqArgs A = make_args(prm, &io);
  if (use_pol_kernel(prm, io.n_streams)) return launch_aeq_pol(st, A, s);
  if (prm.forward == FNTGPU_AEQ_FWD_DIRECT) return launch_fwd<FNTGPU_AEQ_FWD_DIRECT>(st, A, s);
  return launch_fwd<FNTGPU_AEQ_FWD_FNT>(st, A, s);
}

cudaError_t launch_aeq_update_once(fntgpu_aeq_state* st, const fntgpu_aeq_params& prm,
                                   const int64_t* xblk, const double* y, double mu, double* err,
                                   cudaStream_t s) {
  const AeqArgs A = make_args(prm, nullptr);
  k_aeq_update_once<<<1, 32, 0, s>>>(st, A, xblk, y, mu, err);
  return cudaGetLastError();
}

// Self-check of div_D and the threshold ring decision against the IEEE slow path.
// Division: every numerator in [lo, hi). Ring: r2 = y0^2 + y1^2 for y0 = n / D and
// y1 = (n * 2654435761 mod 2^20 - 2^19) / D, plus r2 at and one ulp below each
// threshold.
__global__ void k_aeq_selfcheck(const __grid_constant__ AeqArgs A, int64_t lo, int64_t hi,
                                unsigned long long* mism) {
  unsigned long long bad_div = 0, bad_ring = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t n = lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; n < hi; n += stride) {
    const double q = div_D((int32_t)n, A);
    const double ref = __ddiv_rn((double)n, A.D);
    bad_div += __double_as_longlong(q) != __double_as_longlong(ref);
    if (A.fast_rde) {
      const int32_t m = (int32_t)(((uint32_t)n * 2654435761u) & 0xfffffu) - (1 << 19);
      const double y1 = __ddiv_rn((double)m, A.D);
      AeqArgs B = A;
      B.fast_rde = 0;
      bad_ring += __double_as_longlong(rde(ref, y1, A)) != __double_as_longlong(rde(ref, y1, B));
    }
  }
  if (A.fast_rde && blockIdx.x == 0 && threadIdx.x < 8) {
    const int k = threadIdx.x;
    if (k >= 1 && k < A.prm.n_radii && isfinite(A.T[k]) && A.T[k] > 0.0) {
      for (int d = -1; d <= 1; ++d) {
        const double r2 = __longlong_as_double(__double_as_longlong(A.T[k]) + d);
        // rde of (sqrt-free y_I, 0) reproduces the ring of r2 only if y_I^2 == r2;
        // compare the decisions directly instead
        int fast = 0, slow = 0;
        for (int i = 1; i < A.prm.n_radii; ++i) fast += r2 >= A.T[i];
        const double r = __dsqrt_rn(r2);
        double bd = fabs(dsub(r, A.prm.radii[0]));
        for (int i = 1; i < A.prm.n_radii; ++i) {
          const double dd = fabs(dsub(r, A.prm.radii[i]));
          if (dd < bd) { bd = dd; slow = i; }
        }
        bad_ring += A.R2[fast] != A.R2[slow];
      }
    }
  }
  if (bad_div) atomicAdd(&mism[0], bad_div);
  if (bad_ring) atomicAdd(&mism[1], bad_ring);
}

cudaError_t launch_aeq_selfcheck(const fntgpu_aeq_params& prm, int64_t lo, int64_t hi,
                                 unsigned long long* mismatches, cudaStream_t s) {
  const AeqArgs A = make_args(prm, nullptr);
  k_aeq_selfcheck<<<148 * 8, 256, 0, s>>>(A, lo, hi, mismatches);
  return cudaGetLastError();
}

}  // namespace fntgpu
