// k_aeq_pol.cu -- FNT-AEQ, latency form: two warps per stream, one per
// polarization.
//
// Reference: fntdsp/aeq.py:118-190 (equalize_block, update_taps, process).
//
// Why: k_aeq.cu runs one warp per stream, which saturates the SMs only with >= 12
// streams per SM; with fewer streams (config 3's six SNR points, a single FntAeq,
// config 5 sharded over many GPUs) each stream runs on the latency of its per-block
// recurrence taps -> forward -> error -> gradient -> taps (aeq.py:182-189). The two
// polarizations of a stream are independent inside a block: outputs {XI, XQ} use
// only the taps w[0:2] and the error e_x, {YI, YQ} only w[2:4] and e_y
// (aeq.py:155-164); they share only the read-only inputs. Warp p of the CTA owns
// output streams s = 2p, 2p + 1, so each warp's recurrence carries about 60% of
// the one-warp form's instructions (the input transforms are computed by both). The
// one cross-warp quantity, the err_trace mean over both polarizations, meets every
// POL_ERR_K blocks through a shared ring in numpy's pairwise order.
//
// Lane roles inside warp p (s' = s - 2p):
//   forward  (s', t, g, h) = lane bits (4, 3:2, 1, 0): digit g of filter (s, t),
//            transform bins k = 2 j + h (the first DIF stage of the 32-point
//            transform splits it into two 16-point ones: bins of parity h are
//            FNT16_{alpha=4}(d[n] 2^(n h)));
//   inverse  (s', g, k1 = 2 t + h): bins k = k1 + 8 k2 summed over the 4 input
//            streams (exact range test as k_aeq.cu fused_ok), a 4-point inverse,
//            twiddles 2^(-n k1);
//   output   (s', m = lane & 15): y[s][m], its error, e * y;
//   update   (s', t, g, h): taps k in [8g + 4h, 8g + 4h + 4) of filter (s, t).
// Each lane publishes the digit variants of its 4 taps to shared memory after the
// update, so the next block's forward reads its 16 transform inputs ready-made.
//
// Measured (config 5 chain, 512 streams on one B200): 24.7 ms vs 25.0 ms for the
// one-warp form -- at ~3.5 streams per SM both are latency-bound at about the same
// SM issue rate. A one-block look-ahead variant (block b+1's
// FNT forward with block b's taps overlapped with block b's float64 update, plus an
// exact integer correction for the tap change) was bit-exact but slower (27.1 ms):
// the correction's ~130 instructions per block outweigh the extra overlap.
#ifndef FNT_CARRY_MODE
// end-around carries as madc / complements as IMAD (fermat.cuh): 512 streams 22.85 -> 22.42 ms
#define FNT_CARRY_MODE 2
#endif
#include "aeq_common.cuh"

namespace fntgpu {

#ifndef AEQ_POL_ERR_K
#define AEQ_POL_ERR_K 4
#endif
constexpr int POL_ERR_K = AEQ_POL_ERR_K;  // blocks between the two warps' err_trace meetings
static_assert(POL_ERR_K % 4 == 0, "err_trace means are formed four blocks per pass");
constexpr int POL_BUF_P = 40;   // product row pitch (words): conflict-free (see below)
constexpr int POL_PART_P = 20;  // partial-inverse row pitch (words)
constexpr int POL_TV_P = 20;    // tap-variant row pitch (words)
constexpr int POL_XI_P = 136;   // 4-slot input ring, stored twice (128 words) + pad

struct __align__(16) PolWarp {
  uint32_t buf[32 * POL_BUF_P];        // products, then partial inverses
  uint32_t tv[32 * POL_TV_P];          // tap digit variants, row = reader lane
  double xf[4][66];                    // x / sig_scale ring (as k_aeq.cu AeqScratch.xf)
  int32_t xi[4][POL_XI_P];             // input integers: block b at 16 (b mod 4) and 64 + 16 (b mod 4)
  uint32_t X[4][36];                   // input spectra, canonical, [t][xm_index(k)] = X_t[k]
  int32_t traw[2][4][16];              // 14-bit taps w_int[s'][t][k] (reference-group forward)
  double ey[2][AEQ_L];                 // e * y per output stream of this polarization
};

struct __align__(16) PolScratch {
  PolWarp w[2];
  double eabs[2 * POL_ERR_K][32];      // |e| ring: [block slot][pol * 16 + m]
};

// 32-point forward transform of x_block[tq] = [ring slot a | ring slot b], four-step
// form across 8 lanes per stream (k_aeq.cu warp_input_fnt). Lane n1 ends with
// X[k2 + 4 k1], k1 = bitrev3(n1), N^-1 = 2^-5 folded in.
__device__ __forceinline__ void pol_input_fnt(const PolWarp& S, int lane, int off_prev, int off_cur,
                                              uint32_t (&v)[4]) {
  const int tq = lane >> 3, n1 = lane & 7;
  const int32_t* xr = S.xi[tq];
  const uint32_t a0 = f4_enc_small(xr[off_prev + n1]), a1 = f4_enc_small(xr[off_prev + n1 + 8]);
  const uint32_t a2 = f4_enc_small(xr[off_cur + n1]), a3 = f4_enc_small(xr[off_cur + n1 + 8]);
  const uint32_t s02 = m_add(a0, a2), d02 = m_sub(a0, a2);
  const uint32_t s13 = m_add(a1, a3), d13 = m_rot(m_sub(a1, a3), 8);
  v[0] = m_add(s02, s13);
  v[1] = m_add(d02, d13);
  v[2] = m_sub(s02, s13);
  v[3] = m_sub(d02, d13);
#pragma unroll
  for (int k2 = 1; k2 < 4; ++k2) {
    const int e = n1 * k2;
    const uint32_t r = __funnelshift_l(v[k2], v[k2], e & 15);
    v[k2] = (e & 16) ? ~r : r;
  }
#pragma unroll
  for (int st = 2; st >= 0; --st) {
    const int hh = 1 << st;
    const bool upper = (n1 & hh) != 0;
    const uint32_t mask = upper ? 0xffffffffu : 0u;
    const int e = upper ? (n1 & (hh - 1)) * (16 >> st) : 0;
#pragma unroll
    for (int k2 = 0; k2 < 4; ++k2) {
      const uint32_t o = __shfl_xor_sync(0xffffffffu, v[k2], hh);
      const uint32_t tt = m_add(v[k2] ^ mask, o);
      v[k2] = st > 0 ? __funnelshift_l(tt, tt, e) : tt;
    }
  }
}

// canonical residues (< 2^17, so the 64-bit multiply-accumulates of the stream sum
// cannot overflow) stored by bin k at X[t][4 (k mod 8) + k / 8]: the 4 bins an inverse
// lane k1 needs (k1 + 8 k2) are one 16-byte row
__device__ __host__ constexpr int xm_index(int k) { return 4 * (k & 7) + (k >> 3); }
__device__ __forceinline__ void pol_store_X(PolWarp& S, int lane, const uint32_t (&v)[4]) {
  const int tq = lane >> 3, n1 = lane & 7;
  const int k1 = (int)(__brev((unsigned)n1) >> 29);  // lane holds bins k2 + 4 k1
#pragma unroll
  for (int k2 = 0; k2 < 4; ++k2)
    S.X[tq][4 * (k2 + 4 * (k1 & 1)) + (k1 >> 1)] = f4_mod(m_rot(v[k2], 27));
}
// X_t[2 j + h] (bin parity h) in that layout: 4 h + 8 (j mod 4) + j / 4
__device__ __forceinline__ uint32_t pol_x(const PolWarp& S, int t, int h, int j) {
  return S.X[t][4 * h + 8 * (j & 3) + (j >> 2)];
}

// Digit variants of this lane's 4 taps (k = kb + kk): row (s', t, g, h) of S.tv is
// what forward lane (s', t, g, h) transforms: digit g (balanced base 64, the
// k_aeq.cu pack_taps<true> split w = 64 a + b: a, then b) times 2^(k h). Also the
// raw 14-bit taps for the reference-group forward. Returns sum |a| of the 4 taps.
__device__ __forceinline__ uint32_t publish_taps(PolWarp& S, int sp, int t, int kb,
                                                 const int32_t (&c)[4]) {
  uint32_t va[4], vb[4], wa[4], wb[4], asum = 0;
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) {
    const int32_t a = (c[kk] + 32) >> 6;
    const int32_t b = c[kk] - 64 * a;
    asum += (uint32_t)abs(a);
    va[kk] = (uint32_t)a;
    vb[kk] = (uint32_t)b;
    wa[kk] = (uint32_t)a << (kb + kk);     // |a| <= 256: exact in int32 for k < 16
    wb[kk] = (uint32_t)b << (kb + kk);
  }
  uint32_t* base = S.tv + (16 * sp + 4 * t) * POL_TV_P + kb;
  *reinterpret_cast<uint4*>(base + 0 * POL_TV_P) = make_uint4(va[0], va[1], va[2], va[3]);
  *reinterpret_cast<uint4*>(base + 1 * POL_TV_P) = make_uint4(wa[0], wa[1], wa[2], wa[3]);
  *reinterpret_cast<uint4*>(base + 2 * POL_TV_P) = make_uint4(vb[0], vb[1], vb[2], vb[3]);
  *reinterpret_cast<uint4*>(base + 3 * POL_TV_P) = make_uint4(wb[0], wb[1], wb[2], wb[3]);
  *reinterpret_cast<int4*>(&S.traw[sp][t][kb]) = make_int4(c[0], c[1], c[2], c[3]);
  return asum;
}

// 16-point forward transform (alpha = 4), natural order in and out: the first stage
// in plain int32 (|v| <= 2^23 from the variants), then Z/M stages.
__device__ __forceinline__ void fnt16_taps(uint32_t (&v)[16]) {
  to_bitrev<16>(v);
  // |u +- w| <= 2^24 < F4_BIAS = 65537 * 256: non-negative residues of Z/M after
  fnt_stage_plain<16, RADIX4, 0, 1, F4_BIAS>(v);
  fnt_stage<16, RADIX4, false, false, false, 1, -1>(v);
}

// tap spectra of this lane's (filter, digit, bin parity) from the published variants
__device__ __forceinline__ void load_tap_spectrum(const PolWarp& S, int lane, uint32_t (&W)[16]) {
  const uint4* tv = reinterpret_cast<const uint4*>(S.tv + lane * POL_TV_P);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint4 v = tv[q];
    W[4 * q] = v.x; W[4 * q + 1] = v.y; W[4 * q + 2] = v.z; W[4 * q + 3] = v.w;
  }
  fnt16_taps(W);
}

// the lane's 16 tap-spectrum bins (parity h), written to row `lane` of S.buf in groups
// q = j mod 4 (entries j = q + 4 k2) at group slot q ^ t_lo: with the 40-word pitch
// the 8 lanes of every store / load phase hit 8 distinct 4-bank groups
__device__ __forceinline__ void store_spectrum(PolWarp& S, int lane, const uint32_t (&W)[16]) {
  uint32_t* rowp = S.buf + lane * POL_BUF_P;
  const int swz = (lane >> 2) & 1;
#pragma unroll
  for (int q = 0; q < 4; ++q)
    reinterpret_cast<uint4*>(rowp)[q ^ swz] = make_uint4(W[q], W[q + 4], W[q + 8], W[q + 12]);
}

// inverse role (s', g, k1 = 2t + h): bins k1 + 8 k2 of sum_t'' X_t'' W_st''g as 64-bit
// multiply-accumulates (X canonical < 2^17, W < 2^32: below 2^51), folded once per bin
// (2^32 == 1 mod 2^32 - 1); +32768 on the DC bin (decode offset on every output),
// 4-point inverse, twiddles 2^(-(16 + mm) k1) for the 16 kept outputs
__device__ __forceinline__ void partial_inverse(const PolWarp& S, int sp, int t, int g, int h,
                                                uint32_t (&o)[16]) {
  const int k1 = 2 * t + h;
  uint64_t acc[4];
#pragma unroll
  for (int tt = 0; tt < 4; ++tt) {
    const int r = 16 * sp + 4 * tt + 2 * g + h;
    const uint4 w = reinterpret_cast<const uint4*>(S.buf + r * POL_BUF_P)[t ^ (tt & 1)];
    const uint4 x = *reinterpret_cast<const uint4*>(&S.X[tt][4 * k1]);
    const uint32_t wv[4] = {w.x, w.y, w.z, w.w}, xv[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const uint64_t pr = (uint64_t)xv[e] * wv[e];
      acc[e] = tt == 0 ? pr : acc[e] + pr;
    }
  }
  uint32_t Q[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) Q[e] = m_add((uint32_t)acc[e], (uint32_t)(acc[e] >> 32));
  Q[0] = m_add(Q[0], k1 == 0 ? 32768u : 0u);
  to_bitrev<4>(Q);
  fnt_dit<4, RADIX256, true>(Q);
#pragma unroll
  for (int mm = 0; mm < 16; ++mm) o[mm] = __funnelshift_l(Q[mm & 3], Q[mm & 3], ((16 - mm) * k1) & 31);
}

__device__ __forceinline__ void store_row16(uint32_t* prow, const uint32_t (&o)[16]) {
#pragma unroll
  for (int q = 0; q < 4; ++q)
    reinterpret_cast<uint4*>(prow)[q] = make_uint4(o[4 * q], o[4 * q + 1], o[4 * q + 2], o[4 * q + 3]);
}

// output role (s', m): y_int = 64 dec(sum_k1 digit a) + dec(sum_k1 digit b)
__device__ __forceinline__ int32_t fused_output(const PolWarp& S, int sp, int m) {
  uint32_t u0[8], u1[8];
#pragma unroll
  for (int kq = 0; kq < 8; ++kq) {
    const int r = 16 * sp + 4 * (kq >> 1) + (kq & 1);  // lane (s', t = kq/2, g, h = kq&1)
    u0[kq] = S.buf[r * POL_PART_P + 16 * sp + m];
    u1[kq] = S.buf[(r + 2) * POL_PART_P + 16 * sp + m];
  }
#pragma unroll
  for (int w = 4; w > 0; w >>= 1) {
#pragma unroll
    for (int i = 0; i < w; ++i) {
      u0[i] = m_add(u0[i], u0[i + w]);
      u1[i] = m_add(u1[i], u1[i + w]);
    }
  }
  return 64 * (int32_t)f4_mod(u0[0]) + (int32_t)f4_mod(u1[0]) - 65 * 32768;
}

// The whole forward of one block with the taps published in S.tv / S.traw and the
// spectra in S.X (aeq.py:118-144): the transform-domain stream sum when `fused`, else
// the reference's per-(s, t, group) residue convolutions (split_taps groups). Enters
// and leaves with the warp converged; uses S.buf.
__device__ __forceinline__ int32_t pol_forward(PolWarp& S, int lane, bool fused) {
  const int sp = lane >> 4, t = (lane >> 2) & 3, g = (lane >> 1) & 1, h = lane & 1, m = lane & 15;
  uint32_t P[16];
  if (fused) {
    load_tap_spectrum(S, lane, P);
  } else {
    const int4* tw = reinterpret_cast<const int4*>(S.traw[sp][t]);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int4 v = tw[q];
      const int32_t w4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) P[4 * q + i] = (uint32_t)tap_group(w4[i], g) << ((4 * q + i) * h);
    }
    fnt16_taps(P);
  }
  if (fused) {
    store_spectrum(S, lane, P);
    __syncwarp();
    uint32_t o[16];
    partial_inverse(S, sp, t, g, h, o);
    __syncwarp();
    store_row16(S.buf + lane * POL_PART_P + 16 * sp, o);
    __syncwarp();
    const int32_t yi = fused_output(S, sp, m);
    __syncwarp();
    return yi;
  }
  // per (s, t, group): the lane's 16 products of parity h through a 16-point inverse
  // (alpha^-2), twiddle 2^(-(16 + mm) h), summed over h when decoding
#pragma unroll
  for (int j = 0; j < 16; ++j) P[j] = m_mul(P[j], pol_x(S, t, h, j));
  P[0] = m_add(P[0], h == 0 ? 32768u : 0u);
  to_bitrev<16>(P);
  fnt_dit<16, RADIX4, true>(P);
  uint32_t o[16];
#pragma unroll
  for (int mm = 0; mm < 16; ++mm) o[mm] = __funnelshift_l(P[mm], P[mm], ((16 - mm) * h) & 31);
  __syncwarp();
  store_row16(S.buf + lane * POL_PART_P + 16 * sp, o);
  __syncwarp();
  int32_t a = -4 * 129 * 32768;
#pragma unroll
  for (int tt = 0; tt < 4; ++tt) {
#pragma unroll
    for (int gg = 0; gg < 2; ++gg) {
      const int r = 16 * sp + 4 * tt + 2 * gg;
      const uint32_t u = m_add(S.buf[r * POL_PART_P + 16 * sp + m], S.buf[(r + 1) * POL_PART_P + 16 * sp + m]);
      a += (gg == 0 ? 128 : 1) * (int32_t)f4_mod(u);
    }
  }
  __syncwarp();
  return a;
}

template <int IN_MODE, typename TIN, bool QUICK>
__global__ void __launch_bounds__(64, 4) k_aeq_pol(fntgpu_aeq_state* __restrict__ st,
                                                   const __grid_constant__ AeqArgs A) {
  constexpr bool NARROW = sizeof(TIN) == 1;
  extern __shared__ __align__(16) unsigned char pol_dyn_smem[];
  PolScratch& SS = *reinterpret_cast<PolScratch*>(pol_dyn_smem);
  __shared__ double lut[2 * XF_LUT + 1];
  __shared__ long long sat_sh[2];
  for (int i = threadIdx.x; i < 2 * XF_LUT + 1; i += blockDim.x)
    lut[i] = __ddiv_rn((double)(i - XF_LUT), A.prm.sig_scale);
  __syncthreads();

  const fntgpu_aeq_io& io = A.io;
  const int64_t S_idx = blockIdx.x;  // one stream per CTA
  if (S_idx >= io.n_streams) return;
  const int p = threadIdx.x >> 5, lane = threadIdx.x & 31;
  PolWarp& S = SS.w[p];
  fntgpu_aeq_state& state = st[S_idx];

  const int sp = lane >> 4, s = 2 * p + sp;
  const int t = (lane >> 2) & 3, g = (lane >> 1) & 1, h = lane & 1;
  const int kb = 8 * g + 4 * h;   // this lane's taps (update role)
  const int m = lane & 15;        // output role
  const int tq = lane >> 3, iq = 2 * (lane & 7);  // input-loader role

  double wf[4];
  int32_t c[4];
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) {
    wf[kk] = state.w[s][t][kb + kk];
    c[kk] = state.w_int[s][t][kb + kk];
  }
  uint32_t asum = publish_taps(S, sp, t, kb, c);
  uint32_t sat = 0;
  int32_t v0 = state.hist[tq][iq], v1 = state.hist[tq][iq + 1];  // samples of the latest block
  auto put_int = [&](int64_t blk, int32_t a, int32_t b) {  // input ring slot blk mod 4 (stored twice)
    const int o = AEQ_L * (int)(blk & 3) + iq;
    *reinterpret_cast<int2*>(S.xi[tq] + o) = make_int2(a, b);
    *reinterpret_cast<int2*>(S.xi[tq] + 64 + o) = make_int2(a, b);
  };
  auto put_xf = [&](int64_t blk, double f0, double f1) {  // x / sig ring, parity slot (stored twice)
    double* xr = &S.xf[tq][1 + AEQ_L * (int)(blk & 1) + iq];
    xr[0] = f0;
    xr[1] = f1;
    xr[32] = f0;
    xr[33] = f1;
  };
  put_int(-1, v0, v1);
  put_xf(-1, xf_of<false>(v0, lut, A.prm.sig_scale), xf_of<false>(v1, lut, A.prm.sig_scale));

  const char* row;
  uint32_t sel0 = 0, sel1 = 1;
  if (IN_MODE == FNTGPU_AEQ_IN_PLANAR) {
    row = reinterpret_cast<const char*>(reinterpret_cast<const TIN*>(io.x) + S_idx * io.x_stream_stride +
                                        tq * io.x_row_stride);
  } else {
    const int8_t* plane = (tq & 1) ? io.qi : io.qr;
    row = reinterpret_cast<const char*>(plane + (2 * S_idx + (tq >> 1)) * io.q_stride);
    const uint32_t ph = (uint32_t)io.phase[S_idx];
    sel0 = ph;
    sel1 = 2 + ph;
  }
  constexpr int64_t IN_STEP = IN_MODE == FNTGPU_AEQ_IN_DECIM ? 2 * AEQ_L : (int64_t)sizeof(TIN) * AEQ_L;
  row += IN_MODE == FNTGPU_AEQ_IN_DECIM ? 2 * iq : (int64_t)sizeof(TIN) * iq;
  auto fetch = [&](const char* ptr) -> uint2 {
    if (IN_MODE == FNTGPU_AEQ_IN_DECIM) {
      return make_uint2(__ldg(reinterpret_cast<const uint32_t*>(ptr)), 0u);
    } else if (NARROW) {
      return make_uint2(__ldg(reinterpret_cast<const uint16_t*>(ptr)), 0u);
    } else {
      const int2 v = __ldg(reinterpret_cast<const int2*>(ptr));
      return make_uint2((uint32_t)v.x, (uint32_t)v.y);
    }
  };
  auto decode = [&](uint2 raw, int32_t& a, int32_t& b) {
    if (IN_MODE == FNTGPU_AEQ_IN_DECIM) {
      a = sbyte(raw.x, sel0);
      b = sbyte(raw.x, sel1);
    } else if (NARROW) {
      a = sbyte(raw.x, 0);
      b = sbyte(raw.x, 1);
    } else {
      a = (int32_t)raw.x;
      b = (int32_t)raw.y;
    }
  };
  auto mag = [](int32_t v) -> uint32_t { return v < 0 ? 0u - (uint32_t)v : (uint32_t)v; };

  const int64_t nb = io.n_blocks;
  const double* mu_p = io.mu_blocks;
  double* err_out = io.err ? io.err + S_idx * io.err_stream_stride : nullptr;
  const bool adapt = QUICK || io.adapt;
  const bool want_err = adapt && (QUICK || err_out != nullptr);
  double* yp = io.y + S_idx * io.y_stream_stride + s * io.y_row_stride + m;
  long long sat64 = 0;
  // Block b+1's input transforms are computed inside block b's update (they do not
  // depend on the taps): the float64 gradient leaves integer issue slots free. The
  // input ring therefore holds 4 blocks (b - 1 .. b + 1 in use); X holds X_b until
  // block b's forward has read it.
  uint2 raw = make_uint2(0u, 0u);
  double mu_next = mu_p && nb > 0 ? mu_p[0] : A.prm.mu;
  uint32_t amax_cur = 0;  // max |x| over the current block's window (all four streams)
  if (nb > 0) {
    int32_t a0, a1;
    decode(fetch(row), a0, a1);
    const uint32_t a_hist = max(mag(v0), mag(v1));
    v0 = a0;
    v1 = a1;
    put_int(0, v0, v1);
    if (adapt) put_xf(0, xf_of<NARROW>(v0, lut, A.prm.sig_scale), xf_of<NARROW>(v1, lut, A.prm.sig_scale));
    amax_cur = __reduce_max_sync(0xffffffffu, max(max(mag(v0), mag(v1)), a_hist));
    if (nb > 1) {
      row += IN_STEP;
      raw = fetch(row);
    }
    __syncwarp();
    uint32_t xv[4];
    pol_input_fnt(S, lane, AEQ_L * 3, 0, xv);
    pol_store_X(S, lane, xv);
    __syncwarp();
  }

  for (int64_t b0 = 0; b0 < nb; b0 += (int64_t)1 << 24) {
    const int64_t b1 = nb - b0 < ((int64_t)1 << 24) ? nb : b0 + ((int64_t)1 << 24);
    for (int64_t b = b0; b < b1; ++b) {
      const bool more = b + 1 < nb;
      const double mu = mu_next;
      const uint32_t asum_w = __reduce_add_sync(0xffffffffu, asum);
      // ---- forward (aeq.py:118-144) with X_b
      const int32_t yi = pol_forward(S, lane, amax_cur <= 16u && asum_w * amax_cur <= 32768u);
      const double y0 = div_D<QUICK>(yi, A);  // y_int / (sig_scale * tap_scale)
      yp[AEQ_L * b] = y0;
      // ---- block b+1's samples into the ring (the last block re-reads its own)
      int32_t n0, n1;
      decode(raw, n0, n1);
      if (QUICK) {
        row += (b + 2 < nb) ? IN_STEP : 0;
        raw = fetch(row);
        mu_next = mu_p[more ? b + 1 : b];
      } else {
        if (b + 2 < nb) {
          row += IN_STEP;
          raw = fetch(row);
        }
        if (more && mu_p) mu_next = mu_p[b + 1];
      }
      if (!more) { n0 = v0; n1 = v1; }
      put_int(b + 1, n0, n1);
      const uint32_t amax_next =
          __reduce_max_sync(0xffffffffu, max(max(mag(n0), mag(n1)), max(mag(v0), mag(v1))));
      uint32_t xv[4];
      const int off4 = AEQ_L * (int)(b & 3);  // x_block_{b+1} = [slot b | slot b+1]
      if (adapt) {
        // ---- update_taps (aeq.py:148-170) for this polarization
        const double yo = __shfl_xor_sync(0xffffffffu, y0, 16);
        const double yI = sp == 0 ? y0 : yo, yQ = sp == 0 ? yo : y0;  // one branch-free ring decision
        const double e = rde<QUICK>(yI, yQ, A);
        S.ey[sp][m] = dmul(e, y0);
        if (want_err && sp == 0) SS.eabs[b % (2 * POL_ERR_K)][16 * p + m] = fabs(e);
        __syncwarp();
        if (mu != 0.0) {
          pol_input_fnt(S, lane, off4, off4 + AEQ_L, xv);  // interleaved with the gradient
          // gradient of taps k = kb + kk: sum_m ey[s'][m] x_block[t][16 + m - k] in
          // numpy's einsum order (aeq_common.cuh einsum_m, two chains per tap);
          // x_block[t][16 + m - k] = xs[3 - kk + m], xs + me 16-byte aligned
          const double* xs = S.xf[t] + 1 + AEQ_L * (int)((b & 1) ^ 1) + 13 - kb;
          const double2* eyv = reinterpret_cast<const double2*>(S.ey[sp]);
          double c0[4], c1[4];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int me = (i < 4 ? 6 : 22) - 2 * i;  // 6, 4, 2, 0, 14, 12, 10, 8
            const double2 e2 = eyv[me / 2];
            const double2 p0 = reinterpret_cast<const double2*>(xs + me)[0];
            const double2 p1 = reinterpret_cast<const double2*>(xs + me)[1];
            const double xw[5] = {p0.x, p0.y, p1.x, p1.y, xs[me + 4]};
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              const double pe = dmul(e2.x, xw[3 - kk]), po = dmul(e2.y, xw[4 - kk]);
              c0[kk] = i == 0 ? pe : dadd(pe, c0[kk]);
              c1[kk] = i == 0 ? po : dadd(po, c1[kk]);
            }
          }
          uint32_t smask = 0;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const double w = dadd(wf[kk], dmul(mu, dadd(c0[kk], c1[kk])));
            wf[kk] = w;
            const double pq = dmul(w, A.prm.tap_scale);
            const int32_t i = __double2int_rn(pq);
            c[kk] = min(max(i, -AEQ_TAP_MAX), AEQ_TAP_MAX);
            smask |= (uint32_t)!(fabs(pq) < 16383.5) << kk;  // clipped (rint half-even), or NaN
          }
          sat += __popc(smask);
          if (__any_sync(0xffffffffu, smask != 0u)) {
            // rare: a clipped tap whose rint is not an int64 (numpy: INT64_MIN, NaN
            // included) becomes -16383 and is not counted (aeq.py:165-168)
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              if ((smask >> kk) & 1u) {
                if (!(fabs(dmul(wf[kk], A.prm.tap_scale)) < 9.2233720368547758e18)) {
                  sat -= 1;
                  c[kk] = -AEQ_TAP_MAX;
                }
              }
            }
          }
          asum = publish_taps(S, sp, t, kb, c);
        } else {
          pol_input_fnt(S, lane, off4, off4 + AEQ_L, xv);
        }
        if (want_err && ((b + 1) % POL_ERR_K == 0 || !more)) {
          // both polarizations' |e| of the last <= POL_ERR_K blocks are in the ring:
          // warp 0 forms the means in numpy's pairwise order (k_aeq.cu lane_update)
          __syncthreads();
          if (p == 0) {
            // four blocks per pass, one per group of 8 lanes
#pragma unroll
            for (int q = 0; q < POL_ERR_K; q += 4) {
              const int64_t bb = b - (b % POL_ERR_K) + q + (lane >> 3);
              const int j = lane & 7;
              double r = 0.0;
              if (bb <= b) {
                const double* a = SS.eabs[bb % (2 * POL_ERR_K)];
                r = dadd(dadd(dadd(a[j], a[j + 8]), a[j + 16]), a[j + 24]);
              }
              r = dadd(r, __shfl_xor_sync(0xffffffffu, r, 1));
              r = dadd(r, __shfl_xor_sync(0xffffffffu, r, 2));
              r = dadd(r, __shfl_xor_sync(0xffffffffu, r, 4));
              if (j == 0 && bb <= b) err_out[bb] = dmul(r, 1.0 / 32.0);
            }
          }
        }
        // block b's gradient has read its window: block b+1's x / sig may land
        put_xf(b + 1, xf_of<NARROW>(n0, lut, A.prm.sig_scale), xf_of<NARROW>(n1, lut, A.prm.sig_scale));
      } else {
        pol_input_fnt(S, lane, off4, off4 + AEQ_L, xv);
      }
      pol_store_X(S, lane, xv);  // X_{b+1}: block b's forward has read X_b
      amax_cur = amax_next;
      if (more) { v0 = n0; v1 = n1; }
      __syncwarp();
    }
    sat64 += sat;
    sat = 0;
  }

  // write back the stream state
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) {
    state.w[s][t][kb + kk] = wf[kk];
    state.w_int[s][t][kb + kk] = c[kk];
  }
  long long sw = sat64;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) sw += __shfl_xor_sync(0xffffffffu, sw, off);
  if (lane == 0) sat_sh[p] = sw;
  __syncthreads();
  if (p == 0) {
    if (io.n_blocks > 0) {
      state.hist[tq][iq] = v0;
      state.hist[tq][iq + 1] = v1;
    }
    if (lane == 0) {
      state.saturations += sat_sh[0] + sat_sh[1];
      state.symbols += io.n_blocks * AEQ_L;
      if (io.adapt) state.n_err += io.n_blocks;
    }
  }
}

template <int IN_MODE, typename TIN, bool QUICK>
static cudaError_t launch_pol_one(fntgpu_aeq_state* st, const AeqArgs& A, cudaStream_t s) {
  constexpr size_t smem = sizeof(PolScratch);
  auto* k = k_aeq_pol<IN_MODE, TIN, QUICK>;
  if (smem > 48 * 1024) {
    const cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  k<<<(unsigned)A.io.n_streams, 64, smem, s>>>(st, A);
  return cudaGetLastError();
}

template <bool QUICK>
static cudaError_t launch_pol_q(fntgpu_aeq_state* st, const AeqArgs& A, cudaStream_t s) {
  if (A.io.in_mode == FNTGPU_AEQ_IN_DECIM) return launch_pol_one<FNTGPU_AEQ_IN_DECIM, int8_t, QUICK>(st, A, s);
  if (A.io.in_dtype == FNTGPU_I8) return launch_pol_one<FNTGPU_AEQ_IN_PLANAR, int8_t, QUICK>(st, A, s);
  if (A.io.in_dtype == FNTGPU_I32) return launch_pol_one<FNTGPU_AEQ_IN_PLANAR, int32_t, QUICK>(st, A, s);
  return cudaErrorInvalidValue;
}

cudaError_t launch_aeq_pol(fntgpu_aeq_state* st, const AeqArgs& A, cudaStream_t s) {
  const bool quick = A.fast_rde && A.prm.n_radii == 3 && A.fast_div && A.io.adapt &&
                     A.io.err != nullptr && A.io.mu_blocks != nullptr;
  return quick ? launch_pol_q<true>(st, A, s) : launch_pol_q<false>(st, A, s);
}

}  // namespace fntgpu
