/*
 * fntdsp_oracle.c -- CPU restatement of the reference hot path, used ONLY as a
 * checker (tests/, __graft_entry__.smoke(), bench.py cpu_baseline / --impl
 * reference). Nothing in the product path links or calls this file.
 *
 * Parity status: PINNED. tests/test_oracle_golden.py checks every function
 * below against fixtures produced by the unmodified reference (`fntdsp`,
 * tests/golden/make_golden.py) before any GPU result is compared with it.
 *
 * Restated reference functions (all paths under /root/reference/pkg/src/fntdsp):
 *   or_plan_init          fnt.py:60-83    make_plan / _stage_twiddles / _bit_reverse_permutation
 *   or_fnt                fnt.py:86-114   _butterflies (radix-2 DIT, bit-reversal pre-permutation), fnt, ifnt
 *   or_cyclic_real        fnt.py:117-125  cyclic_convolve_real
 *   or_cyclic_complex     fnt.py:128-161  cyclic_convolve_complex (Eqs. 7-8)
 *   or_quantize_real      fixedpoint.py:51-60 _round_half_away + quantize_real
 *   or_cdc_process_int    cdc.py:89-95, 141-175 overlap-save FNT-CDC
 *   or_cdc_direct         SURVEY a19: out[n] = sum_k h[k] x[n+c-k] reduced mod F (second oracle)
 *   or_aeq_*              aeq.py:53-58, 118-190 FntAeq (float64 update in numpy's einsum order,
 *                         SURVEY Appendix A; compile with -ffp-contract=off)
 *   or_decimation_phase   linksim.py:249-260 _decimation_phase
 *   or_pairwise_sum       numpy's pairwise summation (np.add.reduce on contiguous float64)
 *
 * Build: make -C oracle   (gcc -O2 -ffp-contract=off -fno-fast-math)
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef int64_t i64;

/* ------------------------------------------------------------------------ */
/* ring Z/F, F = 2^(2^t) + 1 (fermat.py:22-53)                                */

static i64 pmod(i64 a, i64 m) { i64 r = a % m; return r < 0 ? r + m : r; }

static i64 mulmod(i64 a, i64 b, i64 m) { return (i64)(((__int128)a * b) % m); }

static i64 powmod(i64 a, i64 e, i64 m) {
  i64 r = 1 % m; a = pmod(a, m);
  while (e > 0) { if (e & 1) r = mulmod(r, a, m); a = mulmod(a, a, m); e >>= 1; }
  return r;
}

typedef struct {
  int t, n, log2n;
  i64 F, alpha, alpha_inv, n_inv;
  i64 bitrev[65536];
  /* stage s twiddles: tw[(1<<s)-1 + j] = root^(j * n / 2^(s+1)), j < 2^s */
  i64 fwd[65536];
  i64 inv[65536];
} or_plan;

size_t or_plan_size(void) { return sizeof(or_plan); }

/* make_plan (fnt.py:60-83). Returns 0, or -1 length, -2 radix range,
 * -3 alpha^n != 1, -4 alpha^(n/2) != -1, -5 unsupported size/index. */
int or_plan_init(or_plan* p, int t, int n, i64 alpha) {
  if (t < 0 || t > 4) return -5;
  if (n < 2 || (n & (n - 1))) return -1;
  if (n > 65536) return -5;
  i64 F = ((i64)1 << (1 << t)) + 1;
  if (!(alpha > 0 && alpha < F)) return -2;
  if (powmod(alpha, n, F) != 1) return -3;
  if (powmod(alpha, n / 2, F) != F - 1) return -4;
  p->t = t; p->n = n; p->F = F; p->alpha = alpha;
  int lg = 0; while ((1 << lg) < n) ++lg;
  p->log2n = lg;
  p->alpha_inv = powmod(alpha, F - 2, F);
  p->n_inv = powmod(n, F - 2, F);
  for (int i = 0; i < n; ++i) {
    int r = 0, v = i;
    for (int b = 0; b < lg; ++b) { r = (r << 1) | (v & 1); v >>= 1; }
    p->bitrev[i] = r;
  }
  for (int s = 0; s < lg; ++s) {
    int half = 1 << s; int step = n >> (s + 1);
    for (int j = 0; j < half; ++j) {
      p->fwd[half - 1 + j] = powmod(alpha, (i64)j * step, F);
      p->inv[half - 1 + j] = powmod(p->alpha_inv, (i64)j * step, F);
    }
  }
  return 0;
}

/* _butterflies (fnt.py:86-103) on one vector; input any int64 (reduced mod F). */
static void fnt1(const or_plan* p, const i64* x, i64* y, int inverse) {
  const i64 F = p->F; const int n = p->n;
  i64* a = y;
  for (int i = 0; i < n; ++i) a[i] = pmod(x[p->bitrev[i]], F);
  for (int s = 0; s < p->log2n; ++s) {
    int half = 1 << s;
    const i64* tw = (inverse ? p->inv : p->fwd) + half - 1;
    for (int g = 0; g < n; g += 2 * half) {
      for (int j = 0; j < half; ++j) {
        i64 u = a[g + j];
        i64 v = (a[g + j + half] * tw[j]) % F;
        a[g + j] = (u + v) % F;
        a[g + j + half] = pmod(u - v, F);
      }
    }
  }
  if (inverse) for (int i = 0; i < n; ++i) a[i] = (a[i] * p->n_inv) % F;
}

/* fnt / ifnt (fnt.py:106-114), batched over leading axes. */
void or_fnt(const or_plan* p, const i64* x, i64* y, i64 batch, int inverse) {
  for (i64 b = 0; b < batch; ++b) fnt1(p, x + b * p->n, y + b * p->n, inverse);
}

/* cyclic_convolve_real (fnt.py:117-125); h_stride = 0 broadcasts one tap vector. */
void or_cyclic_real(const or_plan* p, const i64* x, const i64* h, i64 h_stride, i64* z, i64 batch) {
  const int n = p->n; const i64 F = p->F;
  i64* X = (i64*)malloc(sizeof(i64) * n);
  i64* H = (i64*)malloc(sizeof(i64) * n);
  for (i64 b = 0; b < batch; ++b) {
    fnt1(p, x + b * n, X, 0);
    fnt1(p, h + b * h_stride, H, 0);
    for (int k = 0; k < n; ++k) X[k] = (X[k] * H[k]) % F;
    fnt1(p, X, z + b * n, 1);
  }
  free(X); free(H);
}

/* cyclic_convolve_complex (fnt.py:128-161). */
void or_cyclic_complex(const or_plan* p, const i64* xr, const i64* xi, const i64* yr,
                       const i64* yi, i64 y_stride, i64* zr, i64* zi, i64 batch) {
  const int n = p->n; const i64 F = p->F; const int q = 1 << p->t;
  const i64 j = (i64)1 << (q / 2);
  const i64 c_re = pmod(F - powmod(2, q - 1, F), F);
  const i64 c_im = pmod(F - powmod(2, q / 2 - 1, F), F);
  i64 *Xr = malloc(sizeof(i64) * n), *Xi = malloc(sizeof(i64) * n);
  i64 *Yr = malloc(sizeof(i64) * n), *Yi = malloc(sizeof(i64) * n);
  i64 *S = malloc(sizeof(i64) * n), *D = malloc(sizeof(i64) * n);
  for (i64 b = 0; b < batch; ++b) {
    fnt1(p, xr + b * n, Xr, 0); fnt1(p, xi + b * n, Xi, 0);
    fnt1(p, yr + b * y_stride, Yr, 0); fnt1(p, yi + b * y_stride, Yi, 0);
    for (int k = 0; k < n; ++k) {
      i64 ap = (Xr[k] + j * Xi[k]) % F, am = pmod(Xr[k] - j * Xi[k], F);
      i64 bp = (Yr[k] + j * Yi[k]) % F, bm = pmod(Yr[k] - j * Yi[k], F);
      i64 up = (ap * bp) % F, um = (am * bm) % F;
      S[k] = (up + um) % F; D[k] = pmod(up - um, F);
    }
    fnt1(p, S, zr + b * n, 1); fnt1(p, D, zi + b * n, 1);
    for (int k = 0; k < n; ++k) {
      zr[b * n + k] = (zr[b * n + k] * c_re) % F;
      zi[b * n + k] = (zi[b * n + k] * c_im) % F;
    }
  }
  free(Xr); free(Xi); free(Yr); free(Yi); free(S); free(D);
}

/* ------------------------------------------------------------------------ */
/* quantizer (fixedpoint.py:51-60): v = sign(x*s)*floor(|x*s|+0.5), clip.    */

i64 or_quantize_real(const double* x, i64 n, double scale, i64 max_int, i64* q) {
  i64 clipped = 0;
  for (i64 i = 0; i < n; ++i) {
    double v = x[i] * scale;
    double a = floor(fabs(v) + 0.5);
    double r = v > 0 ? a : (v < 0 ? -a : 0.0);
    if (fabs(r) > (double)max_int) ++clipped;
    if (r > (double)max_int) r = (double)max_int;
    if (r < -(double)max_int) r = -(double)max_int;
    q[i] = (i64)r;
  }
  return clipped;
}

/* ------------------------------------------------------------------------ */
/* FNT-CDC (cdc.py:89-95, 124-175)                                            */

static i64 decode_signed(i64 r, i64 F) { return r <= (F - 1) / 2 ? r : r - F; }
static i64 encode_signed(i64 v, i64 F) { return v >= 0 ? v : F + v; }

/* Overlap-save through the plan: 50% blocks with a hop = n/2 zero lead-in;
 * output aligned by c = n_taps // 2. Taps length n_taps <= n/2 + 1. */
void or_cdc_process_int(const or_plan* p, const i64* tap_re, const i64* tap_im, int n_taps,
                        const i64* xr, const i64* xi, i64 L, i64* yr, i64* yi) {
  const int n = p->n, hop = n / 2; const i64 F = p->F; const int q = 1 << p->t;
  const i64 j = (i64)1 << (q / 2);
  const i64 c_re = pmod(F - powmod(2, q - 1, F), F);
  const i64 c_im = pmod(F - powmod(2, q / 2 - 1, F), F);
  i64 *hr = calloc(n, sizeof(i64)), *hi = calloc(n, sizeof(i64));
  i64 *Hr = malloc(sizeof(i64) * n), *Hi = malloc(sizeof(i64) * n);
  i64 *bp = malloc(sizeof(i64) * n), *bm = malloc(sizeof(i64) * n);
  for (int k = 0; k < n_taps; ++k) { hr[k] = encode_signed(tap_re[k], F); hi[k] = encode_signed(tap_im[k], F); }
  fnt1(p, hr, Hr, 0); fnt1(p, hi, Hi, 0);
  for (int k = 0; k < n; ++k) { bp[k] = (Hr[k] + j * Hi[k]) % F; bm[k] = pmod(Hr[k] - j * Hi[k], F); }
  i64 n_blocks = (L + hop + hop - 1) / hop;
  i64 *br = malloc(sizeof(i64) * n), *bi = malloc(sizeof(i64) * n);
  i64 *Xr = malloc(sizeof(i64) * n), *Xi = malloc(sizeof(i64) * n);
  i64 *S = malloc(sizeof(i64) * n), *D = malloc(sizeof(i64) * n);
  i64 *zr = malloc(sizeof(i64) * n), *zi = malloc(sizeof(i64) * n);
  const i64 c = n_taps / 2;
  for (i64 b = 0; b < n_blocks; ++b) {
    for (int i = 0; i < n; ++i) {
      i64 idx = b * hop - hop + i;
      i64 vr = (idx >= 0 && idx < L) ? xr[idx] : 0, vi = (idx >= 0 && idx < L) ? xi[idx] : 0;
      br[i] = encode_signed(vr, F); bi[i] = encode_signed(vi, F);
    }
    fnt1(p, br, Xr, 0); fnt1(p, bi, Xi, 0);
    for (int k = 0; k < n; ++k) {
      i64 up = ((Xr[k] + j * Xi[k]) % F) * bp[k] % F;
      i64 um = (pmod(Xr[k] - j * Xi[k], F)) * bm[k] % F;
      S[k] = (up + um) % F; D[k] = pmod(up - um, F);
    }
    fnt1(p, S, zr, 1); fnt1(p, D, zi, 1);
    for (int i = hop; i < n; ++i) {
      i64 m = b * hop + (i - hop) - c; /* yr_full[b*hop + i - hop] -> out[m] */
      if (m >= 0 && m < L) {
        yr[m] = decode_signed(zr[i] * c_re % F, F);
        yi[m] = decode_signed(zi[i] * c_im % F, F);
      }
    }
  }
  free(hr); free(hi); free(Hr); free(Hi); free(bp); free(bm); free(br); free(bi);
  free(Xr); free(Xi); free(S); free(D); free(zr); free(zi);
}

/* Direct-FIR oracle: out[n] = decode( sum_k h[k] x[n+c-k] mod F ), complex. */
void or_cdc_direct(i64 F, const i64* tap_re, const i64* tap_im, int n_taps, const i64* xr,
                   const i64* xi, i64 L, i64* yr, i64* yi) {
  const i64 c = n_taps / 2;
  for (i64 m = 0; m < L; ++m) {
    i64 ar = 0, ai = 0;
    for (int k = 0; k < n_taps; ++k) {
      i64 idx = m + c - k;
      if (idx < 0 || idx >= L) continue;
      ar += tap_re[k] * xr[idx] - tap_im[k] * xi[idx];
      ai += tap_re[k] * xi[idx] + tap_im[k] * xr[idx];
    }
    yr[m] = decode_signed(pmod(ar, F), F);
    yi[m] = decode_signed(pmod(ai, F), F);
  }
}

/* ------------------------------------------------------------------------ */
/* numpy pairwise summation (np.add.reduce over contiguous float64)           */

double or_pairwise_sum(const double* a, i64 n) {
  if (n < 8) {
    double r = 0.0;
    for (i64 i = 0; i < n; ++i) r += a[i];
    return r;
  } else if (n <= 128) {
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    i64 i;
    for (i = 8; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; ++j) r[j] += a[i + j];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += a[i];
    return res;
  } else {
    i64 n2 = n / 2;
    n2 -= n2 % 8;
    return or_pairwise_sum(a, n2) + or_pairwise_sum(a + n2, n - n2);
  }
}

/* ------------------------------------------------------------------------ */
/* FNT-AEQ (aeq.py:84-190) -- 4x4 real MIMO, N = 32 block, L = 16 taps       */

#define AEQ_L 16
#define AEQ_TAP_MAX 16383

typedef struct {
  double w[4][4][AEQ_L];
  i64 w_int[4][4][AEQ_L];
  i64 hist[4][AEQ_L];
  i64 saturations;
  i64 symbols;
  i64 n_err;
  double sig_scale, tap_scale, mu;
  double radii[8];
  int n_radii;
} or_aeq;

size_t or_aeq_size(void) { return sizeof(or_aeq); }

/* FntAeq.__init__ (aeq.py:87-104): centre spike round(tap_scale) at k = L/2. */
void or_aeq_init(or_aeq* q, double sig_scale, double tap_scale, double mu, const double* radii,
                 int n_radii) {
  memset(q, 0, sizeof(*q));
  q->sig_scale = sig_scale; q->tap_scale = tap_scale; q->mu = mu;
  q->n_radii = n_radii;
  for (int i = 0; i < n_radii; ++i) q->radii[i] = radii[i];
  i64 spike = (i64)nearbyint(tap_scale);
  for (int s = 0; s < 4; ++s) {
    q->w_int[s][s][AEQ_L / 2] = spike;
    q->w[s][s][AEQ_L / 2] = (double)spike / tap_scale;
  }
}

/* split_taps (fixedpoint.py:111-121): sign-magnitude 7-bit groups. */
static void split_tap(i64 w, i64* hi, i64* lo) {
  i64 sg = (w > 0) - (w < 0); i64 m = w < 0 ? -w : w;
  *hi = sg * (m >> 7); *lo = sg * (m & 127);
}

/* equalize_block (aeq.py:118-144): y_int via per-group residue convolution,
 * computed directly (the cyclic conv of a 16-tap filter over a 32-block has no
 * wrap in outputs 16..31), reduced mod F and decoded per group as the
 * reference does, then recombined 128*hi + lo and summed over input streams. */
static void aeq_forward(const or_aeq* q, const i64 xb[4][2 * AEQ_L], i64 y_int[4][AEQ_L]) {
  const i64 F = 65537;
  for (int s = 0; s < 4; ++s)
    for (int m = 0; m < AEQ_L; ++m) y_int[s][m] = 0;
  for (int s = 0; s < 4; ++s)
    for (int t = 0; t < 4; ++t) {
      i64 hi[AEQ_L], lo[AEQ_L];
      for (int k = 0; k < AEQ_L; ++k) split_tap(q->w_int[s][t][k], &hi[k], &lo[k]);
      for (int m = 0; m < AEQ_L; ++m) {
        i64 ah = 0, al = 0;
        for (int k = 0; k < AEQ_L; ++k) {
          i64 xv = xb[t][AEQ_L + m - k];
          ah += hi[k] * xv; al += lo[k] * xv;
        }
        y_int[s][m] += 128 * decode_signed(pmod(ah, F), F) + decode_signed(pmod(al, F), F);
      }
    }
}

/* rde_error (aeq.py:53-58) for one (yI, yQ) pair. */
static double rde1(double yi, double yq, const double* radii, int nr) {
  double a = yi * yi;
  double b = yq * yq;
  double r2 = a + b;
  double r = sqrt(r2);
  int best = 0; double bd = fabs(r - radii[0]);
  for (int i = 1; i < nr; ++i) { double d = fabs(r - radii[i]); if (d < bd) { bd = d; best = i; } }
  double R = radii[best];
  return R * R - r2;
}

/* einsum("sm,tmk->stk") reduction over m = 0..15 in numpy's SSE2 order
 * (two lanes = even/odd m, unrolled by 4). */
static double einsum_m(const double P[AEQ_L]) {
  double c[2];
  for (int L = 0; L < 2; ++L) {
    double v = P[L + 6];
    v = P[L + 4] + v; v = P[L + 2] + v; v = P[L + 0] + v;
    v = P[L + 14] + v; v = P[L + 12] + v; v = P[L + 10] + v; v = P[L + 8] + v;
    c[L] = v;
  }
  return c[0] + c[1];
}

/* update_taps (aeq.py:148-170). */
static void aeq_update(or_aeq* q, const i64 xb[4][2 * AEQ_L], double y[4][AEQ_L], double mu,
                       double* err_out) {
  double xf[4][2 * AEQ_L];
  for (int t = 0; t < 4; ++t)
    for (int j = 0; j < 2 * AEQ_L; ++j) xf[t][j] = (double)xb[t][j] / q->sig_scale;
  double e[2][AEQ_L];
  for (int p = 0; p < 2; ++p)
    for (int m = 0; m < AEQ_L; ++m) e[p][m] = rde1(y[2 * p][m], y[2 * p + 1][m], q->radii, q->n_radii);
  double ab[2 * AEQ_L];
  for (int p = 0; p < 2; ++p)
    for (int m = 0; m < AEQ_L; ++m) ab[p * AEQ_L + m] = fabs(e[p][m]);
  *err_out = or_pairwise_sum(ab, 2 * AEQ_L) / (double)(2 * AEQ_L);
  q->n_err++;
  if (mu == 0.0) return;
  double ey[4][AEQ_L];
  for (int s = 0; s < 4; ++s)
    for (int m = 0; m < AEQ_L; ++m) ey[s][m] = e[s >> 1][m] * y[s][m];
  for (int s = 0; s < 4; ++s)
    for (int t = 0; t < 4; ++t)
      for (int k = 0; k < AEQ_L; ++k) {
        double P[AEQ_L];
        for (int m = 0; m < AEQ_L; ++m) P[m] = ey[s][m] * xf[t][AEQ_L + m - k];
        double g = einsum_m(P);
        double step = mu * g;
        q->w[s][t][k] = q->w[s][t][k] + step;
        double r = nearbyint(q->w[s][t][k] * q->tap_scale);
        i64 wi;
        if (!(fabs(r) < 9223372036854775808.0)) {
          /* numpy: rint of NaN / |r| >= 2^63 casts to INT64_MIN (x86-64), whose abs is
           * still negative, so it is not counted, and clip gives -16383 (aeq.py:165-168) */
          wi = -AEQ_TAP_MAX;
        } else {
          wi = (i64)r;
          if ((wi < 0 ? -wi : wi) > AEQ_TAP_MAX) {
            q->saturations++;
            wi = wi < 0 ? -AEQ_TAP_MAX : AEQ_TAP_MAX;
          }
        }
        q->w_int[s][t][k] = wi;
      }
}

/* equalize_block alone: x_new (4,16) -> y (4,16), x_block (4,32). */
void or_aeq_equalize_block(or_aeq* q, const i64* x_new, double* y_out, i64* xblk_out) {
  i64 xb[4][2 * AEQ_L];
  for (int t = 0; t < 4; ++t)
    for (int j = 0; j < AEQ_L; ++j) { xb[t][j] = q->hist[t][j]; xb[t][AEQ_L + j] = x_new[t * AEQ_L + j]; }
  for (int t = 0; t < 4; ++t)
    for (int j = 0; j < AEQ_L; ++j) q->hist[t][j] = xb[t][AEQ_L + j];
  i64 y_int[4][AEQ_L];
  aeq_forward(q, (const i64(*)[2 * AEQ_L])xb, y_int);
  const double D = q->sig_scale * q->tap_scale;
  for (int s = 0; s < 4; ++s)
    for (int m = 0; m < AEQ_L; ++m) y_out[s * AEQ_L + m] = (double)y_int[s][m] / D;
  memcpy(xblk_out, xb, sizeof(xb));
  q->symbols += AEQ_L;
}

void or_aeq_update_taps(or_aeq* q, const i64* xblk, const double* y, double mu, double* err_out) {
  double yy[4][AEQ_L];
  memcpy(yy, y, sizeof(yy));
  aeq_update(q, (const i64(*)[2 * AEQ_L])xblk, yy, mu, err_out);
}

/* process (aeq.py:172-190). x is (4, n) row-major with row stride ld.
 * mu_blocks[b] = step size of block b (NULL -> q->mu). Writes y (4, n_blocks*16)
 * row-major with row stride ldy and one err value per adapted block. Returns
 * the number of blocks processed. */
i64 or_aeq_process(or_aeq* q, const i64* x, i64 n, i64 ld, int adapt, const double* mu_blocks,
                   double* y, i64 ldy, double* err) {
  i64 nb = n / AEQ_L;
  for (i64 b = 0; b < nb; ++b) {
    i64 xn[4 * AEQ_L];
    for (int t = 0; t < 4; ++t)
      for (int j = 0; j < AEQ_L; ++j) xn[t * AEQ_L + j] = x[t * ld + b * AEQ_L + j];
    double yb[4 * AEQ_L]; i64 xblk[4 * 2 * AEQ_L];
    or_aeq_equalize_block(q, xn, yb, xblk);
    for (int s = 0; s < 4; ++s)
      for (int m = 0; m < AEQ_L; ++m) y[s * ldy + b * AEQ_L + m] = yb[s * AEQ_L + m];
    if (adapt) {
      double mu = mu_blocks ? mu_blocks[b] : q->mu;
      or_aeq_update_taps(q, xblk, yb, mu, err ? &err[b] : &(double){0});
    }
  }
  return nb;
}

/* ------------------------------------------------------------------------ */
/* CDC -> AEQ glue (linksim.py:249-260, 306-308, 399-404; cdc.py:177-180)     */

/* _decimation_phase over n_streams complex streams (interleaved re,im). */
int or_decimation_phase(const double* const* streams, const i64* lens, int n_streams, int sps) {
  double best = 0.0; int best_phase = 0; int have = 0;
  for (int ph = 0; ph < sps; ++ph) {
    double metric = 0.0;
    for (int s = 0; s < n_streams; ++s) {
      i64 L = lens[s]; i64 m = (L - ph + sps - 1) / sps;
      if (m <= 0) continue;
      double* a2 = malloc(sizeof(double) * m);
      double* a4 = malloc(sizeof(double) * m);
      for (i64 i = 0; i < m; ++i) {
        double re = streams[s][2 * (ph + i * sps)], im = streams[s][2 * (ph + i * sps) + 1];
        double a = hypot(re, im);
        a2[i] = a * a;
        a4[i] = pow(a, 4.0);
      }
      double p2 = or_pairwise_sum(a2, m) / (double)m;
      double p4 = or_pairwise_sum(a4, m) / (double)m;
      metric += p4 / (p2 * p2);
      free(a2); free(a4);
    }
    if (!have || metric < best) { best = metric; best_phase = ph; have = 1; }
  }
  return best_phase;
}
