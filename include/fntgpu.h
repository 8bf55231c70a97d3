/*
 * fntgpu.h -- C ABI of libfntgpu.so, the B200 (sm_100a) implementation of the
 * integer FNT receiver-DSP hot path of arXiv 2405.04253 (reference: the `fntdsp`
 * package, /root/reference/pkg/src/fntdsp).
 *
 * Every entry point replaces one reference interface; the comment above each
 * declaration cites it (file:line in fntdsp). Conventions:
 *   - plain C types only; all data pointers are DEVICE pointers owned by the
 *     caller; `stream` is a cudaStream_t passed as void* (NULL = legacy stream);
 *   - no allocation inside the compute calls (only plan_create allocates);
 *   - return 0 on success, < 0 on error, with fntgpu_last_error() describing it
 *     (thread-local). Argument errors are reported before anything is launched;
 *   - there is no CPU fallback: a missing/unsupported GPU is an error.
 */
#ifndef FNTGPU_H
#define FNTGPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FNTGPU_ABI_VERSION 1

/* return codes */
#define FNTGPU_OK 0
#define FNTGPU_EINVAL (-1)       /* bad argument (ValueError in the reference) */
#define FNTGPU_ECUDA (-2)        /* CUDA runtime / launch error */
#define FNTGPU_EUNSUPPORTED (-3) /* valid for the reference, not implemented on the GPU */
/* InvalidPlanError reasons (fnt.py:63-72) */
#define FNTGPU_EPLAN_LENGTH (-10) /* length must be a power of two >= 2 */
#define FNTGPU_EPLAN_RADIX (-11)  /* radix is not a canonical nonzero residue */
#define FNTGPU_EPLAN_ORDER (-12)  /* alpha^n != 1 (mod F) */
#define FNTGPU_EPLAN_SUBORD (-13) /* alpha^(n/2) != -1 (mod F): order < n */
#define FNTGPU_EPLAN_MODULUS (-14) /* t not in {0..4} (fermat.py:18-44) */

/* element types */
#define FNTGPU_NONE 0
#define FNTGPU_I8 1
#define FNTGPU_I16 2
#define FNTGPU_I32 3
#define FNTGPU_I64 4
#define FNTGPU_F64 5
#define FNTGPU_C128 6 /* interleaved (re, im) float64 == numpy complex128 */

/* flags */
#define FNTGPU_DECODE_SIGNED 1 /* decode residues r > (F-1)/2 to r - F (fermat.py:131-133) */

int fntgpu_abi_version(void);
const char* fntgpu_last_error(void);
/* number of visible CUDA devices (0 -> every compute call fails) */
int fntgpu_device_count(void);
/* Plumbing for the host-buffer (end-to-end) path: a strided 2-D copy of `height`
 * rows of `width` bytes (row pitches in bytes) between host and device memory,
 * asynchronous on `stream` (cudaMemcpy2DAsync with cudaMemcpyDefault). Lets a
 * time segment of the (links, 4, n) float64 equalizer output stream back while
 * the next segment is computed. */
int fntgpu_copy2d_async(void* dst, int64_t dpitch, const void* src, int64_t spitch,
                        int64_t width, int64_t height, void* stream);

/* ------------------------------------------------------------------------ */
/* Transform plans -- TransformPlan / make_plan (fnt.py:24-33, 60-83).        */
/* Validates that alpha has order exactly n modulo F = 2^(2^t) + 1 and         */
/* uploads the per-stage twiddle tables. The two shipped shift-add plans       */
/* (aeq32: t=4, alpha=2, n=32; cdc64: t=4, alpha=4080, n=64) run register-     */
/* resident shift/rotate kernels; any other valid plan runs a shared-memory    */
/* kernel with general products.                                               */
typedef struct fntgpu_plan fntgpu_plan;

int fntgpu_plan_create(int t, int n, int64_t alpha, fntgpu_plan** out);
int fntgpu_plan_destroy(fntgpu_plan* plan);
/* Replace the twiddle tables (host int64, stage-concatenated, n-1 entries each,
 * in the layout of TransformPlan.fwd_twiddles / inv_twiddles). Non-canonical
 * tables (e.g. the CLI selftest --fault-inject negative control, cli.py:84-86)
 * switch the plan to the table-driven kernel so the corruption is observed. */
int fntgpu_plan_set_twiddles(fntgpu_plan* plan, const int64_t* fwd, const int64_t* inv);
/* alpha^-1, n^-1 (fnt.py:73-80) and the kernel kind (0 generic, 1 aeq32, 2 cdc64) */
int fntgpu_plan_info(const fntgpu_plan* plan, int64_t* alpha_inv, int64_t* n_inv, int* kind);

/* fnt / ifnt (fnt.py:106-114): batch vectors of length n, any int64 input
 * (reduced mod F as the reference does implicitly), canonical residues out
 * (or signed with FNTGPU_DECODE_SIGNED). x and y may alias. */
int fntgpu_fnt(const fntgpu_plan* plan, int inverse, const int64_t* x, int64_t* y, int64_t batch,
               int flags, void* stream);

/* cyclic_convolve_real (fnt.py:117-125). h_stride = 0 broadcasts one tap
 * vector over the batch, = n gives per-vector taps. */
int fntgpu_cyclic_convolve_real(const fntgpu_plan* plan, const int64_t* x, const int64_t* h,
                                int64_t h_stride, int64_t* z, int64_t batch, int flags,
                                void* stream);

/* cyclic_convolve_complex (fnt.py:128-161, Eqs. 7-8): two general products per bin. */
int fntgpu_cyclic_convolve_complex(const fntgpu_plan* plan, const int64_t* x_re,
                                   const int64_t* x_im, const int64_t* y_re, const int64_t* y_im,
                                   int64_t y_stride, int64_t* z_re, int64_t* z_im, int64_t batch,
                                   int flags, void* stream);

/* encode_signed_array / decode_signed_array (fermat.py:124-133) elementwise on
 * int64: decode = 0 maps v < 0 to v + F (the caller checks |v| <= (F-1)/2 first,
 * as the reference does), decode = 1 maps r > (F-1)/2 to r - F. */
int fntgpu_residue_map(int t, int decode, const int64_t* in, int64_t* out, int64_t n, void* stream);

/* sizeof() of the ABI structs in declaration order (cdc_taps, cdc_io, decim_io,
 * aeq_params, aeq_state, aeq_io, td_aeq_io) so bindings can verify their layouts.
 * Returns 7. */
int fntgpu_struct_sizes(int64_t* out, int n);

/* ------------------------------------------------------------------------ */
/* quantize_real (fixedpoint.py:51-60): q = sign(v)*floor(|v|+0.5), v = x*scale,
 * clipped to +-max_int; *clipped (device counter) += #(|q| > max_int).
 * out_dtype: FNTGPU_I8 | FNTGPU_I32 | FNTGPU_I64. */
int fntgpu_quantize_real(const double* x, int64_t n, double scale, int32_t max_int, int out_dtype,
                         void* q, unsigned long long* clipped, void* stream);

/* ------------------------------------------------------------------------ */
/* FNT-CDC -- FntCdcEngine (cdc.py:98-180) on the cdc64 plan.                  */
typedef struct fntgpu_cdc_taps {
  uint32_t b_plus[64];  /* (H_r + 2^8 H_i) mod F  (cdc.py:124-135, _b_plus) */
  uint32_t b_minus[64]; /* (H_r - 2^8 H_i) mod F  (_b_minus) */
  int32_t n_taps;       /* output alignment c = n_taps // 2 (cdc.py:174) */
  int32_t kernel;       /* FNTGPU_CDC_KERNEL_*: 0 auto (the measured-faster kernel:
                         * tcgen05 form for int8 planes with int16 / int8-requantized /
                         * statistics outputs, shift-add otherwise), 1 shift-add FNT
                         * kernel, 2 tensor-core split-integer matrix form on mma.sync,
                         * 3 the same on tcgen05 (int8 planes; other dtypes run the
                         * shift-add kernel) */
} fntgpu_cdc_taps;
#define FNTGPU_CDC_KERNEL_AUTO 0
#define FNTGPU_CDC_KERNEL_SHIFT 1
#define FNTGPU_CDC_KERNEL_TC 2
#define FNTGPU_CDC_KERNEL_UMMA 3

typedef struct fntgpu_cdc_io {
  int32_t n_streams;          /* independent streams (polarizations / channels) */
  int32_t in_dtype;           /* FNTGPU_I8 | FNTGPU_I32 | FNTGPU_I64 | FNTGPU_F64 (quantized on load) */
  const void* xr;             /* stream s real part at xr + s * x_stride (elements) */
  const void* xi;
  int64_t x_stride;
  int64_t x_first;            /* global sample index held at xr[0] (range shards) */
  int64_t x_count;            /* samples present: global [x_first, x_first + x_count) */
  int64_t length;             /* stream length L; samples outside [0, L) are zero (cdc.py:89-95) */
  int64_t out_first;          /* global output range [out_first, out_first + out_count) */
  int64_t out_count;
  int32_t out_dtype;          /* FNTGPU_NONE | I16 | I32 | I64 (process_int) | C128 (process) */
  int32_t pad0;
  void* yr;                   /* stream s output at yr + s * y_stride; y[0] <-> out_first */
  void* yi;                   /* unused for C128 (yr holds interleaved complex) */
  int64_t y_stride;
  double inv_scale;           /* C128: y = y_int * (1.0 / output_scale)  (cdc.py:180) */
  /* optional fused AEQ-input requantization (linksim.py:283-308, 399-404):
   * q = clip(round_half_away((y_int * inv_scale) * q_scale), +-q_max) as int8 */
  int8_t* qr;
  int8_t* qi;
  int64_t q_stride;
  double q_scale;
  int32_t q_max;
  int32_t pad1;
  /* optional fused decimation-phase statistics (linksim.py:249-260): per
   * stream s and phase p = (global index & 1): acc[(s*2+p)*4 + 0] += sum |y|^2,
   * acc[... + 1..3] += 32-bit limbs of sum |y|^4 (exact integer sums). */
  unsigned long long* decim_acc;
  /* optional exact integer form of the requantization, valid when
   * q_scale * inv_scale == 2^-q_shift up to rounding (q_scale = the engine's
   * signal scale, tap scale 2^q_shift, cdc.py:80-86): q = round_half_away(y / 2^k)
   * except for exact ties |y| = 2^(k-1) + j 2^k, whose float64 results the caller
   * precomputes in q_tie[j] (j <= q_max). q_shift = -1 selects the float64 path. */
  int32_t q_shift;
  int32_t pad2;
  int8_t q_tie[128];
  /* float64 input (in_dtype FNTGPU_F64): the front-end samples are quantized on
   * load, q = clip(sign(v) floor(|v| + 0.5), +-in_max) with v = x * in_scale
   * (quantize_real, fixedpoint.py:51-60, as linksim.py:290-291 applies it before
   * process_int); in_max <= 127. *in_clipped (device counter, optional) += the
   * number of |q| > in_max among the samples [32 b_lo, 32 (b_hi + 1)) of the
   * launched overlap-save blocks, within [0, length) and the given input window --
   * the whole stream once for a full-range call (cdc.py:165-175). */
  double in_scale;
  int32_t in_max;
  int32_t pad3;
  unsigned long long* in_clipped;
} fntgpu_cdc_io;

/* process_int / process (cdc.py:165-180), any output sub-range of any number
 * of streams in one launch. Output is bit-exact with the reference for every
 * input accepted by encode_signed_array (|x| <= 32768). */
int fntgpu_cdc64_process(const fntgpu_cdc_taps* taps, const fntgpu_cdc_io* io, void* stream);

/* _decimation_phase (linksim.py:249-260) from the fused statistics: link l
 * owns CDC streams 2l (pol X) and 2l+1 (pol Y). */
typedef struct fntgpu_decim_io {
  int32_t n_links;
  int32_t sps;                /* must be 2 */
  const unsigned long long* acc;
  int64_t length;             /* per-stream length L */
  int32_t* phase;             /* out: chosen phase per link */
  double* gap;                /* out (optional): |m0 - m1| / max(m0, m1) tie guard */
} fntgpu_decim_io;
int fntgpu_decim_phase(const fntgpu_decim_io* io, void* stream);

/* ------------------------------------------------------------------------ */
/* FNT-AEQ -- FntAeq (aeq.py:84-190): 4x4 real MIMO, 32-point FNT blocks,   */
/* 16 taps, float64 radius-directed block update, one state per stream.     */
#define FNTGPU_AEQ_FWD_FNT 0    /* forward path in the FNT domain (aeq.py:134-141) */
#define FNTGPU_AEQ_FWD_DIRECT 1 /* exact time-domain integer MIMO FIR, same bits */

typedef struct fntgpu_aeq_params {
  double sig_scale;   /* AeqConfig.sig_spec.scale (aeq.py:42) */
  double tap_scale;   /* AeqConfig.tap_scale (aeq.py:43) */
  double mu;          /* AeqConfig.mu, used when mu_blocks == NULL */
  double radii[8];    /* sorted ring radii (aeq.py:50) */
  int32_t n_radii;    /* 1..8 */
  int32_t forward;    /* FNTGPU_AEQ_FWD_* */
  int32_t kernel;     /* FNTGPU_AEQ_KERNEL_*: stream layout of fntgpu_aeq_process */
  int32_t reserved;
} fntgpu_aeq_params;
/* Stream layout of the FNT-forward equalizer (same bits either way):
 * AUTO  the polarization-split form when there are too few streams to fill the
 *       GPU with one warp each (fewer than ~8 per SM), else one warp per stream;
 * WARP  one warp per stream (k_aeq.cu), the throughput form;
 * POL   two warps per stream, one per polarization's output pair (k_aeq_pol.cu),
 *       the latency form. The DIRECT forward always runs one warp per stream. */
#define FNTGPU_AEQ_KERNEL_AUTO 0
#define FNTGPU_AEQ_KERNEL_WARP 1
#define FNTGPU_AEQ_KERNEL_POL 2

typedef struct fntgpu_aeq_state { /* device memory, one per stream */
  double w[4][4][16];             /* float taps (aeq.py:99) */
  int32_t w_int[4][4][16];        /* 14-bit taps (aeq.py:98, RvMimoTaps.w_int) */
  int32_t hist[4][16];            /* overlap history (aeq.py:100) */
  int64_t saturations;            /* aeq.py:102 */
  int64_t symbols;                /* symbols_processed (aeq.py:103) */
  int64_t n_err;                  /* len(err_trace) */
  int64_t reserved;
} fntgpu_aeq_state;

#define FNTGPU_AEQ_IN_PLANAR 0 /* x: (4, n) rows of in_dtype per stream */
#define FNTGPU_AEQ_IN_DECIM 1  /* int8 requantized CDC planes (fntgpu_cdc_io.qr/qi) */

typedef struct fntgpu_aeq_io {
  int32_t n_streams;
  int32_t in_mode;            /* FNTGPU_AEQ_IN_* */
  int32_t in_dtype;           /* planar: FNTGPU_I8 | I32 | I64 */
  int32_t adapt;              /* process(adapt=...) (aeq.py:172) */
  const void* x;              /* planar: row r of stream s at x + s*x_stream_stride + r*x_row_stride */
  int64_t x_stream_stride;
  int64_t x_row_stride;
  /* decim mode: stream s rows = [qr[2s], qi[2s], qr[2s+1], qi[2s+1]] sampled at phase[s] + 2 i,
   * plane p at q + p * q_stride (linksim.py:306-308, 399) */
  const int8_t* qr;
  const int8_t* qi;
  int64_t q_stride;
  const int32_t* phase;
  int64_t n_blocks;           /* 16-symbol blocks to run (trailing remainder dropped, aeq.py:182) */
  const double* mu_blocks;    /* step size of each block (mu_schedule(16 b)) or NULL -> params.mu */
  double* y;                  /* out: (4, 16*n_blocks) per stream */
  int64_t y_stream_stride;
  int64_t y_row_stride;
  double* err;                /* out (adapt): err_trace entries, one per block */
  int64_t err_stream_stride;
} fntgpu_aeq_io;

/* FntAeq.__init__ (aeq.py:87-104): centre-spike taps, zero history. */
int fntgpu_aeq_init(fntgpu_aeq_state* state, int n_streams, const fntgpu_aeq_params* params,
                    void* stream);
/* FntAeq.process (aeq.py:172-190) for n_streams independent streams. */
int fntgpu_aeq_process(fntgpu_aeq_state* state, const fntgpu_aeq_params* params,
                       const fntgpu_aeq_io* io, void* stream);
/* FntAeq.update_taps (aeq.py:148-170) for one stream with caller-given
 * x_block (4, 32) int64 and y (4, 16) float64; *err receives the err_trace entry. */
int fntgpu_aeq_update_taps(fntgpu_aeq_state* state, const fntgpu_aeq_params* params,
                           const int64_t* x_block, const double* y, double mu, double* err,
                           void* stream);
/* ------------------------------------------------------------------------ */
/* Float per-symbol 4x4 RDE comparator -- td_aeq_float / _td_rde_kernel      */
/* (aeq.py:193-249); not on the FNT path. 16 taps per filter.                 */
typedef struct fntgpu_td_aeq_io {
  int32_t n_streams;
  int32_t n_radii;            /* 1..8, sorted (aeq.py:50) */
  int64_t n;                  /* symbols per stream */
  const double* x;            /* stream s, input row r at x + s * x_stream_stride + r * x_row_stride */
  int64_t x_stream_stride;
  int64_t x_row_stride;
  double* w;                  /* (n_streams, 4, 4, 16) float64 taps, updated in place */
  const double* mu;           /* (n,) step size of every symbol (mu_schedule(m)) */
  double radii[8];
  double* y;                  /* (n_streams, 4, >= n) float64 outputs */
  int64_t y_stream_stride;
  int64_t y_row_stride;
} fntgpu_td_aeq_io;

int fntgpu_td_aeq(const fntgpu_td_aeq_io* io, void* stream);

/* Self-check of the AEQ kernel's two arithmetic shortcuts for these params (no
 * reference counterpart; used by the tests and the CLI selftest): over every int32
 * numerator in [lo, hi), y = y_int / D by reciprocal + one correction step against
 * IEEE division, and for r2 = y^2 + y'^2 on a dense sweep the threshold ring decision
 * against sqrt + first argmin. mismatches: device uint64[2] {division, ring},
 * accumulated (caller zeroes). */
int fntgpu_aeq_selfcheck(const fntgpu_aeq_params* params, int64_t lo, int64_t hi,
                         unsigned long long* mismatches, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* FNTGPU_H */
