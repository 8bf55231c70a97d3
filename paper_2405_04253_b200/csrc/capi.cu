// capi.cu -- extern "C" entry points of libfntgpu.so (declared in include/fntgpu.h).
//
// Argument validation mirrors the reference's error behaviour (fnt.py:63-72
// InvalidPlanError, fnt.py:91 length errors are raised by the Python shim before
// calling in). Errors are reported through return codes + fntgpu_last_error().
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <new>
#include <vector>

#include "internal.h"

namespace fntgpu {
cudaError_t launch_aeq_update_once(fntgpu_aeq_state* st, const fntgpu_aeq_params& prm,
                                   const int64_t* xblk, const double* y, double mu, double* err,
                                   cudaStream_t s);
cudaError_t launch_aeq_selfcheck(const fntgpu_aeq_params& prm, int64_t lo, int64_t hi,
                                 unsigned long long* mismatches, cudaStream_t s);
cudaError_t launch_td_aeq(const fntgpu_td_aeq_io& io, cudaStream_t s);
}

using namespace fntgpu;

static thread_local char g_err[512] = "";

static int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

static int cuda_rc(cudaError_t e, const char* where) {
  if (e == cudaSuccess) return FNTGPU_OK;
  return fail(FNTGPU_ECUDA, "%s: %s", where, cudaGetErrorString(e));
}

static int check_device(const char* where) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0)
    return fail(FNTGPU_ECUDA, "%s: no CUDA device available (%s); there is no CPU fallback", where,
                e == cudaSuccess ? "0 devices" : cudaGetErrorString(e));
  return FNTGPU_OK;
}

static inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

struct fntgpu_plan {
  DevPlan dev;
  int64_t alpha, alpha_inv, n_inv;
  uint32_t* d_tw;  // fwd (n-1) then inv (n-1)
  std::vector<uint32_t> canon;  // canonical tables (host copy)
  int fast_kind;
};

static uint64_t powmod(uint64_t a, uint64_t e, uint64_t m) {
  uint64_t r = 1 % m;
  a %= m;
  while (e) {
    if (e & 1) r = r * a % m;
    a = a * a % m;
    e >>= 1;
  }
  return r;
}

extern "C" {

int fntgpu_abi_version(void) { return FNTGPU_ABI_VERSION; }

const char* fntgpu_last_error(void) { return g_err; }

int fntgpu_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

int fntgpu_copy2d_async(void* dst, int64_t dpitch, const void* src, int64_t spitch,
                        int64_t width, int64_t height, void* stream) {
  if (!dst || !src) return fail(FNTGPU_EINVAL, "copy2d_async: NULL argument");
  if (width < 0 || height < 0 || dpitch < width || spitch < width)
    return fail(FNTGPU_EINVAL, "copy2d_async: bad extent");
  if (width == 0 || height == 0) return FNTGPU_OK;
  return cuda_rc(cudaMemcpy2DAsync(dst, (size_t)dpitch, src, (size_t)spitch, (size_t)width,
                                   (size_t)height, cudaMemcpyDefault, S(stream)),
                 "copy2d_async");
}

int fntgpu_plan_create(int t, int n, int64_t alpha, fntgpu_plan** out) {
  if (!out) return fail(FNTGPU_EINVAL, "plan_create: out is NULL");
  *out = nullptr;
  if (t < 0 || t > 4) return fail(FNTGPU_EPLAN_MODULUS, "t must be in (0, 1, 2, 3, 4), got %d", t);
  const uint64_t F = (1ull << (1 << t)) + 1;
  if (n < 2 || (n & (n - 1)))
    return fail(FNTGPU_EPLAN_LENGTH, "length must be a power of two >= 2, got %d", n);
  if (!(alpha > 0 && (uint64_t)alpha < F))
    return fail(FNTGPU_EPLAN_RADIX, "radix %lld is not a canonical nonzero residue", (long long)alpha);
  if (powmod((uint64_t)alpha, (uint64_t)n, F) != 1)
    return fail(FNTGPU_EPLAN_ORDER, "radix %lld does not satisfy alpha^%d = 1 (mod %llu)",
                (long long)alpha, n, (unsigned long long)F);
  if (powmod((uint64_t)alpha, (uint64_t)(n / 2), F) != F - 1)
    return fail(FNTGPU_EPLAN_SUBORD, "radix %lld has order < %d mod %llu (alpha^%d != -1)",
                (long long)alpha, n, (unsigned long long)F, n / 2);
  int rc = check_device("plan_create");
  if (rc) return rc;
  fntgpu_plan* p = new (std::nothrow) fntgpu_plan();
  if (!p) return fail(FNTGPU_EINVAL, "plan_create: out of host memory");
  p->alpha = alpha;
  p->alpha_inv = (int64_t)powmod((uint64_t)alpha, F - 2, F);
  p->n_inv = (int64_t)powmod((uint64_t)n, F - 2, F);
  int lg = 0;
  while ((1 << lg) < n) ++lg;
  p->dev.t = t;
  p->dev.n = n;
  p->dev.lg = lg;
  p->dev.F = (uint32_t)F;
  p->dev.n_inv = (uint32_t)p->n_inv;
  p->dev.kind = KIND_GENERIC;
  if (t == 4 && n == 32 && alpha == 2) p->dev.kind = KIND_RADIX2_32;
  if (t == 4 && n == 64 && alpha == 4080) p->dev.kind = KIND_SQRT2_64;
  // stage twiddles root^(j * n / 2^(s+1)), j < 2^s (fnt.py:_stage_twiddles)
  uint32_t* h = new uint32_t[2 * (n - 1)];
  for (int s = 0; s < lg; ++s) {
    const int half = 1 << s, step = n >> (s + 1);
    for (int j = 0; j < half; ++j) {
      h[half - 1 + j] = (uint32_t)powmod((uint64_t)alpha, (uint64_t)j * step, F);
      h[(n - 1) + half - 1 + j] = (uint32_t)powmod((uint64_t)p->alpha_inv, (uint64_t)j * step, F);
    }
  }
  p->canon.assign(h, h + 2 * (n - 1));
  p->fast_kind = p->dev.kind;
  cudaError_t e = cudaMalloc(&p->d_tw, sizeof(uint32_t) * 2 * (n - 1));
  if (e == cudaSuccess) e = cudaMemcpy(p->d_tw, h, sizeof(uint32_t) * 2 * (n - 1), cudaMemcpyHostToDevice);
  delete[] h;
  if (e != cudaSuccess) {
    delete p;
    return cuda_rc(e, "plan_create");
  }
  p->dev.tw_fwd = p->d_tw;
  p->dev.tw_inv = p->d_tw + (n - 1);
  *out = p;
  return FNTGPU_OK;
}

int fntgpu_plan_set_twiddles(fntgpu_plan* p, const int64_t* fwd, const int64_t* inv) {
  if (!p || !fwd || !inv) return fail(FNTGPU_EINVAL, "plan_set_twiddles: NULL argument");
  const int n = p->dev.n;
  uint32_t* h = new uint32_t[2 * (n - 1)];
  bool canonical = true;
  std::vector<uint32_t> ref(2 * (n - 1));
  cudaError_t e = cudaMemcpy(ref.data(), p->d_tw, sizeof(uint32_t) * 2 * (n - 1), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) { delete[] h; return cuda_rc(e, "plan_set_twiddles"); }
  for (int i = 0; i < n - 1; ++i) {
    // tables are used modulo F exactly like numpy's (a * tw) % F
    const int64_t F = (int64_t)p->dev.F;
    int64_t a = fwd[i] % F, b = inv[i] % F;
    h[i] = (uint32_t)(a < 0 ? a + F : a);
    h[(n - 1) + i] = (uint32_t)(b < 0 ? b + F : b);
    if (h[i] != p->canon[i] || h[(n - 1) + i] != p->canon[(n - 1) + i]) canonical = false;
  }
  e = cudaMemcpy(p->d_tw, h, sizeof(uint32_t) * 2 * (n - 1), cudaMemcpyHostToDevice);
  delete[] h;
  if (e != cudaSuccess) return cuda_rc(e, "plan_set_twiddles");
  // the register kernels hard-code the canonical shift twiddles
  p->dev.kind = canonical ? p->fast_kind : KIND_GENERIC;
  return FNTGPU_OK;
}

int fntgpu_plan_destroy(fntgpu_plan* p) {
  if (!p) return FNTGPU_OK;
  cudaFree(p->d_tw);
  delete p;
  return FNTGPU_OK;
}

int fntgpu_plan_info(const fntgpu_plan* p, int64_t* alpha_inv, int64_t* n_inv, int* kind) {
  if (!p) return fail(FNTGPU_EINVAL, "plan_info: NULL plan");
  if (alpha_inv) *alpha_inv = p->alpha_inv;
  if (n_inv) *n_inv = p->n_inv;
  if (kind) *kind = p->dev.kind;
  return FNTGPU_OK;
}

static int check_generic_size(const fntgpu_plan* p, int arrays, const char* where) {
  if (p->dev.kind != KIND_GENERIC) return FNTGPU_OK;
  const size_t per = p->dev.n >= 1024 ? 1 : 1024 / p->dev.n;
  const size_t bytes = (size_t)arrays * per * p->dev.n * sizeof(uint32_t);
  if (bytes > 200 * 1024)
    return fail(FNTGPU_EUNSUPPORTED, "%s: generic plan length %d too large for the shared-memory kernel",
                where, p->dev.n);
  return FNTGPU_OK;
}

int fntgpu_fnt(const fntgpu_plan* p, int inverse, const int64_t* x, int64_t* y, int64_t batch,
               int flags, void* stream) {
  if (!p || (!x && batch) || (!y && batch) || batch < 0) return fail(FNTGPU_EINVAL, "fnt: bad arguments");
  int rc = check_generic_size(p, 1, "fnt");
  if (rc) return rc;
  if ((rc = check_device("fnt"))) return rc;
  return cuda_rc(launch_fnt(p->dev, inverse, x, y, batch, flags, S(stream)), "fnt");
}

int fntgpu_cyclic_convolve_real(const fntgpu_plan* p, const int64_t* x, const int64_t* h,
                                int64_t h_stride, int64_t* z, int64_t batch, int flags,
                                void* stream) {
  if (!p || batch < 0 || (batch && (!x || !h || !z)) || (h_stride != 0 && h_stride != p->dev.n))
    return fail(FNTGPU_EINVAL, "cyclic_convolve_real: bad arguments");
  int rc = check_generic_size(p, 2, "cyclic_convolve_real");
  if (rc) return rc;
  if ((rc = check_device("cyclic_convolve_real"))) return rc;
  return cuda_rc(launch_conv_real(p->dev, x, h, h_stride, z, batch, flags, S(stream)),
                 "cyclic_convolve_real");
}

int fntgpu_cyclic_convolve_complex(const fntgpu_plan* p, const int64_t* xr, const int64_t* xi,
                                   const int64_t* yr, const int64_t* yi, int64_t y_stride,
                                   int64_t* zr, int64_t* zi, int64_t batch, int flags,
                                   void* stream) {
  if (!p || batch < 0 || (batch && (!xr || !xi || !yr || !yi || !zr || !zi)) ||
      (y_stride != 0 && y_stride != p->dev.n))
    return fail(FNTGPU_EINVAL, "cyclic_convolve_complex: bad arguments");
  if ((1 << p->dev.t) < 2)
    return fail(FNTGPU_EINVAL, "complex decomposition needs b >= 2, got b=%d", 1 << p->dev.t);
  int rc = check_generic_size(p, 4, "cyclic_convolve_complex");
  if (rc) return rc;
  if ((rc = check_device("cyclic_convolve_complex"))) return rc;
  return cuda_rc(launch_conv_complex(p->dev, xr, xi, yr, yi, y_stride, zr, zi, batch, flags,
                                     S(stream)),
                 "cyclic_convolve_complex");
}

int fntgpu_quantize_real(const double* x, int64_t n, double scale, int32_t max_int, int out_dtype,
                         void* q, unsigned long long* clipped, void* stream) {
  if (n < 0 || (n && (!x || !q)) || max_int < 1 ||
      (out_dtype != FNTGPU_I8 && out_dtype != FNTGPU_I32 && out_dtype != FNTGPU_I64))
    return fail(FNTGPU_EINVAL, "quantize_real: bad arguments");
  if (out_dtype == FNTGPU_I8 && max_int > 127)
    return fail(FNTGPU_EINVAL, "quantize_real: max_int %d does not fit int8", max_int);
  if (!(scale > 0)) return fail(FNTGPU_EINVAL, "scale must be positive");
  int rc = check_device("quantize_real");
  if (rc) return rc;
  return cuda_rc(launch_quantize(x, n, scale, max_int, out_dtype, q, clipped, S(stream)),
                 "quantize_real");
}

int fntgpu_residue_map(int t, int decode, const int64_t* in, int64_t* out, int64_t n, void* stream) {
  if (t < 0 || t > 4) return fail(FNTGPU_EPLAN_MODULUS, "t must be in (0, 1, 2, 3, 4), got %d", t);
  if (n < 0 || (n && (!in || !out))) return fail(FNTGPU_EINVAL, "residue_map: bad arguments");
  int rc = check_device("residue_map");
  if (rc) return rc;
  const int64_t F = (int64_t)((1ull << (1 << t)) + 1);
  return cuda_rc(launch_residue_map(in, out, n, F, decode, S(stream)), "residue_map");
}

int fntgpu_struct_sizes(int64_t* out, int n) {
  const int64_t sz[7] = {(int64_t)sizeof(fntgpu_cdc_taps), (int64_t)sizeof(fntgpu_cdc_io),
                         (int64_t)sizeof(fntgpu_decim_io), (int64_t)sizeof(fntgpu_aeq_params),
                         (int64_t)sizeof(fntgpu_aeq_state), (int64_t)sizeof(fntgpu_aeq_io),
                         (int64_t)sizeof(fntgpu_td_aeq_io)};
  for (int i = 0; i < n && i < 7; ++i) out[i] = sz[i];
  return 7;
}

int fntgpu_cdc64_process(const fntgpu_cdc_taps* taps, const fntgpu_cdc_io* io, void* stream) {
  if (!taps || !io) return fail(FNTGPU_EINVAL, "cdc64_process: NULL argument");
  if (taps->kernel < FNTGPU_CDC_KERNEL_AUTO || taps->kernel > FNTGPU_CDC_KERNEL_UMMA)
    return fail(FNTGPU_EINVAL, "cdc64_process: unknown kernel selector %d", taps->kernel);
  if (taps->n_taps < 1 || taps->n_taps > 33)
    return fail(FNTGPU_EINVAL, "n_taps=%d exceeds overlap-save validity 33 for block_n=64", taps->n_taps);
  if (io->n_streams < 0 || io->length < 0 || io->out_count < 0 || io->x_count < 0)
    return fail(FNTGPU_EINVAL, "cdc64_process: negative size");
  if (io->out_count == 0 || io->n_streams == 0) return FNTGPU_OK;
  if (io->out_first < 0 || io->out_first + io->out_count > io->length)
    return fail(FNTGPU_EINVAL, "cdc64_process: output range [%lld, %lld) outside [0, %lld)",
                (long long)io->out_first, (long long)(io->out_first + io->out_count),
                (long long)io->length);
  if (io->in_dtype != FNTGPU_I8 && io->in_dtype != FNTGPU_I32 && io->in_dtype != FNTGPU_I64 &&
      io->in_dtype != FNTGPU_F64)
    return fail(FNTGPU_EINVAL, "cdc64_process: in_dtype must be I8, I32, I64 or F64");
  if (io->in_dtype == FNTGPU_F64 && (io->in_max < 0 || io->in_max > 127))
    return fail(FNTGPU_EINVAL, "cdc64_process: float64 input needs 0 <= in_max <= 127 (int8 staging)");
  if (!io->xr || !io->xi) return fail(FNTGPU_EINVAL, "cdc64_process: NULL input");
  // every input sample the range needs (x[n - 16 .. n + 16] for c = 16, widened to
  // whole overlap-save blocks) must be present where it lies inside [0, L)
  const int c = taps->n_taps / 2;
  const int64_t b_lo = (io->out_first + c) / 32, b_hi = (io->out_first + io->out_count - 1 + c) / 32;
  int64_t need_lo = b_lo * 32 - 32, need_hi = b_hi * 32 + 32;  // [lo, hi)
  // the staging window of a CTA extends to the CTA's last block; clamp to the stream
  if (need_lo < 0) need_lo = 0;
  if (need_hi > io->length) need_hi = io->length;
  if (need_lo < need_hi && (need_lo < io->x_first || need_hi > io->x_first + io->x_count))
    return fail(FNTGPU_EINVAL,
                "cdc64_process: input samples [%lld, %lld) needed, only [%lld, %lld) provided",
                (long long)need_lo, (long long)need_hi, (long long)io->x_first,
                (long long)(io->x_first + io->x_count));
  switch (io->out_dtype) {
    case FNTGPU_NONE: case FNTGPU_I16: case FNTGPU_I32: case FNTGPU_I64: case FNTGPU_C128: break;
    default: return fail(FNTGPU_EINVAL, "cdc64_process: bad out_dtype %d", io->out_dtype);
  }
  if (io->out_dtype != FNTGPU_NONE && (!io->yr || (io->out_dtype != FNTGPU_C128 && !io->yi)))
    return fail(FNTGPU_EINVAL, "cdc64_process: NULL output");
  if ((io->qr != nullptr) != (io->qi != nullptr) || (io->qr && (io->q_max < 1 || io->q_max > 127)))
    return fail(FNTGPU_EINVAL, "cdc64_process: bad requantization arguments");
  int rc = check_device("cdc64_process");
  if (rc) return rc;
  return cuda_rc(launch_cdc64(*taps, *io, S(stream)), "cdc64_process");
}

int fntgpu_decim_phase(const fntgpu_decim_io* io, void* stream) {
  if (!io || io->n_links < 0 || (io->n_links && (!io->acc || !io->phase)) || io->sps != 2 ||
      io->length < 2)
    return fail(FNTGPU_EINVAL, "decim_phase: bad arguments (sps must be 2, length >= 2)");
  int rc = check_device("decim_phase");
  if (rc) return rc;
  return cuda_rc(launch_decim_phase(*io, S(stream)), "decim_phase");
}

static int check_aeq_params(const fntgpu_aeq_params* prm, const char* where) {
  if (!prm) return fail(FNTGPU_EINVAL, "%s: NULL params", where);
  if (prm->n_radii < 1 || prm->n_radii > 8)
    return fail(FNTGPU_EINVAL, "%s: n_radii must be in [1, 8]", where);
  if (!(prm->sig_scale > 0) || !(prm->tap_scale > 0))
    return fail(FNTGPU_EINVAL, "%s: scales must be positive", where);
  if (prm->mu < 0) return fail(FNTGPU_EINVAL, "mu must be >= 0");
  if (prm->forward != FNTGPU_AEQ_FWD_FNT && prm->forward != FNTGPU_AEQ_FWD_DIRECT)
    return fail(FNTGPU_EINVAL, "%s: bad forward mode", where);
  if (prm->kernel < FNTGPU_AEQ_KERNEL_AUTO || prm->kernel > FNTGPU_AEQ_KERNEL_POL)
    return fail(FNTGPU_EINVAL, "%s: bad kernel selector", where);
  return FNTGPU_OK;
}

int fntgpu_aeq_init(fntgpu_aeq_state* st, int n_streams, const fntgpu_aeq_params* prm, void* stream) {
  int rc = check_aeq_params(prm, "aeq_init");
  if (rc) return rc;
  if (n_streams < 0 || (n_streams && !st)) return fail(FNTGPU_EINVAL, "aeq_init: bad arguments");
  if (prm->tap_scale > 16383.0)
    return fail(FNTGPU_EINVAL, "aeq_init: tap_scale spike exceeds the 14-bit tap range");
  if ((rc = check_device("aeq_init"))) return rc;
  return cuda_rc(launch_aeq_init(st, n_streams, *prm, S(stream)), "aeq_init");
}

static bool aligned(const void* p, size_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

int fntgpu_aeq_process(fntgpu_aeq_state* st, const fntgpu_aeq_params* prm, const fntgpu_aeq_io* io,
                       void* stream) {
  int rc = check_aeq_params(prm, "aeq_process");
  if (rc) return rc;
  if (!io || io->n_streams < 0 || io->n_blocks < 0) return fail(FNTGPU_EINVAL, "aeq_process: bad io");
  if (io->n_streams == 0 || io->n_blocks == 0) return FNTGPU_OK;
  if (!st || !io->y) return fail(FNTGPU_EINVAL, "aeq_process: NULL state or output");
  if (!aligned(io->y, 16) || (io->y_row_stride % 2) || (io->y_stream_stride % 2))
    return fail(FNTGPU_EINVAL, "aeq_process: y must be 16-byte aligned with even strides");
  if (io->in_mode == FNTGPU_AEQ_IN_PLANAR) {
    const size_t es = io->in_dtype == FNTGPU_I8 ? 1 : io->in_dtype == FNTGPU_I32 ? 4 : 0;
    if (!es) return fail(FNTGPU_EINVAL, "aeq_process: planar in_dtype must be I8 or I32");
    if (!io->x || !aligned(io->x, 16) || (io->x_row_stride * es) % 16 || (io->x_stream_stride * es) % 16)
      return fail(FNTGPU_EINVAL, "aeq_process: x must be 16-byte aligned with 16-byte row strides");
  } else if (io->in_mode == FNTGPU_AEQ_IN_DECIM) {
    if (!io->qr || !io->qi || !io->phase || !aligned(io->qr, 16) || !aligned(io->qi, 16) ||
        io->q_stride % 16)
      return fail(FNTGPU_EINVAL, "aeq_process: decim planes must be 16-byte aligned");
  } else {
    return fail(FNTGPU_EINVAL, "aeq_process: bad in_mode");
  }
  if ((rc = check_device("aeq_process"))) return rc;
  return cuda_rc(launch_aeq_process(st, *prm, *io, S(stream)), "aeq_process");
}

int fntgpu_aeq_update_taps(fntgpu_aeq_state* st, const fntgpu_aeq_params* prm,
                           const int64_t* x_block, const double* y, double mu, double* err,
                           void* stream) {
  int rc = check_aeq_params(prm, "aeq_update_taps");
  if (rc) return rc;
  if (!st || !x_block || !y || !err) return fail(FNTGPU_EINVAL, "aeq_update_taps: NULL argument");
  if (mu < 0) return fail(FNTGPU_EINVAL, "mu must be >= 0");
  if ((rc = check_device("aeq_update_taps"))) return rc;
  return cuda_rc(launch_aeq_update_once(st, *prm, x_block, y, mu, err, S(stream)), "aeq_update_taps");
}

int fntgpu_td_aeq(const fntgpu_td_aeq_io* io, void* stream) {
  if (!io) return fail(FNTGPU_EINVAL, "td_aeq: NULL argument");
  if (io->n_streams < 0 || io->n < 0) return fail(FNTGPU_EINVAL, "td_aeq: negative size");
  if (io->n_radii < 1 || io->n_radii > 8) return fail(FNTGPU_EINVAL, "td_aeq: 1..8 ring radii");
  if (io->n_streams > 0 && io->n > 0 && (!io->x || !io->w || !io->mu || !io->y))
    return fail(FNTGPU_EINVAL, "td_aeq: NULL buffer");
  int rc;
  if ((rc = check_device("td_aeq"))) return rc;
  return cuda_rc(launch_td_aeq(*io, S(stream)), "td_aeq");
}

int fntgpu_aeq_selfcheck(const fntgpu_aeq_params* prm, int64_t lo, int64_t hi,
                         unsigned long long* mismatches, void* stream) {
  int rc = check_aeq_params(prm, "aeq_selfcheck");
  if (rc) return rc;
  if (!mismatches) return fail(FNTGPU_EINVAL, "aeq_selfcheck: NULL argument");
  if (lo < INT32_MIN || hi > (int64_t)INT32_MAX + 1 || lo > hi)
    return fail(FNTGPU_EINVAL, "aeq_selfcheck: range must lie within int32");
  if ((rc = check_device("aeq_selfcheck"))) return rc;
  return cuda_rc(launch_aeq_selfcheck(*prm, lo, hi, mismatches, S(stream)), "aeq_selfcheck");
}

}  // extern "C"
