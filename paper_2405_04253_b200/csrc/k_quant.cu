// k_quant.cu -- quantize_real (fixedpoint.py:51-60) on the GPU.
//
// v = x * scale ; q = sign(v) * floor(|v| + 0.5) ; clipped += (|q| > max_int) ;
// q = clip(q, -max_int, max_int). All float64 steps use explicit round-to-nearest
// intrinsics so the result is bit-identical to numpy's elementwise sequence.
#include "internal.h"

namespace fntgpu {

template <typename T>
__global__ void k_quantize(const double* __restrict__ x, int64_t n, double scale, int32_t max_int,
                           T* __restrict__ q, unsigned long long* clipped) {
  unsigned long long c = 0;
  const double mx = (double)max_int;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double v = __dmul_rn(x[i], scale);
    const double a = floor(__dadd_rn(fabs(v), 0.5));
    double r = v > 0 ? a : (v < 0 ? -a : 0.0);
    if (fabs(r) > mx) ++c;
    r = r > mx ? mx : (r < -mx ? -mx : r);
    q[i] = (T)(long long)r;
  }
  if (clipped) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) c += __shfl_xor_sync(0xffffffffu, c, off);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(clipped, c);
  }
}

cudaError_t launch_quantize(const double* x, int64_t n, double scale, int32_t max_int,
                            int out_dtype, void* q, unsigned long long* clipped, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  switch (out_dtype) {
    case FNTGPU_I8:
      k_quantize<int8_t><<<(unsigned)blocks, 256, 0, st>>>(x, n, scale, max_int, (int8_t*)q, clipped);
      break;
    case FNTGPU_I32:
      k_quantize<int32_t><<<(unsigned)blocks, 256, 0, st>>>(x, n, scale, max_int, (int32_t*)q, clipped);
      break;
    case FNTGPU_I64:
      k_quantize<int64_t><<<(unsigned)blocks, 256, 0, st>>>(x, n, scale, max_int, (int64_t*)q, clipped);
      break;
    default:
      return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

// encode_signed_array / decode_signed_array (fermat.py:124-133): elementwise
// v < 0 -> v + F (encode) ; r > half -> r - F (decode). Not a modular reduction:
// the reference applies exactly one conditional correction.
__global__ void k_residue_map(const int64_t* __restrict__ in, int64_t* __restrict__ out, int64_t n,
                              int64_t F, int64_t half, int decode) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = in[i];
    out[i] = decode ? (v <= half ? v : v - F) : (v >= 0 ? v : v + F);
  }
}

cudaError_t launch_residue_map(const int64_t* in, int64_t* out, int64_t n, int64_t F, int decode,
                               cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  k_residue_map<<<(unsigned)blocks, 256, 0, st>>>(in, out, n, F, (F - 1) / 2, decode);
  return cudaGetLastError();
}

}  // namespace fntgpu
