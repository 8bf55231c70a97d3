// internal.h -- launchers shared between the kernel translation units and capi.cu.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

#include "../../include/fntgpu.h"

namespace fntgpu {

// Device-side copy of a validated TransformPlan (fnt.py:24-33).
struct DevPlan {
  int t, n, lg, kind;      // kind: 0 generic, 1 RADIX2 (F4, alpha=2, n=32), 2 SQRT2 (F4, 4080, n=64)
  uint32_t F, n_inv;
  const uint32_t* tw_fwd;  // n-1 entries, stage-concatenated (fnt.py:_stage_twiddles)
  const uint32_t* tw_inv;
};

enum PlanKind { KIND_GENERIC = 0, KIND_RADIX2_32 = 1, KIND_SQRT2_64 = 2 };

cudaError_t launch_fnt(const DevPlan& p, int inverse, const int64_t* x, int64_t* y, int64_t batch,
                       int flags, cudaStream_t st);
cudaError_t launch_conv_real(const DevPlan& p, const int64_t* x, const int64_t* h, int64_t h_stride,
                             int64_t* z, int64_t batch, int flags, cudaStream_t st);
cudaError_t launch_conv_complex(const DevPlan& p, const int64_t* xr, const int64_t* xi,
                                const int64_t* yr, const int64_t* yi, int64_t y_stride,
                                int64_t* zr, int64_t* zi, int64_t batch, int flags,
                                cudaStream_t st);
cudaError_t launch_cdc64(const fntgpu_cdc_taps& taps, const fntgpu_cdc_io& io, cudaStream_t st);
cudaError_t launch_quantize(const double* x, int64_t n, double scale, int32_t max_int,
                            int out_dtype, void* q, unsigned long long* clipped, cudaStream_t st);
cudaError_t launch_residue_map(const int64_t* in, int64_t* out, int64_t n, int64_t F, int decode,
                               cudaStream_t st);
cudaError_t launch_aeq_init(fntgpu_aeq_state* st, int n_streams, const fntgpu_aeq_params& prm,
                            cudaStream_t s);
cudaError_t launch_aeq_process(fntgpu_aeq_state* st, const fntgpu_aeq_params& prm,
                               const fntgpu_aeq_io& io, cudaStream_t s);
cudaError_t launch_decim_phase(const fntgpu_decim_io& io, cudaStream_t s);

}  // namespace fntgpu
