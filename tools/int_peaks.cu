// Integer / FP64 pipe peak microbenchmark for the FNT hot path roofline.
//
// MEASURED_PEAKS.json (driver-written) has only HBM copy bandwidth and bf16 GEMM
// rates. The FNT-CDC / FNT-AEQ kernels are integer-ALU bound (shift/add/IMAD
// Fermat arithmetic) with an FP64 tap update, so their roofline denominators are
// measured here on the same B200s:
//   alu_iadd3    : IADD3-class adds (ALU pipe)
//   alu_shf      : funnel-shift rotates (ALU pipe)
//   fma_imad     : IMAD (FMA pipe)
//   mixed        : IADD3 + IMAD interleaved (both pipes), the integer peak
//   modm_bfly    : one mod-(2^32-1) butterfly = SHF.W + 2x(add.cc/addc), 5 int ops
//   fp64_dfma / fp64_dadd / fp64_dmul
// Each kernel runs 8 independent dependency chains per thread on a grid of
// 148*8 CTAs x 256 threads and is timed with CUDA events (best of 5).
// Output: one JSON object on stdout.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); return 1; } } while (0)

constexpr int ITERS = 4096;

__global__ void k_iadd(uint32_t* out, uint32_t seed) {
  uint32_t a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = seed + threadIdx.x * 8 + i;
  uint32_t c = seed | 1u;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("add.u32 %0, %0, %1;" : "+r"(a[i]) : "r"(c));
  }
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s ^= a[i];
  if (s == 0x12345678u) out[0] = s;
}

__global__ void k_shf(uint32_t* out, uint32_t seed) {
  uint32_t a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = seed + threadIdx.x * 8 + i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("shf.l.wrap.b32 %0, %0, %0, 7;" : "+r"(a[i]));
  }
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s ^= a[i];
  if (s == 0x12345678u) out[0] = s;
}

__global__ void k_imad(uint32_t* out, uint32_t seed) {
  uint32_t a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = seed + threadIdx.x * 8 + i;
  uint32_t m = seed * 2u + 3u, c = seed + 11u;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[i]) : "r"(m), "r"(c));
  }
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s ^= a[i];
  if (s == 0x12345678u) out[0] = s;
}

__global__ void k_mixed(uint32_t* out, uint32_t seed) {
  uint32_t a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = seed + threadIdx.x * 8 + i;
  uint32_t m = seed * 2u + 3u, c = seed + 11u;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; i += 2) {
      asm volatile("add.u32 %0, %0, %1;" : "+r"(a[i]) : "r"(c));
      asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[i + 1]) : "r"(m), "r"(c));
    }
  }
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s ^= a[i];
  if (s == 0x12345678u) out[0] = s;
}

// One radix-2 butterfly modulo 2^32-1: v = rot(b, 5); a' = a + v (end-around); b' = a - v.
__global__ void k_bfly(uint32_t* out, uint32_t seed) {
  uint32_t a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = seed + threadIdx.x * 8 + i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; i += 2) {
      uint32_t u = a[i], v, s, d;
      asm volatile("shf.l.wrap.b32 %0, %1, %1, 5;" : "=r"(v) : "r"(a[i + 1]));
      asm volatile("{\n\t.reg .u32 t;\n\tadd.cc.u32 t, %1, %2;\n\taddc.u32 %0, t, 0;\n\t}" : "=r"(s) : "r"(u), "r"(v));
      asm volatile("{\n\t.reg .u32 t;\n\tsub.cc.u32 t, %1, %2;\n\tsubc.u32 %0, t, 0;\n\t}" : "=r"(d) : "r"(u), "r"(v));
      a[i] = s; a[i + 1] = d;
    }
  }
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s ^= a[i];
  if (s == 0x12345678u) out[0] = s;
}

__global__ void k_dfma(double* out, double seed) {
  double a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = seed + threadIdx.x + i;
  double m = 1.0000001, c = 1e-9;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(a[i]) : "d"(m), "d"(c));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 1.2345) out[0] = s;
}

__global__ void k_dadd(double* out, double seed) {
  double a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = seed + threadIdx.x + i;
  double c = 1e-9;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(a[i]) : "d"(c));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 1.2345) out[0] = s;
}

__global__ void k_dmul(double* out, double seed) {
  double a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = seed + threadIdx.x + i;
  double m = 1.0000001;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("mul.rn.f64 %0, %0, %1;" : "+d"(a[i]) : "d"(m));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 1.2345) out[0] = s;
}

template <typename F>
static float time_best(F launch, int reps = 5) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  launch();  // warm-up
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(a);
    launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  cudaEventDestroy(a); cudaEventDestroy(b);
  return best;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int sms = p.multiProcessorCount;
  int clk_khz = 0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  uint32_t* du; double* dd;
  CK(cudaMalloc(&du, 64)); CK(cudaMalloc(&dd, 64));
  const int threads = 256, blocks = sms * 8;
  const double thr = double(threads) * blocks;
  const double ops_per_thread = 8.0 * ITERS;  // instructions per thread
  struct R { const char* name; double ops_per_inst; float ms; } rs[16];
  int n = 0;
  rs[n++] = {"alu_iadd3", 1.0, time_best([&] { k_iadd<<<blocks, threads>>>(du, 1u); })};
  rs[n++] = {"alu_shf", 1.0, time_best([&] { k_shf<<<blocks, threads>>>(du, 1u); })};
  rs[n++] = {"fma_imad", 1.0, time_best([&] { k_imad<<<blocks, threads>>>(du, 1u); })};
  rs[n++] = {"mixed_iadd_imad", 1.0, time_best([&] { k_mixed<<<blocks, threads>>>(du, 1u); })};
  // k_bfly: 4 butterflies per 8-chain iteration, each 5 int instructions -> 20 instr / 8 "slots"
  rs[n++] = {"modm_bfly", 20.0 / 8.0, time_best([&] { k_bfly<<<blocks, threads>>>(du, 1u); })};
  rs[n++] = {"fp64_dfma", 1.0, time_best([&] { k_dfma<<<blocks, threads>>>(dd, 1.0); })};
  rs[n++] = {"fp64_dadd", 1.0, time_best([&] { k_dadd<<<blocks, threads>>>(dd, 1.0); })};
  rs[n++] = {"fp64_dmul", 1.0, time_best([&] { k_dmul<<<blocks, threads>>>(dd, 1.0); })};
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"clock_khz_attr\": %d, \"threads\": %.0f, \"iters\": %d", p.name, sms,
         clk_khz, thr, ITERS);
  for (int i = 0; i < n; ++i) {
    double insts = thr * ops_per_thread * rs[i].ops_per_inst;
    double tops = insts / (rs[i].ms * 1e-3) / 1e12;
    printf(", \"%s\": {\"ms\": %.4f, \"Tinst_per_s\": %.3f}", rs[i].name, rs[i].ms, tops);
  }
  printf("}\n");
  return 0;
}
