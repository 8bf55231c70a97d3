// Butterfly-formulation microbenchmark for the Z/(2^32-1) FNT arithmetic: time per
// radix-2 butterfly (u, v) -> (u + 2^e v, u - 2^e v) for several instruction
// selections, to pick the fastest pipe mix (ALU: IADD3/SHF/LOP3, FMA: IMAD*).
// 8 independent butterfly chains per thread, 148*8 CTAs x 256 threads.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int ITERS = 2048;

__device__ __forceinline__ uint32_t add_c(uint32_t a, uint32_t b) {  // add.cc + addc
  uint32_t r;
  asm volatile("{\n\t.reg .u32 t;\n\tadd.cc.u32 t, %1, %2;\n\taddc.u32 %0, t, 0;\n\t}" : "=r"(r) : "r"(a), "r"(b));
  return r;
}
__device__ __forceinline__ uint32_t add_m(uint32_t a, uint32_t b) {  // add.cc + madc (IMAD.X)
  uint32_t r;
  asm volatile("{\n\t.reg .u32 t;\n\tadd.cc.u32 t, %1, %2;\n\tmadc.lo.u32 %0, t, 1, 0;\n\t}" : "=r"(r) : "r"(a), "r"(b));
  return r;
}
__device__ __forceinline__ uint32_t sub_c(uint32_t a, uint32_t b) {
  uint32_t r;
  asm volatile("{\n\t.reg .u32 t;\n\tsub.cc.u32 t, %1, %2;\n\tsubc.u32 %0, t, 0;\n\t}" : "=r"(r) : "r"(a), "r"(b));
  return r;
}
__device__ __forceinline__ uint32_t rot(uint32_t a, int j) {
  uint32_t r;
  asm volatile("shf.l.wrap.b32 %0, %1, %1, %2;" : "=r"(r) : "r"(a), "r"(j));
  return r;
}
// rotation through the FMA pipe: (hi:lo) = a * 2^j; lo | hi == lo + hi
__device__ __forceinline__ void rotw(uint32_t a, uint32_t p2, uint32_t& lo, uint32_t& hi) {
  asm volatile("{\n\t.reg .u64 p;\n\tmul.wide.u32 p, %2, %3;\n\tmov.b64 {%0, %1}, p;\n\t}" : "=r"(lo), "=r"(hi) : "r"(a), "r"(p2));
}

// ~a on the FMA pipe: a * 0xFFFFFFFF + 0xFFFFFFFF = -a - 1
__device__ __forceinline__ uint32_t not_f(uint32_t a, uint32_t m1) {
  uint32_t r;
  asm volatile("mad.lo.u32 %0, %1, %2, %2;" : "=r"(r) : "r"(a), "r"(m1));
  return r;
}

template <int V>
__global__ void k(uint32_t* out, uint32_t seed, int j, uint32_t p2, uint32_t m1) {
  uint32_t a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = seed + threadIdx.x * 8 + i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; i += 2) {
      uint32_t u = a[i], v = a[i + 1], s, d;
      if (V == 0) {        // SHF + add.cc/addc + sub.cc/subc
        uint32_t w = rot(v, j); s = add_c(u, w); d = sub_c(u, w);
      } else if (V == 1) { // SHF + add/madc + sub = add(u, ~w)
        uint32_t w = rot(v, j); s = add_m(u, w); d = add_m(u, ~w);
      } else if (V == 2) { // two rotates (mod F4: -2^e v == 2^(e+16) v), two madc adds
        uint32_t w = rot(v, j), x = rot(v, j + 16); s = add_m(u, w); d = add_m(u, x);
      } else if (V == 3) { // FMA-pipe rotate, lo+hi on FMA (IMAD), add/madc, sub.cc/subc
        uint32_t lo, hi; rotw(v, p2, lo, hi);
        uint32_t w; asm volatile("mad.lo.u32 %0, %1, 1, %2;" : "=r"(w) : "r"(lo), "r"(hi));
        s = add_m(u, w); d = sub_c(u, w);
      } else if (V == 4) { // SHF + add.cc/madc + sub.cc/subc
        uint32_t w = rot(v, j); s = add_m(u, w); d = sub_c(u, w);
      } else if (V == 5) { // no twiddle: add.cc/madc + sub.cc/subc
        s = add_m(u, v); d = sub_c(u, v);
      } else if (V == 6) { // SHF + madc add + (IMAD not, madc add): 3 ALU + 3 FMA
        uint32_t w = rot(v, j); s = add_m(u, w); d = add_m(u, not_f(w, m1));
      } else if (V == 7) { // no twiddle, IMAD not
        s = add_m(u, v); d = add_m(u, not_f(v, m1));
      }
      a[i] = s; a[i + 1] = d;
    }
  }
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s ^= a[i];
  if (s == 0x12345678u) out[0] = s;
}

template <int V>
float run(uint32_t* d) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    k<V><<<148 * 8, 256>>>(d, 1u + r, 5, 32u, 0xFFFFFFFFu);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  uint32_t* d; cudaMalloc(&d, 64);
  const double nb = 148.0 * 8 * 256 * ITERS * 4;  // butterflies
  const char* names[] = {"shf+addc+subc", "shf+madc+madc(~w)", "2shf+2madc(mod F4)", "imadwide+imad+madc+subc",
                         "shf+madc+subc", "noshf madc+subc", "shf+madc+imadnot+madc", "noshf madc+imadnot+madc"};
  float t[8] = {run<0>(d), run<1>(d), run<2>(d), run<3>(d), run<4>(d), run<5>(d), run<6>(d), run<7>(d)};
  printf("{");
  for (int i = 0; i < 8; ++i) printf("%s\"%s\": {\"ms\": %.4f, \"Gbfly_per_s\": %.1f}", i ? ", " : "", names[i], t[i], nb / (t[i] * 1e-3) / 1e9);
  printf("}\n");
  return cudaDeviceSynchronize() != cudaSuccess;
}
