// imma_bench.cu -- throughput of the legacy warp-level int8 MMA (mma.sync
// m16n8k32 s8, SASS IMMA.16832) on this GPU: many warps, 8 independent
// accumulator chains each. Used to size the tensor-core form of the FNT-CDC.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int CH>
__global__ void k_imma(const uint32_t* a, int* out, int iters) {
  uint32_t A0 = a[threadIdx.x & 31], A1 = A0 ^ 0x01010101u, A2 = A0 + 3u, A3 = A0 * 7u;
  uint32_t B0 = A0 ^ 0x5a5a5a5au, B1 = A1 + 11u;
  int d[CH][4];
#pragma unroll
  for (int c = 0; c < CH; ++c) d[c][0] = d[c][1] = d[c][2] = d[c][3] = c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c)
      asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+r"(d[c][0]), "+r"(d[c][1]), "+r"(d[c][2]), "+r"(d[c][3])
                   : "r"(A0), "r"(A1), "r"(A2), "r"(A3), "r"(B0), "r"(B1));
  }
  int s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint32_t* a;
  int* out;
  cudaMalloc(&a, 128);
  cudaMemset(a, 1, 128);
  cudaMalloc(&out, 64 << 20);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4096;
  for (int warps : {4, 8, 16, 32}) {
    const int threads = 128;
    const int blocks = sms * warps / 4;
    k_imma<8><<<blocks, threads>>>(a, out, 16);
    cudaEventRecord(e0);
    k_imma<8><<<blocks, threads>>>(a, out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double mma = (double)blocks * (threads / 32) * iters * 8;
    const double macs = mma * 16 * 8 * 32;
    printf("{\"warps_per_sm\": %d, \"ms\": %.3f, \"imma_per_s\": %.4e, \"tmac_per_s\": %.1f, \"cycles_per_imma_per_smsp\": %.2f}\n",
           warps, ms, mma / (ms * 1e-3), macs / (ms * 1e-3) / 1e12,
           (ms * 1e-3) * 1.965e9 * sms * 4 / mma);
  }
  return 0;
}
