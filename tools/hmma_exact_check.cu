// Exactness probe for the FP16 tensor-core form of the AEQ tap transform
// (K3): mma.sync m16n8k16 f16 x f16 -> f32 with integer operands
// (A = digit + 1536 in [1024, 2047], B = +-2^j, j <= 7) accumulated onto the magic
// 1.5 * 2^23, against exact integer dot products. Prints the mismatch count.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/hmma_exact_check.cu
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>

__device__ uint32_t rng(uint64_t& s) { s = s * 6364136223846793005ull + 1442695040888963407ull; return (uint32_t)(s >> 33); }

__global__ void k(unsigned long long* bad, unsigned long long* tot, int iters) {
  const int lane = threadIdx.x & 31, g = lane >> 2, tig = lane & 3;
  uint64_t s = 0x9E3779B97F4A7C15ull * (blockIdx.x * blockDim.x + threadIdx.x + 1);
  __shared__ int A[4][16][16];   // per warp: 16 x 16 digits (+1536 applied on conversion)
  __shared__ int B[4][16][8];    // 16 x 8 powers of two with sign
  const int w = threadIdx.x >> 5;
  for (int it = 0; it < iters; ++it) {
    // each lane fills 8 A entries and 4 B entries
    for (int i = lane; i < 256; i += 32) {
      int d = (int)(rng(s) % 513) - 256;
      if ((rng(s) & 15) == 0) d = (rng(s) & 1) ? 256 : -256;
      A[w][i >> 4][i & 15] = d;
    }
    for (int i = lane; i < 128; i += 32) {
      const int j = rng(s) % 8;
      B[w][i >> 3][i & 7] = ((rng(s) & 1) ? -1 : 1) * (1 << j);
    }
    __syncwarp();
    auto h = [](int v) -> uint32_t { return (uint32_t)__half_as_ushort(__int2half_rn(v)); };
    // A fragment (row-major 16x16): a0 = (g, 2tig..+1), a1 = (g+8, 2tig..), a2 = (g, 2tig+8..), a3 = (g+8, 2tig+8..)
    uint32_t a[4];
    const int rr[4] = {g, g + 8, g, g + 8}, cc[4] = {2 * tig, 2 * tig, 2 * tig + 8, 2 * tig + 8};
    for (int q = 0; q < 4; ++q)
      a[q] = h(A[w][rr[q]][cc[q]] + 1536) | (h(A[w][rr[q]][cc[q] + 1] + 1536) << 16);
    // B fragment (col, 16x8): b0 = (k = 2tig..+1, n = g), b1 = (k = 2tig+8..+9, n = g)
    uint32_t b[2];
    b[0] = h(B[w][2 * tig][g]) | (h(B[w][2 * tig + 1][g]) << 16);
    b[1] = h(B[w][2 * tig + 8][g]) | (h(B[w][2 * tig + 9][g]) << 16);
    const float m = 12582912.f;
    float d[4];
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%10,%10,%10,%10};"
                 : "=f"(d[0]), "=f"(d[1]), "=f"(d[2]), "=f"(d[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]), "f"(m));
    // C fragment: c0 = (g, 2tig), c1 = (g, 2tig+1), c2 = (g+8, 2tig), c3 = (g+8, 2tig+1)
    const int cr[4] = {g, g, g + 8, g + 8}, cn[4] = {2 * tig, 2 * tig + 1, 2 * tig, 2 * tig + 1};
    unsigned long long nb = 0;
    for (int q = 0; q < 4; ++q) {
      long long want = 0;
      for (int kk = 0; kk < 16; ++kk) want += (long long)(A[w][cr[q]][kk] + 1536) * B[w][kk][cn[q]];
      const long long got = (long long)__float_as_uint(d[q]) - (long long)__float_as_uint(m);
      nb += got != want;
    }
    atomicAdd(bad, nb);
    atomicAdd(tot, 4ull);
    __syncwarp();
  }
}

int main() {
  unsigned long long *d, h[2];
  cudaMalloc(&d, 16);
  cudaMemset(d, 0, 16);
  k<<<1184, 128>>>(d, d + 1, 256);
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("hmma exactness: %llu mismatches of %llu dot products (%s)\n", h[0], h[1], cudaGetErrorString(cudaGetLastError()));
  return h[0] != 0;
}
