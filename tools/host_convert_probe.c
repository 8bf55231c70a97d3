/* Host-side int32 -> float64 (y_int / D) conversion bandwidth probe (DESIGN.md section 6,
 * e2e row): would shipping y_int over PCIe and dividing on the host beat the float64
 * D2H? Build: gcc -O3 -march=x86-64-v3 -pthread tools/host_convert_probe.c */
#define _GNU_SOURCE
#include <pthread.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>
#include <unistd.h>
static int32_t* src; static double* dst; static size_t N; static int T; static double D = 1234.5678;
static void* work(void* a) {
  size_t t = (size_t)a, lo = N * t / T, hi = N * (t + 1) / T;
  for (size_t i = lo; i < hi; ++i) dst[i] = (double)src[i] / D;
  return 0;
}
static double now(void) { struct timespec ts; clock_gettime(CLOCK_MONOTONIC, &ts); return ts.tv_sec + 1e-9 * ts.tv_nsec; }
int main(int argc, char** argv) {
  N = (size_t)1 << 28;  /* 1 GiB int32 -> 2 GiB double */
  src = aligned_alloc(64, N * 4); dst = aligned_alloc(64, N * 8);
  for (size_t i = 0; i < N; ++i) src[i] = (int32_t)(i * 2654435761u) >> 10;
  memset(dst, 0, N * 8);
  printf("nproc %ld\n", sysconf(_SC_NPROCESSORS_ONLN));
  int ts[] = {1, 4, 8, 16, 32, 64};
  for (int k = 0; k < 6; ++k) {
    T = ts[k]; pthread_t th[64];
    double best = 1e9;
    for (int rep = 0; rep < 3; ++rep) {
      double t0 = now();
      for (int t = 0; t < T; ++t) pthread_create(&th[t], 0, work, (void*)(size_t)t);
      for (int t = 0; t < T; ++t) pthread_join(th[t], 0);
      double dt = now() - t0; if (dt < best) best = dt;
    }
    printf("threads %d: %.3f s  out %.1f GB/s  in+out %.1f GB/s\n", T, best, N * 8 / best / 1e9, N * 12 / best / 1e9);
  }
  double t0 = now(); memcpy(dst, src, N * 4); printf("memcpy 1GiB %.1f GB/s\n", N * 4 / (now() - t0) / 1e9);
  return 0;
}
