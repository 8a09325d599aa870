/* Dev: host-side cost per library call, from C (no Python): wall time per call of loops of
 * calls at a small shape (the GPU work is a few microseconds, so the loop is host-bound), and
 * the synchronous protected call's round trip.  build + run: tools/host_cost.sh */
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <time.h>
#include "ftblas.h"

static double now_us(void) {
  struct timespec t;
  clock_gettime(CLOCK_MONOTONIC, &t);
  return t.tv_sec * 1e6 + t.tv_nsec * 1e-3;
}

int main(int argc, char **argv) {
  const int64_t N = argc > 1 ? atoll(argv[1]) : 256;
  const int reps = 400;
  double *A, *B, *C;
  cudaMalloc((void **)&A, sizeof(double) * N * N);
  cudaMalloc((void **)&B, sizeof(double) * N * N);
  cudaMalloc((void **)&C, sizeof(double) * N * N);
  cudaMemset(A, 0, sizeof(double) * N * N);
  cudaMemset(B, 0, sizeof(double) * N * N);
  ftblas_event_t ev[64];
  ftblas_err_report_t r = {0};
  r.events = ev;
  r.events_capacity = 64;
  const char *names[] = {"quick return (m = 0)", "noft", "protected, no report", "protected + report"};
  for (int mode = 0; mode < 4; ++mode) {
    for (int pass = 0; pass < 2; ++pass) {
      cudaDeviceSynchronize();
      const double t0 = now_us();
      for (int i = 0; i < reps; ++i) {
        int st = 0;
        if (mode == 0) st = ftblas_dgemm_noft('N', 'N', 0, N, N, 1.0, A, N, B, N, 0.0, C, N);
        if (mode == 1) st = ftblas_dgemm_noft('N', 'N', N, N, N, 1.0, A, N, B, N, 0.0, C, N);
        if (mode == 2) st = ftblas_dgemm('N', 'N', N, N, N, 1.0, A, N, B, N, 0.0, C, N, NULL);
        if (mode == 3) st = ftblas_dgemm('N', 'N', N, N, N, 1.0, A, N, B, N, 0.0, C, N, &r);
        if (st) { printf("status %d\n", st); return 1; }
      }
      const double t1 = now_us();
      cudaDeviceSynchronize();
      const double t2 = now_us();
      if (pass) printf("%-24s n=%lld: %.2f us per call issued, %.2f us per call incl. drain\n", names[mode], (long long)N,
                       (t1 - t0) / reps, (t2 - t0) / reps);
    }
  }
  return 0;
}
