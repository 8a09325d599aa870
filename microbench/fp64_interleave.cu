// How much does interleaving SIMT FP64 (DFMA/DADD) with DMMA in the same warp cost?
// Each iteration: 32 independent DMMA.8x8x4 then X independent DFMA (or DADD).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}
template <int X, bool ADD>
__global__ void k(int iters, double* out) {
  double acc[32][2];
  for (int t = 0; t < 32; ++t) acc[t][0] = acc[t][1] = 0;
  double c[16];
  for (int t = 0; t < 16; ++t) c[t] = threadIdx.x + t;
  double a = 1.0 + blockIdx.x * 1e-12, b = 1.0 - 1e-12;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int t = 0; t < 32; ++t) dmma(acc[t], a, b);
#pragma unroll
    for (int x = 0; x < X; ++x) c[x & 15] = ADD ? c[x & 15] + a : fma(c[x & 15], b, a);
  }
  double s = 0;
  for (int t = 0; t < 32; ++t) s += acc[t][0] + acc[t][1];
  for (int t = 0; t < 16; ++t) s += c[t];
  if (s == 1.2345) out[0] = s;
}
template <int X, bool ADD>
float t(int warps, double* out) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<X, ADD><<<148, 32 * warps>>>(2000, out); cudaDeviceSynchronize();
  float best = 1e9;
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(e0); k<X, ADD><<<148, 32 * warps>>>(2000, out); cudaEventRecord(e1);
    cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  return best;
}
int main() {
  double* out; cudaMalloc(&out, 8);
  for (int w : {8, 16}) {
    float base = t<0, false>(w, out);
    printf("{\"warps\": %d, \"X0_ms\": %.3f", w, base);
#define P(X) printf(", \"dfma%d\": %.3f, \"dadd%d\": %.3f", X, t<X, false>(w, out) / base, X, t<X, true>(w, out) / base);
    P(1) P(2) P(4) P(8) P(16) P(32) P(64)
    printf("}\n");
  }
  return 0;
}
