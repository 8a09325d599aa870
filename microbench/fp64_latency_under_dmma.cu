// Latency of a dependent SIMT chain (DADD / DFMA / FFMA / IADD / SHFL) issued by one warp while
// N other warps of the same SM saturate the FP64 pipe with DMMA.8x8x4.  Tells whether the
// checksum warps' dependent FP64 chains stall behind the DMMA stream.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}
__device__ volatile int g_stop;
template <int KIND>
__global__ void k(int n_dmma_warps, int chain, long long* out, double* sink) {
  int w = threadIdx.x >> 5;
  if (w < n_dmma_warps) {   // load warps
    double acc[16][2];
    for (int t = 0; t < 16; ++t) acc[t][0] = acc[t][1] = 0;
    double a = 1.0 + 1e-12 * threadIdx.x, b = 1.0;
    for (int it = 0; it < 4000; ++it) {
#pragma unroll
      for (int t = 0; t < 16; ++t) dmma(acc[t], a, b);
    }
    double s = 0; for (int t = 0; t < 16; ++t) s += acc[t][0];
    if (s == 1.23) sink[0] = s;
    return;
  }
  // chain warp (the last warp)
  for (volatile int spin = 0; spin < 20000; ++spin) {}  // let the DMMA stream fill the pipe
  double x = 1.0 + threadIdx.x * 1e-9, y = 1e-30;
  float fx = 1.0f + threadIdx.x, fy = 1e-30f;
  int ix = threadIdx.x, iy = 3;
  long long t0 = clock64();
  for (int i = 0; i < chain; ++i) {
    if (KIND == 0) x = x + y;
    else if (KIND == 1) x = fma(x, 1.0, y);
    else if (KIND == 2) fx = fmaf(fx, 1.0f, fy);
    else if (KIND == 3) ix = ix + iy;
    else x = __shfl_xor_sync(0xffffffffu, x, 1);
  }
  long long t1 = clock64();
  if ((threadIdx.x & 31) == 0) out[blockIdx.x] = (t1 - t0);
  if (x == 3.3 || fx == 3.3f || ix == 7) sink[1] = x + fx + ix;
}
int main() {
  long long* out; double* sink; cudaMalloc(&out, 8 * 148); cudaMalloc(&sink, 16);
  const char* names[] = {"DADD", "DFMA", "FFMA", "IADD", "SHFL64"};
  const int chain = 2000;
  printf("{");
  for (int kind = 0; kind < 5; ++kind) {
    for (int nd : {0, 2, 4, 8}) {
      long long h[148];
      int threads = 32 * (nd + 1);
      switch (kind) {
        case 0: k<0><<<148, threads>>>(nd, chain, out, sink); break;
        case 1: k<1><<<148, threads>>>(nd, chain, out, sink); break;
        case 2: k<2><<<148, threads>>>(nd, chain, out, sink); break;
        case 3: k<3><<<148, threads>>>(nd, chain, out, sink); break;
        case 4: k<4><<<148, threads>>>(nd, chain, out, sink); break;
      }
      cudaDeviceSynchronize();
      cudaMemcpy(h, out, 8 * 148, cudaMemcpyDeviceToHost);
      double avg = 0; for (int i = 0; i < 148; ++i) avg += h[i]; avg /= 148;
      printf("\"%s_dmmawarps%d\": %.1f, ", names[kind], nd, avg / chain);
    }
  }
  printf("\"unit\": \"clk per dependent op\"}\n");
  return 0;
}
