// Which instruction classes, issued by a side warp on the same SM sub-partition, slow a
// saturated DMMA.8x8x4 stream?  8 DMMA warps (2 per SMSP) + 4 side warps (1 per SMSP).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}
__device__ int g_stop;
template <int KIND>
__global__ void __launch_bounds__(384, 1) k(int iters, double* sink, int* flag) {
  __shared__ double sm[4096];
  int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 4096; i += 384) sm[i] = i * 0.5;
  __syncthreads();
  if (w >= 4) {   // DMMA warps 4..11
    double acc[16][2];
    for (int t = 0; t < 16; ++t) acc[t][0] = acc[t][1] = 0;
    double a = 1.0 + 1e-12 * threadIdx.x, b = 1.0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int t = 0; t < 16; ++t) dmma(acc[t], a, b);
    }
    double s = 0; for (int t = 0; t < 16; ++t) s += acc[t][0];
    if (s == 1.23) sink[0] = s;
    if (lane == 0) atomicAdd(flag + blockIdx.x, 1);
    return;
  }
  if (KIND == 0) return;
  // side warps: run until all DMMA warps are done
  unsigned x0 = threadIdx.x, x1 = threadIdx.x * 3 + 1, x2 = 7, x3 = 11;
  double d0 = 1.0, d1 = 2.0, d2 = 3.0, d3 = 4.0;
  long long acc = 0;
  int it = 0;
  while (*(volatile int*)(flag + blockIdx.x) < 8) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      if (KIND == 1) { x0 = x0 * 3u + x1; x1 = (x1 << 3) ^ x2; x2 = x2 + x3; x3 = __funnelshift_l(x3, x0, 5); }  // int mix
      if (KIND == 2) { double vx, vy; asm volatile("ld.shared.v2.f64 {%0,%1}, [%2];" : "=d"(vx), "=d"(vy) : "r"((unsigned)__cvta_generic_to_shared(&sm[((lane + u * 32 + it) * 2) & 4095]))); x0 += (unsigned)__double_as_longlong(vx) ^ (unsigned)__double_as_longlong(vy); }       // LDS.128 (+1 DADD)
      if (KIND == 3) { x0 = __shfl_xor_sync(0xffffffffu, x0, 1) + 1; }                                      // SHFL
      if (KIND == 4) { d0 = fma(d0, 1.0000001, 1e-9); d1 = fma(d1, 1.0000001, 1e-9); d2 = fma(d2, 1.0000001, 1e-9); d3 = fma(d3, 1.0000001, 1e-9); } // 4 indep DFMA
      if (KIND == 5) { x0 = x0 + x1; x1 = x1 ^ x2; x2 = x2 + 7; x3 = x3 ^ x0; }  // pure ALU (IADD3/LOP3)
      if (KIND == 6) { x0 = x0 * 3u + x1; x1 = x1 * 5u + x2; x2 = x2 * 7u + x3; x3 = x3 * 9u + x0; }  // IMAD only
    }
    ++it;
  }
  if (x0 + x1 + x2 + x3 == 12345u || d0 + d1 + d2 + d3 == 1.5) sink[1] = x0 + d0 + acc;
  if (lane == 0 && w == 0) sink[2 + blockIdx.x] = it;
}
template <int KIND>
float run(double* sink, int* flag) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e9;
  for (int r = 0; r < 3; ++r) {
    cudaMemset(flag, 0, sizeof(int) * 148);
    cudaEventRecord(e0);
    k<KIND><<<148, 384>>>(3000, sink, flag);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  return best;
}
int main() {
  double* sink; int* flag;
  cudaMalloc(&sink, 8 * 512); cudaMalloc(&flag, 4 * 148);
  // per-block flag: pass flag + blockIdx via pointer offset trick is overkill; use one global counter per launch
  float base = run<0>(sink, flag);
  printf("{\"none_ms\": %.3f", base);
  const char* nm[] = {"", "int_mix", "lds128", "shfl", "dfma4", "alu", "imad"};
  float t1 = run<1>(sink, flag), t2 = run<2>(sink, flag), t3 = run<3>(sink, flag), t4 = run<4>(sink, flag), t5 = run<5>(sink, flag), t6 = run<6>(sink, flag);
  printf(", \"%s\": %.3f, \"%s\": %.3f, \"%s\": %.3f, \"%s\": %.3f, \"%s\": %.3f, \"%s\": %.3f}\n", nm[1], t1 / base, nm[2], t2 / base, nm[3], t3 / base, nm[4], t4 / base, nm[5], t5 / base, nm[6], t6 / base);
  return 0;
}
