// FP64 ceiling microbenchmarks for sm_100a.
// Measures: DFMA (SIMT FP64 pipe), DMMA (mma.sync m8n8k4 f64 -> SASS DMMA.8x8x4),
// and a concurrent mix (half the warps DMMA, half DFMA) to learn whether the two
// share an issue pipe. Prints one JSON object.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

constexpr int NACC_DMMA = 8;   // independent 8x8 accumulators per warp
constexpr int NCH_DFMA = 8;    // independent DFMA chains per thread

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}

__device__ __forceinline__ void run_dmma(int iters, double* out, double seed) {
  double acc[NACC_DMMA][2];
#pragma unroll
  for (int t = 0; t < NACC_DMMA; ++t) { acc[t][0] = 0.0; acc[t][1] = 0.0; }
  double a = 1.0 + seed * 1e-9, b = 1.0 - seed * 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int t = 0; t < NACC_DMMA; ++t) dmma(acc[t], a, b);
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < NACC_DMMA; ++t) s += acc[t][0] + acc[t][1];
  if (s == 12345.678) out[threadIdx.x] = s;
}

__device__ __forceinline__ void run_dfma(int iters, double* out, double seed) {
  double c[NCH_DFMA];
#pragma unroll
  for (int t = 0; t < NCH_DFMA; ++t) c[t] = seed + t;
  double a = 0.9999999, b = 1e-7;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int t = 0; t < NCH_DFMA; ++t) c[t] = fma(c[t], a, b);
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < NCH_DFMA; ++t) s += c[t];
  if (s == 12345.678) out[threadIdx.x] = s;
}

// mode 0: all DMMA; 1: all DFMA; 2: warp-interleaved mix (even warps DMMA, odd DFMA)
__global__ void k_bench(int mode, int it_dmma, int it_dfma, double* out) {
  int w = threadIdx.x >> 5;
  double seed = (double)blockIdx.x;
  if (mode == 0 || (mode == 2 && (w & 1) == 0)) run_dmma(it_dmma, out, seed);
  else run_dfma(it_dfma, out, seed);
}

static float time_it(int mode, int blocks, int threads, int itm, int itf, double* out) {
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  k_bench<<<blocks, threads>>>(mode, itm, itf, out);  // warm
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    CK(cudaEventRecord(e0));
    k_bench<<<blocks, threads>>>(mode, itm, itf, out);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1)); if (ms < best) best = ms;
  }
  return best;
}

int main(int argc, char** argv) {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int sms = p.multiProcessorCount;
  double* out; CK(cudaMalloc(&out, 1024 * sizeof(double)));
  const int itm = 20000, itf = 20000;
  printf("{\"device\": \"%s\", \"sms\": %d, \"results\": [\n", p.name, sms);
  bool first = true;
  for (int wps : {4, 8, 16, 32}) {           // warps per SM (one block per SM)
    int threads = 32 * wps, blocks = sms;
    float tm = time_it(0, blocks, threads, itm, itf, out);
    float tf = time_it(1, blocks, threads, itm, itf, out);
    float tx = time_it(2, blocks, threads, itm, itf, out);
    double fl_dmma = 2.0 * 256 * NACC_DMMA * (double)itm * wps * blocks;        // per warp: 256 FMA per DMMA
    double fl_dfma = 2.0 * 32 * 4 * NCH_DFMA * (double)itf * wps * blocks;      // per thread FMAs
    double fl_mix = 0.5 * fl_dmma + 0.5 * fl_dfma;
    printf("%s {\"warps_per_sm\": %d, \"dmma_ms\": %.3f, \"dmma_tflops\": %.2f, \"dfma_ms\": %.3f, \"dfma_tflops\": %.2f, "
           "\"mix_ms\": %.3f, \"mix_tflops\": %.2f, \"mix_vs_sum_of_halves\": %.3f}\n",
           first ? "" : ",", wps, tm, fl_dmma / tm / 1e9, tf, fl_dfma / tf / 1e9, tx, fl_mix / tx / 1e9,
           tx / (0.5 * tm + 0.5 * tf));
    first = false;
  }
  printf("]}\n");
  return 0;
}
