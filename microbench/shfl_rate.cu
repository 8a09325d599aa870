// SHFL.IDX throughput per SM (64-bit values = 2 SHFL each), 16 warps per SM, independent chains.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double *out, int iters) {
  double v[8];
  for (int i = 0; i < 8; ++i) v[i] = threadIdx.x * 1.0 + i;
  int src = (threadIdx.x * 7) & 31;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __shfl_sync(0xffffffffu, v[i], (src + i) & 31);
  }
  double s = 0; for (int i = 0; i < 8; ++i) s += v[i];
  if (s == 1.2345) out[0] = s;
}
__global__ void k32(int *out, int iters) {
  int v[8];
  for (int i = 0; i < 8; ++i) v[i] = threadIdx.x + i;
  int src = (threadIdx.x * 7) & 31;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __shfl_sync(0xffffffffu, v[i], (src + i) & 31);
  }
  int s = 0; for (int i = 0; i < 8; ++i) s += v[i];
  if (s == 12345) out[0] = s;
}
int main() {
  double *o; cudaMalloc(&o, 64);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int iters = 20000;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a); k<<<sms, 512>>>(o, iters); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double warp_shfl = (double)sms * 16 * iters * 8 * 2;  // 64-bit = 2 SHFL
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    float ms2; cudaEventRecord(a); k32<<<sms, 512>>>((int *)o, iters); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms2, a, b);
    if (rep) printf("{\"shfl64_ms\": %.3f, \"warp_shfl_per_clk_per_sm\": %.3f, \"shfl32_warp_per_clk_per_sm\": %.3f}\n", ms,
                    warp_shfl / sms / (ms * 1e-3 * 1.965e9), (double)sms * 16 * iters * 8 / sms / (ms2 * 1e-3 * 1.965e9));
  }
  return 0;
}
