// dmr.cuh — Level-1/2 BLAS with dual modular redundancy.
//
// FT-BLAS protects its memory-bound routines by duplicating the computing instructions,
// comparing the two results and only then storing (§IV: "we duplicate and
// verify computing instructions instead of memory instructions"; comparison reduction over
// several results before one branch, §IV.D; a third computation resolves a mismatch and is
// itself verified, §IV.E).  On B200 these routines are HBM-bound (DSCAL 1/16 FLOP/B, DGEMV
// 1/4 FLOP/B against a 37 TF / 6.5 TB/s machine), so the duplicate FP64 work hides under the
// memory stream.  The GPU form:
//   - both copies come from inline-asm FP64 instructions on the same loaded registers (no
//     common-subexpression merging), the original one carries the fault-injection hook;
//   - the verdict is reduced per warp with a vote (__any_sync) — one branch per warp-step
//     instead of one per element;
//   - on a mismatch the lane computes a third copy: equal to either copy -> corrected (the
//     third value is stored), else uncorrectable (stored, counted).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace ftd {

struct DmrFault {  // sorted by index
  int64_t index, step;
  double delta;
};

enum { D_DETECTED = 0, D_CORRECTED, D_UNCORRECTABLE, D_N };

__device__ __forceinline__ double v_mul(double a, double b) {
  double r;
  asm volatile("mul.rn.f64 %0, %1, %2;" : "=d"(r) : "d"(a), "d"(b));
  return r;
}
__device__ __forceinline__ double v_fma(double a, double b, double c) {
  double r;
  asm volatile("fma.rn.f64 %0, %1, %2, %3;" : "=d"(r) : "d"(a), "d"(b), "d"(c));
  return r;
}
__device__ __forceinline__ double v_add(double a, double b) {
  double r;
  asm volatile("add.rn.f64 %0, %1, %2;" : "=d"(r) : "d"(a), "d"(b));
  return r;
}
__device__ __forceinline__ bool differ(double a, double b) { return __double_as_longlong(a) != __double_as_longlong(b); }

__device__ __forceinline__ int64_t vidx(int64_t i, int64_t n, int64_t inc) { return inc > 0 ? i * inc : (n - 1 - i) * (-inc); }

// Delta of the fault on output `index` (0 if none); faults sorted by index, binary search.
__device__ __forceinline__ double fault_delta(const DmrFault *f, int nf, int64_t index, int64_t step) {
  int lo = 0, hi = nf;
  while (lo < hi) { const int mid = (lo + hi) >> 1; if (f[mid].index < index) lo = mid + 1; else hi = mid; }
  double d = 0.0;
  for (; lo < nf && f[lo].index == index; ++lo)
    if (f[lo].step == step) d += f[lo].delta;
  return d;
}

// Settle a mismatch with a third computation r3; returns the value to store.
__device__ __forceinline__ double settle(double r1, double r2, double r3, unsigned long long *cnt) {
  atomicAdd(&cnt[D_DETECTED], 1ull);
  if (!differ(r3, r2) || !differ(r3, r1)) atomicAdd(&cnt[D_CORRECTED], 1ull);
  else atomicAdd(&cnt[D_UNCORRECTABLE], 1ull);
  return r3;
}

// ---------------------------------------------------------------- DSCAL: x := alpha x
// FLT: the launch carries armed faults (the fault hook is compiled in only then, so the
// production path keeps its registers for loads in flight).
// Residency: 6 x 256-thread CTAs per SM (40 registers) for both the DMR kernels and their
// unprotected twins (at 32 registers the DMR variants spill; the twins measured no faster at
// 8).  The host sizes grid-stride launches to exactly one wave.
constexpr int resident_ctas(bool dmr) { return dmr ? 6 : 6; }

template <bool DMR, bool FLT>
__global__ void __launch_bounds__(256, resident_ctas(DMR)) dscal_kernel(int64_t n, double alpha, double *__restrict__ x, int64_t incx,
                                                    const DmrFault *__restrict__ f, int nf,
                                                    unsigned long long *__restrict__ cnt) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * 4;
  for (int64_t base = ((int64_t)blockIdx.x * blockDim.x) * 4 + threadIdx.x; base < n; base += stride) {
    double xv[4], r[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t i = base + (int64_t)u * blockDim.x;
      xv[u] = i < n ? x[vidx(i, n, incx)] : 0.0;
    }
    bool bad = false;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      r[u] = v_mul(alpha, xv[u]);
      if (DMR) {
        if (FLT) {
          const int64_t i = base + (int64_t)u * blockDim.x;
          if (i < n) { const double d = fault_delta(f, nf, i, 0); if (d != 0.0) r[u] = v_add(r[u], d); }
        }
        bad |= differ(r[u], v_mul(alpha, xv[u]));  // the duplicate
      }
    }
    if (DMR && __any_sync(__activemask(), bad)) {  // rare: redo the duplicate, settle by a third
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double r2 = v_mul(alpha, xv[u]);
        if (differ(r[u], r2)) r[u] = settle(r[u], r2, v_mul(alpha, xv[u]), cnt);
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t i = base + (int64_t)u * blockDim.x;
      if (i < n) x[vidx(i, n, incx)] = r[u];
    }
  }
}

// ---------------------------------------------------------------- DAXPY: y := alpha x + y
template <bool DMR, bool FLT>
__global__ void __launch_bounds__(256, resident_ctas(DMR)) daxpy_kernel(int64_t n, double alpha, const double *__restrict__ x, int64_t incx,
                                                    double *__restrict__ y, int64_t incy,
                                                    const DmrFault *__restrict__ f, int nf,
                                                    unsigned long long *__restrict__ cnt) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * 4;
  for (int64_t base = ((int64_t)blockIdx.x * blockDim.x) * 4 + threadIdx.x; base < n; base += stride) {
    double xv[4], yv[4], r[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t i = base + (int64_t)u * blockDim.x;
      xv[u] = i < n ? x[vidx(i, n, incx)] : 0.0;
      yv[u] = i < n ? y[vidx(i, n, incy)] : 0.0;
    }
    bool bad = false;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      r[u] = v_fma(alpha, xv[u], yv[u]);
      if (DMR) {
        if (FLT) {
          const int64_t i = base + (int64_t)u * blockDim.x;
          if (i < n) { const double d = fault_delta(f, nf, i, 0); if (d != 0.0) r[u] = v_add(r[u], d); }
        }
        bad |= differ(r[u], v_fma(alpha, xv[u], yv[u]));  // the duplicate
      }
    }
    if (DMR && __any_sync(__activemask(), bad)) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double r2 = v_fma(alpha, xv[u], yv[u]);
        if (differ(r[u], r2)) r[u] = settle(r[u], r2, v_fma(alpha, xv[u], yv[u]), cnt);
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t i = base + (int64_t)u * blockDim.x;
      if (i < n) y[vidx(i, n, incy)] = r[u];
    }
  }
}

// ---------------------------------------------------------------- unit-stride fast paths
// x (and y) contiguous and 16-byte aligned: every thread owns VU 16-byte pairs of one block's
// 2 VU * 256-element chunk (pair u at u * 256 + threadIdx.x: one LDG.128 per pair, a warp reads
// 512 contiguous bytes), all loads issued before any FP64 work; one chunk per CTA, so the
// hardware overlaps the tail of a block with the next block's loads (no loop-carried
// dependence through a grid-stride loop).  Same DMR arithmetic and fault hook per element.
constexpr int VU = 4;                   // 16-byte pairs per thread
constexpr int VCHUNK = 2 * VU * 256;    // elements per CTA

template <bool DMR, bool FLT>
__device__ __forceinline__ double dmr_scal1(double alpha, double xv, int64_t i, const DmrFault *f, int nf, bool &bad) {
  double r = v_mul(alpha, xv);
  if (DMR) {
    if (FLT) { const double d = fault_delta(f, nf, i, 0); if (d != 0.0) r = v_add(r, d); }
    bad |= differ(r, v_mul(alpha, xv));  // the duplicate
  }
  return r;
}
template <bool DMR, bool FLT>
__device__ __forceinline__ double dmr_axpy1(double alpha, double xv, double yv, int64_t i, const DmrFault *f, int nf,
                                            bool &bad) {
  double r = v_fma(alpha, xv, yv);
  if (DMR) {
    if (FLT) { const double d = fault_delta(f, nf, i, 0); if (d != 0.0) r = v_add(r, d); }
    bad |= differ(r, v_fma(alpha, xv, yv));  // the duplicate
  }
  return r;
}

template <bool DMR, bool FLT>
__global__ void __launch_bounds__(256) dscal_vec_kernel(int64_t n, double alpha, double *__restrict__ x,
                                                        const DmrFault *__restrict__ f, int nf,
                                                        unsigned long long *__restrict__ cnt) {
  const int64_t c0 = (int64_t)blockIdx.x * VCHUNK;
  double2 *x2 = reinterpret_cast<double2 *>(x + c0);
  const bool full = c0 + VCHUNK <= n;
  double2 xv[VU];
#pragma unroll
  for (int u = 0; u < VU; ++u) {
    const int64_t i = c0 + 2 * (u * 256 + threadIdx.x);
    if (full) xv[u] = x2[u * 256 + threadIdx.x];
    else xv[u] = make_double2(i < n ? x[i] : 0.0, i + 1 < n ? x[i + 1] : 0.0);
  }
  double2 r[VU];
  bool bad = false;
#pragma unroll
  for (int u = 0; u < VU; ++u) {
    const int64_t i = c0 + 2 * (u * 256 + threadIdx.x);
    r[u].x = dmr_scal1<DMR, FLT>(alpha, xv[u].x, i, f, nf, bad);
    r[u].y = dmr_scal1<DMR, FLT>(alpha, xv[u].y, i + 1, f, nf, bad);
  }
  if (DMR && __any_sync(0xffffffffu, bad)) {  // rare: redo the duplicate, settle by a third
#pragma unroll
    for (int u = 0; u < VU; ++u) {
      double r2 = v_mul(alpha, xv[u].x);
      if (differ(r[u].x, r2)) r[u].x = settle(r[u].x, r2, v_mul(alpha, xv[u].x), cnt);
      r2 = v_mul(alpha, xv[u].y);
      if (differ(r[u].y, r2)) r[u].y = settle(r[u].y, r2, v_mul(alpha, xv[u].y), cnt);
    }
  }
#pragma unroll
  for (int u = 0; u < VU; ++u) {
    const int64_t i = c0 + 2 * (u * 256 + threadIdx.x);
    if (full) {
      x2[u * 256 + threadIdx.x] = r[u];
    } else {
      if (i < n) x[i] = r[u].x;
      if (i + 1 < n) x[i + 1] = r[u].y;
    }
  }
}

template <bool DMR, bool FLT>
__global__ void __launch_bounds__(256) daxpy_vec_kernel(int64_t n, double alpha, const double *__restrict__ x,
                                                        double *__restrict__ y, const DmrFault *__restrict__ f, int nf,
                                                        unsigned long long *__restrict__ cnt) {
  const int64_t c0 = (int64_t)blockIdx.x * VCHUNK;
  const double2 *x2 = reinterpret_cast<const double2 *>(x + c0);
  double2 *y2 = reinterpret_cast<double2 *>(y + c0);
  const bool full = c0 + VCHUNK <= n;
  double2 xv[VU], yv[VU];
#pragma unroll
  for (int u = 0; u < VU; ++u) {
    const int64_t i = c0 + 2 * (u * 256 + threadIdx.x);
    if (full) {
      xv[u] = x2[u * 256 + threadIdx.x];
      yv[u] = y2[u * 256 + threadIdx.x];
    } else {
      xv[u] = make_double2(i < n ? x[i] : 0.0, i + 1 < n ? x[i + 1] : 0.0);
      yv[u] = make_double2(i < n ? y[i] : 0.0, i + 1 < n ? y[i + 1] : 0.0);
    }
  }
  double2 r[VU];
  bool bad = false;
#pragma unroll
  for (int u = 0; u < VU; ++u) {
    const int64_t i = c0 + 2 * (u * 256 + threadIdx.x);
    r[u].x = dmr_axpy1<DMR, FLT>(alpha, xv[u].x, yv[u].x, i, f, nf, bad);
    r[u].y = dmr_axpy1<DMR, FLT>(alpha, xv[u].y, yv[u].y, i + 1, f, nf, bad);
  }
  if (DMR && __any_sync(0xffffffffu, bad)) {
#pragma unroll
    for (int u = 0; u < VU; ++u) {
      double r2 = v_fma(alpha, xv[u].x, yv[u].x);
      if (differ(r[u].x, r2)) r[u].x = settle(r[u].x, r2, v_fma(alpha, xv[u].x, yv[u].x), cnt);
      r2 = v_fma(alpha, xv[u].y, yv[u].y);
      if (differ(r[u].y, r2)) r[u].y = settle(r[u].y, r2, v_fma(alpha, xv[u].y, yv[u].y), cnt);
    }
  }
#pragma unroll
  for (int u = 0; u < VU; ++u) {
    const int64_t i = c0 + 2 * (u * 256 + threadIdx.x);
    if (full) {
      y2[u * 256 + threadIdx.x] = r[u];
    } else {
      if (i < n) y[i] = r[u].x;
      if (i + 1 < n) y[i + 1] = r[u].y;
    }
  }
}

// ---------------------------------------------------------------- DGEMV
// 'N': y_i = alpha sum_j A_ij x_j + beta y_i.  A CTA of GN_W = 16 warps owns 32 rows (one
// per lane); warp w accumulates the columns j = w (mod 16) (coalesced 256-byte column
// segments), the 16 partial sums of a row are combined in warp order by warp 0.
constexpr int GN_W = 8;
constexpr int GN_U = 8;  // columns of a warp's set per loop iteration (loads in flight)
struct GemvParams {
  int64_t m, n;
  double alpha, beta;
  const double *A;
  int64_t lda;
  const double *x;
  int64_t incx;
  double *y;
  int64_t incy;
  const DmrFault *f;
  int nf;
  unsigned long long *cnt;
};

// LPR lanes share a row (LPR = 1, 2, 4: 32, 16, 8 rows per CTA, so moderate m still fills the
// machine); lane part q of warp w sums the columns j = w LPR + q (mod GN_W LPR) in order, the
// LPR parts combine by a fixed xor butterfly (commutative: every lane of the row gets the same
// value), then the warps in order.
template <int LPR>
__device__ __forceinline__ double gemv_n_row(const GemvParams &P, int64_t i) {  // third computation, same order
  constexpr int S = GN_W * LPR;
  double acc = 0.0;
  for (int w = 0; w < GN_W; ++w) {
    double part[LPR];
#pragma unroll
    for (int q = 0; q < LPR; ++q) {
      part[q] = 0.0;
      for (int64_t j = w * LPR + q; j < P.n; j += S) part[q] = v_fma(P.A[i + j * P.lda], P.x[vidx(j, P.n, P.incx)], part[q]);
    }
    double t = part[0];
    if (LPR == 2) t = v_add(part[0], part[1]);
    if (LPR == 4) t = v_add(v_add(part[0], part[1]), v_add(part[2], part[3]));
    acc = w == 0 ? t : v_add(acc, t);
  }
  return acc;
}

template <bool DMR, bool FLT, int LPR>
__global__ void __launch_bounds__(GN_W * 32, 4) dgemv_n_kernel(const GemvParams P) {
  constexpr int RPC = 32 / LPR, S = GN_W * LPR;  // rows per CTA, column stride of a lane part
  __shared__ double part[2][GN_W][RPC];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, r = lane / LPR, q = lane % LPR;
  const int64_t i = (int64_t)blockIdx.x * RPC + r;
  const bool row_ok = i < P.m;
  const int64_t ir = row_ok ? i : 0;
  const int64_t j0 = w * LPR + q;  // this lane's first column
  double a1 = 0.0, a2 = 0.0;
  // This lane's fault (row i, term `step` in this lane's column set), if any.
  int64_t fstep = -1;
  double fdel = 0.0;
  if (DMR && FLT && row_ok) {
    int lo = 0, hi = P.nf;
    while (lo < hi) { const int mid = (lo + hi) >> 1; if (P.f[mid].index < i) lo = mid + 1; else hi = mid; }
    for (; lo < P.nf && P.f[lo].index == i; ++lo)
      if (P.f[lo].step < P.n && (P.f[lo].step % S) == j0) { fstep = P.f[lo].step; fdel += P.f[lo].delta; }
  }
  const double *Ai = P.A + ir;
  int64_t j = j0;
  for (; j + (GN_U - 1) * S < P.n; j += GN_U * S) {  // GN_U columns of this lane's set
    double av[GN_U], xv[GN_U];
#pragma unroll
    for (int u = 0; u < GN_U; ++u) {
      av[u] = Ai[(j + S * u) * P.lda];
      xv[u] = P.x[vidx(j + S * u, P.n, P.incx)];
    }
#pragma unroll
    for (int u = 0; u < GN_U; ++u) {
      if (DMR && FLT && (j + S * u) == fstep) a1 = v_add(a1, fdel);
      a1 = v_fma(av[u], xv[u], a1);
      if (DMR) a2 = v_fma(av[u], xv[u], a2);
    }
  }
  for (; j < P.n; j += S) {
    const double av = Ai[j * P.lda], xv = P.x[vidx(j, P.n, P.incx)];
    if (DMR && FLT && j == fstep) a1 = v_add(a1, fdel);
    a1 = v_fma(av, xv, a1);
    if (DMR) a2 = v_fma(av, xv, a2);
  }
#pragma unroll
  for (int o = 1; o < LPR; o <<= 1) {  // the row's lane parts: fixed butterfly
    a1 = v_add(a1, __shfl_xor_sync(0xffffffffu, a1, o));
    if (DMR) a2 = v_add(a2, __shfl_xor_sync(0xffffffffu, a2, o));
  }
  if (q == 0) {
    part[0][w][r] = a1;
    part[1][w][r] = a2;
  }
  __syncthreads();
  if (w != 0 || q != 0) return;
  double s1 = part[0][0][r], s2 = part[1][0][r];
#pragma unroll
  for (int u = 1; u < GN_W; ++u) {
    s1 = v_add(s1, part[0][u][r]);
    if (DMR) s2 = v_add(s2, part[1][u][r]);
  }
  if (!row_ok) return;
  if (DMR && FLT) s1 = v_add(s1, fault_delta(P.f, P.nf, i, P.n));  // faults after the last term
  double *yi = P.y + vidx(i, P.m, P.incy);
  const double yb = P.beta != 0.0 ? v_mul(P.beta, *yi) : 0.0;
  double r1 = v_fma(P.alpha, s1, yb);
  if (DMR) {
    const double yb2 = P.beta != 0.0 ? v_mul(P.beta, *yi) : 0.0;
    const double r2 = v_fma(P.alpha, s2, yb2);
    if (__any_sync(__activemask(), differ(r1, r2)) && differ(r1, r2))
      r1 = settle(r1, r2, v_fma(P.alpha, gemv_n_row<LPR>(P, i), yb2), P.cnt);
  }
  *yi = r1;
}

// 'T': y_j = alpha sum_i A_ij x_i + beta y_j.  One warp per column j; lane l sums the rows
// i = l (mod 32) in order, then a fixed butterfly combines the lanes.
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = v_add(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// This lane's part of column j's dot product, a1 (plus the duplicate a2 when TWO).  Every
// computation of the column -- the two DMR copies and the third one that settles a mismatch --
// goes through this function, so all three use the same partition and order: lanes own
// elements {b + 64u + 2 lane, +1} of each 512-element block of the unit-stride, 16-byte aligned
// fast path, then rows i = lane (mod 32) of the remainder.  A fault (FLT) at element fstep is
// added to a1 before that element's term by the lane that owns it.
__device__ __forceinline__ int64_t gemv_t_fast_end(const GemvParams &P, const double *Aj) {
  const bool fast = P.incx == 1 && ((reinterpret_cast<uintptr_t>(Aj) | reinterpret_cast<uintptr_t>(P.x)) & 15) == 0;
  return fast ? (P.m / 512) * 512 : 0;
}
__device__ __forceinline__ int gemv_t_owner(int64_t e, int64_t bfast) { return e < bfast ? (int)((e & 63) >> 1) : (int)(e & 31); }

template <bool TWO, bool FLT>
__device__ __forceinline__ void dgemv_t_lane(const GemvParams &P, const double *Aj, int lane, int64_t bfast,
                                             int64_t fstep, double fdel, double &a1, double &a2) {
  a1 = 0.0;
  a2 = 0.0;
  for (int64_t b = 0; b < bfast; b += 512) {
    double2 av[8], xv[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      av[u] = *reinterpret_cast<const double2 *>(Aj + b + 64 * u + 2 * lane);
      xv[u] = *reinterpret_cast<const double2 *>(P.x + b + 64 * u + 2 * lane);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int64_t e = b + 64 * u + 2 * lane;
      if (FLT && e == fstep) a1 = v_add(a1, fdel);
      a1 = v_fma(av[u].x, xv[u].x, a1);
      if (FLT && e + 1 == fstep) a1 = v_add(a1, fdel);
      a1 = v_fma(av[u].y, xv[u].y, a1);
      if (TWO) {
        a2 = v_fma(av[u].x, xv[u].x, a2);
        a2 = v_fma(av[u].y, xv[u].y, a2);
      }
    }
  }
  int64_t i = bfast + lane;
  for (; i + 96 < P.m; i += 128) {
    double av[4], xv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      av[u] = Aj[i + 32 * u];
      xv[u] = P.x[vidx(i + 32 * u, P.m, P.incx)];
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (FLT && (i + 32 * u) == fstep) a1 = v_add(a1, fdel);
      a1 = v_fma(av[u], xv[u], a1);
      if (TWO) a2 = v_fma(av[u], xv[u], a2);
    }
  }
  for (; i < P.m; i += 32) {
    const double av = Aj[i], xv = P.x[vidx(i, P.m, P.incx)];
    if (FLT && i == fstep) a1 = v_add(a1, fdel);
    a1 = v_fma(av, xv, a1);
    if (TWO) a2 = v_fma(av, xv, a2);
  }
}

template <bool DMR, bool FLT>
__device__ __forceinline__ void dgemv_t_column(const GemvParams &P, int64_t j, int lane) {
  const double *Aj = P.A + j * P.lda;
  const int64_t bfast = gemv_t_fast_end(P, Aj);
  int64_t fstep = -1;
  double fdel = 0.0;
  if (DMR && FLT) {
    int lo = 0, hi = P.nf;
    while (lo < hi) { const int mid = (lo + hi) >> 1; if (P.f[mid].index < j) lo = mid + 1; else hi = mid; }
    for (; lo < P.nf && P.f[lo].index == j; ++lo)
      if (P.f[lo].step < P.m && gemv_t_owner(P.f[lo].step, bfast) == lane) { fstep = P.f[lo].step; fdel += P.f[lo].delta; }
  }
  double a1, a2;
  dgemv_t_lane<DMR, DMR && FLT>(P, Aj, lane, bfast, fstep, fdel, a1, a2);
  double s1 = warp_sum(a1), s2 = DMR ? warp_sum(a2) : 0.0;
  if (DMR && FLT) s1 = v_add(s1, fault_delta(P.f, P.nf, j, P.m));
  double *yj = P.y + vidx(j, P.n, P.incy);
  const double yb = P.beta != 0.0 ? v_mul(P.beta, *yj) : 0.0;
  double r1 = v_fma(P.alpha, s1, yb);
  if (DMR) {
    const double yb2 = P.beta != 0.0 ? v_mul(P.beta, *yj) : 0.0;
    const double r2 = v_fma(P.alpha, s2, yb2);
    if (differ(r1, r2)) {  // warp-uniform: every lane holds the butterfly result
      double a3, unused;
      dgemv_t_lane<false, false>(P, Aj, lane, bfast, -1, 0.0, a3, unused);  // same partition and order
      const double r3 = v_fma(P.alpha, warp_sum(a3), yb2);
      if (lane == 0) r1 = settle(r1, r2, r3, P.cnt);
      else r1 = r3;
    }
  }
  if (lane == 0) *yj = r1;
}

constexpr int GT_CTAS = 4;  // resident 256-thread CTAs per SM of dgemv_t (64 registers: 16 loads in flight)
template <bool DMR, bool FLT>
__global__ void __launch_bounds__(256, GT_CTAS) dgemv_t_kernel(const GemvParams P) {
  const int lane = threadIdx.x & 31;
  for (int64_t j = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5); j < P.n; j += (int64_t)gridDim.x * 8)
    dgemv_t_column<DMR, FLT>(P, j, lane);
}

}  // namespace ftd
