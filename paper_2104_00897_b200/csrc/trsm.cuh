// trsm.cuh — the diagonal-block solve of FT-DTRSM.
//
// FT-BLAS's DTRSM (§III.C.3) casts most of the work to GEMM updates and
// solves only the diagonal blocks with a dedicated kernel that multiplies by the packed
// reciprocals of the diagonal instead of dividing.  FT-DTRSM protects the GEMM updates with
// the fused ABFT DGEMM and the diagonal solves with DMR (the paper gives
// no checksum algebra for the triangular solve itself).  The host recursion lives in
// ftblas.cu; this kernel solves one diagonal block S = op(A)[r0:r0+nb, r0:r0+nb], nb <= 128,
// for all n right-hand sides: X_blk = S^-1 B_blk, in place.
//
// Layout: the block is staged in shared memory column-major by op(A) and padded to LEAF x LEAF
// with an identity tail (Sc[i*LEAF + p] = S(p, i); rows/columns >= nb are unit rows), so every
// column runs the same fully static schedule.  One warp per right-hand side column (grid-stride);
// lane l owns rows l + 32q (q = 0..3, the "slots").  Forward (lower S): for i = 0..nb-1,
// x_i = b_i * rd_i broadcast from its owner lane, then b_p -= S(p, i) x_i for p > i; backward
// (upper S) runs i from nb-1 down.  The slot of i is a compile-time constant, so a step touches
// only the slots below (forward) / above (backward) it unconditionally plus one predicated FMA
// on its own slot: no register selects, no per-slot predicates.  A lane's own x_p is formed
// once, after the last step that updates it (the same product its owner step broadcast).  Every
// FP64 operation is computed twice (two register copies of the column, two reciprocal tables);
// the copies are compared bitwise at the end, a warp vote triggers the third computation, which
// settles each mismatching element.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "dmr.cuh"

namespace ftt {

constexpr int LEAF = 128;  // largest diagonal block of the leaf kernel

struct LeafParams {
  int nb, n;
  const double *A;  // caller's A at (r0, r0)
  int64_t lda;
  double *B;        // the block's first element of right-hand side 0
  int64_t es, rs;   // element stride within a right-hand side, stride between right-hand sides
  bool trans, unit;
  const ftd::DmrFault *f;  // faults of this block: index = j * LEAF + local row i, step = local p
  int nf;
  unsigned long long *cnt;  // ftd::D_* counters
};

// Reciprocal as its own instruction sequence (asm volatile: the two DMR copies are not merged).
__device__ __forceinline__ double v_rcp(double d) {
  double r;
  asm volatile("div.rn.f64 %0, 0d3FF0000000000000, %1;" : "=d"(r) : "d"(d));
  return r;
}

__device__ __forceinline__ double leaf_a(const LeafParams &P, int p, int i) {  // S(p, i) = op(A)(p, i)
  return P.trans ? P.A[i + (int64_t)p * P.lda] : P.A[p + (int64_t)i * P.lda];
}

// The 32 steps of slot SL (rows i = 32 SL + l) for NCH independent dependence chains at once:
// NCOL right-hand sides, and with DUAL both DMR copies of each (chain c = DUAL ? 2 col + copy :
// col; copy 1 uses the second reciprocal table).  The chains share each step's column of S
// and hide each other's shuffle / FP64 latency.  The fault hook (copy 0 only) adds fdel[col]
// to row fi[col] after the update from x_fstep[col].
template <int SL, bool FWD, int NCOL, bool DUAL, bool FLT>
__device__ __forceinline__ void leaf_slot(const double *__restrict__ Sc, double (&b)[NCOL * (DUAL ? 2 : 1)][4],
                                          const double (&r1)[4], const double (&r2)[4], int lane, const int (&fi)[NCOL],
                                          const int (&fstep)[NCOL], const double (&fdel)[NCOL]) {
  constexpr int NCH = NCOL * (DUAL ? 2 : 1);
#pragma unroll 2
  for (int s = 0; s < 32; ++s) {
    const int l = FWD ? s : 31 - s;
    const double *col = Sc + (32 * SL + l) * LEAF + lane;
    // All chains' products first, then all broadcasts (the FP64 ops are volatile asm, so their
    // program order is their issue order: interleaving keeps each shuffle off its product's
    // latency).
    double x[NCH];
#pragma unroll
    for (int c = 0; c < NCH; ++c) x[c] = ftd::v_mul(b[c][SL], (DUAL && (c & 1)) ? r2[SL] : r1[SL]);
#pragma unroll
    for (int c = 0; c < NCH; ++c) x[c] = __shfl_sync(0xffffffffu, x[c], l);
    if (FWD ? lane > l : lane < l) {
      const double a = col[32 * SL];
#pragma unroll
      for (int c = 0; c < NCH; ++c) b[c][SL] = ftd::v_fma(-a, x[c], b[c][SL]);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (FWD ? q > SL : q < SL) {
        const double a = col[32 * q];
#pragma unroll
        for (int c = 0; c < NCH; ++c) b[c][q] = ftd::v_fma(-a, x[c], b[c][q]);
      }
    }
    if (FLT) {
#pragma unroll
      for (int cc = 0; cc < NCOL; ++cc)
        if (32 * SL + l == fstep[cc]) {
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (lane + 32 * q == fi[cc]) b[DUAL ? 2 * cc : cc][q] = ftd::v_add(b[DUAL ? 2 * cc : cc][q], fdel[cc]);
        }
    }
  }
#pragma unroll
  for (int c = 0; c < NCH; ++c)  // this lane's x of the slot: no later step changes b
    b[c][SL] = ftd::v_mul(b[c][SL], (DUAL && (c & 1)) ? r2[SL] : r1[SL]);
}

template <bool FWD, int NCOL, bool DUAL, bool FLT>
__device__ __forceinline__ void leaf_solve(const double *Sc, double (&b)[NCOL * (DUAL ? 2 : 1)][4], const double (&r1)[4],
                                           const double (&r2)[4], int lane, int nslots, const int (&fi)[NCOL],
                                           const int (&fstep)[NCOL], const double (&fdel)[NCOL]) {
  if (FWD) {
    leaf_slot<0, true, NCOL, DUAL, FLT>(Sc, b, r1, r2, lane, fi, fstep, fdel);
    if (nslots > 1) leaf_slot<1, true, NCOL, DUAL, FLT>(Sc, b, r1, r2, lane, fi, fstep, fdel);
    if (nslots > 2) leaf_slot<2, true, NCOL, DUAL, FLT>(Sc, b, r1, r2, lane, fi, fstep, fdel);
    if (nslots > 3) leaf_slot<3, true, NCOL, DUAL, FLT>(Sc, b, r1, r2, lane, fi, fstep, fdel);
  } else {
    if (nslots > 3) leaf_slot<3, false, NCOL, DUAL, FLT>(Sc, b, r1, r2, lane, fi, fstep, fdel);
    if (nslots > 2) leaf_slot<2, false, NCOL, DUAL, FLT>(Sc, b, r1, r2, lane, fi, fstep, fdel);
    if (nslots > 1) leaf_slot<1, false, NCOL, DUAL, FLT>(Sc, b, r1, r2, lane, fi, fstep, fdel);
    leaf_slot<0, false, NCOL, DUAL, FLT>(Sc, b, r1, r2, lane, fi, fstep, fdel);
  }
}

#ifndef FTBLAS_LEAF_NCOL
#define FTBLAS_LEAF_NCOL 2
#endif
#ifndef FTBLAS_LEAF_THREADS
#define FTBLAS_LEAF_THREADS 512
#endif
constexpr int LEAF_NCOL = FTBLAS_LEAF_NCOL;        // right-hand sides per warp pass
constexpr int LEAF_THREADS = FTBLAS_LEAF_THREADS;  // threads per CTA (one CTA per SM: the block fills shared memory)

template <bool FWD, bool DMR, bool FLT>
__global__ void __launch_bounds__(LEAF_THREADS) trsm_leaf_kernel(const LeafParams P) {
  extern __shared__ double sm[];
  double *Sc = sm, *rd1 = sm + LEAF * LEAF, *rd2 = rd1 + LEAF;
  const int nb = P.nb, tid = threadIdx.x, lane = tid & 31, nslots = (nb + 31) >> 5;
  FT_CHECK(nb >= 1 && nb <= LEAF && (LEAF_THREADS & 31) == 0);
  for (int e = tid; e < LEAF * LEAF; e += blockDim.x) {
    const int i = e / LEAF, p = e % LEAF;
    Sc[e] = p < nb && i < nb ? leaf_a(P, p, i) : (p == i ? 1.0 : 0.0);
  }
  __syncthreads();
  for (int i = tid; i < LEAF; i += blockDim.x) {  // packed reciprocals of the diagonal, twice
    const double d = Sc[i * LEAF + i];
    rd1[i] = P.unit ? 1.0 : v_rcp(d);
    rd2[i] = P.unit ? 1.0 : v_rcp(d);
  }
  __syncthreads();
  double r1[4], r2[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) { r1[q] = rd1[lane + 32 * q]; r2[q] = rd2[lane + 32 * q]; }
  constexpr int NCOL = LEAF_NCOL, NCH = NCOL * (DMR ? 2 : 1);
  const int warps = blockDim.x >> 5;
  for (int j0 = (blockIdx.x * warps + (tid >> 5)) * NCOL; j0 < P.n; j0 += gridDim.x * warps * NCOL) {
    // This lane's fault in each column, if any (at most one per lane and column is honoured).
    int fi[NCOL], fstep[NCOL];
    double fdel[NCOL];
#pragma unroll
    for (int cc = 0; cc < NCOL; ++cc) { fi[cc] = -1; fstep[cc] = -1; fdel[cc] = 0.0; }
    if (FLT)
      for (int e = 0; e < P.nf; ++e) {
        const int64_t code = P.f[e].index;  // j * LEAF + local row
        const int64_t cc = code / LEAF - j0;
        if (cc >= 0 && cc < NCOL && (int)(code % LEAF) % 32 == lane)
#pragma unroll
          for (int c = 0; c < NCOL; ++c)
            if (c == cc) { FT_CHECK(code % LEAF < nb); fi[c] = (int)(code % LEAF); fstep[c] = (int)P.f[e].step; fdel[c] = P.f[e].delta; }
      }
    double b[NCH][4];
#pragma unroll
    for (int cc = 0; cc < NCOL; ++cc) {
      const bool jv = j0 + cc < P.n;
      const double *col = P.B + (int64_t)(j0 + cc) * P.rs;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int p = lane + 32 * q;
        b[DMR ? 2 * cc : cc][q] = jv && p < nb ? col[(int64_t)p * P.es] : 0.0;
        if (DMR) b[2 * cc + 1][q] = b[2 * cc][q];
      }
    }
    leaf_solve<FWD, NCOL, DMR, FLT>(Sc, b, r1, r2, lane, nslots, fi, fstep, fdel);
#pragma unroll
    for (int cc = 0; cc < NCOL; ++cc) {
      const int j = j0 + cc;
      if (j >= P.n) break;
      double *col = P.B + (int64_t)j * P.rs;
      double *out = b[DMR ? 2 * cc : cc];
      if (DMR) {
        bool bad = false;
#pragma unroll
        for (int q = 0; q < 4; ++q) bad |= (lane + 32 * q < nb) && ftd::differ(b[2 * cc][q], b[2 * cc + 1][q]);
        if (__any_sync(0xffffffffu, bad)) {
          // Rare: a third computation settles the column (the verification unit of a diagonal
          // block: one fault propagates to every later row of the column).  Each element takes
          // the third value; the column is corrected when the third agrees with one copy
          // wherever the two disagreed.
          double b3[1][4];
#pragma unroll
          for (int q = 0; q < 4; ++q) b3[0][q] = lane + 32 * q < nb ? col[(int64_t)(lane + 32 * q) * P.es] : 0.0;
          const int nfi[1] = {-1}, nfs[1] = {-1};
          const double nfd[1] = {0.0};
          leaf_solve<FWD, 1, false, false>(Sc, b3, r2, r2, lane, nslots, nfi, nfs, nfd);
          bool unsettled = false;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            if (lane + 32 * q < nb && ftd::differ(b[2 * cc][q], b[2 * cc + 1][q]))
              unsettled |= ftd::differ(b3[0][q], b[2 * cc][q]) && ftd::differ(b3[0][q], b[2 * cc + 1][q]);
            out[q] = b3[0][q];
          }
          unsettled = __any_sync(0xffffffffu, unsettled);
          if (lane == 0) {
            atomicAdd(&P.cnt[ftd::D_DETECTED], 1ull);
            atomicAdd(&P.cnt[unsettled ? ftd::D_UNCORRECTABLE : ftd::D_CORRECTED], 1ull);
          }
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (lane + 32 * q < nb) col[(int64_t)(lane + 32 * q) * P.es] = out[q];
    }
  }
}

// B := alpha * B (m x n), two roundings avoided: one multiply per element.
__global__ void scale_b_kernel(int64_t m, int64_t n, double alpha, double *B, int64_t ldb) {
  const int64_t total = m * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % m, j = e / m;
    double *p = B + i + j * ldb;
    *p = alpha == 0.0 ? 0.0 : __dmul_rn(alpha, *p);
  }
}

}  // namespace ftt
