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
// Layout: the block is staged in shared memory column-major by op(A) (Sc[i*nb + p] =
// S(p, i)), so the update of step i reads one contiguous column across the lanes (conflict
// free).  One warp per right-hand side column (grid-stride); lane l owns rows l, l+32, l+64,
// l+96.  Forward (lower S): x_i = b_i * rd_i, then b_p -= S(p,i) x_i for p > i; backward
// (upper S) runs i from nb-1 down.  Every FP64 operation is computed twice (two register
// copies of the column, two reciprocal tables); the copies are compared bitwise at the end,
// a warp vote triggers the third computation, which settles each mismatching element.
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
  double *B;        // B at row r0
  int64_t ldb;
  bool trans, unit, fwd, dmr;
  const ftd::DmrFault *f;  // faults of this block: index = local row i, step = local p (p < i fwd)
  int nf;
  unsigned long long *cnt;  // ftd::D_* counters
};

__device__ __forceinline__ double leaf_a(const LeafParams &P, int p, int i) {  // S(p, i) = op(A)(p, i)
  return P.trans ? P.A[i + (int64_t)p * P.lda] : P.A[p + (int64_t)i * P.lda];
}

// One column's solve, both DMR copies in the same pass (two independent dependence chains
// interleaved: x1 / x2 broadcast by two shuffles per step); the step's column of S is loaded
// first so the shared-memory latency overlaps the shuffle.  The fault hook (original copy
// only) adds delta to b_fi after the update from x_fstep.
template <bool DUAL>
__device__ __forceinline__ void leaf_column(const LeafParams &P, const double *Sc, const double *rd1,
                                            const double *rd2, double (&b1)[4], double (&b2)[4], int lane, int fi,
                                            int fstep, double fdel) {
  const int nb = P.nb;
  for (int s = 0; s < nb; ++s) {
    const int i = P.fwd ? s : nb - 1 - s;
    const int owner = i & 31, slot = i >> 5;
    double sv[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) sv[q] = lane + 32 * q < nb ? Sc[i * nb + lane + 32 * q] : 0.0;
    double bi1 = b1[0], bi2 = b2[0];
#pragma unroll
    for (int q = 1; q < 4; ++q) {
      bi1 = slot == q ? b1[q] : bi1;
      if (DUAL) bi2 = slot == q ? b2[q] : bi2;
    }
    const double x1 = __shfl_sync(0xffffffffu, P.unit ? bi1 : ftd::v_mul(bi1, rd1[i]), owner);
    const double x2 = DUAL ? __shfl_sync(0xffffffffu, P.unit ? bi2 : ftd::v_mul(bi2, rd2[i]), owner) : 0.0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int p = lane + 32 * q;
      if (q == slot && lane == owner) {
        b1[q] = x1;
        if (DUAL) b2[q] = x2;
      }
      const bool upd = P.fwd ? (p > i && p < nb) : (p < i);
      if (upd) {
        b1[q] = ftd::v_fma(-sv[q], x1, b1[q]);
        if (DUAL) b2[q] = ftd::v_fma(-sv[q], x2, b2[q]);
      }
      if (p == fi && i == fstep) b1[q] = ftd::v_add(b1[q], fdel);
    }
  }
}

__global__ void __launch_bounds__(512) trsm_leaf_kernel(const LeafParams P) {
  extern __shared__ double sm[];
  double *Sc = sm, *rd1 = sm + LEAF * LEAF, *rd2 = rd1 + LEAF;
  const int nb = P.nb, tid = threadIdx.x, lane = tid & 31;
  for (int e = tid; e < nb * nb; e += blockDim.x) {
    const int i = e / nb, p = e % nb;
    Sc[i * nb + p] = leaf_a(P, p, i);
  }
  __syncthreads();
  for (int i = tid; i < nb; i += blockDim.x) {  // packed reciprocals of the diagonal, twice
    rd1[i] = 1.0 / Sc[i * nb + i];
    rd2[i] = 1.0 / Sc[i * nb + i];
  }
  __syncthreads();
  const int warps = blockDim.x >> 5;
  for (int j = blockIdx.x * warps + (tid >> 5); j < P.n; j += gridDim.x * warps) {
    double *col = P.B + (int64_t)j * P.ldb;
    // This lane's fault in column j, if any (at most one per lane is honoured).
    int fi = -1, fstep = -1;
    double fdel = 0.0;
    for (int e = 0; e < P.nf; ++e) {
      const int64_t code = P.f[e].index;  // j * LEAF + local row
      if (code / LEAF == j && (int)(code % LEAF) % 32 == lane) { fi = (int)(code % LEAF); fstep = (int)P.f[e].step; fdel = P.f[e].delta; }
    }
    double b1[4], b2[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int p = lane + 32 * q;
      b1[q] = p < nb ? col[p] : 0.0;
      b2[q] = b1[q];
    }
    if (P.dmr) leaf_column<true>(P, Sc, rd1, rd2, b1, b2, lane, fi, fstep, fdel);
    else leaf_column<false>(P, Sc, rd1, rd2, b1, b2, lane, -1, -1, 0.0);
    bool bad = false;
    if (P.dmr)
#pragma unroll
    for (int q = 0; q < 4; ++q) bad |= (lane + 32 * q < nb) && ftd::differ(b1[q], b2[q]);
    if (__any_sync(0xffffffffu, bad)) {
      // Rare: a third computation settles the column (the verification unit of a diagonal
      // block: one fault propagates to every later row of the column).  Each element takes
      // the third value; the column is corrected when the third agrees with one copy wherever
      // the two disagreed.
      double b3[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) b3[q] = lane + 32 * q < nb ? col[lane + 32 * q] : 0.0;
      double b4[4];
      leaf_column<false>(P, Sc, rd2, rd2, b3, b4, lane, -1, -1, 0.0);
      bool unsettled = false;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (lane + 32 * q < nb && ftd::differ(b1[q], b2[q]))
          unsettled |= ftd::differ(b3[q], b1[q]) && ftd::differ(b3[q], b2[q]);
        b1[q] = b3[q];
      }
      unsettled = __any_sync(0xffffffffu, unsettled);
      if (lane == 0) {
        atomicAdd(&P.cnt[ftd::D_DETECTED], 1ull);
        atomicAdd(&P.cnt[unsettled ? ftd::D_UNCORRECTABLE : ftd::D_CORRECTED], 1ull);
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (lane + 32 * q < nb) col[lane + 32 * q] = b1[q];
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
