// unfused.cuh — kernels of the UNFUSED ABFT baseline.
//
// The paper's comparison point for its fused design is the classic unfused ABFT DGEMM
// (§V.A, the overhead model (6 + 2K/Kc) P_mm / (n P_mv); §V.B
// "the reference checksums ... were the main cost of unfused ABFT"): checksums are encoded
// by separate memory passes, the product is an ordinary GEMM, the carried checksums
// (e^T A)B and A(Be) are separate (skinny) GEMMs, and the reference checksums e^T C, C e are
// another memory pass over C before a verify / locate / correct step.  Here every piece is a
// B200 kernel of this library (the GEMMs are the unprotected DMMA kernel of dgemm_abft.cuh),
// with the same verification unit semantics as the fused path but on 128 x 128 units (no
// C^f tile: the checksums live outside C).
//
// With a verification interval Kc < k ("for each rank-Kc update") the product
// and the carried checksums are formed Kc updates at a time and C is verified after each:
// the reference row sums C e first (one memory pass), the column sums e^T C only when a row
// mismatched (the paper's "C^r first, C^c only on mismatch"), then locate / correct.
//
//   block_sum_kernel   S[xb + p*lds] = sum_{x in block xb} X(x, p)   (+ running max |hi|)
//                      used for e^T A_I (x = i), B_J e (x = j), e^T C_IJ and C_IJ e
//   row_check_kernel   one thread per (row i, column block J): C_J e against A (B_J e); marks
//                      the unit and raises the "mismatch" flag that enables the e^T C pass
//   verify_kernel      one CTA per flagged unit: residuals, threshold, classify, correct in place
//   axpby_kernel       C = alpha*T + beta*C0 when the verified product lives in scratch
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace ftu {

constexpr int UB = 128;  // unit rows / columns of the unfused path

// Sum of the bs-long (127 or 128) x-blocks of X(x, p), element at X[x*sx + p*sp] with sx == 1 (XC) or
// sp == 1 (!XC).  One CTA of 256 threads per (x-block, 32 p) for XC, (x-block, 256 p) for
// !XC; every global read is coalesced.  hmax (optional) receives max over the block of the
// high word of |X| (reading R1': maxima tracked on 32-bit words, non-finite -> DBL_MAX's).
template <bool XC>
__global__ void __launch_bounds__(256) block_sum_kernel(const double *__restrict__ X, int64_t ld, int64_t nx,
                                                        int64_t np, double *__restrict__ S, int64_t lds,
                                                        unsigned int *__restrict__ hmax, int bs,
                                                        const int *__restrict__ enable) {
  if (enable && *enable == 0) return;  // a pass that runs only on mismatch (e^T C)
  const int64_t xb = blockIdx.x, x0 = xb * bs;  // block size bs <= 128
  const int xn = (int)min((int64_t)bs, nx - x0);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  unsigned int hm = 0;
  if (XC) {
    // element (x, p) at X[x + p*ld]: a warp sums 4 columns p of 128 contiguous x.
    const int64_t pbase = (int64_t)blockIdx.y * 32 + warp * 4;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int64_t p = pbase + q;
      if (p >= np) break;  // warp-uniform
      const double *col = X + p * ld + x0;
      double s = 0.0;
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int x = lane + 32 * r;
        const double v = x < xn ? col[x] : 0.0;
        s += v;
        hm = max(hm, (unsigned)__double2hiint(v) & 0x7FFFFFFFu);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) S[xb + p * lds] = s;
    }
    if (hm >= 0x7FF00000u) hm = 0x7FEFFFFFu;  // non-finite -> DBL_MAX (R1')
  } else {
    // element (x, p) at X[x*ld + p]: thread t sums column p = p0 + t over the block's x.
    const int64_t p = (int64_t)blockIdx.y * 256 + tid;
    if (p < np) {
      double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
      const double *base = X + x0 * ld + p;
      int x = 0;
      for (; x + 4 <= xn; x += 4) {
        const double v0 = base[(int64_t)x * ld], v1 = base[(int64_t)(x + 1) * ld];
        const double v2 = base[(int64_t)(x + 2) * ld], v3 = base[(int64_t)(x + 3) * ld];
        s0 += v0; s1 += v1; s2 += v2; s3 += v3;
        if (hmax) {
          unsigned h0 = (unsigned)__double2hiint(v0) & 0x7FFFFFFFu, h1 = (unsigned)__double2hiint(v1) & 0x7FFFFFFFu;
          unsigned h2 = (unsigned)__double2hiint(v2) & 0x7FFFFFFFu, h3 = (unsigned)__double2hiint(v3) & 0x7FFFFFFFu;
          hm = max(hm, max(max(h0, h1), max(h2, h3)));
        }
      }
      for (; x < xn; ++x) {
        const double v = base[(int64_t)x * ld];
        s0 += v;
        hm = max(hm, (unsigned)__double2hiint(v) & 0x7FFFFFFFu);
      }
      S[xb + p * lds] = (s0 + s1) + (s2 + s3);
      if (hm >= 0x7FF00000u) hm = 0x7FEFFFFFu;  // non-finite -> DBL_MAX (R1')
    }
  }
  if (hmax) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) hm = max(hm, __shfl_xor_sync(0xffffffffu, hm, o));
    if (lane == 0) atomicMax(hmax + xb, hm);
  }
}

struct VerifyParams {
  int64_t m, n, k;   // k: updates accumulated so far (the end of the interval being verified)
  int interval;      // verification interval index t
  const int *unit_flag;  // row-check marks (null: verify every unit)
  char ta, tb;
  const double *A;
  int64_t lda;
  const double *B;
  int64_t ldb;
  double *T;  // the product op(A) op(B) being verified (C itself when alpha == 1, beta == 0)
  int64_t ldt;
  const double *Rc, *CSc;  // e^T C_I (nbm x n, ld ldm), (e^T A_I) B (same layout)
  int64_t ldm;
  const double *Rr;        // C_J e as Rr[J + i*ldn]
  int64_t ldn;
  const double *CSr;       // A (B_J e) as CSr[i + J*ldr]
  int64_t ldr;
  const unsigned int *amax_hi, *bmax_hi;
  // the encoded block sums (e^T A_I as Ac[I + p*ldm], B_J e as Br[J + p*ldn]) and the carried
  // checksums to re-form for a recomputed unit (null when there is no later interval)
  const double *Ac, *Br;
  double *CSc_w, *CSr_w;
  int nbm, nbn;
  int correct_mode;
  unsigned long long *counters;  // [detected, corrected, recomputed, events] (ftk::CNT_*)
  void *events;                  // ftk::EventDev[ev_cap]
  long long ev_cap;
};

struct EventU {  // layout-identical to ftk::EventDev
  long long i, j;
  int kind, interval;
  double residual_row, residual_col;
};

__device__ __forceinline__ double opA(const VerifyParams &P, int64_t i, int64_t p) {
  return (P.ta == 'N' || P.ta == 'n') ? P.A[i + p * P.lda] : P.A[p + i * P.lda];
}
__device__ __forceinline__ double opB(const VerifyParams &P, int64_t p, int64_t j) {
  return (P.tb == 'N' || P.tb == 'n') ? P.B[p + j * P.ldb] : P.B[j + p * P.ldb];
}

// One CTA (256 threads) per 128 x 128 unit (I, J): thread t < 128 owns column J*128 + t,
// thread 128 + t row I*128 + t.  Same threshold, classification and correction as the fused
// epilogue (R1, R1', R4, R6).
__global__ void __launch_bounds__(256) verify_kernel(const VerifyParams P) {
  __shared__ double dres[256];
  __shared__ double red[8];
  __shared__ int first_row, first_col;
  const int unit = blockIdx.x, I = unit % P.nbm, J = unit / P.nbm;
  if (P.unit_flag && P.unit_flag[unit] == 0) return;  // its rows matched: clean
  const int tid = threadIdx.x, lane = tid & 31;
  const int64_t i0 = (int64_t)I * UB, j0 = (int64_t)J * UB;
  const int bm = (int)min((int64_t)UB, P.m - i0), bn = (int)min((int64_t)UB, P.n - j0);
  if (tid == 0) { first_row = 0x7fffffff; first_col = 0x7fffffff; }
  __syncthreads();
  const bool is_row = tid >= 128;
  const int c = tid & 127;
  const bool valid = is_row ? c < bm : c < bn;
  double d = 0.0;
  if (valid) {
    if (is_row) {
      const int64_t i = i0 + c;
      d = P.Rr[J + i * P.ldn] - P.CSr[i + J * P.ldr];
    } else {
      const int64_t j = j0 + c;
      d = P.Rc[I + j * P.ldm] - P.CSc[I + j * P.ldm];
    }
  }
  const double amx = __longlong_as_double((long long)(((unsigned long long)P.amax_hi[I] << 32) | 0xFFFFFFFFull));
  const double bmx = __longlong_as_double((long long)(((unsigned long long)P.bmax_hi[J] << 32) | 0xFFFFFFFFull));
  const int len = is_row ? bn : bm;
  const double nu = (double)(P.k + len) * 0x1p-53;
  const double tau = fmin(2.0 * (nu / (1.0 - nu)) * (double)P.k * (double)len * amx * bmx, 0x1.fffffffffffffp1023);  // R1, R13
  const bool flag = valid && !(fabs(d) <= tau);
  dres[tid] = d;
  if (flag) atomicMin(is_row ? &first_row : &first_col, c);
  const int nfr = __syncthreads_count(flag && is_row);
  const int nfc = __syncthreads_count(flag && !is_row);
  if (nfr == 0 && nfc == 0) return;
  const bool multi = !(nfr == 1 && nfc == 1);
  const int fr = first_row, fc = first_col;
  if (!multi) {
    FT_CHECK(fr < bm && fc < bn);
    const int64_t gi = i0 + fr, gj = j0 + fc;
    double *tij = P.T + gi + gj * P.ldt;
    if (P.correct_mode == 1) {
      if (tid == 0) *tij -= dres[fc];  // subtract d_col
    } else {
      double part = 0.0;  // recompute (R4)
      for (int64_t p = tid; p < P.k; p += 256) part = fma(opA(P, gi, p), opB(P, p, gj), part);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
      if (lane == 0) red[tid >> 5] = part;
      __syncthreads();
      if (tid == 0) {
        double v = 0.0;
#pragma unroll
        for (int q = 0; q < 8; ++q) v += red[q];
        *tij = v;
      }
    }
  } else {
    // Out of the one-error model: recompute the unit once, no re-verification (R6); with
    // later intervals to come its carried checksums are re-formed too (R6').
    for (int e = tid; e < bm * bn; e += 256) {
      const int64_t gi = i0 + e % bm, gj = j0 + e / bm;
      double v = 0.0;
      for (int64_t p = 0; p < P.k; ++p) v = fma(opA(P, gi, p), opB(P, p, gj), v);
      P.T[gi + gj * P.ldt] = v;
    }
    if (P.Ac) {
      for (int c = tid; c < bn + bm; c += 256) {
        double v = 0.0;
        if (c < bn) {  // (e^T A_I) B_J, column j0 + c
          for (int64_t p = 0; p < P.k; ++p) v = fma(P.Ac[I + p * P.ldm], opB(P, p, j0 + c), v);
          P.CSc_w[I + (j0 + c) * P.ldm] = v;
        } else {       // A_I (B_J e), row i0 + c - bn
          const int64_t gi = i0 + c - bn;
          for (int64_t p = 0; p < P.k; ++p) v = fma(opA(P, gi, p), P.Br[J + p * P.ldn], v);
          P.CSr_w[gi + J * P.ldr] = v;
        }
      }
    }
  }
  if (tid == 0) {
    atomicAdd(&P.counters[0], 1ull);
    atomicAdd(&P.counters[multi ? 2 : 1], 1ull);
    const unsigned long long slot = atomicAdd(&P.counters[3], 1ull);
    EventU *ev = reinterpret_cast<EventU *>(P.events);
    if ((long long)slot < P.ev_cap)
      ev[slot] = multi ? EventU{(long long)i0, (long long)j0, 2, P.interval, nfr ? dres[128 + fr] : 0.0, nfc ? dres[fc] : 0.0}
                       : EventU{(long long)(i0 + fr), (long long)(j0 + fc), 1, P.interval, dres[128 + fr], dres[fc]};
  }
}

// The reference row checksums first: one thread per (row i, column block J)
// compares (C_J e)_i with (A (B_J e))_i against the row threshold of unit (i / 128, J); a
// mismatch marks the unit and enables the e^T C pass and the verify kernel.
__global__ void row_check_kernel(int64_t m, int64_t n, int64_t kt, const double *__restrict__ Rr, int64_t ldn,
                                 const double *__restrict__ CSr, int64_t ldr, const unsigned int *__restrict__ amax_hi,
                                 const unsigned int *__restrict__ bmax_hi, int nbm, int nbn, int *__restrict__ unit_flag,
                                 int *__restrict__ any) {
  const int64_t total = m * nbn;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % m;
    const int J = (int)(e / m), I = (int)(i / UB);
    const int bn = (int)min((int64_t)UB, n - (int64_t)J * UB);
    const double d = Rr[J + i * ldn] - CSr[i + J * ldr];
    const double amx = __longlong_as_double((long long)(((unsigned long long)amax_hi[I] << 32) | 0xFFFFFFFFull));
    const double bmx = __longlong_as_double((long long)(((unsigned long long)bmax_hi[J] << 32) | 0xFFFFFFFFull));
    const double nu = (double)(kt + bn) * 0x1p-53;
    const double tau = fmin(2.0 * (nu / (1.0 - nu)) * (double)kt * (double)bn * amx * bmx, 0x1.fffffffffffffp1023);
    if (!(fabs(d) <= tau)) {
      unit_flag[I + (int64_t)J * nbm] = 1;
      *any = 1;
    }
  }
}

// C = alpha*T + beta*C0 (C0 not read when beta == 0), two roundings, no contraction.
__global__ void axpby_kernel(int64_t m, int64_t n, double alpha, const double *__restrict__ T, int64_t ldt,
                             double beta, double *__restrict__ C, int64_t ldc) {
  const int64_t total = m * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % m, j = e / m;
    const double v = __dmul_rn(alpha, T[i + j * ldt]);
    double *c = C + i + j * ldc;
    *c = beta != 0.0 ? __dadd_rn(v, __dmul_rn(beta, *c)) : v;
  }
}

}  // namespace ftu
