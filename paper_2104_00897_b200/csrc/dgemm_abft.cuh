// dgemm_abft.cuh — sm_100a kernels of the online ABFT DGEMM (FT-BLAS, arXiv 2104.00897).
//
// One CTA computes one BM x BN tile of C = alpha*op(A)*op(B) + beta*C and is one
// verification unit (§II.A restricted to the tile; R5):
//
//   mainloop  (per BK-deep stage s, 256 threads = 8 MMA warps in a 2 x 4 grid of 64x32
//              warp tiles; cp.async multistage ring in shared memory)
//     - operand staging: every element of the A/B tiles is loaded from global memory
//       ONCE into shared memory and reused by the MMA, by the checksum encode and by
//       the checksum carry ("each B element reused three times", §V.B)
//     - encode(s):  a_sum[p] = sum_{i in I} op(A)_ip   (e^T A)
//                   b_sum[p] = sum_{j in J} op(B)_pj   (B e)
//                   running max|op(A)_I|, max|op(B)_J| for the threshold (R1)
//     - carry(s-1): cs_col[j] += a_sum[p]*op(B)_pj,  cs_row[i] += op(A)_ip*b_sum[p]
//                   (outer-product checksum maintenance), one stage behind
//                   the encode so that a single barrier per stage suffices
//     - fault hook: injected deltas land in the owning accumulator at stage boundaries
//     - update:     acc += A_tile * B_tile with DMMA.8x8x4 (mma.sync m8n8k4 f64), the only
//                   FP64 tensor instruction sm_100a provides (tcgen05 has no f64 kind)
//   epilogue
//     - stage acc through shared memory; reference checksums r_col = e^T C_IJ and
//       r_row = C_IJ e reuse the computed C ("reuse the computed C elements ... to update
//       the reference checksums")
//     - residuals d = r - cs, flag where not |d| <= tau, classify with block counts:
//       exactly one row and one column -> locate and correct in place;
//       any other pattern -> recompute the tile once (R6)
//     - C = alpha*acc + beta*C0 (C0 not read when beta == 0), coalesced column stores
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace ftk {

constexpr int BM = 128, BN = 128, BK = 16;
constexpr int STAGES = 5;               // shared-memory ring depth
constexpr int LOOKAHEAD = STAGES - 2;   // stages in flight (carry lags the encode by one)
constexpr int NTHREADS = 256;           // 8 MMA warps
constexpr int LD_MN = 130;              // MN-major tile pitch (doubles): conflict-free LDS.128
constexpr int TILE_ELEMS = BK * LD_MN;  // >= 128*BK (K-major tile, dense + XOR swizzle)
constexpr int STAGE_ELEMS = 2 * TILE_ELEMS;
constexpr int LDC_S = 129;              // epilogue C-tile pitch (doubles)
static_assert(BM * LDC_S <= STAGES * STAGE_ELEMS, "C tile must fit in the stage ring");

struct FaultDev {        // one armed fault, sorted by (tile, stage)
  int32_t tile, stage;   // tile = ti + tj*tiles_m; stage = floor(step / BK)
  int32_t li, lj;        // tile-local row / column
  double delta;
};

struct EventDev {
  long long i, j;
  int kind, interval;
  double residual_row, residual_col;
};

enum { CNT_DETECTED = 0, CNT_CORRECTED, CNT_RECOMPUTED, CNT_EVENTS, CNT_N };

struct Params {
  int64_t m, n, k;
  double alpha, beta;
  const double *A;
  int64_t lda;
  const double *B;
  int64_t ldb;
  double *C;
  int64_t ldc;
  int tiles_m, tiles_n, nk;
  const FaultDev *faults;
  int nfaults;
  int correct_mode;               // 0 recompute, 1 subtract
  unsigned long long *counters;   // [CNT_N]
  EventDev *events;
  long long ev_cap;
};

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ void dmma_8x8x4(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

__device__ __forceinline__ int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }
__device__ __forceinline__ int64_t max64(int64_t a, int64_t b) { return a > b ? a : b; }

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// 16-byte async copy, zero-filling bytes beyond src_bytes (0, 8 or 16).
__device__ __forceinline__ void cp_async16(void *sdst, const void *gsrc, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(sdst)), "l"(gsrc),
               "r"(src_bytes));
}
// 8-byte async copy, zero-fill when src_bytes == 0.
__device__ __forceinline__ void cp_async8(void *sdst, const void *gsrc, int src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(sdst)), "l"(gsrc),
               "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// |x| as ordered bits; NaN contributes 0 (the oracle's fabs(a) > amax ignores NaN too).
__device__ __forceinline__ unsigned long long absbits(double x) {
  unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(x)) & 0x7FFFFFFFFFFFFFFFull;
  return b <= 0x7FF0000000000000ull ? b : 0ull;
}
__device__ __forceinline__ unsigned long long umax64(unsigned long long a, unsigned long long b) {
  return a > b ? a : b;
}

// ------------------------------------------------------------------ shared-memory layouts
// An operand tile X holds the 128 x BK block X(x, p), x the M (or N) index, p the K index.
//  MN-major (x contiguous in global memory: op(A) with 'N', op(B) with 'T'):
//     X(x,p) at [p*LD_MN + x]; LD_MN = 130 makes the fragment LDS.128 conflict-free.
//  K-major  (p contiguous in global memory: op(A) with 'T', op(B) with 'N'):
//     X(x,p) at [x*16 + 2*((p/2) ^ ((x&1)<<2)) + (p&1)]: dense 128-byte rows, 16-byte
//     chunks XOR-swizzled by row parity so the fragment LDS.128 is conflict-free.
template <bool KM>
__device__ __forceinline__ int sidx(int x, int p) {
  if (KM) return x * 16 + ((((p >> 1) ^ ((x & 1) << 2))) << 1) + (p & 1);
  return p * LD_MN + x;
}

// Asynchronously load the X tile for rows [x0, x0+128) and k in [k0, k0+BK).
// Global element (x, p) is g[(x0+x) + (k0+p)*ld] (MN-major) or g[(k0+p) + (x0+x)*ld]
// (K-major).  Out-of-range elements are zero-filled (zeros contribute exactly nothing to
// the product, the checksums or the maxima; R14).
template <bool KM, bool V16>
__device__ __forceinline__ void load_tile(double *s, const double *g, int64_t ld, int64_t x0,
                                          int64_t xlim, int64_t k0, int64_t k, int tid) {
  if (V16) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int c = tid + NTHREADS * r;  // 1024 16-byte chunks per tile
      int x, p;
      if (KM) { x = c >> 3; p = (c & 7) * 2; }
      else    { p = c >> 6; x = (c & 63) * 2; }
      const int64_t gx = x0 + x, gp = k0 + p;
      int nval;
      const double *src;
      if (KM) {
        nval = (gx < xlim) ? (int)min64(max64(k - gp, 0), 2) : 0;
        src = g + gp + gx * ld;
      } else {
        nval = (gp < k) ? (int)min64(max64(xlim - gx, 0), 2) : 0;
        src = g + gx + gp * ld;
      }
      cp_async16(s + sidx<KM>(x, p), nval ? src : g, nval * 8);
    }
  } else {
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const int c = tid + NTHREADS * r;  // 2048 elements per tile
      int x, p;
      if (KM) { x = c >> 4; p = c & 15; }
      else    { p = c >> 7; x = c & 127; }
      const int64_t gx = x0 + x, gp = k0 + p;
      const bool ok = gx < xlim && gp < k;
      const double *src = KM ? g + gp + gx * ld : g + gx + gp * ld;
      cp_async8(s + sidx<KM>(x, p), ok ? src : g, ok ? 8 : 0);
    }
  }
}

// ------------------------------------------------------------------ register fragments
// k-slot mapping inside a BK=16 stage: k-step s (0..3), lane slot t (0..3) <-> p =
// 8*(s>>1) + 2t + (s&1).  Both operands use it, so the MMA sums the same p's.
// Warp tile: 64 rows (8 m-tiles of 8) x 32 cols (4 n-tiles of 8).
// Row of m-tile mt, fragment row g:   MN-major: 16*(mt>>1) + 2g + (mt&1);  K-major: 8*mt + g.
// Same mapping for columns of B's n-tiles.
template <bool KM, int NT>
__device__ __forceinline__ void load_frags(const double *s, int xw, int h, int g, int t,
                                           double (&f)[2][NT]) {
  if (KM) {
#pragma unroll
    for (int r = 0; r < NT; ++r) {
      const int x = xw + 8 * r + g;
      const double2 v = *reinterpret_cast<const double2 *>(s + x * 16 + (((4 * h + t) ^ ((x & 1) << 2)) << 1));
      f[0][r] = v.x;
      f[1][r] = v.y;
    }
  } else {
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int p = 8 * h + 2 * t + e;
#pragma unroll
      for (int q = 0; q < NT / 2; ++q) {
        const double2 v = *reinterpret_cast<const double2 *>(s + p * LD_MN + xw + 16 * q + 2 * g);
        f[e][2 * q] = v.x;
        f[e][2 * q + 1] = v.y;
      }
    }
  }
}

template <bool KM>
__device__ __forceinline__ int tile_row(int r, int g) {  // r: m/n-tile index, g: index in tile
  return KM ? 8 * r + g : 16 * (r >> 1) + 2 * g + (r & 1);
}

// ------------------------------------------------------------------ fused encode
// Warp w reduces p = 2w and 2w+1 over all 128 rows of an operand tile.
// Writes xsum[2w], xsum[2w+1]; folds |x| into the running max bits.
template <bool KM>
__device__ __forceinline__ void encode_tile(const double *s, int warp, int lane, double *xsum,
                                            unsigned long long &xmax) {
  if (KM) {
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int x = lane + 32 * r;
      const double2 v = *reinterpret_cast<const double2 *>(s + x * 16 + ((warp ^ ((x & 1) << 2)) << 1));
      s0 += v.x;
      s1 += v.y;
      xmax = umax64(xmax, umax64(absbits(v.x), absbits(v.y)));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      s0 += __shfl_xor_sync(0xffffffffu, s0, o);
      s1 += __shfl_xor_sync(0xffffffffu, s1, o);
    }
    if (lane == 0) { xsum[2 * warp] = s0; xsum[2 * warp + 1] = s1; }
  } else {
    const int p = 2 * warp + (lane >> 4), l16 = lane & 15;
    double acc = 0.0;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const double2 v = *reinterpret_cast<const double2 *>(s + p * LD_MN + 2 * l16 + 32 * r);
      acc += v.x + v.y;
      xmax = umax64(xmax, umax64(absbits(v.x), absbits(v.y)));
    }
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (l16 == 0) xsum[p] = acc;
  }
}

// Carry for one stage: thread (c = tid & 127, half h = tid >> 7) accumulates
// cs_col[c] += sum_{p in half} a_sum[p]*B(p,c) and cs_row[c] += sum_p A(c,p)*b_sum[p].
template <bool AKM, bool BKM>
__device__ __forceinline__ void carry_stage(const double *sA, const double *sB, const double *asum,
                                            const double *bsum, int c, int h, double &cs_col,
                                            double &cs_row) {
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int p = 8 * h + q;
    cs_col = fma(asum[p], sB[sidx<BKM>(c, p)], cs_col);
    cs_row = fma(sA[sidx<AKM>(c, p)], bsum[p], cs_row);
  }
}

// ------------------------------------------------------------------ the kernel
struct SmemTail {
  double asum[2][BK], bsum[2][BK];
  double cs_part[2][2][128];      // [col/row][half][index]
  double dres[NTHREADS];          // residuals d (0..127 columns, 128..255 rows)
  double red[NTHREADS / 32];
  unsigned long long amax, bmax;
  int first_row, first_col;
};
constexpr size_t SMEM_BYTES = sizeof(double) * STAGES * STAGE_ELEMS + sizeof(SmemTail);

template <bool AKM, bool BKM, bool FT, bool V16>
__global__ void __launch_bounds__(NTHREADS, 1) dgemm_abft_kernel(const Params P) {
  extern __shared__ __align__(16) double smem[];
  double *const ring = smem;
  SmemTail &tl = *reinterpret_cast<SmemTail *>(smem + STAGES * STAGE_ELEMS);
  double *const ctile = smem;  // epilogue reuse of the ring

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp >> 2, wn = warp & 3;  // 2 x 4 warp grid
  const int ti = blockIdx.x, tj = blockIdx.y;
  const int tile = ti + tj * P.tiles_m;
  const int64_t i0 = (int64_t)ti * BM, j0 = (int64_t)tj * BN;
  const int bm_eff = (int)min64(BM, P.m - i0), bn_eff = (int)min64(BN, P.n - j0);
  const int nk = P.nk;

  // Faults of this tile: [f_lo, f_hi) in the (tile, stage)-sorted list.
  int f_lo = 0, f_hi = 0;
  if (P.nfaults > 0) {
    int lo = 0, hi = P.nfaults;
    while (lo < hi) { const int mid = (lo + hi) >> 1; if (P.faults[mid].tile < tile) lo = mid + 1; else hi = mid; }
    f_lo = lo;
    hi = P.nfaults;
    while (lo < hi) { const int mid = (lo + hi) >> 1; if (P.faults[mid].tile <= tile) lo = mid + 1; else hi = mid; }
    f_hi = lo;
  }

  double acc[8][4][2];
  for (int attempt = 0;; ++attempt) {
    const bool verify = FT && attempt == 0;
    const bool inject = attempt == 0 && f_lo < f_hi;
    int fnext = f_lo;
    int next_stage = inject ? P.faults[fnext].stage : 0x7fffffff;

#pragma unroll
    for (int a = 0; a < 8; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
    double cs_col = 0.0, cs_row = 0.0;
    unsigned long long amax = 0ull, bmax = 0ull;
    if (tid == 0) { tl.amax = 0ull; tl.bmax = 0ull; tl.first_row = 0x7fffffff; tl.first_col = 0x7fffffff; }

    auto load_stage = [&](int s) {
      if (s < nk) {
        double *sa = ring + (s % STAGES) * STAGE_ELEMS;
        load_tile<AKM, V16>(sa, P.A, P.lda, i0, P.m, (int64_t)s * BK, P.k, tid);
        load_tile<BKM, V16>(sa + TILE_ELEMS, P.B, P.ldb, j0, P.n, (int64_t)s * BK, P.k, tid);
      }
      cp_async_commit();
    };
    auto apply_faults = [&](int s) {
      while (s == next_stage) {
        const FaultDev f = P.faults[fnext];
        const int lr = f.li & 63, lc = f.lj & 31;
        const int fmt = AKM ? (lr >> 3) : 2 * (lr >> 4) + (lr & 1);
        const int fg = AKM ? (lr & 7) : ((lr & 15) >> 1);
        const int fnt = BKM ? (lc >> 3) : 2 * (lc >> 4) + (lc & 1);
        const int cc = BKM ? (lc & 7) : ((lc & 15) >> 1);
        // Register index of the owning accumulator, -1 for every other thread.  Select-based
        // (no dynamic register indexing) so the accumulators stay in registers.
        const bool owner = (f.li >> 6) == wm && (f.lj >> 5) == wn && lane == fg * 4 + (cc >> 1);
        const int fidx = owner ? (fmt * 4 + fnt) * 2 + (cc & 1) : -1;
#pragma unroll
        for (int a = 0; a < 8; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const double v = acc[a][b][e];
              acc[a][b][e] = ((a * 4 + b) * 2 + e == fidx) ? v + f.delta : v;
            }
        ++fnext;
        next_stage = fnext < f_hi ? P.faults[fnext].stage : 0x7fffffff;
      }
    };

    // Prologue.
#pragma unroll
    for (int s = 0; s < LOOKAHEAD; ++s) load_stage(s);

    for (int s = 0; s < nk; ++s) {
      cp_async_wait<LOOKAHEAD - 1>();
      __syncthreads();
      load_stage(s + LOOKAHEAD);
      const double *sA = ring + (s % STAGES) * STAGE_ELEMS;
      const double *sB = sA + TILE_ELEMS;
      if (verify) {
        encode_tile<AKM>(sA, warp, lane, tl.asum[s & 1], amax);
        encode_tile<BKM>(sB, warp, lane, tl.bsum[s & 1], bmax);
        if (s > 0) {
          const double *pA = ring + ((s - 1) % STAGES) * STAGE_ELEMS;
          carry_stage<AKM, BKM>(pA, pA + TILE_ELEMS, tl.asum[(s - 1) & 1], tl.bsum[(s - 1) & 1],
                                tid & 127, tid >> 7, cs_col, cs_row);
        }
      }
      if (inject) apply_faults(s);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        double af[2][8], bf[2][4];
        load_frags<AKM, 8>(sA, wm * 64, h, g, t, af);
        load_frags<BKM, 4>(sB, wn * 32, h, g, t, bf);
#pragma unroll
        for (int e = 0; e < 2; ++e)
#pragma unroll
          for (int a = 0; a < 8; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) dmma_8x8x4(acc[a][b], af[e][a], bf[e][b]);
      }
    }
    cp_async_wait<0>();
    __syncthreads();
    if (verify && nk > 0) {
      const double *pA = ring + ((nk - 1) % STAGES) * STAGE_ELEMS;
      carry_stage<AKM, BKM>(pA, pA + TILE_ELEMS, tl.asum[(nk - 1) & 1], tl.bsum[(nk - 1) & 1],
                            tid & 127, tid >> 7, cs_col, cs_row);
    }
    if (inject) apply_faults(nk);  // faults with step_q == k
    __syncthreads();               // ring no longer read: reuse it as the C tile

    // Stage the accumulator tile through shared memory: ctile[col*LDC_S + row].
#pragma unroll
    for (int a = 0; a < 8; ++a) {
      const int row = wm * 64 + tile_row<AKM>(a, g);
#pragma unroll
      for (int b = 0; b < 4; ++b)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int col = wn * 32 + tile_row<BKM>(b, 2 * t + e);
          ctile[col * LDC_S + row] = acc[a][b][e];
        }
    }
    if (verify) {
      tl.cs_part[0][tid >> 7][tid & 127] = cs_col;
      tl.cs_part[1][tid >> 7][tid & 127] = cs_row;
      // CTA-wide maxima for the threshold.
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        amax = umax64(amax, __shfl_xor_sync(0xffffffffu, amax, o));
        bmax = umax64(bmax, __shfl_xor_sync(0xffffffffu, bmax, o));
      }
      if (lane == 0) { atomicMax(&tl.amax, amax); atomicMax(&tl.bmax, bmax); }
    }
    __syncthreads();

    if (!verify) break;

    // ---- verification: reference checksums from the computed tile.
    const int c = tid & 127;
    const bool is_row = tid >= 128;
    double r = 0.0;
    if (is_row) {
#pragma unroll 8
      for (int j = 0; j < BN; ++j) r += ctile[j * LDC_S + c];
    } else {
#pragma unroll 8
      for (int i = 0; i < BM; ++i) r += ctile[c * LDC_S + i];
    }
    const double cs = tl.cs_part[is_row][0][c] + tl.cs_part[is_row][1][c];
    const double d = r - cs;
    const double amx = __longlong_as_double((long long)tl.amax), bmx = __longlong_as_double((long long)tl.bmax);
    const int64_t kt = P.k;
    const int len = is_row ? bn_eff : bm_eff;
    const double nu = (double)(kt + len) * 0x1p-53;
    const double tau = 2.0 * (nu / (1.0 - nu)) * (double)kt * (double)len * amx * bmx;  // DESIGN.md R1
    const bool valid = is_row ? (c < bm_eff) : (c < bn_eff);
    const bool flag = valid && !(fabs(d) <= tau);
    tl.dres[tid] = d;
    if (flag) atomicMin(is_row ? &tl.first_row : &tl.first_col, c);
    const int nfr = __syncthreads_count(flag && is_row);
    const int nfc = __syncthreads_count(flag && !is_row);
    if (nfr == 0 && nfc == 0) break;  // clean unit

    const int fr = tl.first_row, fc = tl.first_col;
    if (nfr == 1 && nfc == 1) {
      // Single error at the intersection (i0+fr, j0+fc): correct in place.
      if (P.correct_mode == 1) {
        if (tid == 0) ctile[fc * LDC_S + fr] -= tl.dres[fc];  // subtract d_col
      } else {
        // Recompute C_ij with a fresh k-long dot product (R4).
        const int64_t gi = i0 + fr, gj = j0 + fc;
        double part = 0.0;
        for (int64_t p = tid; p < P.k; p += NTHREADS) {
          const double av = AKM ? P.A[p + gi * P.lda] : P.A[gi + p * P.lda];
          const double bv = BKM ? P.B[p + gj * P.ldb] : P.B[gj + p * P.ldb];
          part = fma(av, bv, part);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
        if (lane == 0) tl.red[warp] = part;
        __syncthreads();
        if (tid == 0) {
          double v = 0.0;
#pragma unroll
          for (int w = 0; w < NTHREADS / 32; ++w) v += tl.red[w];
          ctile[fc * LDC_S + fr] = v;
        }
      }
      if (tid == 0) {
        atomicAdd(&P.counters[CNT_DETECTED], 1ull);
        atomicAdd(&P.counters[CNT_CORRECTED], 1ull);
        const unsigned long long slot = atomicAdd(&P.counters[CNT_EVENTS], 1ull);
        if ((long long)slot < P.ev_cap)
          P.events[slot] = EventDev{(long long)(i0 + fr), (long long)(j0 + fc), 1, 0,
                                    tl.dres[128 + fr], tl.dres[fc]};
      }
      __syncthreads();
      break;
    }
    // Out of the one-error model: record, then recompute the whole tile once.
    if (tid == 0) {
      atomicAdd(&P.counters[CNT_DETECTED], 1ull);
      atomicAdd(&P.counters[CNT_RECOMPUTED], 1ull);
      const unsigned long long slot = atomicAdd(&P.counters[CNT_EVENTS], 1ull);
      if ((long long)slot < P.ev_cap)
        P.events[slot] = EventDev{(long long)i0, (long long)j0, 2, 0,
                                  nfr ? tl.dres[128 + fr] : 0.0, nfc ? tl.dres[fc] : 0.0};
    }
    __syncthreads();
  }

  // ---- store: C = alpha*acc + beta*C0 (two roundings each, no contraction).
  {
    const int i = tid & 127;
    const double alpha = P.alpha, beta = P.beta;
    if (i < bm_eff) {
      double *crow = P.C + (i0 + i) + j0 * P.ldc;
#pragma unroll 4
      for (int j = tid >> 7; j < bn_eff; j += 2) {
        const double v = __dmul_rn(alpha, ctile[j * LDC_S + i]);
        double *dst = crow + (int64_t)j * P.ldc;
        *dst = (beta != 0.0) ? __dadd_rn(v, __dmul_rn(beta, *dst)) : v;
      }
    }
  }
}

// C = beta*C (beta == 0: C = 0 without reading C).
__global__ void scale_kernel(int64_t m, int64_t n, double beta, double *C, int64_t ldc) {
  const int64_t total = m * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % m, j = e / m;
    double *p = C + i + j * ldc;
    *p = (beta == 0.0) ? 0.0 : __dmul_rn(beta, *p);
  }
}

}  // namespace ftk
