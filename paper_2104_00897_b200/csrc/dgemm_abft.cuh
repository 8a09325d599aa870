// dgemm_abft.cuh — sm_100a kernel of the online ABFT DGEMM (FT-BLAS, arXiv 2104.00897).
//
// One CTA computes one BM x BN = 128 x 128 tile of C = alpha*op(A)*op(B) + beta*C; the tile
// is one verification unit (§II.A restricted to the tile; R5).
//
// Warp-specialised (384 threads = 3 warpgroups):
//   warpgroup 0  (warps 0-3, 152 registers): "checksum warps".  Warp 0 lane 0 is also the
//                TMA producer: it streams the BK = 16 deep A and B tiles of every stage into
//                a 5-deep shared-memory ring (cp.async.bulk.tensor, 128-byte swizzle,
//                mbarrier complete_tx).  In the protected kernel each checksum warp c owns
//                k-slots p = 4c..4c+3 of every stage and, from the SAME staged tiles the MMA
//                reads ("each B element reused three times", §V.B):
//                  encode  a_sum[p] = sum_{i in I} op(A)_ip,  b_sum[p] = sum_{j in J} op(B)_pj
//                          (e^T A, B e) and the running max|op(A)_I|, max|op(B)_J|
//                  carry   cs_col[j] += a_sum[p] op(B)_pj,  cs_row[i] += op(A)_ip b_sum[p]
//                          (outer-product maintenance)
//   warpgroups 1-2 (warps 4-11, 176 registers): 8 MMA warps in a 2 x 4 grid of 64 x 32 warp
//                tiles; acc += A_tile*B_tile with DMMA.8x8x4 (mma.sync m8n8k4 f64 — the only
//                FP64 tensor instruction of sm_100a; tcgen05 has no f64 kind).  They also host
//                the fault-injection hook (a delta added to the owning accumulator when the
//                k-loop reaches the fault's quantised step).
//   Every consumer warp waits on the stage's full barrier and arrives on its empty barrier:
//   no CTA-wide barrier inside the k-loop, so warps drift and hide each other's latency.
//
// Epilogue (all warps): stage the accumulator through shared memory; reference checksums
// r_col = e^T C_IJ, r_row = C_IJ e from the computed C; residuals
// d = r - cs; flag where not |d| <= tau (R1); exactly one flagged row and column
// -> locate and correct in place; any other pattern -> recompute the
// tile once (R6).  Store C = alpha*acc + beta*C0 (C0 not read when beta == 0).
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace ftk {

constexpr int BM = 128, BN = 128, BK = 16;  // MMA tile (C^f tile) and k-stage depth
constexpr int DM = 127;                     // data rows/cols per tile; row/col DM is the checksum
constexpr int TM = DM, TN = DM;             // verification unit (tile stride in C)
constexpr int STAGES = 6;                 // shared-memory ring depth (6 x 32 KB)
constexpr int NTHREADS = 384;             // 12 warps
constexpr int N_CS_WARPS = 4;             // checksum warps (warpgroup 0)
constexpr int N_MMA_WARPS = 8;            // MMA warps (warpgroups 1-2)
constexpr int TILE_ELEMS = 128 * BK;      // one operand tile: 16 KB
constexpr int STAGE_ELEMS = 2 * TILE_ELEMS;
constexpr int STAGE_BYTES = STAGE_ELEMS * 8;
constexpr int LDC_S = 129;                // epilogue C-tile pitch (doubles)
constexpr int REG_CS = 152, REG_MMA = 176; // setmaxnreg split: 128*152 + 256*176 = 384*168
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
  unsigned long long *dev_prof;   // development only: per-CTA [warp][wait, work] clock64 sums (null = off)
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
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ bool mbar_test(uint64_t *bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n.reg .pred p;\nmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void tma_load_2d(void *sdst, const CUtensorMap *map, int c0, int c1, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          smem_u32(sdst)),
      "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap *map) {
  asm volatile("prefetch.tensormap [%0];\n" ::"l"(map) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void setmaxnreg_inc() { asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(N)); }
template <int N>
__device__ __forceinline__ void setmaxnreg_dec() { asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(N)); }

// ------------------------------------------------------------------ shared-memory layouts
// Operand tile X(x, p): x the M (or N) index in [0,128), p the k index in [0,16).  Both are
// written by TMA with the 128-byte swizzle (16-byte chunk c of a 128-byte row r lands at
// chunk c ^ (r & 7)); buffers are 1024-byte aligned.
//  K-major (p contiguous in global: op(A) 'T', op(B) 'N'): one box {16 p, 128 x};
//     row x holds X(x, 0..15).
//  MN-major (x contiguous: op(A) 'N', op(B) 'T'): eight boxes {16 x, 16 p}, one per x-block
//     xb = x/16 (2 KB each); row p of block xb holds X(16xb .. 16xb+15, p).
template <bool KM>
__device__ __forceinline__ int sidx(int x, int p) {
  if (KM) return x * 16 + (((p >> 1) ^ (x & 7)) << 1) + (p & 1);
  return (x >> 4) * 256 + p * 16 + ((((x & 15) >> 1) ^ (p & 7)) << 1) + (x & 1);
}

// MMA fragment rows.  k-slot mapping in a stage: k-step s (0..3), lane slot t (0..3) <-> p =
// 8*(s>>1) + 2t + (s&1) for both operands.  Row of m/n-tile r for fragment index g:
//   K-major : 8r + ((g&1)<<2) + (g>>1)   (rows of lanes g, g+1 differ by 4 -> swizzle
//             chunks in complementary halves: conflict-free LDS.128)
//   MN-major: 16(r>>1) + 2g + (r&1)      (one LDS.128 feeds the tile pair 2q, 2q+1)
template <bool KM>
__device__ __forceinline__ int tile_row(int r, int g) {
  return KM ? 8 * r + ((g & 1) << 2) + (g >> 1) : 16 * (r >> 1) + 2 * g + (r & 1);
}

template <bool KM, int NT>
__device__ __forceinline__ void load_frags(const double *s, int xw, int h, int g, int t, double (&f)[2][NT]) {
  if (KM) {
#pragma unroll
    for (int r = 0; r < NT; ++r) {
      const int x = xw + tile_row<true>(r, g);
      const double2 v = *reinterpret_cast<const double2 *>(s + x * 16 + (((4 * h + t) ^ (x & 7)) << 1));
      f[0][r] = v.x;
      f[1][r] = v.y;
    }
  } else {
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int p = 8 * h + 2 * t + e;
#pragma unroll
      for (int q = 0; q < NT / 2; ++q) {
        const int xb = (xw >> 4) + q;
        const double2 v = *reinterpret_cast<const double2 *>(s + xb * 256 + p * 16 + ((g ^ (p & 7)) << 1));
        f[e][2 * q] = v.x;
        f[e][2 * q + 1] = v.y;
      }
    }
  }
}

// Checksum-warp view of an operand tile: lane l owns 4 x-rows (cs_row_of(l, 0..3)) and the
// warp's 4 k-slots p = 4c..4c+3; v[r][q] = X(cs_row_of(l, r), 4c + q).  Conflict-free LDS.128.
template <bool KM>
__device__ __forceinline__ int cs_row_of(int lane, int r) {
  return KM ? lane + 32 * r : 2 * (lane & 7) + 16 * (lane >> 3) + 64 * (r >> 1) + (r & 1);
}
template <bool KM>
__device__ __forceinline__ void cs_load(const double *s, int c, int lane, double (&v)[4][4]) {
  if (KM) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int x = lane + 32 * r;
#pragma unroll
      for (int hq = 0; hq < 2; ++hq) {
        const double2 w = *reinterpret_cast<const double2 *>(s + x * 16 + (((2 * c + hq) ^ (x & 7)) << 1));
        v[r][2 * hq] = w.x;
        v[r][2 * hq + 1] = w.y;
      }
    }
  } else {
#pragma unroll
    for (int rr = 0; rr < 2; ++rr) {
      const int xb = (lane >> 3) + 4 * rr;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int p = 4 * c + q;
        const double2 w = *reinterpret_cast<const double2 *>(s + xb * 256 + p * 16 + (((lane & 7) ^ (p & 7)) << 1));
        v[2 * rr][q] = w.x;
        v[2 * rr + 1][q] = w.y;
      }
    }
  }
}

// ---------------- integer (fixed-point) encode: no SIMT FP64 next to the DMMA stream.
// A dependent DADD behind a saturated DMMA stream takes ~1000 clk on sm_100a
// (profiles/fp64_latency_under_dmma.json), so the column / row sums e^T A, B e are formed on
// the integer pipes: each element x = (-1)^s m 2^(e-1075) (m with the hidden bit, e >= 1) is
// aligned to the largest biased exponent E of the warp's stage slice as the integer
// floor-toward-zero(m 2^(e-E)) (53 significant bits for the largest element), and 128 of them
// sum without overflow in a signed 64-bit word.  Per-element truncation is below
// 2^(E-1075) <= 2^-52 max|x|, far inside the rounding budget of the threshold (R1).
// Non-finite elements clamp the stage maximum to that of DBL_MAX (reading R1'): such a unit's
// residuals are NaN or Inf and it is flagged whatever the threshold.

__device__ __forceinline__ void split_hi_lo(double x, uint32_t &hi, uint32_t &lo) {
  asm("mov.b64 {%0, %1}, %2;\n" : "=r"(lo), "=r"(hi) : "d"(x));
}

// One operand slice: v[r][q] for the lane's 4 rows and the warp's 4 k-slots.  Returns the sum
// for k-slot 4c + lane/8 in every lane; folds the slice's max |hi word| into hmax.
__device__ __forceinline__ double cs_encode_fx(const double (&v)[4][4], int lane, uint32_t &hmax) {
  uint32_t hi[4][4], lo[4][4], ex[4][4];
  uint32_t emax = 0, hm = 0;
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      split_hi_lo(v[r][q], hi[r][q], lo[r][q]);
      ex[r][q] = (hi[r][q] >> 20) & 0x7FFu;
      hm = max(hm, hi[r][q] & 0x7FFFFFFFu);
    }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) hm = max(hm, __shfl_xor_sync(0xffffffffu, hm, o));
  hm = min(hm, 0x7FEFFFFFu);  // Inf/NaN -> largest finite (R1')
  hmax = max(hmax, hm);
  emax = max(hm >> 20, 1u);
  long long sum[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    unsigned long long acc = 0ull;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const uint32_t e = ex[r][q];
      const uint32_t mhi = (hi[r][q] & 0x000FFFFFu) | (e ? 0x00100000u : 0u);
      const uint32_t d = min(emax - max(e, 1u), 63u);  // e <= emax for finite elements
      const unsigned long long m = ((unsigned long long)mhi << 32) | lo[r][q];
      const unsigned long long sgn = (unsigned long long)(long long)(int)hi[r][q] >> 63;  // 0 or 1
      acc += ((m >> d) ^ (0ull - sgn)) + sgn;  // +/- (m >> d), two's complement
    }
    sum[q] = (long long)acc;
  }
  const bool b4 = (lane >> 4) & 1, b3 = (lane >> 3) & 1;
  auto sx = [](long long x, int o) { return (long long)__shfl_xor_sync(0xffffffffu, x, o); };
  const long long w0 = (b4 ? sum[2] : sum[0]) + sx(b4 ? sum[0] : sum[2], 16);  // keep q in {2b4, 2b4+1}
  const long long w1 = (b4 ? sum[3] : sum[1]) + sx(b4 ? sum[1] : sum[3], 16);
  long long z = (b3 ? w1 : w0) + sx(b3 ? w0 : w1, 8);                          // keep q = 2b4 + b3
  z += sx(z, 4);
  z += sx(z, 2);
  z += sx(z, 1);
  // z * 2^(emax - 1075) as a double, truncated to 53 bits; integer ops only.
  if (z == 0) return 0.0;
  const unsigned long long sg = z < 0 ? (1ull << 63) : 0ull;
  const unsigned long long a = z < 0 ? (unsigned long long)(-z) : (unsigned long long)z;
  const int lz = __clzll((long long)a);
  const int biased = (int)emax + 11 - lz;  // exponent of the leading bit, biased
  const unsigned long long norm = a << lz;  // leading one at bit 63
  unsigned long long bits;
  if (biased >= 2047) bits = 0x7FF0000000000000ull;                                    // overflow
  else if (biased >= 1) bits = ((unsigned long long)biased << 52) | ((norm >> 11) & 0xFFFFFFFFFFFFFull);
  else bits = (1 - biased) < 53 ? ((norm >> 11) >> (1 - biased)) : 0ull;               // subnormal
  return __longlong_as_double((long long)(sg | bits));
}

// ------------------------------------------------------------------ the kernel
struct SmemTail {
  uint64_t full[STAGES], enc[STAGES], empty[STAGES];
  double dres[256];                // residuals: 0..127 columns, 128..255 rows
  double red[NTHREADS / 32];
  unsigned int amax_hi, bmax_hi;   // max finite |op(A)|, |op(B)| high words (R1')
  int first_row, first_col;
  int retry;
};
constexpr size_t SMEM_BYTES = 1024 + sizeof(double) * STAGES * STAGE_ELEMS + sizeof(SmemTail);

// Named barriers (id 0 is __syncthreads).  Both roles execute the same sequence of the
// CTA-wide ones; the 256-thread ones are private to the MMA warpgroups.
enum { BAR_RING_FREE = 1, BAR_CTILE = 2, BAR_FLAGS_R = 3, BAR_FLAGS_C = 4, BAR_DECIDE = 5, BAR_RED = 6 };
__device__ __forceinline__ void bar_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ int bar_popc(int id, int count, bool pred) {
  int r;
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.u32 p, %1, 0;\nbar.red.popc.u32 %0, %2, %3, p;\n}\n"
      : "=r"(r)
      : "r"((int)pred), "r"(id), "r"(count)
      : "memory");
  return r;
}

struct Ctx {
  double *ring;
  SmemTail *tl;
  int tid, lane, warp, tile, i0, j0, bm_eff, bn_eff, nk, f_lo, f_hi;
  // Protected tiles: TMA boxes start at the even coordinate xs = x0 - (x0 & 1) (the contiguous
  // dimension of a TMA box must start 16-byte aligned), so tile-local data row i sits in
  // staged row i + o (o = x0 & 1) and the checksum row/column takes the free row cr.
  int oa, ob, cra, crb;
};

// ---------------- warpgroup 0: TMA producer (warp 0 lane 0) + checksum-encode warps
// Checksum warp c encodes k-slots 4c..4c+3 of every stage: it waits for the stage's TMA
// bytes, forms a_sum[p] = sum_{i<127} op(A)_ip and b_sum[p] = sum_{j<127} op(B)_pj on the
// integer pipes, writes them into row 127 of the staged A tile and row 127 (= column 127 of
// op(B)) of the staged B tile, and arrives on the stage's `enc` barrier.  The DMMA stream
// then computes C^f = [A; e^T A][B, B e] tile by tile: acc(127, j) is the
// carried column checksum (e^T A_I) B_J and acc(i, 127) the carried row checksum A_I (B_J e)
// (outer-product maintenance), at no SIMT FP64 cost.
template <bool AKM, bool BKM, bool FT>
__device__ __forceinline__ void checksum_role(const CUtensorMap &tmA, const CUtensorMap &tmB, const Params &P,
                                              const Ctx &x) {
  SmemTail &tl = *x.tl;
  double *const ring = x.ring;
  const int lane = x.lane, warp = x.warp, c = warp, nk = x.nk;
  int stage_base = 0;
  for (int attempt = 0;; ++attempt) {
    const bool verify = FT && attempt == 0;
    int produced = 0;
    // Issue stages [produced, min(lim, nk)).  Blocking for stages below `must` (the checksum
    // warps need them next); beyond that only while ring slots are already free, so the
    // producer never stalls warp 0's encode behind the MMA warps.
    auto produce_upto = [&](int lim, int must) {
      for (; produced < lim && produced < nk; ++produced) {
        const int gs = stage_base + produced, slot = gs % STAGES;
        if (gs >= STAGES) {
          const uint32_t par = ((gs / STAGES) - 1) & 1;
          if (produced < must) mbar_wait(&tl.empty[slot], par);
          else if (!mbar_test(&tl.empty[slot], par)) break;
        }
        double *sa = ring + slot * STAGE_ELEMS;
        mbar_arrive_expect_tx(&tl.full[slot], STAGE_BYTES);
        const int k0 = produced * BK;
        const int xa = x.i0 - x.oa, xbj = x.j0 - x.ob;  // even box origins
        if (AKM) {
          tma_load_2d(sa, &tmA, k0, xa, &tl.full[slot]);
        } else {
#pragma unroll
          for (int xb = 0; xb < 8; ++xb) tma_load_2d(sa + xb * 256, &tmA, xa + 16 * xb, k0, &tl.full[slot]);
        }
        double *sb = sa + TILE_ELEMS;
        if (BKM) {
          tma_load_2d(sb, &tmB, k0, xbj, &tl.full[slot]);
        } else {
#pragma unroll
          for (int xb = 0; xb < 8; ++xb) tma_load_2d(sb + xb * 256, &tmB, xbj + 16 * xb, k0, &tl.full[slot]);
        }
      }
    };
    if (verify) {
      uint32_t amax_hi = 0u, bmax_hi = 0u;
      for (int s = 0; s < nk; ++s) {
        if (warp == 0 && lane == 0) produce_upto(s + STAGES, s + 1);
        __syncwarp();
        const int gs = stage_base + s, slot = gs % STAGES;
        const long long t0 = P.dev_prof ? clock64() : 0;
        mbar_wait(&tl.full[slot], (gs / STAGES) & 1);
        const long long t1 = P.dev_prof ? clock64() : 0;
        double *sA = ring + slot * STAGE_ELEMS, *sB = sA + TILE_ELEMS;
        double v[4][4];
        // The checksum row cr (127, or 0 for odd tiles) holds a neighbour tile's data: it is
        // staged row 127 = lane 31 / r 3, or staged row 0 = lane 0 / r 0, in both layouts.
        const bool xa_l = x.cra ? lane == 31 : lane == 0, xb_l = x.crb ? lane == 31 : lane == 0;
        const int xa_r = x.cra ? 3 : 0, xb_r = x.crb ? 3 : 0;
        cs_load<AKM>(sA, c, lane, v);  // encode A: e^T A_I over the 127 data rows
#pragma unroll
        for (int r = 0; r < 4; ++r)  // constant indices only: v must stay in registers
#pragma unroll
          for (int q = 0; q < 4; ++q) v[r][q] = (xa_l && r == xa_r) ? 0.0 : v[r][q];
        const double asum = cs_encode_fx(v, lane, amax_hi);
        cs_load<BKM>(sB, c, lane, v);  // encode B: B_J e over the 127 data columns
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int q = 0; q < 4; ++q) v[r][q] = (xb_l && r == xb_r) ? 0.0 : v[r][q];
        const double bsum = cs_encode_fx(v, lane, bmax_hi);
        if ((lane & 7) == 0) {  // lanes 8q hold the sums of k-slot 4c+q
          const int p = 4 * c + (lane >> 3);
          sA[sidx<AKM>(x.cra, p)] = asum;
          sB[sidx<BKM>(x.crb, p)] = bsum;
        }
        fence_proxy_async();  // generic writes into a TMA-filled buffer that TMA will refill
        __syncwarp();
        if (lane == 0) mbar_arrive(&tl.enc[slot]);
        if (P.dev_prof && lane == 0) {
          const long long t2 = clock64();
          unsigned long long *dp = P.dev_prof + ((size_t)(blockIdx.x + blockIdx.y * gridDim.x) * 12 + warp) * 2;
          dp[0] += (unsigned long long)(t1 - t0);
          dp[1] += (unsigned long long)(t2 - t1);
        }
      }
      if (lane == 0) { atomicMax(&tl.amax_hi, amax_hi); atomicMax(&tl.bmax_hi, bmax_hi); }
    } else if (warp == 0 && lane == 0) {
      produce_upto(nk, nk);
    }
    stage_base += nk;
    bar_sync(BAR_RING_FREE, NTHREADS);  // ring consumed by everyone; maxima visible
    if (!verify) return;
    bar_sync(BAR_DECIDE, NTHREADS);     // MMA warps decided: clean / corrected / recompute
    if (!tl.retry) return;
  }
}

// ---------------- warpgroups 1-2: MMA warps (+ epilogue)
template <bool AKM, bool BKM, bool FT>
__device__ __forceinline__ void mma_role(const Params &P, const Ctx &x) {
  SmemTail &tl = *x.tl;
  double *const ring = x.ring;
  double *const ctile = ring;  // epilogue reuse of the ring
  const int lane = x.lane, nk = x.nk;
  const int mw = x.warp - N_CS_WARPS, wm = mw >> 2, wn = mw & 3;
  const int g = lane >> 2, t = lane & 3;
  const int vt = x.tid - N_CS_WARPS * 32;  // 0..255
  double acc[8][4][2];
  int stage_base = 0;
  for (int attempt = 0;; ++attempt) {
    const bool verify = FT && attempt == 0;
    const bool inject = attempt == 0 && x.f_lo < x.f_hi;
    int fnext = x.f_lo;
    int next_stage = inject ? P.faults[fnext].stage : 0x7fffffff;
#pragma unroll
    for (int a = 0; a < 8; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
    auto apply_faults = [&](int s) {
      while (s == next_stage) {
        const FaultDev f = P.faults[fnext];
        const int si = f.li + x.oa, sj = f.lj + x.ob;  // staged row / column
        const int lr = si & 63, lc = sj & 31;
        const int fmt = AKM ? (lr >> 3) : 2 * (lr >> 4) + (lr & 1);
        const int rr = lr & 7;  // K-major: row in the 8-row tile = 4*(g&1) + (g>>1)
        const int fg = AKM ? (((rr & 3) << 1) | (rr >> 2)) : ((lr & 15) >> 1);
        const int fnt = BKM ? (lc >> 3) : 2 * (lc >> 4) + (lc & 1);
        const int cr = lc & 7;  // K-major: column in the 8-column tile, same mapping
        const int cc = BKM ? (((cr & 3) << 1) | (cr >> 2)) : ((lc & 15) >> 1);  // n-index
        // Register index of the owning accumulator, -1 for every other thread.  Select-based
        // (no dynamic register indexing) so the accumulators stay in registers.
        const bool owner = (si >> 6) == wm && (sj >> 5) == wn && lane == fg * 4 + (cc >> 1);
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
        next_stage = fnext < x.f_hi ? P.faults[fnext].stage : 0x7fffffff;
      }
    };
    long long w_wait = 0, w_work = 0;
    for (int s = 0; s < nk; ++s) {
      const int gs = stage_base + s, slot = gs % STAGES;
      const long long t0 = P.dev_prof ? clock64() : 0;
      // The protected pass waits for the encoded stage (TMA bytes + checksum row/column).
      if (verify) mbar_wait(&tl.enc[slot], (gs / STAGES) & 1);
      else mbar_wait(&tl.full[slot], (gs / STAGES) & 1);
      if (P.dev_prof) { const long long t1 = clock64(); w_wait += t1 - t0; w_work -= t1; }
      if (inject) apply_faults(s);
      const double *sA = ring + slot * STAGE_ELEMS, *sB = sA + TILE_ELEMS;
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
      __syncwarp();
      if (lane == 0) mbar_arrive(&tl.empty[slot]);
      if (P.dev_prof) w_work += clock64();
    }
    if (P.dev_prof && lane == 0) {
      unsigned long long *dp = P.dev_prof + ((size_t)(blockIdx.x + blockIdx.y * gridDim.x) * 12 + x.warp) * 2;
      dp[0] += (unsigned long long)w_wait;
      dp[1] += (unsigned long long)w_work;
    }
    if (inject) apply_faults(nk);  // faults with step_q == k
    stage_base += nk;
    bar_sync(BAR_RING_FREE, NTHREADS);  // every stage consumed: the ring is free for the C tile

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
    bar_sync(BAR_CTILE, 256);
    if (!verify) break;

    // ---- verification: reference checksums r from the computed C_IJ against
    // the carried checksums in row / column 127 of C^f.
    // ctile is indexed by staged rows / columns: data row i at i + oa, data column j at j + ob.
    const int cidx = vt & 127;
    const bool is_row = vt >= 128;
    double r = 0.0, cs = 0.0;
    if (cidx < DM) {
      if (is_row) {
        const double *rowp = ctile + (cidx + x.oa);
#pragma unroll 9
        for (int j = 0; j < DM; ++j) r += rowp[(j + x.ob) * LDC_S];
        cs = rowp[x.crb * LDC_S];  // A_I (B_J e)
      } else {
        const double *colp = ctile + (cidx + x.ob) * LDC_S;
#pragma unroll 9
        for (int i = 0; i < DM; ++i) r += colp[i + x.oa];
        cs = colp[x.cra];  // (e^T A_I) B_J
      }
    }
    const double d = r - cs;
    // R1': maxima rounded up to the largest double with the same high word.
    const double amx = __longlong_as_double((long long)(((unsigned long long)tl.amax_hi << 32) | 0xFFFFFFFFull));
    const double bmx = __longlong_as_double((long long)(((unsigned long long)tl.bmax_hi << 32) | 0xFFFFFFFFull));
    const int64_t kt = P.k;
    const int len = is_row ? x.bn_eff : x.bm_eff;
    const double nu = (double)(kt + len) * 0x1p-53;
    const double tau = 2.0 * (nu / (1.0 - nu)) * (double)kt * (double)len * amx * bmx;  // DESIGN.md R1
    const bool valid = is_row ? (cidx < x.bm_eff) : (cidx < x.bn_eff);
    const bool flag = valid && !(fabs(d) <= tau);
    tl.dres[vt] = d;
    if (flag) atomicMin(is_row ? &tl.first_row : &tl.first_col, cidx);
    const int nfr = bar_popc(BAR_FLAGS_R, 256, flag && is_row);
    const int nfc = bar_popc(BAR_FLAGS_C, 256, flag && !is_row);
    const bool multi = !(nfr == 0 && nfc == 0) && !(nfr == 1 && nfc == 1);
    const int fr = tl.first_row, fc = tl.first_col;
    if (nfr == 1 && nfc == 1) {
      // Single error at the intersection (i0+fr, j0+fc): correct in place.
      if (P.correct_mode == 1) {
        if (vt == 0) ctile[(fc + x.ob) * LDC_S + fr + x.oa] -= tl.dres[fc];  // subtract d_col
      } else {
        // Recompute C_ij with a fresh k-long dot product (R4).
        const int64_t gi = x.i0 + fr, gj = x.j0 + fc;
        double part = 0.0;
        for (int64_t p = vt; p < P.k; p += 256) {
          const double av = AKM ? P.A[p + gi * P.lda] : P.A[gi + p * P.lda];
          const double bv = BKM ? P.B[p + gj * P.ldb] : P.B[gj + p * P.ldb];
          part = fma(av, bv, part);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
        if (lane == 0) tl.red[mw] = part;
        bar_sync(BAR_RED, 256);
        if (vt == 0) {
          double v = 0.0;
#pragma unroll
          for (int q = 0; q < N_MMA_WARPS; ++q) v += tl.red[q];
          ctile[(fc + x.ob) * LDC_S + fr + x.oa] = v;
        }
      }
    }
    if (vt == 0 && (nfr | nfc)) {
      atomicAdd(&P.counters[CNT_DETECTED], 1ull);
      atomicAdd(&P.counters[multi ? CNT_RECOMPUTED : CNT_CORRECTED], 1ull);
      const unsigned long long slot = atomicAdd(&P.counters[CNT_EVENTS], 1ull);
      if ((long long)slot < P.ev_cap)
        P.events[slot] = multi ? EventDev{(long long)x.i0, (long long)x.j0, 2, 0, nfr ? tl.dres[128 + fr] : 0.0,
                                          nfc ? tl.dres[fc] : 0.0}
                               : EventDev{(long long)(x.i0 + fr), (long long)(x.j0 + fc), 1, 0, tl.dres[128 + fr],
                                          tl.dres[fc]};
    }
    if (vt == 0) tl.retry = multi ? 1 : 0;
    if (multi) fence_proxy_async();  // generic writes to the ring (C tile) before TMA reuses it
    bar_sync(BAR_DECIDE, NTHREADS);
    if (!multi) break;
    // Out of the one-error model: recompute the whole tile once (no re-verification).
  }

  // ---- store: C = alpha*acc + beta*C0 (two roundings each, no contraction).
  const int i = vt & 127;
  const double alpha = P.alpha, beta = P.beta;
  if (i < x.bm_eff) {
    double *crow = P.C + (int64_t)(x.i0 + i) + (int64_t)x.j0 * P.ldc;
#pragma unroll 4
    for (int j = vt >> 7; j < x.bn_eff; j += 2) {
      const double v = __dmul_rn(alpha, ctile[(j + x.ob) * LDC_S + i + x.oa]);
      double *dst = crow + (int64_t)j * P.ldc;
      *dst = (beta != 0.0) ? __dadd_rn(v, __dmul_rn(beta, *dst)) : v;
    }
  }
}

template <bool AKM, bool BKM, bool FT>
__global__ void __launch_bounds__(NTHREADS, 1)
    dgemm_abft_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                      const Params P) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  Ctx x;
  // 1024-byte alignment by pointer arithmetic on the __shared__ array (an integer round trip
  // would lose the address space and turn every LDS into a generic LD).
  x.ring = reinterpret_cast<double *>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
  x.tl = reinterpret_cast<SmemTail *>(x.ring + STAGES * STAGE_ELEMS);
  SmemTail &tl = *x.tl;
  x.tid = threadIdx.x;
  x.lane = x.tid & 31;
  x.warp = x.tid >> 5;
  const int ti = blockIdx.x, tj = blockIdx.y;
  x.tile = ti + tj * P.tiles_m;
  // Protected tiles advance by the 127 data rows/cols of C^f; the unprotected twin uses the
  // full 128 x 128 MMA tile for data.
  constexpr int tm = FT ? TM : BM, tn = FT ? TN : BN;
  x.i0 = ti * tm;
  x.j0 = tj * tn;
  x.bm_eff = (int)min64(tm, P.m - x.i0);
  x.bn_eff = (int)min64(tn, P.n - x.j0);
  x.oa = FT ? (x.i0 & 1) : 0;
  x.ob = FT ? (x.j0 & 1) : 0;
  x.cra = x.oa ? 0 : DM;
  x.crb = x.ob ? 0 : DM;
  x.nk = P.nk;

  if (x.tid == 0) {
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB);
#pragma unroll
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&tl.full[s], 1);
      mbar_init(&tl.enc[s], N_CS_WARPS);
      mbar_init(&tl.empty[s], N_MMA_WARPS);
    }
    tl.amax_hi = 0u;
    tl.bmax_hi = 0u;
    tl.first_row = 0x7fffffff;
    tl.first_col = 0x7fffffff;
    tl.retry = 0;
    fence_mbar_init();
  }
  // Faults of this tile: [f_lo, f_hi) in the (tile, stage)-sorted list.
  x.f_lo = x.f_hi = 0;
  if (P.nfaults > 0) {
    int lo = 0, hi = P.nfaults;
    while (lo < hi) { const int mid = (lo + hi) >> 1; if (P.faults[mid].tile < x.tile) lo = mid + 1; else hi = mid; }
    x.f_lo = lo;
    hi = P.nfaults;
    while (lo < hi) { const int mid = (lo + hi) >> 1; if (P.faults[mid].tile <= x.tile) lo = mid + 1; else hi = mid; }
    x.f_hi = lo;
  }
  __syncthreads();

  // The two roles never re-converge, so ptxas can give each its own register budget.  The
  // checksum warps take the LOWEST warp ids: the issue arbiter favours high ids, so the DMMA
  // warps always win an issue slot and the integer encode fills the idle ones.
  if (x.warp < N_CS_WARPS) {
    setmaxnreg_dec<REG_CS>();
    checksum_role<AKM, BKM, FT>(tmA, tmB, P, x);
  } else {
    setmaxnreg_inc<REG_MMA>();
    mma_role<AKM, BKM, FT>(P, x);
  }
}

// C = beta*C (beta == 0: C = 0 without reading C).
__global__ void scale_kernel(int64_t m, int64_t n, double beta, double *C, int64_t ldc) {
  const int64_t total = m * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % m, j = e / m;
    double *p = C + i + j * ldc;
    *p = (beta == 0.0) ? 0.0 : __dmul_rn(beta, *p);
  }
}

}  // namespace ftk
