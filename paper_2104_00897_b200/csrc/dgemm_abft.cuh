// dgemm_abft.cuh — sm_100a kernel of the online ABFT DGEMM (FT-BLAS, arXiv 2104.00897).
//
// One CTA computes one BM x BN = 128 x 128 MMA tile of C = alpha*op(A)*op(B) + beta*C.  In the
// protected kernel the tile is the unit's full checksum block C^f = [A_I; e^T A_I][B_J, B_J e]
// restricted to 127 x 127 data rows / columns: staged row cra holds e^T A_I,
// staged column crb holds B_J e, so the DMMA stream that forms C also carries the checksums
// (outer-product maintenance) and the unit is 127 x 127 (R16).
//
// Warp-specialised (384 threads = 3 warpgroups):
//   warps 0-7 (176 registers): MMA warps in a 2 x 4 grid of 64 x 32 warp tiles, acc += A*B
//                with DMMA.8x8x4 (mma.sync m8n8k4 f64 -- the only FP64 tensor instruction of
//                sm_100a; tcgen05 has no f64 kind); the fault hook between fault-free k-loop
//                segments; the online verification from the live accumulators at every
//                interval end (reference sums e^T C and C e, residuals against
//                the carried checksums, tau, locate / correct / recompute) and the epilogue.
//   warps 8-11 (152 registers): encoder warps.  Warp w issues the TMA loads of stages
//                s = w (mod 4) into a 6-deep shared-memory ring (cp.async.bulk.tensor, 128-byte
//                swizzle, mbarrier complete_tx) and, in the protected kernel, writes the stage's
//                16 k-slots of e^T A_I and B_J e into the staged checksum row / column: copied
//                from the tile that published them through L2, or encoded from the staged tile
//                (integer fixed point, R17, R22).
//   No CTA-wide barrier inside the k-loop: MMA warps wait on a stage's `enc` (protected) or
//   `full` (unprotected) mbarrier and arrive on its `empty` one.
// k-split (launches of <= 18 tiles, Kc = k): each tile runs as several CTAs over contiguous
// k ranges; the last to finish sums the partial C^f blocks in split order, verifies and stores.
#pragma once
#include <cstdint>
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>

namespace ftk {

constexpr int BM = 128, BN = 128, BK = 16;  // MMA tile (C^f tile) and k-stage depth
constexpr int DM = 127;                     // data rows/cols per tile; row/col DM is the checksum
constexpr int TM = DM, TN = DM;             // verification unit (tile stride in C)
constexpr int STAGES = 6;                 // shared-memory ring depth (6 x 32 KB)
constexpr int RASTER_G = 12;              // tile rows per raster band (grouped CTA order)
constexpr int NTHREADS = 384;             // 12 warps
constexpr int N_CS_WARPS = 4;             // checksum warps (warpgroup 0)
constexpr int N_MMA_WARPS = 8;            // MMA warps (warpgroups 1-2)
constexpr int TILE_ELEMS = 128 * BK;      // one operand tile: 16 KB
constexpr int STAGE_ELEMS = 2 * TILE_ELEMS;
constexpr int STAGE_BYTES = STAGE_ELEMS * 8;
constexpr int LDC_S = 129;                // epilogue C-tile pitch (doubles)
constexpr int REG_CS = 152, REG_MMA = 176; // setmaxnreg split: 128*152 + 256*176 = 384*168
                                           // (protected TT: 128*136 + 256*184, same total)
static_assert(BM * LDC_S <= STAGES * STAGE_ELEMS, "C tile must fit in the stage ring");

struct FaultDev {        // one armed fault, sorted by (tile, stage)
  int32_t tile, stage;   // tile = ti + tj*tiles_m; stage = floor(step / BK)
  int32_t li, lj;        // tile-local row / column (-1: the checksum row / column)
  double delta;
};

struct EventDev {
  long long i, j;
  int kind, interval;
  double residual_row, residual_col;
};

enum { CNT_DETECTED = 0, CNT_CORRECTED, CNT_RECOMPUTED, CNT_EVENTS, CNT_N };
constexpr int CNT_DONE = 4;  // CTAs finished (device-written report); inside the 64-byte counter slot
constexpr int REP_EVENTS = 32;  // events the device-written report carries (the rest: a read-back)

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
  // Verification intervals: every CTA verifies
  // its tile online after every Kc rank-1 updates (T intervals, the last one ragged), from the
  // live accumulators; Kc is a multiple of BK.
  int64_t Kc;
  int T, ntiles;
  // Launched as 2-CTA clusters (fused encode): consecutive CTAs 2c, 2c+1 hold tiles of one
  // tile column, so they stage the same B_J: each encodes half of its 16 k-slots and the pair
  // swaps halves through distributed shared memory.  `total` = real CTAs of this launch.
  int cluster2, total;
  // k-split of a launch with few tiles (Kc = k only): CTA b runs split q = b % ksplit of tile
  // b / ksplit -- stages [q nk / ksplit, (q+1) nk / ksplit) -- and writes its partial C^f
  // block (data and carried checksums) to part[(tile * ksplit + q) * 16384 + idx * 256 + thread]
  // and its stage maxima to part_max; the last split of a tile to finish (ticket) sums the
  // partials in split order (deterministic), verifies the whole C^f block and stores the tile.
  int ksplit;
  // Encoder CTAs at the head of a few-wave protected launch (R22): blocks [0, enc_head) encode
  // and publish e^T A_I of tile row b (b < tiles_m, when Ash) or B_J e of tile column b - tiles_m
  // and compute nothing else; every tile then copies the published checksums.
  int enc_head;
  int kcoop;  // 1: the splits of a tile are co-resident (cooperative launch): the S splits sum
              // one slice of the block each (distributed reduction) instead of the last one alone
  double *part;
  unsigned *part_max;
  int *tickets;  // per tile, zeroed by the host
  const FaultDev *faults;
  int nfaults;
  int correct_mode;               // 0 recompute, 1 subtract
  // Pre-encoded checksums (encode mode PREPASS; null = encode in the kernel): e^T A_I as
  // Ac[ti + p*ldac], B_J e as Br[tj + p*ldbr], and the per-block maxima (R1' high words).
  const double *Ac, *Br;
  int64_t ldac, ldbr;
  const unsigned int *amax_pre, *bmax_pre;
  // Row-shared fused encode (encode mode FUSED): the tile of tile column 0 encodes e^T A_I from
  // its staged tiles and publishes it per stage through L2 -- Ash[ti*ldash + p] for the 16
  // k-slots (k contiguous: one 128-byte line per stage) and the slice's R1' high-word maximum
  // hmA[ti*nk + sg] (sg = global stage index), relaxed stores into buffers the host filled with
  // all-ones bytes.  Every other tile of row I loads the stage's words before waiting for its
  // TMA bytes and copies them when none reads all-ones; otherwise it encodes that stage itself
  // (same integer encode of the same staged data: bitwise the same checksum), so no CTA ever
  // waits on another.  Null = every CTA encodes A itself.
  double *Ash;
  int64_t ldash;
  unsigned int *hmA;
  // B_J e the same way along tile columns: the tile of tile row 0 publishes Bsh[tj*ldbsh + p]
  // and hmB[tj*nk + sg]; the other tiles of column J copy or encode per stage.  Null = no
  // sharing (cluster-pair launches split the B encode instead).
  double *Bsh;
  int64_t ldbsh;
  unsigned int *hmB;
  // Encode mode FUSED_WAIT: a tile whose stage is not published yet waits for the publisher
  // instead of encoding it itself (every checksum encoded exactly once; tests of the copy paths).
  int wait_pub;
  // Development builds only (-DFTBLAS_DEV, libftblas_dev.so; compiled out of libftblas.so):
  unsigned long long *dev_prof;   // per-CTA [warp][wait, work] clock64 sums (null = off)
  int dev_mode;                   // 1 skip pass 2, 2 skip the encode, 4 never flag, 8 MMA waits for
                                  // the TMA bytes only, 16 encoders skip the TMA wait, 32 unprotected
                                  // kernel on the 127 grid, 128 no clusters, 1024 skip the last check,
                                  // 2048 no proxy fence before slot refills, 4096 no interval maxima
                                  // (timing only)
  unsigned long long *counters;   // [CNT_N] (+ CNT_DONE)
  // Device-written report (ftblas.cu finish_report_mapped): the launch's last CTA copies the
  // counters and the first rep_events events into this mapped pinned host buffer and then
  // writes rep_seq to its word 0; null: the host reads the report back itself.
  unsigned long long *host_rep;
  unsigned long long rep_seq;
  int rep_events;
  int64_t ev_row_off;             // added to event rows (row panels of the host-buffer pipeline)
  int64_t ev_col_off;             // added to event columns (column chunks of the host-buffer pipeline)
  EventDev *events;
  long long ev_cap;
};

// Development switches exist only in -DFTBLAS_DEV builds; in libftblas.so they are constant
// zero, so every development branch is compiled out and nothing reads them at run time.
#ifdef FTBLAS_DEV
#define FT_DEV_MODE(P) ((P).dev_mode)
#define FT_DEV_PROF(P) ((P).dev_prof)
#else
#define FT_DEV_MODE(P) 0
#define FT_DEV_PROF(P) ((unsigned long long *)nullptr)
#endif

// Bounds / invariant assertions of the checked build (-DFTBLAS_CHECKED, libftblas_checked.so,
// the stand-in for compute-sanitizer, which this pool does not run): a failed check prints its
// site and traps, so the test that reached it fails with a sticky launch error.  Compiled out of
// libftblas.so.
#ifdef FTBLAS_CHECKED
#define FT_CHECK(cond)                                                                       \
  do {                                                                                       \
    if (!(cond)) {                                                                           \
      printf("FT_CHECK failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #cond,  \
             (int)blockIdx.x, (int)threadIdx.x);                                             \
      __trap();                                                                              \
    }                                                                                        \
  } while (0)
#else
#define FT_CHECK(cond) \
  do {                 \
  } while (0)
#endif

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ void dmma_8x8x4(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}
__device__ __forceinline__ int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }
// Relaxed (morally strong, unordered) accesses for the checksum publication (R22): every
// published word is validated on its own against the all-ones fill, so no flag, fence or
// acquire is needed and the loads do not block until their values are used.
// The published words are read by every tile of their tile row / column over the whole launch
// while A and B stream through L2: loads and stores carry an L2 evict_last policy so that the
// small publication region stays resident (a consumer's first stage waits for these loads).
#define FT_PUB_POLICY "createpolicy.fractional.L2::evict_last.b64 pol, 1.0;\n"
__device__ __forceinline__ double ld_relaxed_gpu(const double *p) {
  double v;
  asm volatile("{\n.reg .b64 pol;\n" FT_PUB_POLICY "ld.relaxed.gpu.global.L2::cache_hint.f64 %0, [%1], pol;\n}\n"
               : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ unsigned ld_relaxed_gpu(const unsigned *p) {
  unsigned v;
  asm volatile("{\n.reg .b64 pol;\n" FT_PUB_POLICY "ld.relaxed.gpu.global.L2::cache_hint.u32 %0, [%1], pol;\n}\n"
               : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ int ld_acquire_gpu(const int *p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_gpu(double *p, double v) {
  asm volatile("{\n.reg .b64 pol;\n" FT_PUB_POLICY "st.relaxed.gpu.global.L2::cache_hint.f64 [%0], %1, pol;\n}\n"
               ::"l"(p), "d"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_gpu(unsigned *p, unsigned v) {
  asm volatile("{\n.reg .b64 pol;\n" FT_PUB_POLICY "st.relaxed.gpu.global.L2::cache_hint.u32 [%0], %1, pol;\n}\n"
               ::"l"(p), "r"(v) : "memory");
}
// The publication buffers are filled with all-ones bytes before the launch: an all-ones double
// is a NaN that fx_to_double never produces, an all-ones maximum has the sign bit that R1'
// masks off, so a word that reads all-ones is simply not published yet.
__device__ __forceinline__ bool pub_ok(double v) { return __double_as_longlong(v) != -1ll; }
__device__ __forceinline__ bool pub_ok(unsigned v) { return v != 0xFFFFFFFFu; }
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// Volatile 32-bit shared-memory word q of the array at shared address base.
__device__ __forceinline__ int ld_sv(uint32_t base, int q) {
  int v;
  asm volatile("ld.volatile.shared.u32 %0, [%1];\n" : "=r"(v) : "r"(base + 4u * q) : "memory");
  return v;
}
__device__ __forceinline__ void st_sv(uint32_t base, int q, int v) {
  asm volatile("st.volatile.shared.u32 [%0], %1;\n" ::"r"(base + 4u * q), "r"(v) : "memory");
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
#ifdef FTBLAS_WATCHDOG
// Watchdog builds (-DFTBLAS_WATCHDOG, tools/hang_probe.py): every mbarrier wait reports (once) a wait that has
// not completed after ~2^27 polls -- locates a hang instead of timing out silently.
__device__ __forceinline__ bool mbar_try_u32(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
// Host-mapped report slot of the watchdog (set through FTBLAS_DEV_WATCH to a pinned host
// address; a hung kernel never flushes printf, so the host polls this buffer instead).
__device__ unsigned long long *g_dev_watch = nullptr;
__device__ __noinline__ void mbar_watchdog(uint32_t bar, uint32_t parity, int where) {
  long long n = 0;
  while (!mbar_try_u32(bar, parity))
    if (++n == (1ll << 24) && g_dev_watch) {
      volatile unsigned long long *w = g_dev_watch;
      const unsigned long long q = atomicAdd(g_dev_watch, 1ull);
      if (q < 255) {
        w[1 + q] = ((unsigned long long)blockIdx.x << 40) | ((unsigned long long)threadIdx.x << 28) |
                   ((unsigned long long)where << 12) | ((unsigned long long)(bar & 0x7FF) << 1) | parity;
        __threadfence_system();
      }
    }
}
#define FT_WATCH(bar, parity, where) mbar_watchdog((bar), (parity), (where))
#endif
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
#ifdef FTBLAS_WATCHDOG
  FT_WATCH(static_cast<uint32_t>(__cvta_generic_to_shared(bar)), parity, __LINE__);
  return;
#endif
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
__device__ __forceinline__ void mbar_wait_u32(uint32_t bar, uint32_t parity) {
#ifdef FTBLAS_WATCHDOG
  FT_WATCH(bar, parity, __LINE__);
  return;
#endif
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
// Waits of the checksum / producer warps, which run ahead of the MMA warps: poll with a short
// sleep between tests instead of spinning, so their waiting issues next to nothing on the SM
// sub-partitions the DMMA warps share (ncu: the spinning producer wait was 18% of the protected
// kernel's instructions at 8192^3).
__device__ __forceinline__ bool mbar_test(uint64_t *bar, uint32_t parity);
__device__ __forceinline__ void mbar_wait_sleep(uint64_t *bar, uint32_t parity) {
#ifdef FTBLAS_WATCHDOG
  mbar_wait(bar, parity);
#else
  // try_wait with a suspend-time hint: the warp is suspended until the phase completes (or the
  // hint's 20 us pass), instead of polling with test_wait + nanosleep (ncu at 8192^3: the
  // polling loop was more than half of the unprotected kernel's issued instructions).
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAITS_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      "@!p bra WAITS_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(20000)
      : "memory");
#endif
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

// Thread-block cluster helpers (pairs of CTAs sharing an operand's checksum encode).
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ uint32_t mapa_u32(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_cluster_f64(uint32_t addr, double v) {
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(addr), "d"(v) : "memory");
}
__device__ __forceinline__ void st_cluster_u32(uint32_t addr, uint32_t v) {
  asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(addr) : "memory");
}
__device__ __forceinline__ void mbar_wait_acq_cluster(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAITC_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAITC_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

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

// ---------------- checksum encode (e^T A, B e) on the staged tiles.
// One encoder warp owns a whole stage (both operands); per operand it makes two passes over
// the staged tile, on the FP32 and integer pipes only.  (SIMT FP64 is not an option next to
// the DMMA stream: the FP64 pipe is saturated, and a side warp's DADDs only execute when the
// MMA warps stall -- measured ~10k clocks per round trip.)
//  pass 1  max |X| over the 127 data rows: the high word of a double read as a float orders
//          like |x| (FMNMX3.NAN with |.| operands, two elements per instruction).  A NaN
//          result means a non-finite element or one with |x| >= 2^1017; that warp-uniform rare
//          case is redone exactly with integer maxima.
//  pass 2  exponent-aligned fixed point: with c the largest exponent field of the slice and
//          C = c + 2, element x = (-1)^s m 2^(e-1075) contributes (-1)^s trunc(m / 2^(C-e)),
//          i.e. x / 2^(c-1073) truncated toward zero (exact for integer-valued data); 127 terms
//          of |.| < 2^51 sum exactly in 64-bit integers and are converted back by integer
//          ops.  The per-element error < 2^(c-1073) <= 2^-51 max|x| is far inside the rounding
//          budget of the threshold (R1, R17).
// Lane maps (conflict-free LDS.128; each lane sums one or two columns over 64 or 32 rows):
//  MN-major: lane = 16h + p: column p, rows 64h .. 64h+63 (x pairs from one LDS.128).
//  K-major : lane = 8q + c : columns 2c, 2c+1, rows 32q .. 32q+31.
// The checksum row cr (127, or 0 for odd tiles) holds a neighbour tile's data and is excluded.

__device__ __forceinline__ float fmax3_abs_nan(float m, float a, float b) {
  float r;
  asm("{.reg .f32 x, y;\n abs.f32 x, %2;\n abs.f32 y, %3;\n max.NaN.f32 %0, %1, x, y;\n}"
      : "=f"(r)
      : "f"(m), "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float fmax_nan(float a, float b) {
  float r;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float hi_f(double x) { return __int_as_float(__double2hiint(x)); }

template <bool KM>
__device__ __forceinline__ int enc_addr(int lane, int j) {
  if (KM) {
    const int c = lane & 7, q = lane >> 3, x = 32 * q + j;
    return x * 16 + ((c ^ (j & 7)) << 1);
  }
  const int p = lane & 15, h = lane >> 4;
  return (4 * h + (j >> 3)) * 256 + p * 16 + (((j & 7) ^ (p & 7)) << 1);
}
// Element pair j of this lane, with the checksum row cr zeroed.
template <bool KM>
__device__ __forceinline__ double2 enc_ld(const double *s, int lane, int j, int cr) {
  double2 v = *reinterpret_cast<const double2 *>(s + enc_addr<KM>(lane, j));
  if (j == 0 && cr == 0 && (lane >> (KM ? 3 : 4)) == 0) {  // staged row 0
    v.x = 0.0;
    if (KM) v.y = 0.0;
  }
  if (j == 31 && cr == DM && (lane >> (KM ? 3 : 4)) == (KM ? 3 : 1)) {  // staged row 127
    v.y = 0.0;
    if (KM) v.x = 0.0;
  }
  return v;
}

// Element pair jj (0..15, compile time) of half hh of this lane's pairs: pair j = 16 hh + jj
// sits at a constant offset from the half's base (MN-major +512, K-major +256 elements).
template <bool KM>
__device__ __forceinline__ double2 enc_ld_half(const double *s, int lane, int hh, int jj, int cr) {
  double2 v = *reinterpret_cast<const double2 *>(s + hh * (KM ? 256 : 512) + enc_addr<KM>(lane, jj));
  if (jj == 0 && hh == 0 && cr == 0 && (lane >> (KM ? 3 : 4)) == 0) {  // staged row 0
    v.x = 0.0;
    if (KM) v.y = 0.0;
  }
  if (jj == 15 && hh == 1 && cr == DM && (lane >> (KM ? 3 : 4)) == (KM ? 3 : 1)) {  // staged row 127
    v.y = 0.0;
    if (KM) v.x = 0.0;
  }
  return v;
}

// Pass 1: per-lane max (as float bits of |high word|), NaN-propagating.
template <bool KM>
__device__ __forceinline__ float enc_pass1(const double *s, int lane, int cr) {
  float m0 = 0.f, m1 = 0.f;
#pragma unroll
  for (int j = 0; j < 32; j += 2) {
    const double2 v = enc_ld<KM>(s, lane, j, cr), w = enc_ld<KM>(s, lane, j + 1, cr);
    m0 = fmax3_abs_nan(m0, hi_f(v.x), hi_f(v.y));
    m1 = fmax3_abs_nan(m1, hi_f(w.x), hi_f(w.y));
  }
  return fmax_nan(m0, m1);
}
__device__ __forceinline__ float warp_max_nan(float m) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax_nan(m, __shfl_xor_sync(0xffffffffu, m, o));
  return m;
}

// Exact max |high word| of the slice (integer pipes; rare path).
template <bool KM>
__device__ __noinline__ uint32_t enc_exact_hmax(const double *s, int lane, int cr) {
  uint32_t hm = 0;
  for (int j = 0; j < 32; ++j) {
    double2 v = *reinterpret_cast<const double2 *>(s + enc_addr<KM>(lane, j));
    const bool r0 = j == 0 && cr == 0 && (lane >> (KM ? 3 : 4)) == 0;
    const bool r127 = j == 31 && cr == DM && (lane >> (KM ? 3 : 4)) == (KM ? 3 : 1);
    if (r0) { v.x = 0.0; if (KM) v.y = 0.0; }
    if (r127) { v.y = 0.0; if (KM) v.x = 0.0; }
    hm = max(hm, max((uint32_t)__double2hiint(v.x) & 0x7FFFFFFFu, (uint32_t)__double2hiint(v.y) & 0x7FFFFFFFu));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) hm = max(hm, __shfl_xor_sync(0xffffffffu, hm, o));
  return hm;
}

// One element's fixed-point term floor(ones'-complement(x) / 2^(C-e)) = sign(x) trunc(|x| /
// 2^(C-1075)) - [x < 0]; S = -[x < 0] is returned so the caller can add the count back.
// C >= e + 2 for every element of the slice.  EXACT handles subnormals (no hidden bit,
// exponent 1); the fast form gives them a spurious hidden bit, which shifts out entirely once
// C >= 53 (c > 50).
template <bool EXACT>
__device__ __forceinline__ long long fx_term(double x, uint32_t C, int &S) {
  const uint32_t H = (uint32_t)__double2hiint(x), L = (uint32_t)__double2loint(x);
  S = (int)H >> 31;
  uint32_t E = (H >> 20) & 0x7FFu, MH;
  if (EXACT) {
    MH = (H & 0xFFFFFu) | (E ? 0x100000u : 0u);
    E = max(E, 1u);
  } else {
    MH = (H & 0xFFFFFu) | 0x100000u;
  }
  const uint32_t t = min(C - E, 63u);
  const long long m = (long long)(((unsigned long long)(MH ^ (uint32_t)S) << 32) | (L ^ (uint32_t)S));
  return m >> t;
}

// Pass 2: this lane's column sum(s) in fixed point (scale 2^(C-1075)), each term truncated
// toward zero (exact for integer-valued data), already reduced over the lanes that share the
// column(s).
template <bool KM, bool EXACT>
__device__ __forceinline__ void enc_pass2(const double *s, int lane, int cr, uint32_t C, long long &q0, long long &q1) {
  long long a0 = 0, a1 = 0;
  int n0 = 0, n1 = 0;  // minus the number of negative terms (ones' -> two's complement)
  // Two halves in a rolled loop: caps the encoder's register peak (a fully unrolled pass
  // makes ptxas spill the MMA warps' loop state in this same kernel).
#pragma unroll 1
  for (int hh = 0; hh < 2; ++hh)
#pragma unroll
  for (int jj = 0; jj < 16; jj += 2) {
    const double2 v = enc_ld_half<KM>(s, lane, hh, jj, cr), w = enc_ld_half<KM>(s, lane, hh, jj + 1, cr);
    int sv0, sv1, sw0, sw1;
    const long long tv0 = fx_term<EXACT>(v.x, C, sv0), tv1 = fx_term<EXACT>(v.y, C, sv1);
    const long long tw0 = fx_term<EXACT>(w.x, C, sw0), tw1 = fx_term<EXACT>(w.y, C, sw1);
    if (KM) {
      a0 += tv0 + tw0;
      a1 += tv1 + tw1;
      n0 += sv0 + sw0;
      n1 += sv1 + sw1;
    } else {
      a0 += (tv0 + tv1) + (tw0 + tw1);
      n0 += (sv0 + sv1) + (sw0 + sw1);
    }
  }
  a0 -= n0;
  a1 -= n1;
  if (KM) {
#pragma unroll
    for (int o = 8; o <= 16; o <<= 1) {
      a0 += __shfl_xor_sync(0xffffffffu, a0, o);
      a1 += __shfl_xor_sync(0xffffffffu, a1, o);
    }
  } else {
    a0 += __shfl_xor_sync(0xffffffffu, a0, 16);
  }
  q0 = a0;
  q1 = a1;
}
template <bool KM>
__device__ __noinline__ void enc_pass2_exact(const double *s, int lane, int cr, uint32_t C, long long &q0, long long &q1) {
  enc_pass2<KM, true>(s, lane, cr, C, q0, q1);
}

// z * 2^sc as a double, truncated toward zero to 53 bits (integer ops only).
__device__ __forceinline__ double fx_to_double(long long z, int sc) {
  if (z == 0) return 0.0;
  const unsigned long long sg = z < 0 ? (1ull << 63) : 0ull;
  const unsigned long long a = z < 0 ? (unsigned long long)(-z) : (unsigned long long)z;
  const int lz = __clzll((long long)a);
  const int biased = 63 - lz + sc + 1023;   // exponent of the leading bit, biased
  const unsigned long long norm = a << lz;  // leading one at bit 63
  unsigned long long bits;
  if (biased >= 2047) bits = 0x7FF0000000000000ull;                                   // overflow
  else if (biased >= 1) bits = ((unsigned long long)biased << 52) | ((norm >> 11) & 0xFFFFFFFFFFFFFull);
  else bits = (1 - biased) < 53 ? ((norm >> 11) >> (1 - biased)) : 0ull;              // subnormal
  return __longlong_as_double((long long)(sg | bits));
}

// ---------------- half-slice encode (thread-block clusters share an operand tile; each CTA
// of a pair encodes the 8 k-slots hsel*8 .. hsel*8+7 of the 16 and swaps them with its partner)
// Lane maps (conflict-free LDS.128, offsets compile-time per load j = 0..15):
//  K-major: lane = 4q + cc: k-slot pair c = 4 hsel + cc, row x = 8j + q (the 8 rows of one load
//           have distinct x & 7, so the 4-chunk halves of the swizzled rows tile the banks);
//           reduce over q (xor 4, 8, 16).
//  MN-major: lane = 8g + pp: k-slot p = 8 hsel + pp, rows x = 32g + 2j, 2j+1; reduce over g
//           (xor 8, 16).
template <bool KM>
__device__ __forceinline__ double2 enc_ld_h(const double *s, int lane, int hsel, int j, int cr) {
  int off;
  if (KM) {
    const int q = lane >> 2, c = 4 * hsel + (lane & 3);
    off = (8 * j + q) * 16 + ((c ^ q) << 1);
  } else {
    const int g = lane >> 3, p = 8 * hsel + (lane & 7);
    off = (2 * g + (j >> 3)) * 256 + p * 16 + (((j & 7) ^ (p & 7)) << 1);
  }
  double2 v = *reinterpret_cast<const double2 *>(s + off);
  if (KM) {
    const int q = lane >> 2;
    if ((cr == 0 && j == 0 && q == 0) || (cr == DM && j == 15 && q == 7)) v.x = v.y = 0.0;
  } else {
    const int g = lane >> 3;
    if (cr == 0 && j == 0 && g == 0) v.x = 0.0;
    if (cr == DM && j == 15 && g == 3) v.y = 0.0;
  }
  return v;
}

template <bool KM, bool EXACT>
__device__ __forceinline__ void enc_pass2_h(const double *s, int lane, int hsel, int cr, uint32_t C, long long &q0,
                                            long long &q1) {
  long long a0 = 0, a1 = 0;
  int n0 = 0, n1 = 0;
#pragma unroll 1
  for (int hh = 0; hh < 2; ++hh)
#pragma unroll
  for (int jj = 0; jj < 8; jj += 2) {
    const int j = 8 * hh + jj;
    const double2 v = enc_ld_h<KM>(s, lane, hsel, j, cr), w = enc_ld_h<KM>(s, lane, hsel, j + 1, cr);
    int sv0, sv1, sw0, sw1;
    const long long tv0 = fx_term<EXACT>(v.x, C, sv0), tv1 = fx_term<EXACT>(v.y, C, sv1);
    const long long tw0 = fx_term<EXACT>(w.x, C, sw0), tw1 = fx_term<EXACT>(w.y, C, sw1);
    if (KM) {
      a0 += tv0 + tw0;
      a1 += tv1 + tw1;
      n0 += sv0 + sw0;
      n1 += sv1 + sw1;
    } else {
      a0 += (tv0 + tv1) + (tw0 + tw1);
      n0 += (sv0 + sv1) + (sw0 + sw1);
    }
  }
  a0 -= n0;
  a1 -= n1;
#pragma unroll
  for (int o = KM ? 4 : 8; o <= 16; o <<= 1) {
    a0 += __shfl_xor_sync(0xffffffffu, a0, o);
    if (KM) a1 += __shfl_xor_sync(0xffffffffu, a1, o);
  }
  q0 = a0;
  q1 = a1;
}

template <bool KM>
__device__ __noinline__ void enc_pass2_h_exact(const double *s, int lane, int hsel, int cr, uint32_t C, long long &q0,
                                               long long &q1) {
  enc_pass2_h<KM, true>(s, lane, hsel, cr, C, q0, q1);
}

// Encode the half slice hsel: sum0 (sum1) = e^T X for this lane's k-slot(s) (valid in the
// lanes q == 0 / g == 0); hm_half returns the half's R1' high-word maximum.
// The fixed-point scale comes from the maximum of the WHOLE slice (both halves: pass 1 is
// cheap), so each k-slot's sum is bitwise the one a single CTA encoding the whole slice forms
// (the sum of exact fixed-point terms at a common scale does not depend on who adds them).
template <bool KM>
__device__ __forceinline__ void enc_operand_h(const double *s, int lane, int hsel, int cr, double &sum0, double &sum1,
                                              uint32_t &hm_half) {
  uint32_t hm = (uint32_t)__float_as_int(warp_max_nan(enc_pass1<KM>(s, lane, cr)));
  if (hm >= 0x7F800000u) hm = enc_exact_hmax<KM>(s, lane, cr);
  hm_half = min(hm, 0x7FEFFFFFu);
  const uint32_t c = hm >> 20;
  if (c >= 2047u) {
    sum0 = sum1 = __longlong_as_double(0x7FF8000000000000ll);
    return;
  }
  long long q0, q1;
  if (c > 50u) enc_pass2_h<KM, false>(s, lane, hsel, cr, c + 2u, q0, q1);
  else enc_pass2_h_exact<KM>(s, lane, hsel, cr, c + 2u, q0, q1);
  sum0 = fx_to_double(q0, (int)c - 1073);
  sum1 = KM ? fx_to_double(q1, (int)c - 1073) : 0.0;
}

// Encode one operand slice.  sum0 (and sum1 for K-major) receive e^T X for this lane's
// column(s); hmax_acc accumulates the R1' high-word maximum of the data elements.
template <bool KM>
__device__ __forceinline__ void enc_operand(const double *s, int lane, int cr, double &sum0, double &sum1,
                                            uint32_t &hmax_acc) {
  const float mf = warp_max_nan(enc_pass1<KM>(s, lane, cr));
  uint32_t hm = (uint32_t)__float_as_int(mf);
  if (hm >= 0x7F800000u) hm = enc_exact_hmax<KM>(s, lane, cr);  // warp-uniform rare path
  hmax_acc = max(hmax_acc, min(hm, 0x7FEFFFFFu));               // non-finite -> DBL_MAX (R1')
  const uint32_t c = hm >> 20;
  if (c >= 2047u) {  // a non-finite element: the checksums are NaN, the unit will flag
    sum0 = sum1 = __longlong_as_double(0x7FF8000000000000ll);
    return;
  }
  long long q0, q1;
  if (c > 50u) enc_pass2<KM, false>(s, lane, cr, c + 2u, q0, q1);
  else enc_pass2_exact<KM>(s, lane, cr, c + 2u, q0, q1);  // max |x| < 2^-972: subnormals matter
  sum0 = fx_to_double(q0, (int)c - 1073);
  sum1 = KM ? fx_to_double(q1, (int)c - 1073) : 0.0;
}

// ------------------------------------------------------------------ the kernel
// Tile geometry kept in shared memory: the MMA warps re-read it after the k-loop, so none of
// it has to stay live in registers across the DMMA stream.
struct TileGeom {
  int ti, tj, i0, j0, bm_eff, bn_eff, oa, ob, cra, crb;
  int64_t k0, k1;  // the k range [k0, k1) = [0, k)
};
__device__ __forceinline__ TileGeom load_geom(const TileGeom &g) {
  const volatile TileGeom &v = g;
  return TileGeom{v.ti, v.tj, v.i0, v.j0, v.bm_eff, v.bn_eff, v.oa, v.ob, v.cra, v.crb, v.k0, v.k1};
}

constexpr int MAX_FIX = 32;  // distinct corrected cells per tile recomputed in the epilogue (R4)
struct SmemTail {
  TileGeom geo;
  // Cluster-pair B encode: the partner's 8 k-slot sums of B_J e per stage and its half maximum;
  // mfull[s] is arrived by the partner once mail[s] is written, mfree[s] by the partner once it
  // has consumed what this CTA wrote into its mailbox.
  double mail[STAGES][8];
  uint32_t mail_hm[STAGES];
  uint64_t mfull[STAGES], mfree[STAGES];
  int share;  // this CTA encodes half of B and swaps it with its cluster partner
  uint64_t full[STAGES], enc[STAGES], empty[STAGES];
  // Online verification (check_unit): per-warp partial sums, the reference sums, the carried
  // checksums, residuals (0..127 columns, 128..255 rows), dot-product partials.
  double colpart[2][128], rowpart4[4][128], colsum[128], rowsum[128], cs_col[128], cs_row[128];
  double dres[256];
  double red[NTHREADS / 32];
  unsigned int amax_hi, bmax_hi;   // PREPASS: the blocks' whole-k maxima (R1' high words)
  unsigned int int_am[8], int_bm[8];  // per-interval (slot t & 7) stage maxima from the encoders
  unsigned int cum_am, cum_bm;     // maxima of the intervals already verified
  int first_row[2], first_col[2];  // first flagged row / column, by check parity
  int nfix, fix[MAX_FIX];          // corrected cells (staged row | col << 8) to recompute (R4)
  int wstate[N_MMA_WARPS][8];      // per MMA warp: segment state of the k-loop (mma_role)
  int retry;                       // -1: done; else the interval whose check asked for a recompute
  int ticket;                      // k-split: arrival order of this split among the tile's splits
  // tau factors (2 gamma(kt + len) + 8u) kt len of intervals t < TAU_TAB, [0]: columns (len =
  // bm_eff), [1]: rows (len = bn_eff); filled while the first stage loads (check_decide)
  double tau_f[2][64];
};
constexpr size_t SMEM_BYTES = 1024 + sizeof(double) * STAGES * STAGE_ELEMS + sizeof(SmemTail);

// Named barriers (id 0 is __syncthreads).  Both roles execute the same sequence of the
// CTA-wide ones; the 256-thread ones are private to the MMA warpgroups.
enum { BAR_RING_FREE = 1, BAR_CTILE = 2, BAR_FLAGS_R = 3, BAR_FLAGS_C = 4, BAR_DECIDE = 5, BAR_RED = 6, BAR_PART = 7,
       BAR_REPORT = 8 };
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

// Warp roles.  The checksum warpgroup takes the HIGHEST warp ids: the issue arbiter favours
// high ids, so an encoder's few FP64 adds win the FP64 pipe over the saturating DMMA stream
// instead of starving behind it until the MMA warps stall.
constexpr bool CS_HIGH = true;
__device__ __forceinline__ bool is_cs_warp(int w) { return CS_HIGH ? w >= N_MMA_WARPS : w < N_CS_WARPS; }
__device__ __forceinline__ int cs_warp(int w) { return CS_HIGH ? w - N_MMA_WARPS : w; }
__device__ __forceinline__ int mma_warp(int w) { return CS_HIGH ? w : w - N_CS_WARPS; }

struct Ctx {
  double *ring;
  SmemTail *tl;
  int tid, lane, warp, tile, ti, tj, i0, j0, bm_eff, bn_eff, nk, f_lo, f_hi;
  int64_t k0, k1;
  int q, s0, nk_all;  // k-split: this CTA's split and its first global stage; stages of all of k
  int tile_slot;      // the tile's index in launch order (its k-split partials / ticket)
  // Protected tiles: TMA boxes start at the even coordinate xs = x0 - (x0 & 1) (the contiguous
  // dimension of a TMA box must start 16-byte aligned), so tile-local data row i sits in
  // staged row i + o (o = x0 & 1) and the checksum row/column takes the free row cr.
  int oa, ob, cra, crb;
  int enc_only;  // 0: a tile; 1: encoder CTA of e^T A_I (tile row ti); 2: of B_J e (tile column tj)
};

// ---------------- checksum warpgroup: four encoder warps, each also its stages' TMA producer
// Encoder warp w owns stages s = w (mod 4).  It issues the TMA loads of its own stages (lane
// 0: the first ring's worth up front, then stage s + 4 once the MMA warps have released that
// ring slot) and, in the protected pass, waits for stage s's bytes, forms
// a_sum[p] = sum_{i in I} op(A)_ip and b_sum[p] = sum_{j in J} op(B)_pj for the 16 k-slots,
// writes them into the free row cr of the staged A tile and of the staged B tile, and arrives
// on the stage's `enc` barrier (one arrival per operand: a tile's stages 0..3 split their A
// and B encodes between two warps, see the job loop).  The DMMA stream then computes C^f = [A; e^T A][B, B e]
// tile by tile: acc(cr, j) is the carried column checksum (e^T A_I) B_J and
// acc(i, cr) the carried row checksum A_I (B_J e) (outer-product maintenance).
// One encoder per SM sub-partition spreads the encode's issue slots evenly over the four DMMA
// streams, and owning every fourth stage leaves ~4 stage-times per encode job.
constexpr int N_ENC_WARPS = N_CS_WARPS;

template <bool AKM, bool BKM, bool FT>
__device__ __forceinline__ void checksum_role(const CUtensorMap &tmA, const CUtensorMap &tmB, const Params &P,
                                              const Ctx &x) {
  SmemTail &tl = *x.tl;
  double *const ring = x.ring;
  const int lane = x.lane, warp = cs_warp(x.warp);
  // The attempt's k range: this CTA's split first; a recompute (R6) covers the whole k.
  int nk = x.nk;
  int64_t k0 = x.k0, k1 = x.k1;
  const int xa = x.i0 - x.oa, xbj = x.j0 - x.ob;  // even box origins
  int stage_base = 0;
  // Lane 0: load stage s into its ring slot once the slot's previous stage is consumed.
  auto issue = [&](int s) {
    const int gs = stage_base + s, slot = gs % STAGES;
    if (gs >= STAGES) {
      mbar_wait_sleep(&tl.empty[slot], ((gs / STAGES) - 1) & 1);
      // The slot's checksum row / column was written through the generic proxy (encoder warps,
      // acquired here through enc -> MMA warps -> empty); order it before TMA (async proxy)
      // refills the slot.  Issued here, off the path of the stage the MMA warps wait for.
      if (FT && !(FT_DEV_MODE(P) & 2048)) fence_proxy_async();
    }
    double *sa = ring + slot * STAGE_ELEMS;
    mbar_arrive_expect_tx(&tl.full[slot], STAGE_BYTES);
    const int kc = (int)k0 + s * BK;
    if (AKM) {
      tma_load_2d(sa, &tmA, kc, xa, &tl.full[slot]);
    } else {
#pragma unroll
      for (int xb = 0; xb < 8; ++xb) tma_load_2d(sa + xb * 256, &tmA, xa + 16 * xb, kc, &tl.full[slot]);
    }
    double *sb = sa + TILE_ELEMS;
    if (BKM) {
      tma_load_2d(sb, &tmB, kc, xbj, &tl.full[slot]);
    } else {
#pragma unroll
      for (int xb = 0; xb < 8; ++xb) tma_load_2d(sb + xb * 256, &tmB, xbj + 16 * xb, kc, &tl.full[slot]);
    }
  };
  const uint32_t rank = P.cluster2 ? cluster_rank() : 0u;
  // e^T A_I of stage s: tile column 0 encodes it and publishes it; another tile copies the
  // published stage if its flag is already set and otherwise encodes the stage itself.  The
  // flag and the published sums are fetched before the stage's TMA bytes are waited for, so
  // the L2 round trips overlap the TMA latency.
  const bool a_pub = P.Ash && (P.enc_head ? x.enc_only == 1 : x.tj == 0);
  const bool a_sub = P.Ash && (P.enc_head ? x.enc_only == 0 : x.tj != 0);
  const bool b_pub = P.Bsh && (P.enc_head ? x.enc_only == 2 : x.ti == 0);
  struct PubA { bool ok; double a0, a1; uint32_t am; };
  // Relaxed loads of stage s's published e^T A_I words (not used until after the TMA wait).
  // Per attempt (the k range changes for a recompute): this lane's published words of the
  // attempt's first stage and its slot offsets of the checksum row / column (the copy path of
  // ~99% of the stages at C5 then costs a handful of instructions next to the DMMA stream).
  const int pa = AKM ? 2 * lane : lane;  // this lane's k-slot(s) of e^T A_I within a stage
  const double *srcA = nullptr, *srcB = nullptr;
  const unsigned *hmAp = nullptr, *hmBp = nullptr;
  int offA = 0, offB = 0;
  auto attempt_setup = [&]() {
    srcA = P.Ash ? P.Ash + x.ti * P.ldash + k0 + pa : nullptr;
    hmAp = P.hmA ? P.hmA + (size_t)x.ti * P.nk + k0 / BK : nullptr;
    srcB = P.Bsh ? P.Bsh + x.tj * P.ldbsh + k0 + lane : nullptr;
    hmBp = P.hmB ? P.hmB + (size_t)x.tj * P.nk + k0 / BK : nullptr;
    offA = sidx<AKM>(x.cra, AKM ? 2 * (lane & 7) : (lane & 15));
    offB = sidx<BKM>(x.crb, lane & 15);
  };
  attempt_setup();
  auto fetch_a = [&](int s) {
    PubA f{false, 0.0, 0.0, 0xFFFFFFFFu};
    if (!a_sub) return f;
    const int kl = (int)(k1 - k0) - s * BK;  // k-slots of this stage inside k
    const double *src = srcA + s * BK;
    if (AKM) {
      f.a0 = lane < 8 && pa < kl ? ld_relaxed_gpu(src) : 0.0;
      f.a1 = lane < 8 && pa + 1 < kl ? ld_relaxed_gpu(src + 1) : 0.0;
    } else {
      f.a0 = lane < 16 && pa < kl ? ld_relaxed_gpu(src) : 0.0;
    }
    f.am = ld_relaxed_gpu(hmAp + s);
    return f;
  };
  // Whole stage published?  (warp-uniform; encode mode FUSED_WAIT waits for it)
  auto check_a = [&](int s, PubA &f) {
    if (!a_sub) return;
    f.ok = __all_sync(0xffffffffu, pub_ok(f.a0) && pub_ok(f.a1) && pub_ok(f.am));
    while (P.wait_pub && !f.ok) {
      __nanosleep(256);
      f = fetch_a(s);
      f.ok = __all_sync(0xffffffffu, pub_ok(f.a0) && pub_ok(f.a1) && pub_ok(f.am));
    }
  };
  auto enc_a = [&](double *sA, int s, const PubA &f, double &a0, double &a1, uint32_t &amax) {
    if (f.ok) {
      a0 = f.a0;
      a1 = f.a1;
      amax = max(amax, f.am);
      return;
    }
    uint32_t hm = 0u;
    enc_operand<AKM>(sA, lane, x.cra, a0, a1, hm);
    amax = max(amax, hm);
    if (a_pub) {
      const int64_t sg = k0 / BK + s;
      const int p = AKM ? 2 * lane : lane;
      const int64_t pg = k0 + (int64_t)s * BK + p;
      double *dst = P.Ash + x.ti * P.ldash + pg;
      // (pg + 1 is stored only when it is < k1 <= ldash: odd k leaves the pair's second slot out)
      FT_CHECK(x.ti < P.tiles_m && sg < P.nk && k1 <= P.ldash && (pg >= k1 || pg < P.ldash));
      if (AKM) {
        if (lane < 8 && pg < k1) st_relaxed_gpu(dst, a0);
        if (lane < 8 && pg + 1 < k1) st_relaxed_gpu(dst + 1, a1);
      } else if (lane < 16 && pg < k1) {
        st_relaxed_gpu(dst, a0);
      }
      if (lane == 0) st_relaxed_gpu(P.hmA + (size_t)x.ti * P.nk + sg, hm);
    }
  };
  const int KcS = max(1, (int)(P.Kc / BK));
  int t_done = -1;  // intervals <= t_done are not verified again (retry after a recompute decision)
  for (int attempt = 0;; ++attempt) {
    const bool verify = FT && t_done < P.T - 1;
    if (lane == 0)
      for (int s = warp; s < nk && s < STAGES; s += N_ENC_WARPS) issue(s);
    // B_J e published by tile row 0 is copied per stage like e^T A_I.  Publication only
    // happens in launches without clusters, so a cluster pair (share) never copies.
    const bool b_sub = P.Bsh && (P.enc_head ? x.enc_only == 0 : x.ti != 0);
    // Only the first attempt exchanges half encodes with the cluster partner: a recompute pass
    // (this tile alone) encodes its B_J e itself, bitwise the same checksum.
    const bool share = verify && tl.share && attempt == 0;
    // Encode jobs.  Stages 0..3 of the tile: the two operands of a stage go to two warps
    // (warps 0, 2 share stages 0 and 2, warps 1, 3 stages 1 and 3; warps 0, 1 take A of stages
    // 0 / 1 and B of 2 / 3, warps 2, 3 the opposite), so the first stage -- on the critical path
    // at every tile start -- is encoded in about half the time of one warp doing both
    // (dev_timeline at 1016^2 x 256: first-stage wait 10.4k -> 6.3k clk).  From stage 4 on,
    // warp s % 4 encodes both operands of stage s (splitting every stage costs the long
    // shapes 0.2-0.3%).  The TMA issue stays with warp s % 4 throughout.
    bool split = verify;  // the unprotected kernel and recompute passes only issue TMA loads
    for (int s = verify ? (warp & 1) : warp;; s += split ? 2 : N_ENC_WARPS) {
      if (split && s >= N_ENC_WARPS) { split = false; s = warp + N_ENC_WARPS; }
      if (s >= nk) break;
      const bool doA = !split || ((((s >> 1) & 1) == 0) == (warp < 2));
      const bool doB = !split || !doA;
      if (verify) {
        const int gs = stage_base + s, slot = gs % STAGES;
        uint32_t amax_hi = 0u, bmax_hi = 0u;  // this stage's slice maxima (R1' high words)
        const long long t0 = FT_DEV_PROF(P) ? clock64() : 0;
        const bool pubs = !(P.Ac || (FT_DEV_MODE(P) & 3));
        PubA pa_ = pubs && doA ? fetch_a(s) : PubA{false, 0.0, 0.0, 0u};
        // B_J e words of this stage: relaxed loads before the TMA wait as well
        double pb = 0.0;
        uint32_t pbm = 0xFFFFFFFFu;
        auto fetch_b = [&]() {
          pb = lane < 16 && lane < (int)(k1 - k0) - s * BK ? ld_relaxed_gpu(srcB + s * BK) : 0.0;
          pbm = ld_relaxed_gpu(hmBp + s);
        };
        if (pubs && doB && b_sub) fetch_b();
        if (!(FT_DEV_MODE(P) & 16)) mbar_wait_sleep(&tl.full[slot], (gs / STAGES) & 1);
        if (pubs && doA) check_a(s, pa_);
        bool bcopy = false;
        if (pubs && doB && b_sub) {
          bcopy = __all_sync(0xffffffffu, pub_ok(pb) && pub_ok(pbm));
          while (P.wait_pub && !bcopy) {  // FUSED_WAIT: wait for tile row 0
            __nanosleep(256);
            fetch_b();
            bcopy = __all_sync(0xffffffffu, pub_ok(pb) && pub_ok(pbm));
          }
        }
        const long long t1 = FT_DEV_PROF(P) ? clock64() : 0;
        double *sA = ring + slot * STAGE_ELEMS, *sB = sA + TILE_ELEMS;
        double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
        if (P.Ac) {  // PREPASS: copy the pre-encoded 16 k-slots of e^T A_I / B_J e
          const int64_t p = k0 + s * BK + lane;
          if (lane < 16) {
            if (doA) sA[sidx<AKM>(x.cra, lane)] = p < k1 ? P.Ac[x.ti + p * P.ldac] : 0.0;
            if (doB) sB[sidx<BKM>(x.crb, lane)] = p < k1 ? P.Br[x.tj + p * P.ldbr] : 0.0;
          }
        } else if (FT_DEV_MODE(P) & 1) {  // development: pass 1 only
          if (doA) amax_hi = max(amax_hi, (uint32_t)__float_as_int(warp_max_nan(enc_pass1<AKM>(sA, lane, x.cra))));
          if (doB) bmax_hi = max(bmax_hi, (uint32_t)__float_as_int(warp_max_nan(enc_pass1<BKM>(sB, lane, x.crb))));
        } else if ((FT_DEV_MODE(P) & 2) && !share) {
          // development: no encode (checksum rows zero)
        } else {
         if (doA && x.enc_only != 2) {  // (an encoder CTA handles its own operand only)
          enc_a(sA, s, pa_, a0, a1, amax_hi);  // e^T A_I over the 127 data rows
          if (AKM) {
            if (lane < 8) *reinterpret_cast<double2 *>(sA + offA) = make_double2(a0, a1);
          } else {
            if (lane < 16) sA[offA] = a0;
          }
         }
         if (doB && x.enc_only != 1) {
          const int64_t sg = k0 / BK + s;  // global stage index
          if (bcopy) {  // B_J e of this stage as published by tile row 0
            if (lane < 16) sB[offB] = pb;
            bmax_hi = max(bmax_hi, pbm);
          } else {
            uint32_t hmb = 0u;
            if (share) {
              // Cluster pair: the half `rank` of B_J e here, the other half from the partner.
              enc_operand_h<BKM>(sB, lane, (int)rank, x.crb, b0, b1, hmb);
              // own half into the staged tile and into the partner's mailbox (lanes 0..3 hold two
              // k-slots each for a K-major B, lanes 0..7 one each for an MN-major B)
              if (gs >= STAGES && lane == 0) mbar_wait_acq_cluster(&tl.mfree[slot], ((gs / STAGES) - 1) & 1);
              __syncwarp();
              const uint32_t pmail = mapa_u32(smem_u32(&tl.mail[slot][0]), rank ^ 1u);
              if (BKM) {
                if (lane < 4) {
                  *reinterpret_cast<double2 *>(sB + sidx<true>(x.crb, 8 * (int)rank + 2 * lane)) = make_double2(b0, b1);
                  st_cluster_f64(pmail + 8u * (2 * lane), b0);
                  st_cluster_f64(pmail + 8u * (2 * lane + 1), b1);
                }
              } else {
                if (lane < 8) {
                  sB[sidx<false>(x.crb, 8 * (int)rank + lane)] = b0;
                  st_cluster_f64(pmail + 8u * lane, b0);
                }
              }
              if (lane == 0) st_cluster_u32(mapa_u32(smem_u32(&tl.mail_hm[slot]), rank ^ 1u), hmb);
              __syncwarp();
              if (lane == 0) mbar_arrive_remote(mapa_u32(smem_u32(&tl.mfull[slot]), rank ^ 1u));
              // the partner's half
              if (lane == 0) mbar_wait_acq_cluster(&tl.mfull[slot], (gs / STAGES) & 1);
              __syncwarp();
              if (lane < 8) sB[sidx<BKM>(x.crb, 8 * (int)(rank ^ 1u) + lane)] = tl.mail[slot][lane];
              hmb = max(hmb, tl.mail_hm[slot]);
              __syncwarp();
              if (lane == 0) mbar_arrive_remote(mapa_u32(smem_u32(&tl.mfree[slot]), rank ^ 1u));
            } else {
              enc_operand<BKM>(sB, lane, x.crb, b0, b1, hmb);  // B_J e over the 127 data columns
              if (BKM) {
                if (lane < 8) *reinterpret_cast<double2 *>(sB + sidx<true>(x.crb, 2 * lane)) = make_double2(b0, b1);
              } else {
                if (lane < 16) sB[sidx<false>(x.crb, lane)] = b0;
              }
            }
            bmax_hi = max(bmax_hi, hmb);
            if (b_pub) {  // tile row 0: publish this stage's B_J e for the other tile rows
              __syncwarp();
              const int64_t pg = k0 + (int64_t)s * BK + lane;
              FT_CHECK(x.tj < P.tiles_n && sg < P.nk && (pg >= k1 || pg < P.ldbsh));
              if (lane < 16 && pg < k1) st_relaxed_gpu(P.Bsh + x.tj * P.ldbsh + pg, sB[sidx<BKM>(x.crb, lane)]);
              if (lane == 0) st_relaxed_gpu(P.hmB + (size_t)x.tj * P.nk + sg, hmb);
            }
          }
         }
        }
        if (!P.Ac && lane == 0 && !(FT_DEV_MODE(P) & 4096)) {  // the interval's maxima, read by the MMA warps at its check
          const int tint = P.T == 1 ? 0 : min(s / KcS, P.T - 1) & 7;
          if (doA) atomicMax(&tl.int_am[tint], amax_hi);
          if (doB) atomicMax(&tl.int_bm[tint], bmax_hi);
        }
        __syncwarp();
        if (lane == 0) {  // one arrival per operand job (the barrier expects two per stage)
          mbar_arrive(&tl.enc[slot]);
          if (doA && doB) mbar_arrive(&tl.enc[slot]);
        }
        if (FT_DEV_PROF(P) && lane == 0) {
          const long long t2 = clock64();
          unsigned long long *dp = FT_DEV_PROF(P) + ((size_t)blockIdx.x * 12 + warp) * 2;
          dp[0] += (unsigned long long)(t1 - t0);
          dp[1] += (unsigned long long)(t2 - t1);
        }
      }
      const int s2 = s + N_ENC_WARPS;  // the next stage of this warp's TMA ring slots
      if (lane == 0 && (s & 3) == warp && s2 >= STAGES && s2 < nk) issue(s2);
      __syncwarp();
    }
    stage_base += nk;
    bar_sync(BAR_RING_FREE, NTHREADS);  // ring consumed by everyone
    if (!verify) return;
    bar_sync(BAR_DECIDE, NTHREADS);     // MMA warps decided: done, or recompute from k = 0
    const int r = tl.retry;
    if (r < 0) return;
    t_done = r;
    nk = x.nk_all;  // a recompute covers the whole k (a k-split tile is recomputed unsplit)
    k0 = 0;
    k1 = P.k;
    attempt_setup();
  }
}

// ---- online verification (§II.A, 258 §V.A) from the LIVE accumulators.
// The MMA tile is the unit's C^f block: staged row cra holds the carried column checksums
// (e^T A_I) B_J, staged column crb the carried row checksums A_I (B_J e).  At the
// end of verification interval t (after kt = min((t+1) Kc, k) rank-1 updates) the 256 MMA
// threads form the reference checksums e^T C and C e of the partial product held in their
// registers: per thread over its 8 rows / 8 columns of the m8n8k4 accumulator fragments, then
// warp shuffles over the lanes sharing a column (xor 4, 8, 16) or a row (xor 1, 2), then a small
// shared-memory exchange across the 2 x 4 warp grid.  Residuals d = r - cs against tau (DESIGN
// R1, R1', R17, clamped: R13), flags counted with bar.red.popc; exactly one flagged row and one
// flagged column -> the element at their intersection is corrected in its owner's register
// (recompute over [0, kt) or subtract; R4); any other pattern -> the unit is
// recomputed (R6).  Returns true for the latter.
template <bool AKM, bool BKM>
__device__ __forceinline__ int acc_owner_index(int si, int sj, int wm, int wn, int lane) {
  // Register index (a*4 + b)*2 + e of staged element (si, sj) in this thread, or -1.
  const int lr = si & 63, lc = sj & 31;
  const int fmt = AKM ? (lr >> 3) : 2 * (lr >> 4) + (lr & 1);
  const int rr = lr & 7;  // K-major: row in the 8-row tile = 4*(g&1) + (g>>1)
  const int fg = AKM ? (((rr & 3) << 1) | (rr >> 2)) : ((lr & 15) >> 1);
  const int fnt = BKM ? (lc >> 3) : 2 * (lc >> 4) + (lc & 1);
  const int cr = lc & 7;  // K-major: column in the 8-column tile, same mapping
  const int cc = BKM ? (((cr & 3) << 1) | (cr >> 2)) : ((lc & 15) >> 1);  // n-index
  const bool owner = (si >> 6) == wm && (sj >> 5) == wn && lane == fg * 4 + (cc >> 1);
  return owner ? (fmt * 4 + fnt) * 2 + (cc & 1) : -1;
}

// Record a corrected cell (staged row si, column sj) for the epilogue's fresh dot product.
__device__ __forceinline__ void add_fix(SmemTail &tl, int si, int sj) {
  const int cell = si | (sj << 8);
  int q = 0;
  while (q < tl.nfix && tl.fix[q] != cell) ++q;
  if (q == tl.nfix && q < MAX_FIX) tl.fix[tl.nfix++] = cell;
}

struct CheckOut {
  int multi;    // 1: recompute the unit (R6)
  int si, sj;   // single error: the located staged cell (si = -1: none)
  double dcol;  // the located magnitude d_col to subtract from it
};

// DESIGN.md R1, R17: 2 gamma(kt + len) for the two sums plus 2^-50 = 8u for the fixed-point
// encode (per element below 2^-50 max|x|, summed over len rows and kt k-slots), times kt len;
// tau = min(factor * amax * bmax, DBL_MAX) (R13: a NaN or infinite residual always flags).
constexpr int TAU_TAB = 64;
__device__ __forceinline__ double tau_factor(int64_t kt, int len) {
  const double nu = (double)(kt + len) * 0x1p-53;
  return (2.0 * (nu / (1.0 - nu)) + 0x1p-50) * (double)kt * (double)len;
}

// Residuals, threshold, flags, classification and report of one unit at the end of
// interval t, from the reference sums (tl.colsum, tl.rowsum) and the carried checksums
// (tl.cs_col, tl.cs_row) already in shared memory.  All 256 MMA threads.
template <bool AKM, bool BKM>
__device__ __forceinline__ CheckOut check_decide(const Params &P, SmemTail &tl, int t, int64_t kt, int mw, int lane) {
  const int vt = mw * 32 + lane;  // 0..255
  const TileGeom x = load_geom(tl.geo);
  // Cumulative maxima of op(A)_I and op(B)_J over the updates so far (R1'): the running value
  // plus the encoders' maxima of interval t's stages (slot t & 7; PREPASS: whole-k presets).
  const uint32_t amax_hi = max(tl.cum_am, tl.int_am[t & 7]), bmax_hi = max(tl.cum_bm, tl.int_bm[t & 7]);
  // one thread per data column (vt < 128) / data row (vt >= 128): residual, tau, flag
  const int par = t & 1;
  const int cidx = vt & 127;
  const bool is_row = vt >= 128;
  double d = 0.0;
  bool valid = false;
  if (cidx < DM) {
    if (is_row) {
      const int sr = cidx + x.oa;
      valid = cidx < x.bm_eff;
      d = tl.rowsum[sr] - tl.cs_row[sr];
    } else {
      const int sc = cidx + x.ob;
      valid = cidx < x.bn_eff;
      d = tl.colsum[sc] - tl.cs_col[sc];
    }
  }
  // R1': maxima rounded up to the largest double with the same high word.
  const double amx = __longlong_as_double((long long)(((unsigned long long)amax_hi << 32) | 0xFFFFFFFFull));
  const double bmx = __longlong_as_double((long long)(((unsigned long long)bmax_hi << 32) | 0xFFFFFFFFull));
  const int len = is_row ? x.bn_eff : x.bm_eff;
  // (the factor of interval t, formed before the k-loop for t < TAU_TAB: same expression, same
  // rounding; the check's own dependent chain is two products)
  const double fct = t < TAU_TAB ? tl.tau_f[is_row ? 1 : 0][t] : tau_factor(kt, len);
  const double tau = fmin(fct * amx * bmx, 0x1.fffffffffffffp1023);
  const bool flag = valid && !(fabs(d) <= tau) && !(FT_DEV_MODE(P) & 4);
  tl.dres[vt] = d;
  if (flag) atomicMin(is_row ? &tl.first_row[par] : &tl.first_col[par], cidx);
  const int nfr = bar_popc(BAR_FLAGS_R, 256, flag && is_row);
  const int nfc = bar_popc(BAR_FLAGS_C, 256, flag && !is_row);
  if (vt == 0) {  // everyone has read the maxima and the other parity's slots: roll them over
    tl.first_row[par ^ 1] = 0x7fffffff;
    tl.first_col[par ^ 1] = 0x7fffffff;
    tl.cum_am = amax_hi;
    tl.cum_bm = bmax_hi;
    tl.int_am[t & 7] = tl.int_bm[t & 7] = 0u;  // the slot of interval t + 8
  }
  CheckOut out{0, -1, 0, 0.0};
  if (nfr == 0 && nfc == 0) return out;
  const bool multi = !(nfr == 1 && nfc == 1);
  const int fr = tl.first_row[par], fc = tl.first_col[par];
  if (!multi) {  // single error at the intersection (i0+fr, j0+fc)
    out.si = fr + x.oa;
    out.sj = fc + x.ob;
    out.dcol = tl.dres[fc];
  }
  if (vt == 0) {
    atomicAdd(&P.counters[CNT_DETECTED], 1ull);
    atomicAdd(&P.counters[multi ? CNT_RECOMPUTED : CNT_CORRECTED], 1ull);
    const unsigned long long slot = atomicAdd(&P.counters[CNT_EVENTS], 1ull);
    // (a direction without flags keeps its sentinel: a checksum-lane fault flags one direction)
    FT_CHECK((nfr == 0 || (fr >= 0 && fr < 128)) && (nfc == 0 || (fc >= 0 && fc < 128)));
    if ((long long)slot < P.ev_cap)
      P.events[slot] = multi ? EventDev{(long long)(x.i0 + P.ev_row_off), (long long)(x.j0 + P.ev_col_off), 2, t,
                                        nfr ? tl.dres[128 + fr] : 0.0, nfc ? tl.dres[fc] : 0.0}
                             : EventDev{(long long)(x.i0 + fr + P.ev_row_off), (long long)(x.j0 + fc + P.ev_col_off), 1, t,
                                        tl.dres[128 + fr], tl.dres[fc]};
  }
  out.multi = multi ? 1 : 0;
  return out;
}

// Register partials of a check, reduce-scatter form.  Columns: two batches of 4 columns
// q = 4j + i (q = 2b + e), 4 independent chains over this thread's 8 rows; the 8 lanes sharing
// the columns (lane bits 2..4) reduce-scatter them (2 + 1 shuffles, then 1 for the last pair):
// lanes g, g ^ 1 end with column i = h1 + 2 h2.  Rows: two batches of 4 rows a = 4j + i over
// this thread's 8 columns; the 4 lanes sharing the rows (lane bits 0..1) reduce-scatter them
// (2 + 1 shuffles): lane tq ends with row a = 4j + tq.  The checksum row cra / column crb are
// left out of the sums and stored as the carried checksums.  STD: they sit at tile row /
// column 0 or DM (every tile but the partial edge tiles), i.e. in register (a, g) = (0, 0) of
// warp row 0 or (7, 7) of warp row 1 (column: (b, e, tq) = (0, 0, 0) of warp column 0 or
// (3, 1, 3) of warp column 3) in both fragment layouts, so only those registers need a select.
template <bool AKM, bool BKM, bool STD>
__device__ __forceinline__ void partials_rs(SmemTail &tl, const double (&acc)[8][4][2], int lg, int lt, int lwm, int lwn,
                                            int cra, int crb) {
  const bool exA0 = STD && cra == 0 && lwm == 0 && lg == 0, exA7 = STD && cra == DM && lwm == 1 && lg == 7;
  const bool exB0 = STD && crb == 0 && lwn == 0 && lt == 0, exB7 = STD && crb == DM && lwn == 3 && lt == 3;
  {
    const bool h2 = (lg >> 2) & 1, h1 = (lg >> 1) & 1;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      double c[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int b = 2 * j + (i >> 1), e = i & 1;
        double x = 0.0;
#pragma unroll
        for (int a = 0; a < 8; ++a) {
          if (STD) {
            x += ((a == 0 && exA0) || (a == 7 && exA7)) ? 0.0 : acc[a][b][e];
          } else {
            if (lwm * 64 + tile_row<AKM>(a, lg) != cra) x += acc[a][b][e];
            else tl.cs_col[lwn * 32 + tile_row<BKM>(b, 2 * lt + e)] = acc[a][b][e];  // carried (e^T A_I) B_J
          }
        }
        c[i] = x;
      }
      double c2[2];
#pragma unroll
      for (int u = 0; u < 2; ++u)  // i = u + 2 h2
        c2[u] = (h2 ? c[u + 2] : c[u]) + __shfl_xor_sync(0xffffffffu, h2 ? c[u] : c[u + 2], 16);
      double c1 = (h1 ? c2[1] : c2[0]) + __shfl_xor_sync(0xffffffffu, h1 ? c2[0] : c2[1], 8);  // i = h1 + 2 h2
      c1 += __shfl_xor_sync(0xffffffffu, c1, 4);
      if ((lg & 1) == 0) tl.colpart[lwm][lwn * 32 + tile_row<BKM>(2 * j + (h2 ? 1 : 0), 2 * lt + (h1 ? 1 : 0))] = c1;
    }
  }
  {
    const bool h1 = (lt >> 1) & 1, h0 = lt & 1;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      double r[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        double x = 0.0;
#pragma unroll
        for (int b = 0; b < 4; ++b)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            if (STD) {
              x += ((b == 0 && e == 0 && exB0) || (b == 3 && e == 1 && exB7)) ? 0.0 : acc[4 * j + i][b][e];
            } else {
              if (lwn * 32 + tile_row<BKM>(b, 2 * lt + e) != crb) x += acc[4 * j + i][b][e];
              else tl.cs_row[lwm * 64 + tile_row<AKM>(4 * j + i, lg)] = acc[4 * j + i][b][e];  // carried A_I (B_J e)
            }
          }
        r[i] = x;
      }
      double r2[2];
#pragma unroll
      for (int u = 0; u < 2; ++u)  // i = u + 2 h1
        r2[u] = (h1 ? r[u + 2] : r[u]) + __shfl_xor_sync(0xffffffffu, h1 ? r[u] : r[u + 2], 2);
      const double r1 = (h0 ? r2[1] : r2[0]) + __shfl_xor_sync(0xffffffffu, h0 ? r2[0] : r2[1], 1);  // i = tq
      tl.rowpart4[lwn][lwm * 64 + tile_row<AKM>(4 * j + lt, lg)] = r1;
    }
  }
  if (STD) {  // the carried checksums (e^T A_I) B_J and A_I (B_J e)
    if (exA0 || exA7) {
#pragma unroll
      for (int b = 0; b < 4; ++b)
#pragma unroll
        for (int e = 0; e < 2; ++e) tl.cs_col[lwn * 32 + tile_row<BKM>(b, 2 * lt + e)] = exA0 ? acc[0][b][e] : acc[7][b][e];
    }
    if (exB0 || exB7) {
#pragma unroll
      for (int a = 0; a < 8; ++a) tl.cs_row[lwm * 64 + tile_row<AKM>(a, lg)] = exB0 ? acc[a][0][0] : acc[a][3][1];
    }
  }
}

// Check at the end of an intermediate interval (Kc < k), with the accumulators LIVE in
// registers (the k-loop continues): straight from the registers, in two sequential passes with
// few live temporaries -- column partials one n-tile at a time (over this thread's 8 rows, then
// a butterfly over the 8 lanes sharing the column), then row partials one m-tile at a time
// (over its 8 columns, then a butterfly over the 4 lanes sharing the row); the 2 x 4 warp grid's
// partials meet in shared memory (6 KB; no staging of the tile).  The checksum row / column are
// excluded by index.  The loop-carried segment state lives in shared memory, so the DMMA k-loop
// keeps its register allocation (tools/kloop_stats.py).
template <bool AKM, bool BKM, int RS>
__device__ __forceinline__ CheckOut check_unit(const Params &P, SmemTail &tl, const double (&acc)[8][4][2], int t,
                                               int64_t kt, int mw, int wm, int wn, int lane) {
  const int g = lane >> 2, tq = lane & 3;
  const int vt = mw * 32 + lane;  // 0..255
#ifdef FTBLAS_DEV
  const long long dv_t0 = clock64();
#endif
  // Every MMA warp has issued its last DMMA of the interval before anyone sums: a dependent
  // FP64 add next to a running DMMA stream waits ~270-1000 clocks (profiles/
  // fp64_latency_under_dmma.json), ~8 once the FP64 pipe is free (end-of-tile check 7.4k ->
  // see DESIGN.md section 6).
  bar_sync(BAR_PART, 256);
#ifdef FTBLAS_DEV
  const long long dv_ta = clock64();
  // drain probe: a shared store of this warp's last DMMA result issues only once it has landed
  *reinterpret_cast<volatile double *>(&tl.red[mw]) = acc[7][3][1];
  const long long dv_tb = clock64();
#endif
  const int cra = tl.geo.cra, crb = tl.geo.crb;
  // RS 0: the serial form below; 1: the reduce-scatter form for the standard checksum positions,
  // else the serial form; 2: the reduce-scatter form always.  (Chosen per call site and layout
  // so that the DMMA k-loop around an intermediate check keeps its registers.)
  const bool std_geo = (cra == 0 || cra == DM) && (crb == 0 || crb == DM);
  if (RS == 0 || (RS == 1 && !std_geo)) {
    // serial: one column / row chain at a time with full butterflies
#pragma unroll
    for (int b = 0; b < 4; ++b) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int col = wn * 32 + tile_row<BKM>(b, 2 * tq + e);
        double c = 0.0;
#pragma unroll
        for (int a = 0; a < 8; ++a) {
          const double v = acc[a][b][e];
          if (wm * 64 + tile_row<AKM>(a, g) != cra) c += v;
          else tl.cs_col[col] = v;  // carried (e^T A_I) B_J
        }
#pragma unroll
        for (int o = 4; o <= 16; o <<= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
        if (g == 0) tl.colpart[wm][col] = c;
      }
    }
#pragma unroll
    for (int a = 0; a < 8; ++a) {
      const int row = wm * 64 + tile_row<AKM>(a, g);
      double r = 0.0;
#pragma unroll
      for (int b = 0; b < 4; ++b)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const double v = acc[a][b][e];
          if (wn * 32 + tile_row<BKM>(b, 2 * tq + e) != crb) r += v;
          else tl.cs_row[row] = v;  // carried A_I (B_J e)
        }
      r += __shfl_xor_sync(0xffffffffu, r, 1);
      r += __shfl_xor_sync(0xffffffffu, r, 2);
      if (tq == 0) tl.rowpart4[wn][row] = r;
    }
  } else {
    // Lane / warp coordinates laundered here, so the index arithmetic is not hoisted out of the
    // k-loop's segment loop (where it would hold registers across the DMMA stream).
    int lg = g, lt = tq, lwm = wm, lwn = wn;
    asm volatile("" : "+r"(lg), "+r"(lt), "+r"(lwm), "+r"(lwn));
    if (std_geo) partials_rs<AKM, BKM, true>(tl, acc, lg, lt, lwm, lwn, cra, crb);
    else if (RS == 2) partials_rs<AKM, BKM, false>(tl, acc, lg, lt, lwm, lwn, cra, crb);
  }
  bar_sync(BAR_PART, 256);
#ifdef FTBLAS_DEV
  const long long dv_t1 = clock64();
#endif
  if (vt < 128) {
    tl.colsum[vt] = tl.colpart[0][vt] + tl.colpart[1][vt];
  } else {
    const int r = vt - 128;
    tl.rowsum[r] = (tl.rowpart4[0][r] + tl.rowpart4[1][r]) + (tl.rowpart4[2][r] + tl.rowpart4[3][r]);
  }
  bar_sync(BAR_PART, 256);
#ifdef FTBLAS_DEV
  const long long dv_t2 = clock64();
  const CheckOut dv_out = check_decide<AKM, BKM>(P, tl, t, kt, mw, lane);
  if (FT_DEV_PROF(P) && vt == 0) {  // [arrival + register partials, combine], [count, decision]
    unsigned long long *dp = FT_DEV_PROF(P) + ((size_t)blockIdx.x * 12 + 8) * 2;
    const long long t3 = clock64();
    dp[0] += (unsigned long long)(dv_t1 - dv_t0);
    dp[1] += (unsigned long long)(dv_t2 - dv_t1);
    dp[2] += 1ull;
    dp[3] += (unsigned long long)(t3 - dv_t2);
    dp[4] += (unsigned long long)(dv_ta - dv_t0);  // arrival skew (first barrier)
    dp[5] += (unsigned long long)(dv_tb - dv_ta);  // drain of this warp's DMMA stream
  }
  return dv_out;
#else
  return check_decide<AKM, BKM>(P, tl, t, kt, mw, lane);
#endif
}

// k-split with co-resident splits (P.kcoop): wait for the tile's S partial blocks, sum slice q
// of the accumulator registers [64q/S, 64(q+1)/S) over them in split order into partial 0,
// then (split S-1) wait for every slice.  Out of line: it touches memory only, and inlined it
// moved the register allocation of the DMMA k-loops.
__device__ __forceinline__ void ksplit_coop_reduce(const Params &P, SmemTail &tl, const double *p0, int slot, int q,
                                                int S, int vt) {
  if (vt == 0) {
    tl.ticket = q;
    atomicAdd(&P.tickets[slot], 1);
    while (ld_acquire_gpu(&P.tickets[slot]) < S) __nanosleep(32);
  }
  bar_sync(BAR_CTILE, 256);
  double *const sum0 = const_cast<double *>(p0);
  for (int reg = (64 * q) / S; reg < (64 * (q + 1)) / S; ++reg) {
    double v = __ldcg(p0 + reg * 256);
    for (int r = 1; r < S; ++r) v += __ldcg(p0 + (size_t)r * (BM * BN) + reg * 256);
    __stcg(sum0 + reg * 256, v);
  }
  __threadfence();
  bar_sync(BAR_CTILE, 256);
  if (vt == 0) {
    atomicAdd(&P.tickets[slot], 1);
    if (q == S - 1)
      while (ld_acquire_gpu(&P.tickets[slot]) < 2 * S) __nanosleep(32);
  }
  bar_sync(BAR_CTILE, 256);
}

// The DMMA k-loop of a sliver tile's warp over its first NA m-tiles and NB n-tiles only.
template <bool AKM, bool BKM, int NA, int NB>
__device__ __forceinline__ void kloop_narrow(SmemTail &tl, const double *ring, uint32_t ready, int &gs, int gs_end,
                                             int wm, int wn, int g, int t, int lane, double (&acc)[8][4][2]) {
  for (; gs < gs_end; ++gs) {
    const int slot = gs % STAGES;
    mbar_wait_u32(ready + 8u * slot, (gs / STAGES) & 1);
    const double *sA = ring + slot * STAGE_ELEMS, *sB = sA + TILE_ELEMS;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      double af[2][NA], bf[2][NB];
      load_frags<AKM, NA>(sA, wm * 64, h, g, t, af);
      load_frags<BKM, NB>(sB, wn * 32, h, g, t, bf);
#pragma unroll
      for (int e = 0; e < 2; ++e)
#pragma unroll
        for (int a = 0; a < NA; ++a)
#pragma unroll
          for (int b = 0; b < NB; ++b) dmma_8x8x4(acc[a][b], af[e][a], bf[e][b]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&tl.empty[slot]);
  }
}

// ---------------- warpgroups 1-2: MMA warps (+ online verification and epilogue)
template <bool AKM, bool BKM, bool FT>
__device__ __forceinline__ void mma_role(const Params &P, const Ctx &x) {
  SmemTail &tl = *x.tl;
  double *const ring = x.ring;
  double *const ctile = ring;  // epilogue reuse of the ring
  const int lane = x.lane;
  // Warp w runs on SM sub-partition w & 3.  The 64 x 32 quarter (wm, wn) of warp w has
  // wn = (w + 2 wm) & 3, so each warp row spans all four sub-partitions and the two warps of a
  // warp column sit on different ones (a partial edge tile's active warps share the DMMA pipes
  // of at least two sub-partitions).
  const int mw = mma_warp(x.warp), wm = mw >> 2, wn = (mw + 2 * wm) & 3;
  const int g = lane >> 2, t = lane & 3;
  const int vt = mw * 32 + lane;  // 0..255
  // Rows / columns of the MMA tile that carry data or a checksum; in the protected kernel a
  // warp whose quarter holds none of them (partial edge tiles) waits and releases the stages
  // without issuing DMMA.  (The unprotected kernel keeps one loop: the split costs its k-loop
  // codegen and its tiles are only partial at sizes that are not multiples of 128.)
  // SKIP: whether this instantiation has the idle-warp loop.  The protected kernel always; the
  // unprotected K-major-A / MN-major-B one too (ptxas allocates its DMMA loop better with it:
  // 106 instead of 186 non-DMMA instructions per stage, tools/kloop_stats.py); the other
  // unprotected ones keep their single loop.
  constexpr bool SKIP = FT || (AKM && !BKM);
  const bool active = FT ? (!x.enc_only && wm * 64 < max(x.oa + x.bm_eff, x.cra + 1) && wn * 32 < max(x.ob + x.bn_eff, x.crb + 1))
                         : (!SKIP || (wm * 64 < x.bm_eff && wn * 32 < x.bn_eff));
  // Sliver tiles (the last tile row / column of a size that is not a multiple of 127): a warp
  // whose used rows (columns) of its 64 x 32 quarter fit in its first 2 m-tiles (n-tiles) -- 16
  // rows (columns) in either fragment layout -- runs a narrow DMMA loop over those tiles only
  // (bit 0: rows, bit 1: columns); the other accumulators stay zero.
  // (kept in the warp's shared slot W_NARROW: no register held across the DMMA loops)
  double acc[8][4][2];
  // Segment state that changes only between segments lives in this warp's shared-memory slots
  // (lane-uniform), not in registers across the DMMA loop: next fault stage, next interval end,
  // next fault index, the interval of a recompute decision in this attempt.
  // (32-bit shared addresses through volatile ld/st.shared: no generic pointer held in registers)
  const uint32_t ws = smem_u32(&tl.wstate[mw][0]);
  enum { W_NEXT_STAGE = 0, W_NEXT_CHECK, W_FNEXT, W_FAILED, W_BASE, W_NARROW, W_NK, W_SOFF };
  if (lane == 0) {
    st_sv(ws, W_BASE, 0);
    // (bits 4 / 8: the used rows / columns fit in the first m-tile / n-tile of a K-major
    // operand, 8 rows / columns)
    const int ur = max(x.oa + x.bm_eff, x.cra + 1) - wm * 64, uc = max(x.ob + x.bn_eff, x.crb + 1) - wn * 32;
    st_sv(ws, W_NARROW, !FT ? 0
                            : (ur <= 16 ? 1 : 0) | (uc <= 16 ? 2 : 0) | (AKM && ur <= 8 ? 4 : 0) |
                                  (BKM && uc <= 8 ? 8 : 0));
  }
  if (FT) {  // the checks' tau factors, while the first stage loads (the FP64 pipe is idle here)
    const int kcs = max(1, (int)(P.Kc / BK)), nt = min(P.T, TAU_TAB);
    for (int q = vt; q < 2 * nt; q += 256) {
      const int t = q >> 1;
      const int64_t kt = t < P.T - 1 ? (int64_t)(t + 1) * kcs * BK : P.k;  // the check's kt (mma_role calls)
      tl.tau_f[q & 1][t] = tau_factor(kt, (q & 1) ? x.bn_eff : x.bm_eff);
    }
  }
#ifdef FTBLAS_DEV_TIMELINE
  // tools/dev_timeline.py (timeline build, -DFTBLAS_DEV_TIMELINE only): MMA warp 0's
  // [globaltimer at start, first stage ready, k-loop end, role end] (clock64 offsets) in the
  // CTA's dev_prof slots 10..11 (u64 20..23; the start clock parks in 23, so no register is held
  // across the k-loop).
#define FT_TL(i) (P.dev_prof[(size_t)blockIdx.x * 24 + 20 + (i)])
  // (u64 16..18: after the last check, after the ring is released, before the stores)
  if (P.dev_prof && vt == 0) {
    unsigned long long gt;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
    FT_TL(0) = gt;
    FT_TL(3) = (unsigned long long)clock64();
    mbar_wait_u32(smem_u32(tl.full) + (FT ? STAGES * 8u : 0u), 0);
    FT_TL(1) = (unsigned long long)clock64() - FT_TL(3);
  }
#endif
  for (int attempt = 0;; ++attempt) {
    // Interval of the last recompute decision (tl.retry, -1 in the first attempt): intervals
    // <= t_done are neither re-injected nor re-verified (the unit restarts from k = 0).
    const int t_done = tl.retry;
    const bool verify = FT && t_done < P.T - 1;
    if (lane == 0) {
      // The attempt's stages: this CTA's k-split first (local stage 0 = global stage s0); a
      // recompute covers the whole k.  Fault stages are global: compared as stage - s0.
      st_sv(ws, W_NK, attempt == 0 ? x.nk : x.nk_all);
      st_sv(ws, W_SOFF, attempt == 0 ? x.s0 : 0);
      st_sv(ws, W_FNEXT, x.f_lo);
      st_sv(ws, W_NEXT_STAGE, x.f_lo < x.f_hi ? P.faults[x.f_lo].stage - (attempt == 0 ? x.s0 : 0) : 0x7fffffff);
      // Stage index at which the next intermediate verification interval ends (Kc = KcS
      // stages); the last interval is checked after the k-loop, on the staged tile.
      st_sv(ws, W_NEXT_CHECK, verify && !x.enc_only && t_done + 1 < P.T - 1 ? (t_done + 2) * max(1, (int)(P.Kc / BK)) : 0x7fffffff);
      st_sv(ws, W_FAILED, -1);
    }
    __syncwarp();
#pragma unroll
    for (int a = 0; a < 8; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
    // The protected pass waits for the encoded stage (TMA bytes + checksum row/column), the
    // unprotected one for the TMA bytes only.
    // 32-bit shared address of the barrier array to wait on (enc = full + STAGES).
    const uint32_t ready = smem_u32(tl.full) + ((verify && !(FT_DEV_MODE(P) & 8)) ? STAGES * 8u : 0u);
    // The k-loop runs in segments between fault stages and interval ends, so that the DMMA loop
    // body carries neither injection nor verification code (which would make the register
    // allocator shuffle accumulators).
    // Stage counters run on the global stage index gs (ring slot gs % STAGES, parity
    // (gs / STAGES) & 1); this attempt's first stage is kept in the warp's shared slot W_BASE.
    for (int s = 0;;) {
      const int base = ld_sv(ws, W_BASE);
      int gs = base + s;
      const int gs_end = base + __shfl_sync(0xffffffffu, min(min(ld_sv(ws, W_NEXT_STAGE), ld_sv(ws, W_NEXT_CHECK)), ld_sv(ws, W_NK)), 0);
      if (SKIP && !active) {  // nothing of this warp's quarter is used: release the stages only
        for (; gs < gs_end; ++gs) {
          const int slot = gs % STAGES;
          mbar_wait_u32(ready + 8u * slot, (gs / STAGES) & 1);
          __syncwarp();
          if (lane == 0) mbar_arrive(&tl.empty[slot]);
        }
      }
      const int narrow = FT ? ld_sv(ws, W_NARROW) : 0;
      if (FT && narrow) {  // sliver tiles: only the m / n tiles holding used rows / columns
        if (AKM && (narrow & 4)) {
          if (narrow & 2) kloop_narrow<AKM, BKM, 1, 2>(tl, ring, ready, gs, gs_end, wm, wn, g, t, lane, acc);
          else kloop_narrow<AKM, BKM, 1, 4>(tl, ring, ready, gs, gs_end, wm, wn, g, t, lane, acc);
        } else if (BKM && (narrow & 8)) {
          if (narrow & 1) kloop_narrow<AKM, BKM, 2, 1>(tl, ring, ready, gs, gs_end, wm, wn, g, t, lane, acc);
          else kloop_narrow<AKM, BKM, 8, 1>(tl, ring, ready, gs, gs_end, wm, wn, g, t, lane, acc);
        } else if (narrow == 1) kloop_narrow<AKM, BKM, 2, 4>(tl, ring, ready, gs, gs_end, wm, wn, g, t, lane, acc);
        else if (narrow == 2) kloop_narrow<AKM, BKM, 8, 2>(tl, ring, ready, gs, gs_end, wm, wn, g, t, lane, acc);
        else kloop_narrow<AKM, BKM, 2, 2>(tl, ring, ready, gs, gs_end, wm, wn, g, t, lane, acc);
      }
      for (; gs < gs_end; ++gs) {
        const int slot = gs % STAGES;
        mbar_wait_u32(ready + 8u * slot, (gs / STAGES) & 1);
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
      }
      s = gs - ld_sv(ws, W_BASE);
      // At the end of a segment: an interval ends at stage s (its check comes before the faults
      // due at stage s, which belong to the next interval).  One call site each, so the
      // register allocation of the DMMA loop is not disturbed.
      // A correction located by the check is applied like a fault: -d_col at the located cell
      // (one select block for both, so the register allocation of the DMMA loop is undisturbed).
      int pend_si = -1, pend_sj = 0;
      double pend_d = 0.0;
      if (FT && s == ld_sv(ws, W_NEXT_CHECK)) {
        const int kcs = max(1, (int)(P.Kc / BK));
        const int tcur = s / kcs - 1;
        const CheckOut co = check_unit<AKM, BKM, BKM ? 2 : (AKM ? 0 : 1)>(P, tl, acc, tcur, (int64_t)s * BK, mw, wm, wn, lane);
        // A single error is subtracted now, so the next intervals verify the
        // corrected partial product; in recompute mode (R4) the cell is also replaced by a fresh
        // k-long dot product in the epilogue (fix list), which equals the oracle's recomputed
        // partial plus its later updates.
        pend_si = co.si;
        pend_sj = co.sj;
        pend_d = -co.dcol;
        if (vt == 0 && co.si >= 0 && P.correct_mode != 1) add_fix(tl, co.si, co.sj);
        __syncwarp();
        if (lane == 0) {
          if (co.multi) {  // recompute: the rest of this attempt is neither injected nor verified
            st_sv(ws, W_FAILED, tcur);
            st_sv(ws, W_NEXT_CHECK, 0x7fffffff);
            st_sv(ws, W_FNEXT, x.f_hi);
            st_sv(ws, W_NEXT_STAGE, 0x7fffffff);
          } else {
            st_sv(ws, W_NEXT_CHECK, tcur + 1 < P.T - 1 ? (tcur + 2) * kcs : 0x7fffffff);
          }
        }
        __syncwarp();
      }
      // Then the faults due before stage s's updates (s == nk: after the last update).
      for (;;) {
        int si = -1, sj = 0;
        double dv = 0.0;
        if (pend_si >= 0) {
          si = pend_si;
          sj = pend_sj;
          dv = pend_d;
          pend_si = -1;
        } else if (s == ld_sv(ws, W_NEXT_STAGE)) {
          const int fnext = ld_sv(ws, W_FNEXT);
          FT_CHECK(fnext >= x.f_lo && fnext < x.f_hi && x.f_hi <= P.nfaults);
          const FaultDev f = P.faults[fnext];
          FT_CHECK(f.tile == x.tile && f.li < 127 && f.lj < 127 && f.li >= -1 && f.lj >= -1);
          // a fault belongs to interval min(stage / KcS, T - 1); a retry skips the decided ones
          if (min(f.stage / max(1, (int)(P.Kc / BK)), P.T - 1) > tl.retry) {
            const TileGeom gf = load_geom(tl.geo);
            // staged row / column; -1 = the unit's checksum row / column (checksum-lane faults)
            si = f.li < 0 ? gf.cra : f.li + gf.oa;
            sj = f.lj < 0 ? gf.crb : f.lj + gf.ob;
            dv = f.delta;
          }
          __syncwarp();
          if (lane == 0) {
            st_sv(ws, W_FNEXT, fnext + 1);
            st_sv(ws, W_NEXT_STAGE, fnext + 1 < x.f_hi ? P.faults[fnext + 1].stage - ld_sv(ws, W_SOFF) : 0x7fffffff);
          }
          __syncwarp();
        } else {
          break;
        }
        // Register index of the owning accumulator, -1 for every other thread.  Select-based
        // (no dynamic register indexing) so the accumulators stay in registers.
        const int fidx = si >= 0 ? acc_owner_index<AKM, BKM>(si, sj, wm, wn, lane) : -1;
#pragma unroll
        for (int a = 0; a < 8; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const double v = acc[a][b][e];
              acc[a][b][e] = ((a * 4 + b) * 2 + e == fidx) ? v + dv : v;
            }
      }
      if (s >= ld_sv(ws, W_NK)) break;
    }
    __syncwarp();
    if (lane == 0) st_sv(ws, W_BASE, ld_sv(ws, W_BASE) + ld_sv(ws, W_NK));  // the next attempt's first stage
    __syncwarp();
    int failed = ld_sv(ws, W_FAILED);  // the same in every MMA warp (a CTA-wide decision)
    bool owner = true;  // this CTA verifies and stores the tile (k-split: the tile's last split)
    if (P.ksplit > 1 && attempt == 0) {
      // k-split: publish this split's partial C^f block and stage maxima; the tile's last split
      // to finish (ticket) sums all partials in split order and carries on with the whole
      // block, the others are done.
      // (split and tile slot recomputed from blockIdx: nothing extra held across the k-loop)
      const int S = P.ksplit, q = (int)blockIdx.x % S, slot = (int)blockIdx.x / S;
      double *pp = P.part + (size_t)(slot * S + q) * (BM * BN);
#pragma unroll
      for (int a = 0; a < 8; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b)
#pragma unroll
          for (int e = 0; e < 2; ++e) pp[((a * 4 + b) * 2 + e) * 256 + vt] = acc[a][b][e];
      if (FT && vt == 0) {
        P.part_max[2 * (slot * S + q)] = tl.int_am[0];
        P.part_max[2 * (slot * S + q) + 1] = tl.int_bm[0];
      }
      __threadfence();
      bar_sync(BAR_CTILE, 256);
      if (P.kcoop) {
        // Co-resident splits (cooperative launch): split q sums its slice of the accumulator
        // registers over the S partials in split order into partial 0 (the same sum per
        // element as one CTA summing them all), then split S-1 carries on with the whole block.
        // (One CTA reading all S blocks was 12 of C1's 27 us.)
        const double *p0 = P.part + (size_t)slot * S * (BM * BN) + vt;
        ksplit_coop_reduce(P, tl, p0, slot, q, S, vt);
        owner = tl.ticket == S - 1;
        if (owner) {
          __threadfence();
#pragma unroll
          for (int a = 0; a < 8; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b)
#pragma unroll
              for (int e = 0; e < 2; ++e) acc[a][b][e] = __ldcg(p0 + ((a * 4 + b) * 2 + e) * 256);
        }
      } else {
        if (vt == 0) tl.ticket = atomicAdd(&P.tickets[slot], 1);
        bar_sync(BAR_CTILE, 256);
        owner = tl.ticket == S - 1;
        if (owner) {
          __threadfence();
          // (every split's partial from memory, this one's included: the same sum in the same
          // order whichever split arrives last)
          const double *p0 = P.part + (size_t)slot * S * (BM * BN) + vt;
#pragma unroll
          for (int a = 0; a < 8; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b)
#pragma unroll
              for (int e = 0; e < 2; ++e) acc[a][b][e] = __ldcg(p0 + ((a * 4 + b) * 2 + e) * 256);
          for (int r = 1; r < S; ++r) {
            const double *pr = p0 + (size_t)r * (BM * BN);
#pragma unroll
            for (int a = 0; a < 8; ++a)
#pragma unroll
              for (int b = 0; b < 4; ++b)
#pragma unroll
                for (int e = 0; e < 2; ++e) acc[a][b][e] += __ldcg(pr + ((a * 4 + b) * 2 + e) * 256);
          }
        }
      }
      if (owner) {
        // The tile's faults after its last update (stage nk): on the summed block, as the unsplit
        // kernel adds them after its last stage.
        if (P.nfaults > 0) {
          const TileGeom gf = load_geom(tl.geo);
          const int tile = gf.ti + gf.tj * P.tiles_m, nk_all = (int)((P.k + BK - 1) / BK);
          int lo = 0, hi = P.nfaults;
          while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            const FaultDev &f = P.faults[mid];
            if (f.tile < tile || (f.tile == tile && f.stage < nk_all)) lo = mid + 1; else hi = mid;
          }
          for (int fi = lo; fi < P.nfaults && P.faults[fi].tile == tile; ++fi) {
            const FaultDev f = P.faults[fi];
            const int si = f.li < 0 ? gf.cra : f.li + gf.oa, sj = f.lj < 0 ? gf.crb : f.lj + gf.ob;
            const int fidx = acc_owner_index<AKM, BKM>(si, sj, wm, wn, lane);
#pragma unroll
            for (int a = 0; a < 8; ++a)
#pragma unroll
              for (int b = 0; b < 4; ++b)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                  const double v = acc[a][b][e];
                  acc[a][b][e] = ((a * 4 + b) * 2 + e == fidx) ? v + f.delta : v;
                }
          }
        }
        if (FT && vt == 0) {  // the maxima over all of k (R1')
          uint32_t am = 0u, bm = 0u;
          for (int r = 0; r < S; ++r) {
            am = max(am, __ldcg(P.part_max + 2 * (slot * S + r)));
            bm = max(bm, __ldcg(P.part_max + 2 * (slot * S + r) + 1));
          }
          tl.int_am[0] = am;
          tl.int_bm[0] = bm;
        }
        bar_sync(BAR_CTILE, 256);
      }
    }
#ifdef FTBLAS_DEV_TIMELINE
    if (P.dev_prof && vt == 0 && attempt == 0) FT_TL(2) = (unsigned long long)clock64() - FT_TL(3);
#endif
    if (owner && verify && failed < 0 && !x.enc_only && !(FT_DEV_MODE(P) & 1024)) {  // dev 1024: skip the last check (timing)
      // The last interval, verified before C is written, from the registers
      // (its first barrier is also the point where every MMA warp has drained its DMMA stream).
      const CheckOut co = check_unit<AKM, BKM, 2>(P, tl, acc, P.T - 1, P.k, mw, wm, wn, lane);
      if (co.multi) {
        failed = P.T - 1;
      } else if (co.si >= 0) {
        if (P.correct_mode == 1) {  // subtract d_col at the located cell
          const int fidx = acc_owner_index<AKM, BKM>(co.si, co.sj, wm, wn, lane);
#pragma unroll
          for (int a = 0; a < 8; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b)
#pragma unroll
              for (int e = 0; e < 2; ++e) {
                const double v = acc[a][b][e];
                acc[a][b][e] = ((a * 4 + b) * 2 + e == fidx) ? v - co.dcol : v;
              }
        } else if (vt == 0) {
          add_fix(tl, co.si, co.sj);  // R4: fresh dot product in the epilogue
        }
      }
    }
#ifdef FTBLAS_DEV_TIMELINE
    if (P.dev_prof && vt == 0 && attempt == 0) FT_TL(-4) = (unsigned long long)clock64() - FT_TL(3);
#endif
    // Stage the accumulators into the ring as the C tile: every MMA warp has consumed its last
    // stage (and every TMA write and checksum row has landed before that stage was consumed).
    bar_sync(BAR_CTILE, 256);
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
    if (failed >= 0) fence_proxy_async();  // generic writes to the ring before TMA refills it
    bar_sync(BAR_RING_FREE, NTHREADS);  // every stage consumed: the ring is free for the C tile
#ifdef FTBLAS_DEV_TIMELINE
    if (P.dev_prof && vt == 0 && attempt == 0) FT_TL(-3) = (unsigned long long)clock64() - FT_TL(3);
#endif
    if (!verify) break;
    if (vt == 0) {
      tl.retry = failed;
      if (failed >= 0) tl.nfix = 0;  // the recompute re-forms every element
      tl.cum_am = tl.amax_hi;  // the next attempt's maxima: from scratch (PREPASS preset)
      tl.cum_bm = tl.bmax_hi;
#pragma unroll
      for (int q = 0; q < 8; ++q) tl.int_am[q] = tl.int_bm[q] = 0u;
    }
    bar_sync(BAR_DECIDE, NTHREADS);  // encoders learn whether (and from where) to run again
    if (failed < 0) break;  // else out of the one-error model: recompute the unit (R6)
  }
  if (FT && x.enc_only) return;  // an encoder CTA stores nothing
  // k-split: another split of this tile verifies and stores it (a recompute only ever runs in
  // the owner, so the ticket of its first attempt decides)
  if (P.ksplit > 1 && tl.ticket != P.ksplit - 1) return;

  // ---- epilogue: corrected cells (recompute mode), then C = alpha*acc + beta*C0 (two
  // roundings each, no contraction) from the staged tile, coalesced column stores.
  bar_sync(BAR_CTILE, 256);
#ifdef FTBLAS_DEV_TIMELINE
  if (P.dev_prof && vt == 0) FT_TL(-2) = (unsigned long long)clock64() - FT_TL(3);
#endif
  const TileGeom ge = load_geom(tl.geo);
  if (FT) {
    // Recompute mode (R4): each corrected element becomes a fresh dot product over all k.
    const int nfix = tl.nfix;
    for (int q = 0; q < nfix; ++q) {
      const int si = tl.fix[q] & 255, sj = tl.fix[q] >> 8;
      const int64_t gi = ge.i0 + si - ge.oa, gj = ge.j0 + sj - ge.ob;
      FT_CHECK(nfix <= MAX_FIX && gi >= ge.i0 && gi < ge.i0 + ge.bm_eff && gj >= ge.j0 && gj < ge.j0 + ge.bn_eff);
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
        for (int w = 0; w < N_MMA_WARPS; ++w) v += tl.red[w];
        ctile[sj * LDC_S + si] = v;
      }
      bar_sync(BAR_CTILE, 256);
    }
  }
  const int i = vt & 127;
  const double alpha = P.alpha, beta = P.beta;
  if (i < ge.bm_eff) {
    FT_CHECK(ge.i0 + i < P.m && ge.j0 + ge.bn_eff <= P.n && i + ge.oa < 128 && ge.bn_eff + ge.ob <= 128);
    double *crow = P.C + (int64_t)(ge.i0 + i) + (int64_t)ge.j0 * P.ldc;
    if (beta != 0.0) {
      // C0 loaded EPI_B columns at a time ahead of their stores: in a load-then-store loop the
      // compiler cannot hoist a load above the previous (possibly aliasing) store, so every
      // column paid a full memory round trip (~30 us per 2048^3 tile wave).
      constexpr int EPI_B = 8;
      for (int j0 = vt >> 7; j0 < ge.bn_eff; j0 += 2 * EPI_B) {
        double c0[EPI_B];
#pragma unroll
        for (int u = 0; u < EPI_B; ++u) {
          const int j = j0 + 2 * u;
          c0[u] = j < ge.bn_eff ? crow[(int64_t)j * P.ldc] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < EPI_B; ++u) {
          const int j = j0 + 2 * u;
          if (j < ge.bn_eff)
            crow[(int64_t)j * P.ldc] =
                __dadd_rn(__dmul_rn(alpha, ctile[(j + ge.ob) * LDC_S + i + ge.oa]), __dmul_rn(beta, c0[u]));
        }
      }
    } else {
#pragma unroll 4
      for (int j = vt >> 7; j < ge.bn_eff; j += 2)
        crow[(int64_t)j * P.ldc] = __dmul_rn(alpha, ctile[(j + ge.ob) * LDC_S + i + ge.oa]);
    }
  }
#ifdef FTBLAS_DEV_TIMELINE
  if (P.dev_prof && vt == 0) FT_TL(3) = (unsigned long long)clock64() - FT_TL(3);
#undef FT_TL
#endif
}

// The launch's report, written by its last CTA into mapped pinned host memory: every CTA,
// after all its threads' C stores, counter atomics and events (barrier + fences), counts itself
// done; the last one copies the counters and the first rep_events events, then (after a
// system-scope fence) the call's sequence number to word 0, which the host polls instead of a
// device-to-host copy and a stream synchronisation.  Layout: [seq | counters[CNT_N] |
// events as EventDev].
// (Called by each role after its last global write, and by ghost CTAs: the roles run with
// different register budgets and must not re-converge, so each meets the others at barrier
// BAR_REPORT from its own code path; thread 0 -- an MMA thread -- does the counting.)
__device__ __forceinline__ void publish_report(const Params &P) {
  __threadfence();
  bar_sync(BAR_REPORT, NTHREADS);
  if (threadIdx.x != 0) return;
  const unsigned long long done = atomicAdd(&P.counters[CNT_DONE], 1ull);
  if (done != (unsigned long long)gridDim.x - 1) return;
  __threadfence();
  volatile unsigned long long *h = P.host_rep;
  unsigned long long cnt[CNT_N];
#pragma unroll
  for (int i = 0; i < CNT_N; ++i) cnt[i] = __ldcg(&P.counters[i]);
#pragma unroll
  for (int i = 0; i < CNT_N; ++i) h[1 + i] = cnt[i];
  const long long nev = min((long long)cnt[CNT_EVENTS], min((long long)P.rep_events, P.ev_cap));
  const unsigned long long *ev = reinterpret_cast<const unsigned long long *>(P.events);
  constexpr int W = sizeof(EventDev) / 8;
  for (long long q = 0; q < nev * W; ++q) h[1 + CNT_N + q] = __ldcg(ev + q);
  __threadfence_system();
  h[0] = P.rep_seq;
  __threadfence_system();
}

template <bool AKM, bool BKM, bool FT>
__global__ void __launch_bounds__(NTHREADS, 1)
    dgemm_abft_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                      const __grid_constant__ Params P) {
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
  // Grouped raster: CTAs run in bands of RASTER_G tile rows, column by column inside a band,
  // so that one wave of 148 CTAs touches ~12 A row panels and ~12 B column panels (L2 reuse)
  // instead of 148 A panels and one B panel.
  // With checksums shared through L2 (R22) the publishing tiles come first: tile row 0 (B_J e)
  // and tile column 0 (e^T A_I) in the first waves, so nearly every other tile finds both
  // checksums published when it runs.  A partial last tile row / column (cheap: its idle warps
  // skip the DMMA stream) goes last, so the final waves are made of short tiles.
  const int tstr_m = (FT || (FT_DEV_MODE(P) & 32)) ? TM : BM, tstr_n = (FT || (FT_DEV_MODE(P) & 32)) ? TN : BN;
  const bool prow = P.tiles_m > 1 && (P.m % tstr_m) != 0, pcol = P.tiles_n > 1 && (P.n % tstr_n) != 0;
  auto map_tile = [&](int Lg, int &ti_, int &tj_) {
    int L = Lg;
    int r0 = 0, c0 = 0;
    if (FT && P.Ash && P.Bsh) {
      if (L < P.tiles_n) { ti_ = 0; tj_ = L; return; }
      L -= P.tiles_n;
      if (L < P.tiles_m - 1) { ti_ = 1 + L; tj_ = 0; return; }
      L -= P.tiles_m - 1;
      r0 = c0 = 1;
    }
    const int rend = P.tiles_m - (prow ? 1 : 0), cend = P.tiles_n - (pcol ? 1 : 0);
    const int tm = rend - r0, tn = cend - c0;  // interior, in grouped raster
    if (tm > 0 && tn > 0 && L < tm * tn) {
      const int band_tiles = RASTER_G * tn, band = L / band_tiles;
      const int within = L - band * band_tiles, rows = min(RASTER_G, tm - band * RASTER_G);
      ti_ = r0 + band * RASTER_G + within % rows;
      tj_ = c0 + within / rows;
      return;
    }
    L -= max(tm, 0) * max(tn, 0);
    if (prow) {
      if (L < cend - c0) { ti_ = P.tiles_m - 1; tj_ = c0 + L; return; }
      L -= cend - c0;
    }
    ti_ = r0 + L;  // partial last tile column, its rows top to bottom
    tj_ = P.tiles_n - 1;
  };
  const int E = FT ? P.enc_head : 0;
  const int enc_b = (int)blockIdx.x;  // encoder CTAs first
  x.enc_only = enc_b < E ? ((P.Ash && enc_b < P.tiles_m) ? 1 : 2) : 0;
  const int bid = (int)blockIdx.x - E;
  const int Lg = x.enc_only ? 0 : bid / P.ksplit;  // tile in launch order (k-split: P.ksplit CTAs each)
  const bool ghost = P.cluster2 && Lg >= P.total;  // pads an odd grid to whole clusters
  int ti, tj;
  if (x.enc_only == 1) {
    ti = enc_b;
    tj = 0;
  } else if (x.enc_only == 2) {
    ti = 0;
    tj = enc_b - (P.Ash ? P.tiles_m : 0);
  } else {
    map_tile(ghost ? Lg - 1 : Lg, ti, tj);
  }
  // Cluster pair (2c, 2c+1): share the B_J encode when both are real tiles of the same tile
  // column and interval (a band with an odd row count pairs across columns: no sharing).
  bool share = false;
  if (FT && P.cluster2 && !P.Ac && !ghost && (Lg ^ 1) < P.total) {
    int pti, ptj;
    map_tile(Lg ^ 1, pti, ptj);
    share = ptj == tj;
  }
  x.tile = x.enc_only ? -1 : ti + tj * P.tiles_m;  // fault bucket key (encoder CTAs: none)
  x.tile_slot = Lg;
  x.nk_all = (int)((P.k + BK - 1) / BK);
  x.q = x.enc_only ? 0 : bid % P.ksplit;
  x.s0 = (int)((int64_t)x.q * x.nk_all / P.ksplit);
  const int s1 = (int)((int64_t)(x.q + 1) * x.nk_all / P.ksplit);
  x.k0 = (int64_t)x.s0 * BK;
  x.k1 = min64((int64_t)s1 * BK, P.k);
  // Protected tiles advance by the 127 data rows/cols of C^f; the unprotected twin uses the
  // full 128 x 128 MMA tile for data.
  const bool g127 = FT || (FT_DEV_MODE(P) & 32);  // dev mode 32: unprotected kernel on the 127 grid
  const int tm = g127 ? TM : BM, tn = g127 ? TN : BN;
  x.ti = ti;
  x.tj = tj;
  x.i0 = ti * tm;
  x.j0 = tj * tn;
  x.bm_eff = (int)min64(tm, P.m - x.i0);
  x.bn_eff = (int)min64(tn, P.n - x.j0);
  x.oa = g127 ? (x.i0 & 1) : 0;
  x.ob = g127 ? (x.j0 & 1) : 0;
  // Checksum row / column: 0 for odd tiles (data in staged rows 1..127), else 127; a partial
  // even tile at the matrix edge takes the first row / column past its data instead (staged as
  // TMA's out-of-bounds zeros), so its used rows / columns stay contiguous from 0 and the MMA
  // warps whose 64 x 32 quarter holds none of them skip the DMMA stream (mma_role).
  x.cra = x.oa ? 0 : (g127 && x.bm_eff < DM ? x.bm_eff : DM);
  x.crb = x.ob ? 0 : (g127 && x.bn_eff < DM ? x.bn_eff : DM);
  x.nk = (int)((x.k1 - x.k0 + BK - 1) / BK);

  if (x.tid == 0) {
    tl.geo = TileGeom{x.ti, x.tj, x.i0, x.j0, x.bm_eff, x.bn_eff, x.oa, x.ob, x.cra, x.crb, x.k0, x.k1};
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB);
#pragma unroll
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&tl.full[s], 1);
      mbar_init(&tl.enc[s], 2);  // the A and the B encode job
      mbar_init(&tl.empty[s], N_MMA_WARPS);
    }
    tl.amax_hi = P.Ac ? P.amax_pre[ti] : 0u;
    tl.bmax_hi = P.Ac ? P.bmax_pre[tj] : 0u;
    tl.first_row[0] = tl.first_row[1] = 0x7fffffff;
    tl.first_col[0] = tl.first_col[1] = 0x7fffffff;
#pragma unroll
    for (int q = 0; q < 8; ++q) tl.int_am[q] = tl.int_bm[q] = 0u;
    tl.cum_am = tl.amax_hi;
    tl.cum_bm = tl.bmax_hi;
    tl.nfix = 0;
    tl.retry = -1;
    tl.share = share ? 1 : 0;
#pragma unroll
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&tl.mfull[s], 1);
      mbar_init(&tl.mfree[s], 1);
    }
    fence_mbar_init();
  }
  // Faults of this tile: [f_lo, f_hi) in the (tile, stage)-sorted list.
  // (k-split: those with stage in [s0, s1); the last split also takes the faults at stage nk,
  // i.e. after the last update)
  x.f_lo = x.f_hi = 0;
  if (P.nfaults > 0) {
    auto before = [&](const FaultDev &f, int st) { return f.tile < x.tile || (f.tile == x.tile && f.stage < st); };
    int lo = 0, hi = P.nfaults;
    while (lo < hi) { const int mid = (lo + hi) >> 1; if (before(P.faults[mid], x.s0)) lo = mid + 1; else hi = mid; }
    x.f_lo = lo;
    // (the faults after the last update, stage nk, go to the tile's owner in a k-split launch)
    const int s_end = P.ksplit == 1 ? 0x7fffffff : s1;
    hi = P.nfaults;
    while (lo < hi) { const int mid = (lo + hi) >> 1; if (before(P.faults[mid], s_end)) lo = mid + 1; else hi = mid; }
    x.f_hi = lo;
  }
  __syncthreads();
  if (P.cluster2) cluster_sync_all();  // partners' mailbox barriers are initialised
  if (ghost) {
    if (FT && P.host_rep) publish_report(P);
    return;
  }

  // The two roles never re-converge, so ptxas can give each its own register budget.
  if (is_cs_warp(x.warp)) {
    // K-major A with MN-major B (TT) needs 8 more registers in the protected DMMA loop.
    if (FT && AKM && !BKM) setmaxnreg_dec<REG_CS - 16>(); else setmaxnreg_dec<REG_CS>();
    checksum_role<AKM, BKM, FT>(tmA, tmB, P, x);
    if (FT && P.host_rep) publish_report(P);
  } else {
    if (FT && AKM && !BKM) setmaxnreg_inc<REG_MMA + 8>(); else setmaxnreg_inc<REG_MMA>();
    mma_role<AKM, BKM, FT>(P, x);
    if (FT && P.host_rep) publish_report(P);
  }
  // A sharing pair stays resident until the partner has made its last remote access.
  if (share) cluster_sync_all();
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
