// ftblas.cu — host side of libftblas.so: the C ABI declared in include/ftblas.h.
//
// Argument checking (BLAS INFO convention), quick returns, fault bucketing, kernel
// dispatch over (transA, transB, FT, 16-byte vector path), the error-report path and the
// seeded fault generator.  All arithmetic of the method runs in the kernels of
// dgemm_abft.cuh; this file only marshals.
#include "../../include/ftblas.h"
#include "dgemm_abft.cuh"
#include "unfused.cuh"
#include "dmr.cuh"
#include "trsm.cuh"

#include <cudaTypedefs.h>

#include <algorithm>
#include <type_traits>
#include <atomic>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>
#include <map>
#include <functional>

namespace {

thread_local cudaStream_t tl_stream = nullptr;
thread_local std::vector<ftblas_fault_t> tl_armed;
thread_local bool tl_have_armed = false;
// Checksum-lane faults (ftblas_inject_arm_checksum): lane 1 = column checksum, 2 = row checksum.
struct CsFault {
  ftblas_fault_t f;
  int32_t lane;
};
thread_local std::vector<CsFault> tl_armed_cs;
thread_local int tl_correct = FTBLAS_CORRECT_RECOMPUTE;
thread_local int tl_encode = FTBLAS_ENCODE_FUSED;
thread_local int64_t tl_interval = 0;  // Kc; 0 = k (one interval)
thread_local int64_t tl_launches = 0;
thread_local std::string tl_cuda_error;

std::mutex g_init_mu;
bool g_init_done[64] = {false};

int cuda_fail(cudaError_t e) {
  tl_cuda_error = cudaGetErrorString(e);
  return e == cudaErrorMemoryAllocation ? 2 : 1;
}
#define CUDA_TRY(x)                          \
  do {                                       \
    cudaError_t e_ = (x);                    \
    if (e_ != cudaSuccess) return cuda_fail(e_); \
  } while (0)

// Releases what one call acquired on every return path: the stream-ordered allocations (freed
// on the call's stream once the library streams listed in `streams` are drained), events and
// streams.
struct Cleanup {
  cudaStream_t st;
  std::vector<void *> mem;
  std::vector<cudaStream_t> streams;
  std::vector<cudaEvent_t> events;
  explicit Cleanup(cudaStream_t s) : st(s) {}
  Cleanup(const Cleanup &) = delete;
  Cleanup &operator=(const Cleanup &) = delete;
  ~Cleanup() {
    for (cudaStream_t s : streams) cudaStreamSynchronize(s);
    for (void *p : mem) cudaFreeAsync(p, st);
    for (cudaEvent_t e : events) cudaEventDestroy(e);
    for (cudaStream_t s : streams) cudaStreamDestroy(s);
  }
  template <class T>
  cudaError_t alloc(T **p, size_t bytes) {
    const cudaError_t e = cudaMallocAsync(reinterpret_cast<void **>(p), bytes, st);
    if (e == cudaSuccess) mem.push_back(*p);
    else *p = nullptr;
    return e;
  }
  cudaError_t stream(cudaStream_t *s) {
    const cudaError_t e = cudaStreamCreateWithFlags(s, cudaStreamNonBlocking);
    if (e == cudaSuccess) streams.push_back(*s);
    return e;
  }
  cudaError_t event(cudaEvent_t *ev) {
    const cudaError_t e = cudaEventCreateWithFlags(ev, cudaEventDisableTiming);
    if (e == cudaSuccess) events.push_back(*ev);
    return e;
  }
};

bool is_n(char c) { return c == 'N' || c == 'n'; }
bool is_t(char c) { return c == 'T' || c == 't' || c == 'C' || c == 'c'; }

template <bool AKM, bool BKM, bool FT>
int launch_one(const CUtensorMap &ta, const CUtensorMap &tb, const ftk::Params &p0, dim3 grid, cudaStream_t st) {
  auto kfn = ftk::dgemm_abft_kernel<AKM, BKM, FT>;
  static std::atomic<bool> attr_set[64];  // per instantiation and device (idempotent if raced)
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64 || !attr_set[dev].load(std::memory_order_acquire)) {
    CUDA_TRY(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ftk::SMEM_BYTES));
    if (dev >= 0 && dev < 64) attr_set[dev].store(true, std::memory_order_release);
  }
  ftk::Params p = p0;
  p.total = (int)grid.x;
  // Encode mode FUSED_LOCAL (p.cluster2 requested by the caller): 2-CTA clusters share the B_J
  // encode (cluster size 2 packs all 148 SMs).  With the checksums shared through L2 (FUSED,
  // R22) nearly every tile copies B_J e, and pair co-scheduling costs more than the split saves
  // (C5-like 4.0% -> 3.9%, C4a 9.2% -> 7.8%); a single-wave FUSED launch, which skips the
  // sharing, is also faster plain (1016^2 x 256: first-stage wait 10.2k vs 11.6k clocks), so
  // FUSED launches are plain.
  if (FT && p.cluster2 && !p.Ac && !p.Ash && !p.Bsh && !(FT_DEV_MODE(p) & 128)) {
    p.cluster2 = 1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((grid.x + 1) & ~1u);
    cfg.blockDim = dim3(ftk::NTHREADS);
    cfg.dynamicSmemBytes = ftk::SMEM_BYTES;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    CUDA_TRY(cudaLaunchKernelEx(&cfg, kfn, ta, tb, p));
    ++tl_launches;
    return 0;
  }
  p.cluster2 = 0;
  if (p.kcoop) {
    // k-split of a single-wave launch: a cooperative launch makes the splits of a tile
    // co-resident, so they can reduce their partial blocks together (dgemm_abft.cuh); if the
    // driver refuses it, the ticket reduction (the last split sums alone) needs no co-residency.
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(ftk::NTHREADS);
    cfg.dynamicSmemBytes = ftk::SMEM_BYTES;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, kfn, ta, tb, p) == cudaSuccess) {
      ++tl_launches;
      return 0;
    }
    (void)cudaGetLastError();
    p.kcoop = 0;
  }
  kfn<<<grid, ftk::NTHREADS, ftk::SMEM_BYTES, st>>>(ta, tb, p);
  ++tl_launches;
  CUDA_TRY(cudaGetLastError());
  return 0;
}

template <bool FT>
int dispatch(bool akm, bool bkm, const CUtensorMap &ta, const CUtensorMap &tb, const ftk::Params &p, dim3 grid,
             cudaStream_t st) {
  if (akm) return bkm ? launch_one<true, true, FT>(ta, tb, p, grid, st) : launch_one<true, false, FT>(ta, tb, p, grid, st);
  return bkm ? launch_one<false, true, FT>(ta, tb, p, grid, st) : launch_one<false, false, FT>(ta, tb, p, grid, st);
}

// TMA descriptor of one operand.  K-major (k contiguous): dims {k, x}, box {16, 128};
// MN-major (x contiguous): dims {x, k}, box {16, 16}.  128-byte swizzle, zero OOB fill.
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
int make_tmap(CUtensorMap *map, const double *base, int64_t ld, bool kmajor, int64_t xdim, int64_t kdim) {
  if (!g_encode) {
    cudaDriverEntryPointQueryResult q;
    void *fn = nullptr;
    CUDA_TRY(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !fn) { tl_cuda_error = "cuTensorMapEncodeTiled unavailable"; return 1; }
    g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  cuuint64_t dims[2], strides[1] = {(cuuint64_t)ld * sizeof(double)};
  cuuint32_t box[2], estr[2] = {1, 1};
  if (kmajor) { dims[0] = kdim; dims[1] = xdim; box[0] = 16; box[1] = 128; }
  else        { dims[0] = xdim; dims[1] = kdim; box[0] = 16; box[1] = 16; }
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double *>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { tl_cuda_error = "cuTensorMapEncodeTiled failed"; return 1; }
  return 0;
}

int ensure_device_init() {
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_init_mu);
  if (dev >= 0 && dev < 64 && !g_init_done[dev]) {
    // Keep stream-ordered scratch cached in the device's default pool, up to a quarter of the
    // device memory (the C5 host-buffer pipeline's panels fit; larger transient scratch is
    // returned at the next synchronisation instead of staying reserved until ftblas_finalize).
    cudaMemPool_t pool;
    CUDA_TRY(cudaDeviceGetDefaultMemPool(&pool, dev));
    size_t free_b = 0, total_b = 0;
    CUDA_TRY(cudaMemGetInfo(&free_b, &total_b));
    uint64_t thr = (uint64_t)total_b / 4;
    CUDA_TRY(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
    g_init_done[dev] = true;
  }
  return 0;
}

int check_args(char ta, char tb, int64_t m, int64_t n, int64_t k, double alpha, const double *A,
               int64_t lda, const double *B, int64_t ldb, const double *C, int64_t ldc) {
  if (!is_n(ta) && !is_t(ta)) return -1;
  if (!is_n(tb) && !is_t(tb)) return -2;
  if (m < 0) return -3;
  if (n < 0) return -4;
  if (k < 0) return -5;
  const int64_t nrowa = is_n(ta) ? m : k, nrowb = is_n(tb) ? k : n;
  const bool reads_ab = alpha != 0.0 && k > 0 && m > 0 && n > 0;
  if (reads_ab && A == nullptr) return -7;
  if (lda < std::max<int64_t>(1, nrowa)) return -8;
  if (reads_ab && B == nullptr) return -9;
  if (ldb < std::max<int64_t>(1, nrowb)) return -10;
  if (m > 0 && n > 0 && C == nullptr) return -12;
  if (ldc < std::max<int64_t>(1, m)) return -13;
  // Index arithmetic inside the kernels uses int for tile coordinates.
  if ((m + ftk::TM - 1) / ftk::TM > 0x7fffffff) return -3;
  if (((m + ftk::TM - 1) / ftk::TM) * ((n + ftk::TN - 1) / ftk::TN) > 0x7fffffff) return -4;
  return 0;
}

void fill_geometry(ftblas_err_report_t *err, int64_t k) {
  err->unit_rows = ftk::TM;
  err->unit_cols = ftk::TN;
  err->unit_k = (int32_t)std::min<int64_t>(k, INT32_MAX);
  err->step_quantum = ftk::BK;
}

void zero_report(ftblas_err_report_t *err, int64_t k) {
  if (!err) return;
  err->units_checked = err->detected = err->corrected = err->recomputed = err->n_events = 0;
  fill_geometry(err, k);
}

std::vector<CsFault> take_armed_cs() {
  std::vector<CsFault> cs;
  cs.swap(tl_armed_cs);
  return cs;
}
// Entry points other than ftblas_dgemm: armed checksum-lane faults are a bad fault list.
bool reject_armed_cs() { return !take_armed_cs().empty(); }

std::vector<ftblas_fault_t> take_armed() {
  std::vector<ftblas_fault_t> faults;
  if (tl_have_armed) { faults.swap(tl_armed); tl_have_armed = false; }
  return faults;
}

int num_sms();

// Per-thread pinned host buffer for the report read-back (grown on demand, never shrunk).
cudaError_t pinned_report_buffer(size_t bytes, char **out) {
  static thread_local char *buf = nullptr;
  static thread_local size_t cap = 0;
  if (bytes > cap) {
    if (buf) cudaFreeHost(buf);
    buf = nullptr;
    cap = 0;
    const size_t want = std::max<size_t>(bytes, 4096);
    const cudaError_t e = cudaHostAlloc((void **)&buf, want, cudaHostAllocPortable);
    if (e != cudaSuccess) { buf = nullptr; return e; }
    cap = want;
  }
  *out = buf;
  return cudaSuccess;
}

// Per-thread pinned staging for the armed-fault list's host->device copy.  The buffer is reused
// once the event recorded after its last copy has completed (normally long before: the copy is
// the first thing on the stream in the previous call).
struct FaultStage {
  char *buf = nullptr;
  size_t cap = 0;
  cudaEvent_t done = nullptr;
  int dev = -1;
  bool pending = false;
};
thread_local FaultStage tl_fstage;
cudaError_t pinned_fault_stage(size_t bytes, char **out) {
  FaultStage &f = tl_fstage;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (f.pending) {
    if ((e = cudaEventSynchronize(f.done)) != cudaSuccess) return e;
    f.pending = false;
  }
  if (f.done && f.dev != dev) {  // events belong to one device
    cudaEventDestroy(f.done);
    f.done = nullptr;
  }
  if (!f.done) {
    if ((e = cudaEventCreateWithFlags(&f.done, cudaEventDisableTiming)) != cudaSuccess) return e;
    f.dev = dev;
  }
  if (bytes > f.cap) {
    if (f.buf) cudaFreeHost(f.buf);
    f.buf = nullptr;
    f.cap = 0;
    const size_t want = std::max<size_t>(bytes, 4096);
    if ((e = cudaHostAlloc((void **)&f.buf, want, cudaHostAllocPortable)) != cudaSuccess) return e;
    f.cap = want;
  }
  *out = f.buf;
  return cudaSuccess;
}
cudaError_t pinned_fault_release(cudaStream_t st) {
  const cudaError_t e = cudaEventRecord(tl_fstage.done, st);
  tl_fstage.pending = e == cudaSuccess;
  return e;
}

// Sort the events by (interval, i, j) and fill the caller's report.
void fill_report(ftblas_err_report_t *err, const unsigned long long *cnt, std::vector<ftk::EventDev> &ev,
                 int64_t units_checked) {
  const int64_t nev = (int64_t)cnt[ftk::CNT_EVENTS];
  const int64_t nstore = (int64_t)ev.size();
  std::sort(ev.begin(), ev.end(), [](const ftk::EventDev &a, const ftk::EventDev &b) {
    if (a.interval != b.interval) return a.interval < b.interval;
    if (a.i != b.i) return a.i < b.i;
    return a.j < b.j;
  });
  err->units_checked = units_checked;
  err->detected = (int64_t)cnt[ftk::CNT_DETECTED];
  err->corrected = (int64_t)cnt[ftk::CNT_CORRECTED];
  err->recomputed = (int64_t)cnt[ftk::CNT_RECOMPUTED];
  err->n_events = nev;
  if (err->events && err->events_capacity > 0) {
    const int64_t ncopy = std::min<int64_t>(nstore, err->events_capacity);
    for (int64_t e = 0; e < ncopy; ++e) {
      err->events[e].i = ev[e].i;
      err->events[e].j = ev[e].j;
      err->events[e].kind = ev[e].kind;
      err->events[e].interval = ev[e].interval;
      err->events[e].residual_row = ev[e].residual_row;
      err->events[e].residual_col = ev[e].residual_col;
    }
  }
}

// Copy the device counters / events of one call into the caller's report (events sorted by
// (interval, i, j)).  Synchronises the stream.
int finish_report(ftblas_err_report_t *err, const unsigned long long *d_counters, const void *d_events,
                  int64_t ev_cap, int64_t units_checked, cudaStream_t st) {
  // One device->host copy for the counters and (when they follow the counters closely) the
  // first E0 events; a second one only when more events were recorded.
  constexpr int64_t E0 = 32;
  const ptrdiff_t gap = reinterpret_cast<const char *>(d_events) - reinterpret_cast<const char *>(d_counters);
  const bool joint = gap >= (ptrdiff_t)(sizeof(unsigned long long) * ftk::CNT_N) && gap <= 256;
  const int64_t e0 = joint ? std::min<int64_t>(E0, ev_cap) : 0;
  const size_t head_bytes = (size_t)(joint ? gap : 0) + sizeof(ftk::EventDev) * (size_t)e0 + sizeof(unsigned long long) * ftk::CNT_N;
  // Pinned staging (per thread, grown on demand; safe to reuse because this function
  // synchronises before returning): a pageable copy costs a driver staging pass per call.
  char *head = nullptr;
  CUDA_TRY(pinned_report_buffer(head_bytes, &head));
  CUDA_TRY(cudaMemcpyAsync(head, d_counters, joint ? (size_t)gap + sizeof(ftk::EventDev) * (size_t)e0
                                                   : sizeof(unsigned long long) * ftk::CNT_N,
                           cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  unsigned long long cnt[ftk::CNT_N];
  std::memcpy(cnt, head, sizeof cnt);
  const int64_t nev = (int64_t)cnt[ftk::CNT_EVENTS];
  const int64_t nstore = std::min<int64_t>(nev, ev_cap);
  std::vector<ftk::EventDev> ev((size_t)nstore);
  const int64_t have = std::min<int64_t>(nstore, e0);
  if (have > 0) std::memcpy(ev.data(), head + gap, sizeof(ftk::EventDev) * (size_t)have);
  if (nstore > have) {
    CUDA_TRY(cudaMemcpyAsync(ev.data() + have, reinterpret_cast<const ftk::EventDev *>(d_events) + have,
                             sizeof(ftk::EventDev) * (size_t)(nstore - have), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
  }
  fill_report(err, cnt, ev, units_checked);
  return 0;
}

// Per-thread mapped pinned buffer of the device-written report (ftk::publish_report).
struct MappedReport {
  unsigned long long *host = nullptr, *dev = nullptr, seq = 0;
  int device = -1;
};
thread_local MappedReport tl_mrep;
cudaError_t mapped_report_buffer(MappedReport **out) {
  MappedReport &r = tl_mrep;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (!r.host) {
    if ((e = cudaHostAlloc((void **)&r.host, 4096, cudaHostAllocMapped | cudaHostAllocPortable)) != cudaSuccess) {
      r.host = nullptr;
      return e;
    }
    std::memset(r.host, 0, 4096);
  }
  if (r.device != dev) {
    if ((e = cudaHostGetDevicePointer((void **)&r.dev, r.host, 0)) != cudaSuccess) return e;
    r.device = dev;
  }
  *out = &r;
  return cudaSuccess;
}

// The report of a launch that writes it itself (ftk::publish_report): poll the sequence word
// of the mapped buffer instead of a device-to-host copy and a stream synchronisation (all C
// stores and counters of the launch precede it); more than REP_EVENTS events are read back.
// If the stream completes without the word (not expected), the report is read back instead.
int finish_report_mapped(ftblas_err_report_t *err, const MappedReport &mr, unsigned long long seq,
                         const unsigned long long *d_counters, const void *d_events, int64_t ev_cap,
                         int64_t units_checked, cudaStream_t st) {
  volatile unsigned long long *h = mr.host;
  for (uint64_t spin = 1; h[0] != seq; ++spin) {
    if ((spin & 255) == 0) {
      const cudaError_t e = cudaStreamQuery(st);
      if (e == cudaSuccess) {
        if (h[0] == seq) break;
        return finish_report(err, d_counters, d_events, ev_cap, units_checked, st);
      }
      if (e != cudaErrorNotReady) return cuda_fail(e);
    }
  }
  std::atomic_thread_fence(std::memory_order_acquire);
  unsigned long long cnt[ftk::CNT_N];
  for (int i = 0; i < ftk::CNT_N; ++i) cnt[i] = h[1 + i];
  const int64_t nev = (int64_t)cnt[ftk::CNT_EVENTS];
  const int64_t nstore = std::min<int64_t>(nev, ev_cap);
  const int64_t have = std::min<int64_t>(nstore, ftk::REP_EVENTS);
  std::vector<ftk::EventDev> ev((size_t)nstore);
  if (have > 0)
    std::memcpy(ev.data(), const_cast<const unsigned long long *>(mr.host) + 1 + ftk::CNT_N, sizeof(ftk::EventDev) * (size_t)have);
  if (nstore > have) {
    CUDA_TRY(cudaMemcpyAsync(ev.data() + have, reinterpret_cast<const ftk::EventDev *>(d_events) + have,
                             sizeof(ftk::EventDev) * (size_t)(nstore - have), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
  }
  fill_report(err, cnt, ev, units_checked);
  return 0;
}

// Block sums over bs-long x-blocks (encode passes, reference sums): unfused.cuh.
int launch_block_sum(const double *X, bool xc, int64_t ld, int64_t nx, int64_t np, double *S, int64_t lds,
                     unsigned *hm, int bs, cudaStream_t st, const int *enable = nullptr) {
  const int64_t nb = (nx + bs - 1) / bs;
  if (nb == 0 || np == 0) return 0;
  if (xc) {
    const dim3 g((unsigned)nb, (unsigned)((np + 31) / 32));
    ftu::block_sum_kernel<true><<<g, 256, 0, st>>>(X, ld, nx, np, S, lds, hm, bs, enable);
  } else {
    const dim3 g((unsigned)nb, (unsigned)((np + 255) / 256));
    ftu::block_sum_kernel<false><<<g, 256, 0, st>>>(X, ld, nx, np, S, lds, hm, bs, enable);
  }
  ++tl_launches;
  CUDA_TRY(cudaGetLastError());
  return 0;
}

// Where a protected call accumulates its report when it is one piece of a larger call (the
// row panels of the host-buffer pipeline): shared device counters / events, zeroed by the
// caller; no synchronisation inside.
struct ReportSink {
  unsigned long long *counters;
  ftk::EventDev *events;
  int64_t ev_cap;
  int64_t row_off;  // global row of this piece's row 0
  int64_t units;    // out: accumulated units checked
  int64_t col_off = 0;  // global column of this piece's column 0
};

// k-split of few-wave launches with a long k (C4b: 516 full tiles + 134 sliver tiles on 148
// SMs is 3.5 waves of full tiles, i.e. 4 rounds): the split that minimises the launch's makespan,
// estimated by list scheduling the CTAs in launch order (full tiles, then the protected kernel's
// sliver tiles, which the raster puts last) on the SMs, in stage units.  A split CTA costs its
// k-range plus the tile's fixed cost (first stage, check, store: ~3 stages) plus the partial
// block's write and, for the tile's last split, the read of the S partials (~0.6 stage each).
// A sliver tile of the protected kernel (at most 15 data rows / columns: the narrow DMMA loop)
// costs 0.32 of a full one (timeline build at C4b: 701 against 2192 us); the unprotected
// kernel has no narrow loop, all its tiles count as full.  Split only for an estimated gain of
// 3% or more, >= 16 stages per split and at most 8192 split CTAs (1 GB of partial blocks).
int wave_ksplit(bool ft, int64_t m, int64_t n, int tm, int tn, int nk, int nsm) {
  const int64_t tiles_m = (m + tm - 1) / tm, tiles_n = (n + tn - 1) / tn;
  const bool sliver_r = ft && m % tm != 0 && m % tm < 16, sliver_c = ft && n % tn != 0 && n % tn < 16;
  const int64_t full_m = tiles_m - (sliver_r ? 1 : 0), full_n = tiles_n - (sliver_c ? 1 : 0);
  const int64_t nfull = full_m * full_n, nsliver = tiles_m * tiles_n - nfull;
  if (nfull > 16 * (int64_t)nsm) return 1;  // many waves: the last partial wave costs < 1/16
  auto makespan = [&](int S) {
    // SM loads as groups {load: number of SMs}; a batch of identical CTAs fills the least
    // loaded group first (the list schedule of identical CTAs, a few steps per round instead
    // of a heap operation per CTA: this runs on every call)
    std::map<double, int64_t> g;
    g[0.0] = nsm;
    auto run = [&](int64_t cnt, double cost) {
      while (cnt > 0) {
        const auto it = g.begin();
        const double L = it->first;
        const int64_t k = it->second, take = std::min(k, cnt);
        g.erase(it);
        g[L + cost] += take;
        if (k > take) g[L] += k - take;
        cnt -= take;
      }
    };
    const double red = S > 1 ? 0.5 + 0.6 * S : 0.0;
    run(nfull * S, (double)nk / S + 3.0 + red);
    run(nsliver * S, 0.32 * nk / S + 3.0 + red);
    return g.rbegin()->first;
  };
  const double t1 = makespan(1);
  int best = 1;
  double best_t = 0.97 * t1;
  for (int S = 2; S <= 4; ++S) {
    if (nk / S < 16 || (nfull + nsliver) * S > 8192) break;
    const double t = makespan(S);
    if (t < best_t) { best = S; best_t = t; }
  }
  return best;
}

// The core entry: device pointers, protected (FT) or not, explicit fault list.
int dgemm_core(bool ft, const std::vector<ftblas_fault_t> &faults, char ta, char tb, int64_t m, int64_t n,
               int64_t k, double alpha, const double *A, int64_t lda, const double *B, int64_t ldb, double beta,
               double *C, int64_t ldc, ftblas_err_report_t *err, ReportSink *sink = nullptr,
               const std::vector<CsFault> &csf = {}) {
  const int rc = check_args(ta, tb, m, n, k, alpha, A, lda, B, ldb, C, ldc);
  if (rc) return rc;
  zero_report(err, k);
  if (m == 0 || n == 0) return 0;
  if (int e = ensure_device_init()) return e;
  cudaStream_t st = tl_stream;
  if (alpha == 0.0 || k == 0) {
    if (beta == 1.0) return 0;
    const int64_t total = m * n;
    const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
    ftk::scale_kernel<<<blocks, 256, 0, st>>>(m, n, beta, C, ldc);
    ++tl_launches;
    CUDA_TRY(cudaGetLastError());
    return 0;
  }
  for (const auto &f : faults)
    if (f.i < 0 || f.i >= m || f.j < 0 || f.j >= n || f.step < 0 || f.step > k) return 3;
  for (const auto &c : csf)
    if (!ft || c.f.i < 0 || c.f.i >= m || c.f.j < 0 || c.f.j >= n || c.f.step < 0 || c.f.step > k ||
        (c.lane != 1 && c.lane != 2))
      return 3;

  ftk::Params p{};
  p.m = m; p.n = n; p.k = k; p.alpha = alpha; p.beta = beta;
  p.A = A; p.lda = lda; p.B = B; p.ldb = ldb; p.C = C; p.ldc = ldc;
  int dev_mode = 0;
#ifdef FTBLAS_DEV
  if (const char *dm = std::getenv("FTBLAS_DEV_MODE")) dev_mode = std::atoi(dm);
#endif
  const bool g127 = ft || (dev_mode & 32);  // dev mode 32: unprotected kernel on the 127 grid
  const int tm = g127 ? ftk::TM : ftk::BM, tn = g127 ? ftk::TN : ftk::BN;  // tile stride in C
  p.tiles_m = (int)((m + tm - 1) / tm);
  p.tiles_n = (int)((n + tn - 1) / tn);
  p.nk = (int)((k + ftk::BK - 1) / ftk::BK);
  // Verification intervals (NEXT-1): Kc rank-1 updates each, the last one ragged.
  const int64_t Kc = (ft && tl_interval > 0 && tl_interval < k) ? tl_interval : k;
  const int64_t T = (k + Kc - 1) / Kc;
  p.Kc = Kc;
  p.T = (int)T;
  p.ntiles = p.tiles_m * p.tiles_n;
  // k-split of launches of at most half a wave of tiles (C^f partials summed in split order and
  // verified by the tile's last split, dgemm_abft.cuh): up to 8 splits of >= 2 stages each, as
  // many as fit in one wave (C1: 9 tiles x 8; 512^3: 25 x 5; the latency-bound small
  // problems).  The partial sums round differently from one k-loop, so such a call is not
  // bitwise equal to the same tiles computed unsplit, or split another way (a row panel of it),
  // but within the parity bound.  Verification intervals (Kc < k) keep whole tiles.
  p.ksplit = 1;
  if (T == 1 && (int64_t)p.ntiles * 2 <= (int64_t)num_sms()) {
    // single wave: up to 8 splits of >= 2 stages per tile, as many as fit on the SMs
    p.ksplit = (int)std::max<int64_t>(1, std::min<int64_t>(std::min<int64_t>((int64_t)p.nk / 2, 8),
                                                           (int64_t)num_sms() / p.ntiles));
    p.kcoop = p.ksplit > 1 ? 1 : 0;  // the splits reduce together (launch_one)
  }
  else if (T == 1)
    p.ksplit = wave_ksplit(ft, m, n, tm, tn, p.nk, num_sms());
  if (err) err->unit_k = (int32_t)std::min<int64_t>(Kc, INT32_MAX);
  p.correct_mode = tl_correct;
  p.cluster2 = (ft && tl_encode == FTBLAS_ENCODE_FUSED_LOCAL && p.ksplit == 1) ? 1 : 0;  // request; launch_one decides
#ifdef FTBLAS_DEV
#ifdef FTBLAS_WATCHDOG
  if (const char *dw = std::getenv("FTBLAS_DEV_WATCH")) {  // hang watchdog slot (tools/hang_probe.py)
    unsigned long long *w = reinterpret_cast<unsigned long long *>(std::strtoull(dw, nullptr, 0));
    CUDA_TRY(cudaMemcpyToSymbol(ftk::g_dev_watch, &w, sizeof w));
  }
#endif
  // development build only: per-CTA per-warp clock64 wait/work sums (tools/dev_prof.py)
  if (const char *dp = std::getenv("FTBLAS_DEV_PROF")) p.dev_prof = reinterpret_cast<unsigned long long *>(std::strtoull(dp, nullptr, 0));
  p.dev_mode = dev_mode;
#endif
#ifdef FTBLAS_DEV_TIMELINE
  // timeline build only (tools/dev_timeline.py): per-CTA clocks of MMA warp 0
  if (const char *dp = std::getenv("FTBLAS_DEV_PROF")) p.dev_prof = reinterpret_cast<unsigned long long *>(std::strtoull(dp, nullptr, 0));
#endif
  p.wait_pub = (ft && tl_encode == FTBLAS_ENCODE_FUSED_WAIT) ? 1 : 0;

  // Bucket faults by (tile, stage); stable so same-stage faults keep the caller's order.
  std::vector<ftk::FaultDev> fd;
  fd.reserve(faults.size() + csf.size());
  // lane 0: the data accumulator (i, j); 1: the column checksum of column j of (i, j)'s unit
  // (tile-local row -1 = the checksum row); 2: the row checksum of row i (column -1).
  auto bucket = [&](const ftblas_fault_t &f, int lane) {
    const int64_t ti = f.i / tm, tj = f.j / tn;
    // step quantised to BK (R8), applied before stage step_q / BK; it belongs to interval
    // min(step_q / Kc, T - 1) (step_q == k: after the last update of the last interval).
    const int64_t step_q = (f.step / ftk::BK) * ftk::BK;
    fd.push_back(ftk::FaultDev{(int32_t)(ti + tj * p.tiles_m), (int32_t)(step_q / ftk::BK),
                               lane == 1 ? -1 : (int32_t)(f.i - ti * tm), lane == 2 ? -1 : (int32_t)(f.j - tj * tn),
                               f.delta});
  };
  for (const auto &f : faults) bucket(f, 0);
  for (const auto &c : csf) bucket(c.f, c.lane);
  std::stable_sort(fd.begin(), fd.end(), [](const ftk::FaultDev &a, const ftk::FaultDev &b) {
    return a.tile != b.tile ? a.tile < b.tile : a.stage < b.stage;
  });

  // The device event ring holds one event per unit, so it never overflows: the report's events
  // are the first events_capacity of ALL events in sorted order (deterministic).
  const int64_t ev_cap = ft ? std::max<int64_t>(err ? err->events_capacity : 0, (int64_t)p.ntiles * T) : 0;
  static_assert(sizeof(unsigned long long) * ftk::CNT_N <= 64, "counters fit their 64-byte slot");
  const size_t ev_bytes = sizeof(ftk::EventDev) * (size_t)ev_cap;
  const size_t f_bytes = sizeof(ftk::FaultDev) * fd.size();
  // Encode mode PREPASS: e^T A_I, B_J e and the block maxima from two memory passes.
  const bool prepass = ft && tl_encode == FTBLAS_ENCODE_PREPASS;
  auto al256 = [](size_t b) { return (b + 255) & ~size_t(255); };
  // Tile-column-0 / tile-row-0 publication of e^T A_I / B_J e (encode mode FUSED, R22): the
  // slice maxima and the published sums, filled with all-ones bytes (= not yet published).
  // Launches of a single wave skip it (every tile starts together, so a consumer would almost
  // never find a stage published) unless dev modes 256 / 512 force the copy paths.
  const bool one_wave = (int64_t)p.ntiles * p.ksplit <= (int64_t)num_sms() && !p.wait_pub;
  const bool fused_shared = tl_encode == FTBLAS_ENCODE_FUSED || tl_encode == FTBLAS_ENCODE_FUSED_WAIT;
  const bool ashare = ft && fused_shared && p.tiles_n > 1 && !one_wave;
  const bool bshare = ft && fused_shared && p.tiles_m > 1 && !one_wave;
  // Launches of at most 3 waves: encoder CTAs at the head of the grid encode and publish every
  // tile row's e^T A_I and tile column's B_J e (integer passes only, no DMMA: several times the
  // DMMA pace), so no tile of the first wave waits for or repeats an encode (2048^3: the first
  // wave ran at the encoding pace, 294 against 280.5 us per tile).  Longer launches keep the
  // tile row / column 0 publishers (their extra cost is spread over many waves).
  p.enc_head = 0;
  if ((ashare || bshare) && p.ksplit == 1 && !p.cluster2 && (int64_t)p.ntiles <= 3 * (int64_t)num_sms())
    p.enc_head = (ashare ? p.tiles_m : 0) + (bshare ? p.tiles_n : 0);
  const size_t nsg = (size_t)p.nk;  // global stages over the whole k
  // Scratch: [counters (64 B) | events | faults | prepass | hmA Ash | hmB Bsh]: the counters
  // zeroed, the publication region filled with 0xFF; counters and the first events are read
  // back by one copy (finish_report).
  const size_t base_bytes = al256(64 + ev_bytes + f_bytes);
  // k-split: the partial C^f blocks, their stage maxima and the per-tile tickets
  const size_t split_bytes = p.ksplit > 1 ? al256(sizeof(double) * ftk::BM * ftk::BN * (size_t)p.ntiles * p.ksplit) +
                                                al256(sizeof(unsigned) * 2 * (size_t)p.ntiles * p.ksplit) +
                                                al256(sizeof(int) * (size_t)p.ntiles)
                                          : 0;
  const size_t hm_bytes = al256(sizeof(unsigned) * (p.tiles_m + p.tiles_n));
  const size_t pre_bytes = prepass ? hm_bytes + sizeof(double) * (size_t)(p.tiles_m + p.tiles_n) * k : 0;
  const size_t hma_bytes = ashare ? al256(sizeof(unsigned) * (size_t)p.tiles_m * nsg) : 0;
  const size_t ash_bytes = ashare ? hma_bytes + al256(sizeof(double) * (size_t)p.tiles_m * (size_t)k) : 0;
  const size_t hmb_bytes = bshare ? al256(sizeof(unsigned) * (size_t)p.tiles_n * nsg) : 0;
  const size_t bsh_bytes = bshare ? hmb_bytes + sizeof(double) * (size_t)p.tiles_n * (size_t)k : 0;
  Cleanup cl(st);
  char *scratch = nullptr;
  CUDA_TRY(cl.alloc(&scratch, base_bytes + pre_bytes + ash_bytes + bsh_bytes + split_bytes));
  char *const cnt_ptr = scratch;
  if (p.ksplit > 1) {
    char *sp = scratch + base_bytes + pre_bytes + ash_bytes + bsh_bytes;
    p.part = reinterpret_cast<double *>(sp);
    sp += al256(sizeof(double) * ftk::BM * ftk::BN * (size_t)p.ntiles * p.ksplit);
    p.part_max = reinterpret_cast<unsigned *>(sp);
    sp += al256(sizeof(unsigned) * 2 * (size_t)p.ntiles * p.ksplit);
    p.tickets = reinterpret_cast<int *>(sp);
    CUDA_TRY(cudaMemsetAsync(p.tickets, 0, sizeof(int) * (size_t)p.ntiles, st));
  }
  if (ashare) {
    char *sb = scratch + base_bytes + pre_bytes;
    p.hmA = reinterpret_cast<unsigned *>(sb);
    p.Ash = reinterpret_cast<double *>(sb + hma_bytes);
    p.ldash = k;
  }
  if (bshare) {
    char *sb = scratch + base_bytes + pre_bytes + ash_bytes;
    p.hmB = reinterpret_cast<unsigned *>(sb);
    p.Bsh = reinterpret_cast<double *>(sb + hmb_bytes);
    p.ldbsh = k;
  }
  CUDA_TRY(cudaMemsetAsync(scratch, 0, 64, st));
  if (ash_bytes + bsh_bytes)
    CUDA_TRY(cudaMemsetAsync(scratch + base_bytes + pre_bytes, 0xFF, ash_bytes + bsh_bytes, st));
  if (prepass) {
    char *pb = scratch + base_bytes;
    auto *hm = reinterpret_cast<unsigned *>(pb);
    double *Ac = reinterpret_cast<double *>(pb + hm_bytes);
    double *Br = Ac + (size_t)p.tiles_m * k;
    CUDA_TRY(cudaMemsetAsync(hm, 0, sizeof(unsigned) * (p.tiles_m + p.tiles_n), st));
    if (int e = launch_block_sum(A, is_n(ta), lda, m, k, Ac, p.tiles_m, hm, ftk::TM, st)) return e;
    if (int e = launch_block_sum(B, is_t(tb), ldb, n, k, Br, p.tiles_n, hm + p.tiles_m, ftk::TN, st)) return e;
    p.Ac = Ac; p.Br = Br; p.ldac = p.tiles_m; p.ldbr = p.tiles_n;
    p.amax_pre = hm; p.bmax_pre = hm + p.tiles_m;
  }
  p.counters = sink ? sink->counters : reinterpret_cast<unsigned long long *>(cnt_ptr);
  p.events = sink ? sink->events : reinterpret_cast<ftk::EventDev *>(cnt_ptr + 64);
  p.ev_cap = sink ? sink->ev_cap : ev_cap;
  p.ev_row_off = sink ? sink->row_off : 0;
  p.ev_col_off = sink ? sink->col_off : 0;
  if (sink && ft) sink->units += (int64_t)p.ntiles * T;
  // A protected call of at most 4 waves that fills its report: the launch writes it into mapped
  // pinned memory (ftk::publish_report; finish_report_mapped), no read-back copy (C1 call with
  // report 46 -> 41 us, 2048^3 616 -> 604 us).  Longer launches read it back: there the copy is
  // noise, and every CTA's exit fence (its C stores must land before it counts itself done)
  // cost C4a ~1%.
  MappedReport *mrep = nullptr;
  if (ft && err && !sink && (int64_t)p.ntiles * p.ksplit <= 4 * (int64_t)num_sms() &&
      mapped_report_buffer(&mrep) == cudaSuccess) {
    p.host_rep = mrep->dev;
    p.rep_seq = ++mrep->seq;
    p.rep_events = ftk::REP_EVENTS;
  }
  p.faults = fd.empty() ? nullptr : reinterpret_cast<const ftk::FaultDev *>(cnt_ptr + 64 + ev_bytes);
  p.nfaults = (int)fd.size();
  if (!fd.empty()) {
    char *stage = nullptr;
    CUDA_TRY(pinned_fault_stage(f_bytes, &stage));
    std::memcpy(stage, fd.data(), f_bytes);
    CUDA_TRY(cudaMemcpyAsync(cnt_ptr + 64 + ev_bytes, stage, f_bytes, cudaMemcpyHostToDevice, st));
    CUDA_TRY(pinned_fault_release(st));
  }

  const bool akm = is_t(ta), bkm = is_n(tb);
  // TMA needs 16-byte aligned bases and leading dimensions: repack otherwise (device copy
  // into a stream-ordered buffer with an even leading dimension; marshalling only).
  const int64_t ar = is_n(ta) ? m : k, ac = is_n(ta) ? k : m;
  const int64_t br = is_n(tb) ? k : n, bc = is_n(tb) ? n : k;
  double *rA = nullptr, *rB = nullptr;
  auto aligned = [](const double *q, int64_t ld) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0 && ld % 2 == 0; };
  if (!aligned(A, lda)) {
    const int64_t nld = (ar + 1) & ~int64_t(1);
    CUDA_TRY(cl.alloc(&rA, sizeof(double) * nld * ac));
    CUDA_TRY(cudaMemcpy2DAsync(rA, sizeof(double) * nld, A, sizeof(double) * lda, sizeof(double) * ar, ac,
                               cudaMemcpyDeviceToDevice, st));
    p.A = rA; p.lda = nld;
  }
  if (!aligned(B, ldb)) {
    const int64_t nld = (br + 1) & ~int64_t(1);
    CUDA_TRY(cl.alloc(&rB, sizeof(double) * nld * bc));
    CUDA_TRY(cudaMemcpy2DAsync(rB, sizeof(double) * nld, B, sizeof(double) * ldb, sizeof(double) * br, bc,
                               cudaMemcpyDeviceToDevice, st));
    p.B = rB; p.ldb = nld;
  }
  CUtensorMap tmA, tmB;
  if (int e = make_tmap(&tmA, p.A, p.lda, akm, m, k)) return e;
  if (int e = make_tmap(&tmB, p.B, p.ldb, bkm, n, k)) return e;
  // One launch: every CTA verifies its tile online after every Kc updates (T checks).
  const dim3 grid((unsigned)(p.ntiles * p.ksplit + p.enc_head));  // 1-D: grouped raster in the kernel
  const int lrc = ft ? dispatch<true>(akm, bkm, tmA, tmB, p, grid, st) : dispatch<false>(akm, bkm, tmA, tmB, p, grid, st);
  if (lrc) return lrc;

  if (err && !sink) {
    const int64_t units = ft ? (int64_t)p.ntiles * T : 0;
    if (p.host_rep) {
      if (int e = finish_report_mapped(err, *mrep, p.rep_seq, p.counters, p.events, ev_cap, units, st)) return e;
    } else if (int e = finish_report(err, p.counters, p.events, ev_cap, units, st)) {
      return e;
    }
  }
  return 0;
}

int dgemm_impl(bool ft, char ta, char tb, int64_t m, int64_t n, int64_t k, double alpha, const double *A,
               int64_t lda, const double *B, int64_t ldb, double beta, double *C, int64_t ldc,
               ftblas_err_report_t *err) {
  const std::vector<ftblas_fault_t> faults = take_armed();
  const std::vector<CsFault> csf = take_armed_cs();
  return dgemm_core(ft, faults, ta, tb, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, err, nullptr, csf);
}

// The unfused ABFT baseline (kernels in unfused.cuh; PAPER.md:257-261
// §V.A): encode passes, then for every interval of Kc updates: the unprotected GEMM on the
// k-slice (accumulating into C), the two skinny GEMMs carrying the checksums, the reference
// row sums C e, the row check, the column sums e^T C only on a mismatch, verify / locate /
// correct the flagged units.
int unfused_impl(char ta, char tb, int64_t m, int64_t n, int64_t k, double alpha, const double *A, int64_t lda,
                 const double *B, int64_t ldb, double beta, double *C, int64_t ldc, ftblas_err_report_t *err) {
  const std::vector<ftblas_fault_t> faults = take_armed();
  if (reject_armed_cs()) return 3;  // checksum-lane faults: ftblas_dgemm only
  const int rc = check_args(ta, tb, m, n, k, alpha, A, lda, B, ldb, C, ldc);
  if (rc) return rc;
  const int64_t Kc = (tl_interval > 0 && tl_interval < k) ? tl_interval : std::max<int64_t>(k, 1);
  const int64_t T = (k + Kc - 1) / Kc;
  if (err) {
    err->units_checked = err->detected = err->corrected = err->recomputed = err->n_events = 0;
    err->unit_rows = err->unit_cols = ftu::UB;
    err->unit_k = (int32_t)std::min<int64_t>(Kc, INT32_MAX);
    err->step_quantum = ftk::BK;
  }
  if (m == 0 || n == 0) return 0;
  if (alpha == 0.0 || k == 0)  // C = beta*C, no ABFT
    return dgemm_core(false, {}, ta, tb, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, nullptr);
  for (const auto &f : faults)
    if (f.i < 0 || f.i >= m || f.j < 0 || f.j >= n || f.step < 0 || f.step > k) return 3;
  if (int e = ensure_device_init()) return e;
  cudaStream_t st = tl_stream;
  const int64_t nbm = (m + ftu::UB - 1) / ftu::UB, nbn = (n + ftu::UB - 1) / ftu::UB;
  const int64_t ldm = (nbm + 1) & ~int64_t(1), ldn = (nbn + 1) & ~int64_t(1), ldr = (m + 1) & ~int64_t(1);
  const bool direct = alpha == 1.0 && beta == 0.0;  // verify C itself, else a scratch product T
  const int64_t ev_cap = std::max<int64_t>(err ? err->events_capacity : 0, nbm * nbn * T);  // one per unit
  // scratch: counters, events, maxima, Ac, Br, CSc, CSr, Rc, Rr, unit flags (+ T)
  const size_t cnt_b = sizeof(unsigned long long) * ftk::CNT_N, ev_b = sizeof(ftk::EventDev) * ev_cap;
  const size_t hm_b = sizeof(unsigned) * (ldm + ldn);
  const size_t ac_b = sizeof(double) * ldm * k, br_b = sizeof(double) * ldn * k;
  const size_t csc_b = sizeof(double) * ldm * n, csr_b = sizeof(double) * ldr * ldn;
  const size_t rc_b = sizeof(double) * ldm * n, rr_b = sizeof(double) * ldn * m;
  const size_t fl_b = sizeof(int) * (nbm * nbn + 1);
  const size_t t_b = direct ? 0 : sizeof(double) * ldr * n;
  auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
  const size_t total = al(cnt_b) + al(ev_b) + al(hm_b) + al(ac_b) + al(br_b) + al(csc_b) + al(csr_b) + al(rc_b) +
                       al(rr_b) + al(fl_b) + al(t_b);
  Cleanup cl(st);
  char *base = nullptr;
  CUDA_TRY(cl.alloc(&base, total));
  char *q = base;
  auto take = [&](size_t b) { char *r = q; q += al(b); return r; };
  auto *counters = reinterpret_cast<unsigned long long *>(take(cnt_b));
  void *events = take(ev_b);
  auto *hmax = reinterpret_cast<unsigned *>(take(hm_b));
  auto *Ac = reinterpret_cast<double *>(take(ac_b));
  auto *Br = reinterpret_cast<double *>(take(br_b));
  auto *CSc = reinterpret_cast<double *>(take(csc_b));
  auto *CSr = reinterpret_cast<double *>(take(csr_b));
  auto *Rc = reinterpret_cast<double *>(take(rc_b));
  auto *Rr = reinterpret_cast<double *>(take(rr_b));
  auto *flags = reinterpret_cast<int *>(take(fl_b));  // [unit flags | any]
  double *Tm = direct ? C : reinterpret_cast<double *>(take(t_b));
  const int64_t ldt = direct ? ldc : ldr;
  CUDA_TRY(cudaMemsetAsync(counters, 0, cnt_b, st));
  CUDA_TRY(cudaMemsetAsync(hmax, 0, hm_b, st));
  // Zero the padded checksum rows once so the GEMMs on them read defined values.
  if (ldm != nbm) CUDA_TRY(cudaMemsetAsync(Ac, 0, ac_b, st));
  if (ldn != nbn) CUDA_TRY(cudaMemsetAsync(Br, 0, br_b, st));

  auto block_sum = [&](const double *X, bool xc, int64_t ld, int64_t nx, int64_t np, double *S, int64_t lds,
                       unsigned *hm, const int *enable = nullptr) -> int {
    return launch_block_sum(X, xc, ld, nx, np, S, lds, hm, ftu::UB, st, enable);
  };
  // 1. encode: e^T A_I for every row block I (x = i), B_J e for every column block J (x = j).
  if (int e = block_sum(A, is_n(ta), lda, m, k, Ac, ldm, hmax)) return e;
  if (int e = block_sum(B, is_t(tb), ldb, n, k, Br, ldn, hmax + ldm)) return e;
  for (int64_t t = 0; t < T; ++t) {
    const int64_t k0 = t * Kc, k1 = std::min(k0 + Kc, k), kl = k1 - k0;
    const double bt = t ? 1.0 : 0.0;  // accumulate the intervals into C (and the checksums)
    const double *At = is_n(ta) ? A + k0 * lda : A + k0;
    const double *Bt = is_n(tb) ? B + k0 : B + k0 * ldb;
    // 2. the product on the k-slice, unprotected kernel (this interval's faults land here, their
    //    steps local to the slice).
    std::vector<ftblas_fault_t> ft_t;
    for (const auto &f : faults) {
      const int64_t sq = (f.step / ftk::BK) * ftk::BK;
      if (std::min<int64_t>(sq / Kc, T - 1) == t) ft_t.push_back(ftblas_fault_t{f.i, f.j, f.step - k0, f.delta});
    }
    if (int e = dgemm_core(false, ft_t, ta, tb, m, n, kl, 1.0, At, lda, Bt, ldb, bt, Tm, ldt, nullptr)) return e;
    // 3. carried checksums: (e^T A_I) B (nbm x n) and A (B_J e) (m x nbn), two skinny GEMMs.
    if (int e = dgemm_core(false, {}, 'N', tb, ldm, n, kl, 1.0, Ac + k0 * ldm, ldm, Bt, ldb, bt, CSc, ldm, nullptr)) return e;
    if (int e = dgemm_core(false, {}, ta, 'T', m, ldn, kl, 1.0, At, lda, Br + k0 * ldn, ldn, bt, CSr, ldr, nullptr)) return e;
    // 4. reference row checksums C_J e first; the row check marks mismatching units.
    CUDA_TRY(cudaMemsetAsync(flags, 0, fl_b, st));
    if (int e = block_sum(Tm, false, ldt, n, m, Rr, ldn, nullptr)) return e;
    {
      const int blocks = (int)std::min<int64_t>((m * nbn + 255) / 256, 148 * 8);
      ftu::row_check_kernel<<<blocks, 256, 0, st>>>(m, n, k1, Rr, ldn, CSr, ldr, hmax, hmax + ldm, (int)nbm, (int)nbn,
                                                    flags, flags + nbm * nbn);
      ++tl_launches;
      CUDA_TRY(cudaGetLastError());
    }
    // 5. e^T C_I only on a mismatch (the pass returns at once otherwise), then verify / locate /
    //    correct the marked units.
    if (int e = block_sum(Tm, true, ldt, m, n, Rc, ldm, nullptr, flags + nbm * nbn)) return e;
    ftu::VerifyParams vp{};
    vp.m = m; vp.n = n; vp.k = k1; vp.interval = (int)t; vp.unit_flag = flags;
    vp.ta = is_n(ta) ? 'N' : 'T'; vp.tb = is_n(tb) ? 'N' : 'T';
    vp.A = A; vp.lda = lda; vp.B = B; vp.ldb = ldb; vp.T = Tm; vp.ldt = ldt;
    vp.Rc = Rc; vp.CSc = CSc; vp.ldm = ldm; vp.Rr = Rr; vp.ldn = ldn; vp.CSr = CSr; vp.ldr = ldr;
    vp.amax_hi = hmax; vp.bmax_hi = hmax + ldm; vp.nbm = (int)nbm; vp.nbn = (int)nbn;
    vp.Ac = t + 1 < T ? Ac : nullptr; vp.Br = Br; vp.CSc_w = CSc; vp.CSr_w = CSr;
    vp.correct_mode = tl_correct; vp.counters = counters; vp.events = events; vp.ev_cap = ev_cap;
    ftu::verify_kernel<<<(unsigned)(nbm * nbn), 256, 0, st>>>(vp);
    ++tl_launches;
    CUDA_TRY(cudaGetLastError());
  }
  // 6. C = alpha*T + beta*C0 when the product was verified in scratch.
  if (!direct) {
    const int blocks = (int)std::min<int64_t>((m * n + 255) / 256, 148 * 16);
    ftu::axpby_kernel<<<blocks, 256, 0, st>>>(m, n, alpha, Tm, ldt, beta, C, ldc);
    ++tl_launches;
    CUDA_TRY(cudaGetLastError());
  }
  if (err)
    if (int e = finish_report(err, counters, events, ev_cap, nbm * nbn * T, st)) return e;
  return 0;
}

int num_sms();

// Host-buffer variant (the end-to-end API).  B goes to the device once; C is processed in row
// panels (multiples of the 127-row unit, so the verification units are those of one call)
// through a three-stream pipeline: the H2D copy of panel r+1's op(A) rows (and C0 rows) and
// the D2H copy of panel r-1's result overlap the protected GEMM of panel r.  The first and the
// last panel run in column chunks (edges multiples of 2 x 127 columns): the first panel starts
// as soon as its op(A) rows and the first chunk of op(B) are on the device, the rest of B
// streaming in behind it chunk by chunk; the last panel returns its result chunk by chunk.
// When m is small against n (column mode) there is one panel: all of op(A), then op(B) and
// the result in column chunks.
// Faults are routed to their panel / chunk with local indices; counters and events accumulate
// on the device (events carry global indices) and the report is filled once at the end.
int dgemm_host_impl(bool ft, char ta, char tb, int64_t m, int64_t n, int64_t k, double alpha,
                    const double *A, int64_t lda, const double *B, int64_t ldb, double beta,
                    double *C, int64_t ldc, ftblas_err_report_t *err) {
  std::vector<ftblas_fault_t> faults = take_armed();
  if (reject_armed_cs()) return 3;  // checksum-lane faults: ftblas_dgemm only
  const int rc = check_args(ta, tb, m, n, k, alpha, A, lda, B, ldb, C, ldc);
  if (rc) return rc;
  zero_report(err, k);
  if (m == 0 || n == 0) return 0;
  if (int e = ensure_device_init()) return e;
  cudaStream_t st = tl_stream;
  const bool reads_ab = alpha != 0.0 && k > 0;
  if (!reads_ab) {  // C = beta*C: one device round trip, no ABFT
    if (beta == 1.0) return 0;
    Cleanup cl0(st);
    double *dC = nullptr;
    CUDA_TRY(cl0.alloc(&dC, sizeof(double) * m * n));
    if (beta != 0.0)
      CUDA_TRY(cudaMemcpy2DAsync(dC, sizeof(double) * m, C, sizeof(double) * ldc, sizeof(double) * m, n,
                                 cudaMemcpyHostToDevice, st));
    int r = dgemm_core(false, {}, ta, tb, m, n, k, alpha, nullptr, std::max<int64_t>(1, is_n(ta) ? m : k), nullptr,
                       std::max<int64_t>(1, is_n(tb) ? k : n), beta, dC, m, nullptr);
    if (r == 0)
      r = cudaMemcpy2DAsync(C, sizeof(double) * ldc, dC, sizeof(double) * m, sizeof(double) * m, n,
                            cudaMemcpyDeviceToHost, st) == cudaSuccess ? 0 : 1;
    const cudaError_t se = cudaStreamSynchronize(st);
    return r ? r : (se == cudaSuccess ? 0 : cuda_fail(se));
  }
  for (const auto &f : faults)
    if (f.i < 0 || f.i >= m || f.j < 0 || f.j >= n || f.step < 0 || f.step > k) return 3;
  const int64_t Kc = (ft && tl_interval > 0 && tl_interval < k) ? tl_interval : k;
  const int64_t T_units = (k + Kc - 1) / Kc;
  if (err) err->unit_k = (int32_t)std::min<int64_t>(Kc, INT32_MAX);

  // Panels: about m/8 rows, a multiple of 2 x 127 (units intact, even leading dimensions),
  // chosen within [m/11, m/6] to minimise the total number of 148-CTA waves over the panels
  // (ties: closest to m/8); one panel when the problem is small.
  const int64_t unit2 = 2 * ftk::TM;
  int64_t P = m;
  if (m >= 16 * unit2) {
    const int64_t th = ft ? ftk::TM : ftk::BM, tw = ft ? ftk::TN : ftk::BN, sms = num_sms();
    const int64_t tcols = (n + tw - 1) / tw, target = (m + 7) / 8;
    int64_t best_waves = INT64_MAX, best_dist = INT64_MAX;
    for (int64_t c = (m / 11 + unit2 - 1) / unit2 * unit2; c <= m / 6; c += unit2) {
      int64_t waves = 0;
      for (int64_t r0 = 0; r0 < m; r0 += c) waves += (((std::min(c, m - r0) + th - 1) / th) * tcols + sms - 1) / sms;
      const int64_t dist = c > target ? c - target : target - c;
      if (waves < best_waves || (waves == best_waves && dist < best_dist)) { best_waves = waves; best_dist = dist; P = c; }
    }
    if (P == m) P = (target + unit2 - 1) / unit2 * unit2;
  }
  // Column mode: all of op(A) first, then op(B) in column chunks over one panel of m rows.  It
  // wins when waiting for all of op(B) behind the first row panel costs more start-up than
  // copying all of op(A) (m small against n: the row panels of a multi-GPU run).  Estimated in
  // bytes, with ~636 FP64 flops of DMMA time per byte of PCIe Gen5 copy.
  bool colmode = false;
  if (P < m) {
    const double f_per_b = 636.0;
    const double row_idle = 8.0 * (double)P * (double)k +
                            std::max(0.0, 8.0 * (double)k * (double)n - 2.0 * (double)P * (double)n * (double)k / f_per_b);
    const double col_idle = 8.0 * (double)m * (double)k;
    if (col_idle < row_idle) { colmode = true; P = m; }
  }
  const int64_t npan = (m + P - 1) / P;
  const int64_t br = is_n(tb) ? k : n, bc = is_n(tb) ? n : k;

  // Column chunks of a panel of pr rows: uniform chunks of t tile columns (t even, so chunk
  // edges are multiples of 2 tiles: units intact, 16-byte aligned bases), t minimising the
  // panel's time in 148-CTA waves plus the copy of one chunk of op(B) (the pipeline's start-up:
  // a k-deep column takes ~1.2e-3 of a k-deep wave over PCIe Gen5 against the FP64 DMMA rate),
  // at most 16 chunks.  One chunk when there is one panel.
  auto chunking = [&](int64_t pr) {
    std::vector<int64_t> best{0, n};
    if (npan < 2 && !colmode) return best;
    const int64_t tw = ft ? ftk::TN : ftk::BN, th = ft ? ftk::TM : ftk::BM;
    const int64_t trows = (pr + th - 1) / th, tcols = (n + tw - 1) / tw, sms = num_sms();
    double best_cost = 1e300;
    for (int64_t t = 2; t < tcols; t += 2) {
      const int64_t nch = (tcols + t - 1) / t;
      if (nch > 16) continue;
      int64_t waves = 0;
      std::vector<int64_t> e{0};
      for (int64_t c0 = 0; c0 < n; c0 += t * tw) {
        const int64_t c1 = std::min(n, c0 + t * tw);
        waves += (trows * ((c1 - c0 + tw - 1) / tw) + sms - 1) / sms;
        e.push_back(c1);
      }
      const double cost = (double)waves + 1.2e-3 * (double)(t * tw);
      if (cost < best_cost) { best_cost = cost; best = e; }
    }
    return best;
  };

  Cleanup cl(st);
  cudaStream_t sh = nullptr, sd = nullptr;
  CUDA_TRY(cl.stream(&sh));
  CUDA_TRY(cl.stream(&sd));
  cudaEvent_t ev_b, ev_in[2], ev_out[2], ev_free[2];
  CUDA_TRY(cl.event(&ev_b));
  for (int q = 0; q < 2; ++q) {
    CUDA_TRY(cl.event(&ev_in[q]));
    CUDA_TRY(cl.event(&ev_out[q]));
    CUDA_TRY(cl.event(&ev_free[q]));
  }
  // one event slot per unit of the whole problem (never overflows; deterministic report)
  const int64_t ev_cap = ft ? std::max<int64_t>(err ? err->events_capacity : 0,
                                                ((m + ftk::TM - 1) / ftk::TM) * ((n + ftk::TN - 1) / ftk::TN) * T_units)
                            : 0;
  const size_t cnt_bytes = sizeof(unsigned long long) * ftk::CNT_N;
  const size_t ev_bytes = sizeof(ftk::EventDev) * (size_t)std::max<int64_t>(ev_cap, 1);
  const size_t pa = sizeof(double) * (size_t)P * (size_t)k, pc = sizeof(double) * (size_t)P * (size_t)n;
  char *rep_base = nullptr;
  double *dB = nullptr, *dA[2] = {nullptr, nullptr}, *dC[2] = {nullptr, nullptr};
  int r = 0;
  auto fail = [&](cudaError_t e) { if (r == 0 && e != cudaSuccess) r = cuda_fail(e); };
  // Stream-ordered (pooled) staging on the compute stream; the copy streams wait for it.
  fail(cl.alloc(&rep_base, 256 + ev_bytes));
  fail(cl.alloc(&dB, sizeof(double) * br * bc));
  for (int q = 0; q < 2 && q < npan; ++q) {
    fail(cl.alloc(&dA[q], pa));
    fail(cl.alloc(&dC[q], pc));
  }
  fail(cudaEventRecord(ev_b, st));
  fail(cudaStreamWaitEvent(sh, ev_b, 0));
  fail(cudaStreamWaitEvent(sd, ev_b, 0));
  ReportSink sink{reinterpret_cast<unsigned long long *>(rep_base),
                  reinterpret_cast<ftk::EventDev *>(rep_base + 256), ev_cap, 0, 0};
  if (r == 0) fail(cudaMemsetAsync(rep_base, 0, cnt_bytes, st));
  // development only (FTBLAS_DEV_E2E): stream-event timeline of the pipeline, printed at the end
#ifdef FTBLAS_DEV
  const bool dev_e2e = std::getenv("FTBLAS_DEV_E2E") != nullptr;
#else
  const bool dev_e2e = false;
#endif
  std::vector<std::pair<std::string, cudaEvent_t>> dev_ev;
  auto mark = [&](const std::string &what, cudaStream_t s) {
    if (!dev_e2e) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, s);
    dev_ev.emplace_back(what, e);
  };
  mark("start(st)", st);
  // op(B) columns [c0, c1) -> device (dB keeps the stored layout, leading dimension br).
  auto upload_b = [&](int64_t c0, int64_t c1) {
    if (is_n(tb))
      fail(cudaMemcpy2DAsync(dB + c0 * br, sizeof(double) * br, B + c0 * ldb, sizeof(double) * ldb,
                             sizeof(double) * br, c1 - c0, cudaMemcpyHostToDevice, sh));
    else
      fail(cudaMemcpy2DAsync(dB + c0, sizeof(double) * br, B + c0, sizeof(double) * ldb, sizeof(double) * (c1 - c0),
                             bc, cudaMemcpyHostToDevice, sh));
  };
  for (int64_t pi = 0; pi < npan && r == 0; ++pi) {
    const int q = (int)(pi & 1);
    const int64_t r0 = pi * P, pr = std::min<int64_t>(P, m - r0);
    if (pi >= 2) fail(cudaStreamWaitEvent(sh, ev_free[q], 0));  // panel pi-2 left the device
    if (is_n(ta))  // op(A) rows r0.. of an m x k matrix
      fail(cudaMemcpy2DAsync(dA[q], sizeof(double) * pr, A + r0, sizeof(double) * lda, sizeof(double) * pr, k,
                             cudaMemcpyHostToDevice, sh));
    else  // columns r0.. of the k x m stored matrix
      fail(cudaMemcpy2DAsync(dA[q], sizeof(double) * k, A + r0 * lda, sizeof(double) * lda, sizeof(double) * k, pr,
                             cudaMemcpyHostToDevice, sh));
    if (beta != 0.0)
      fail(cudaMemcpy2DAsync(dC[q], sizeof(double) * pr, C + r0, sizeof(double) * ldc, sizeof(double) * pr, n,
                             cudaMemcpyHostToDevice, sh));
    fail(cudaEventRecord(ev_in[q], sh));
    fail(cudaStreamWaitEvent(st, ev_in[q], 0));
    mark("A" + std::to_string(pi) + " in(sh)", sh);
    if (r) break;
    const bool first = pi == 0, last = pi == npan - 1;
    const std::vector<int64_t> edges = (first || last) ? chunking(pr) : std::vector<int64_t>{0, n};
    for (size_t ci = 0; ci + 1 < edges.size() && r == 0; ++ci) {
      const int64_t c0 = edges[ci], c1 = edges[ci + 1];
      if (first) {  // this chunk of op(B) (all of it when unchunked), then compute on it
        upload_b(c0, c1);
        mark("B chunk " + std::to_string(ci) + " in(sh)", sh);
        fail(cudaEventRecord(ev_b, sh));
        fail(cudaStreamWaitEvent(st, ev_b, 0));
        if (r) break;
      }
      std::vector<ftblas_fault_t> pf;
      for (const auto &f : faults)
        if (f.i >= r0 && f.i < r0 + pr && f.j >= c0 && f.j < c1)
          pf.push_back(ftblas_fault_t{f.i - r0, f.j - c0, f.step, f.delta});
      sink.row_off = r0;
      sink.col_off = c0;
      const double *Bc = is_n(tb) ? dB + c0 * br : dB + c0;
      mark("p" + std::to_string(pi) + "c" + std::to_string(ci) + " begin(st)", st);
      r = dgemm_core(ft, pf, ta, tb, pr, c1 - c0, k, alpha, dA[q], is_n(ta) ? pr : k, Bc, br, beta, dC[q] + c0 * pr,
                     pr, nullptr, ft ? &sink : nullptr);
      mark("p" + std::to_string(pi) + "c" + std::to_string(ci) + " end(st)", st);
      if (r) break;
      if (last) {  // return this chunk of the result
        fail(cudaEventRecord(ev_out[q], st));
        fail(cudaStreamWaitEvent(sd, ev_out[q], 0));
        fail(cudaMemcpy2DAsync(C + r0 + c0 * ldc, sizeof(double) * ldc, dC[q] + c0 * pr, sizeof(double) * pr,
                               sizeof(double) * pr, c1 - c0, cudaMemcpyDeviceToHost, sd));
      }
    }
    if (r) break;
    if (!last) {
      fail(cudaEventRecord(ev_out[q], st));
      fail(cudaStreamWaitEvent(sd, ev_out[q], 0));
      fail(cudaMemcpy2DAsync(C + r0, sizeof(double) * ldc, dC[q], sizeof(double) * pr, sizeof(double) * pr, n,
                             cudaMemcpyDeviceToHost, sd));
    }
    fail(cudaEventRecord(ev_free[q], sd));
  }
  mark("last D2H(sd)", sd);
  fail(cudaStreamSynchronize(sd));
  if (dev_e2e) {
    cudaDeviceSynchronize();
    for (auto &pe : dev_ev) {
      float ms = 0.f;
      const cudaError_t ee = cudaEventElapsedTime(&ms, dev_ev[0].second, pe.second);
      std::fprintf(stderr, "[e2e] %8.2f ms  %s%s\n", ms, pe.first.c_str(), ee == cudaSuccess ? "" : cudaGetErrorString(ee));
    }
    for (auto &pe : dev_ev) cudaEventDestroy(pe.second);
  }
  fail(cudaStreamSynchronize(sh));
  fail(cudaStreamSynchronize(st));
  if (r == 0 && err && ft) r = finish_report(err, sink.counters, sink.events, ev_cap, sink.units, st);
  return r;
}

// ---------------------------------------------------------------- Level-1/2 DMR (NEXT-4)
// Device scratch for one DMR call: counters + the armed faults (sorted by output index).
struct DmrScratch {
  char *base = nullptr;
  unsigned long long *cnt = nullptr;
  ftd::DmrFault *f = nullptr;
  int nf = 0;
};

int dmr_prepare(bool ft, std::vector<ftblas_fault_t> &faults, int64_t nout, int64_t maxstep, DmrScratch &sc,
                cudaStream_t st) {
  for (const auto &f : faults)
    if (f.i < 0 || f.i >= nout || f.step < 0 || f.step > maxstep) return 3;
  std::vector<ftd::DmrFault> fd;
  if (ft)
    for (const auto &f : faults) fd.push_back(ftd::DmrFault{f.i, f.step, f.delta});
  std::stable_sort(fd.begin(), fd.end(), [](const ftd::DmrFault &a, const ftd::DmrFault &b) { return a.index < b.index; });
  const size_t cb = sizeof(unsigned long long) * ftd::D_N, fb = sizeof(ftd::DmrFault) * fd.size();
  CUDA_TRY(cudaMallocAsync((void **)&sc.base, 256 + fb, st));
  sc.cnt = reinterpret_cast<unsigned long long *>(sc.base);
  sc.f = fd.empty() ? nullptr : reinterpret_cast<ftd::DmrFault *>(sc.base + 256);
  sc.nf = (int)fd.size();
  cudaError_t e = cudaMemsetAsync(sc.cnt, 0, cb, st);
  if (e == cudaSuccess && !fd.empty()) e = cudaMemcpyAsync(sc.f, fd.data(), fb, cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) {
    cudaFreeAsync(sc.base, st);
    sc.base = nullptr;
    return cuda_fail(e);
  }
  return 0;
}

int dmr_finish(DmrScratch &sc, int64_t checked, ftblas_dmr_report_t *rep, cudaStream_t st) {
  Cleanup cl(st);  // the scratch is released on every path
  if (sc.base) cl.mem.push_back(sc.base);
  sc.base = nullptr;
  CUDA_TRY(cudaGetLastError());
  if (rep) {
    unsigned long long c[ftd::D_N];
    CUDA_TRY(cudaMemcpyAsync(c, sc.cnt, sizeof c, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    rep->checked = checked;
    rep->detected = (int64_t)c[ftd::D_DETECTED];
    rep->corrected = (int64_t)c[ftd::D_CORRECTED];
    rep->uncorrectable = (int64_t)c[ftd::D_UNCORRECTABLE];
  }
  return 0;
}

void dmr_zero(ftblas_dmr_report_t *rep) {
  if (rep) rep->checked = rep->detected = rep->corrected = rep->uncorrectable = 0;
}

// One wave of resident CTAs (8 x 256 threads per SM at <= 32 registers) for grid-stride loops.
int num_sms() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
      sms = 148;
  }
  return sms;
}
bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }
int l1_grid(int64_t n, bool dmr) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((n + 1023) / 1024, (int64_t)num_sms() * ftd::resident_ctas(dmr)));
}

int dscal_impl(bool ft, int64_t n, double alpha, double *x, int64_t incx, ftblas_dmr_report_t *rep) {
  std::vector<ftblas_fault_t> faults = take_armed();
  if (reject_armed_cs()) return 3;  // checksum-lane faults: ftblas_dgemm only
  if (n < 0) return -1;
  if (n > 0 && x == nullptr) return -3;
  if (incx == 0) return -4;
  dmr_zero(rep);
  if (n == 0) return 0;
  if (int e = ensure_device_init()) return e;
  cudaStream_t st = tl_stream;
  DmrScratch sc;
  if (int e = dmr_prepare(ft, faults, n, 0, sc, st)) return e;
  if (incx == 1 && aligned16(x)) {  // unit stride: one 16-byte-vectorised chunk per CTA
    const unsigned g = (unsigned)((n + ftd::VCHUNK - 1) / ftd::VCHUNK);
    if (ft && sc.nf) ftd::dscal_vec_kernel<true, true><<<g, 256, 0, st>>>(n, alpha, x, sc.f, sc.nf, sc.cnt);
    else if (ft) ftd::dscal_vec_kernel<true, false><<<g, 256, 0, st>>>(n, alpha, x, nullptr, 0, sc.cnt);
    else ftd::dscal_vec_kernel<false, false><<<g, 256, 0, st>>>(n, alpha, x, nullptr, 0, sc.cnt);
  } else if (ft && sc.nf) ftd::dscal_kernel<true, true><<<l1_grid(n, true), 256, 0, st>>>(n, alpha, x, incx, sc.f, sc.nf, sc.cnt);
  else if (ft) ftd::dscal_kernel<true, false><<<l1_grid(n, true), 256, 0, st>>>(n, alpha, x, incx, nullptr, 0, sc.cnt);
  else ftd::dscal_kernel<false, false><<<l1_grid(n, false), 256, 0, st>>>(n, alpha, x, incx, nullptr, 0, sc.cnt);
  ++tl_launches;
  return dmr_finish(sc, ft ? n : 0, rep, st);
}

int daxpy_impl(bool ft, int64_t n, double alpha, const double *x, int64_t incx, double *y, int64_t incy,
               ftblas_dmr_report_t *rep) {
  std::vector<ftblas_fault_t> faults = take_armed();
  if (reject_armed_cs()) return 3;  // checksum-lane faults: ftblas_dgemm only
  if (n < 0) return -1;
  if (n > 0 && x == nullptr) return -3;
  if (incx == 0) return -4;
  if (n > 0 && y == nullptr) return -5;
  if (incy == 0) return -6;
  dmr_zero(rep);
  if (n == 0) return 0;
  if (int e = ensure_device_init()) return e;
  cudaStream_t st = tl_stream;
  DmrScratch sc;
  if (int e = dmr_prepare(ft, faults, n, 0, sc, st)) return e;
  if (incx == 1 && incy == 1 && aligned16(x) && aligned16(y)) {  // unit stride: vectorised chunks
    const unsigned g = (unsigned)((n + ftd::VCHUNK - 1) / ftd::VCHUNK);
    if (ft && sc.nf) ftd::daxpy_vec_kernel<true, true><<<g, 256, 0, st>>>(n, alpha, x, y, sc.f, sc.nf, sc.cnt);
    else if (ft) ftd::daxpy_vec_kernel<true, false><<<g, 256, 0, st>>>(n, alpha, x, y, nullptr, 0, sc.cnt);
    else ftd::daxpy_vec_kernel<false, false><<<g, 256, 0, st>>>(n, alpha, x, y, nullptr, 0, sc.cnt);
  } else if (ft && sc.nf) ftd::daxpy_kernel<true, true><<<l1_grid(n, true), 256, 0, st>>>(n, alpha, x, incx, y, incy, sc.f, sc.nf, sc.cnt);
  else if (ft) ftd::daxpy_kernel<true, false><<<l1_grid(n, true), 256, 0, st>>>(n, alpha, x, incx, y, incy, nullptr, 0, sc.cnt);
  else ftd::daxpy_kernel<false, false><<<l1_grid(n, false), 256, 0, st>>>(n, alpha, x, incx, y, incy, nullptr, 0, sc.cnt);
  ++tl_launches;
  return dmr_finish(sc, ft ? n : 0, rep, st);
}

int dgemv_impl(bool ft, char trans, int64_t m, int64_t n, double alpha, const double *A, int64_t lda,
               const double *x, int64_t incx, double beta, double *y, int64_t incy, ftblas_dmr_report_t *rep) {
  std::vector<ftblas_fault_t> faults = take_armed();
  if (reject_armed_cs()) return 3;  // checksum-lane faults: ftblas_dgemm only
  if (!is_n(trans) && !is_t(trans)) return -1;
  if (m < 0) return -2;
  if (n < 0) return -3;
  const bool tr = is_t(trans);
  const int64_t nout = tr ? n : m, len = tr ? m : n;  // outputs, dot length
  if (lda < std::max<int64_t>(1, m)) return -6;
  if (nout > 0 && len > 0 && alpha != 0.0 && A == nullptr) return -5;
  if (nout > 0 && len > 0 && alpha != 0.0 && x == nullptr) return -7;
  if (incx == 0) return -8;
  if (nout > 0 && y == nullptr) return -10;
  if (incy == 0) return -11;
  dmr_zero(rep);
  if (nout == 0) return 0;
  if (int e = ensure_device_init()) return e;
  cudaStream_t st = tl_stream;
  DmrScratch sc;
  if (int e = dmr_prepare(ft, faults, nout, len, sc, st)) return e;
  ftd::GemvParams P{};
  P.m = m; P.n = n; P.alpha = alpha; P.beta = beta; P.A = A; P.lda = lda; P.x = x; P.incx = incx;
  P.y = y; P.incy = incy; P.f = sc.f; P.nf = sc.nf; P.cnt = sc.cnt;
  if (alpha == 0.0 || len == 0) { P.m = tr ? 0 : m; P.n = tr ? n : 0; }  // y = beta*y: empty dot products
  if (!tr) {
    // lanes per row: the smallest of 1, 2, 4 that gives at least 512 CTAs (~3.5 waves); 4 below
    // (8 lanes per row measured slower at m = 2048)
    const int lpr = m >= 512 * 32 ? 1 : (m >= 512 * 16 ? 2 : 4);
    const unsigned g = (unsigned)((m + 32 / lpr - 1) / (32 / lpr));
    auto launch = [&](auto lprc) {
      constexpr int L = decltype(lprc)::value;
      if (ft && sc.nf) ftd::dgemv_n_kernel<true, true, L><<<g, ftd::GN_W * 32, 0, st>>>(P);
      else if (ft) ftd::dgemv_n_kernel<true, false, L><<<g, ftd::GN_W * 32, 0, st>>>(P);
      else ftd::dgemv_n_kernel<false, false, L><<<g, ftd::GN_W * 32, 0, st>>>(P);
    };
    if (lpr == 1) launch(std::integral_constant<int, 1>{});
    else if (lpr == 2) launch(std::integral_constant<int, 2>{});
    else launch(std::integral_constant<int, 4>{});
  } else {
    const unsigned g = (unsigned)std::min<int64_t>((n + 7) / 8, (int64_t)num_sms() * ftd::GT_CTAS);
    if (ft && sc.nf) ftd::dgemv_t_kernel<true, true><<<g, 256, 0, st>>>(P);
    else if (ft) ftd::dgemv_t_kernel<true, false><<<g, 256, 0, st>>>(P);
    else ftd::dgemv_t_kernel<false, false><<<g, 256, 0, st>>>(P);
  }
  ++tl_launches;
  return dmr_finish(sc, ft ? nout : 0, rep, st);
}

// ---------------------------------------------------------------- FT-DTRSM (NEXT-3)

// op(A) X = alpha B, side 'L'.  Recursive blocked solve: a block of more than LEAF rows is
// split (the updated part a multiple of 127, see trsm_rec), the parts are solved recursively and the coupling
// is a GEMM update B2 -= op(A)21 X1 (forward, op(A) lower) or B1 -= op(A)12 X2 (backward, op(A)
// upper) through the protected DMMA kernel (fused ABFT, report accumulated in a sink); the
// leaves are the DMR diagonal-block kernel of trsm.cuh.  A fault (i, j, step = p) perturbs the
// update of B(i, j) by X(p, j): it lands in the GEMM whose rows hold i and whose k-range holds
// p, or in the leaf when i and p share one LEAF block.
struct TrsmCtx {
  bool ft, fwd, trans, unit;
  bool right;    // side 'R': X op(A) = B, the solve runs over B's columns, each row an RHS
  int64_t leaf;  // diagonal block rows (LEAF; 127 for the protected solve measured slower)
  const double *A;
  int64_t lda;
  double *B;
  int64_t ldb, n;  // n: number of right-hand sides (side L: B's columns, side R: B's rows)
  const std::vector<ftblas_fault_t> *faults;
  ReportSink *sink;
  DmrScratch *leaf_sc;  // leaf DMR counters
  cudaStream_t st;
};

// A fault (i, j, step) as (element along the solve, right-hand side): side L (row i of column
// j), side R (column j of row i).
inline int64_t f_elem(const TrsmCtx &c, const ftblas_fault_t &f) { return c.right ? f.j : f.i; }
inline int64_t f_rhs(const TrsmCtx &c, const ftblas_fault_t &f) { return c.right ? f.i : f.j; }

int trsm_leaf(TrsmCtx &c, int64_t r0, int64_t mb) {
  std::vector<ftd::DmrFault> lf;
  if (c.ft)
    for (const auto &f : *c.faults) {
      const int64_t e = f_elem(c, f);
      if (e >= r0 && e < r0 + mb && f.step >= r0 && f.step < r0 + mb)
        lf.push_back(ftd::DmrFault{f_rhs(c, f) * ftt::LEAF + (e - r0), f.step - r0, f.delta});
    }
  Cleanup cl(c.st);
  ftd::DmrFault *df = nullptr;
  if (!lf.empty()) {
    CUDA_TRY(cl.alloc(&df, sizeof(ftd::DmrFault) * lf.size()));
    CUDA_TRY(cudaMemcpyAsync(df, lf.data(), sizeof(ftd::DmrFault) * lf.size(), cudaMemcpyHostToDevice, c.st));
  }
  ftt::LeafParams P{};
  P.nb = (int)mb; P.n = (int)c.n;
  P.A = c.A + r0 + r0 * c.lda; P.lda = c.lda;
  // side L: element p of right-hand side j at B[(r0 + p) + j ldb]; side R: at B[j + (r0 + p) ldb],
  // and the block is solved transposed (x S = b  <=>  S^T x^T = b^T)
  P.es = c.right ? c.ldb : 1;
  P.rs = c.right ? 1 : c.ldb;
  P.B = c.B + r0 * P.es;
  P.trans = c.right ? !c.trans : c.trans; P.unit = c.unit;
  P.f = df; P.nf = (int)lf.size(); P.cnt = c.leaf_sc->cnt;
  const int smem = (int)(sizeof(double) * (ftt::LEAF * ftt::LEAF + 2 * ftt::LEAF));
  constexpr int per_cta = ftt::LEAF_THREADS / 32 * ftt::LEAF_NCOL;  // right-hand sides per CTA pass
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((c.n + per_cta - 1) / per_cta,
                                                              (int64_t)num_sms()));
  using K = void (*)(ftt::LeafParams);
  // [fwd][dmr][faults]
  static const K kernels[2][2][2] = {
      {{ftt::trsm_leaf_kernel<false, false, false>, ftt::trsm_leaf_kernel<false, false, true>},
       {ftt::trsm_leaf_kernel<false, true, false>, ftt::trsm_leaf_kernel<false, true, true>}},
      {{ftt::trsm_leaf_kernel<true, false, false>, ftt::trsm_leaf_kernel<true, false, true>},
       {ftt::trsm_leaf_kernel<true, true, false>, ftt::trsm_leaf_kernel<true, true, true>}}};
  static std::atomic<bool> attr_set[64];  // per device (idempotent if raced)
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64 || !attr_set[dev].load(std::memory_order_acquire)) {
    for (int a = 0; a < 8; ++a)
      CUDA_TRY(cudaFuncSetAttribute(kernels[a >> 2][(a >> 1) & 1][a & 1], cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    if (dev >= 0 && dev < 64) attr_set[dev].store(true, std::memory_order_release);
  }
  kernels[c.fwd][c.ft][c.ft && P.nf > 0]<<<grid, ftt::LEAF_THREADS, smem, c.st>>>(P);
  ++tl_launches;
  CUDA_TRY(cudaGetLastError());
  return 0;
}

// The update rows [R0, R0+mr) of B -= op(A)[R0.., K0..K0+mk] * X[K0.., :].
int trsm_update(TrsmCtx &c, int64_t R0, int64_t mr, int64_t K0, int64_t mk) {
  std::vector<ftblas_fault_t> gf;
  if (c.ft)
    for (const auto &f : *c.faults) {
      const int64_t e = f_elem(c, f);
      if (e >= R0 && e < R0 + mr && f.step >= K0 && f.step < K0 + mk)
        gf.push_back(c.right ? ftblas_fault_t{f.i, e - R0, f.step - K0, f.delta}
                             : ftblas_fault_t{e - R0, f.j, f.step - K0, f.delta});
    }
  if (!c.right) {  // B[R0.., :] -= op(A)[R0.., K0..] X[K0.., :]
    const double *Asub = c.trans ? c.A + K0 + R0 * c.lda : c.A + R0 + K0 * c.lda;
    if (c.sink) { c.sink->row_off = R0; c.sink->col_off = 0; }
    return dgemm_core(c.ft, gf, c.trans ? 'T' : 'N', 'N', mr, c.n, mk, -1.0, Asub, c.lda, c.B + K0, c.ldb, 1.0,
                      c.B + R0, c.ldb, nullptr, c.ft ? c.sink : nullptr);
  }
  // side R: B[:, R0..] -= X[:, K0..] op(A)[K0.., R0..]
  const double *Asub = c.trans ? c.A + R0 + K0 * c.lda : c.A + K0 + R0 * c.lda;
  if (c.sink) { c.sink->row_off = 0; c.sink->col_off = R0; }
  return dgemm_core(c.ft, gf, 'N', c.trans ? 'T' : 'N', c.n, mr, mk, -1.0, c.B + K0 * c.ldb, c.ldb, Asub, c.lda, 1.0,
                    c.B + R0 * c.ldb, c.ldb, nullptr, c.ft ? c.sink : nullptr);
}

int trsm_rec(TrsmCtx &c, int64_t r0, int64_t m) {
  if (m <= c.leaf) return trsm_leaf(c, r0, m);
  // The part the coupling GEMM updates is u = 254 j rows, j = round(m / 508) (reduced until
  // u < m), else 126: whole tile rows of the protected kernel's 127-row grid (a power-of-two
  // split leaves a sliver tile row that costs a wave of its own: 256 x 8192 x 256 87% over
  // the unprotected kernel, 254 x 8192 x 254 10.5%) and even, so every block boundary keeps
  // the operands 16-byte aligned for TMA (an odd one costs a repack copy).  The part solved
  // first takes the rest (leaves <= LEAF).  Both twins use the same split, so their results
  // stay bitwise equal.
  int64_t j = (m + 2 * ftk::TM) / (4 * ftk::TM);
  while (j > 0 && 2 * ftk::TM * j >= m) --j;
  const int64_t u = j > 0 ? 2 * ftk::TM * j : ftk::TM - 1;
  const int64_t m1 = c.fwd ? m - u : u, m2 = m - m1;
  if (c.fwd) {
    if (int e = trsm_rec(c, r0, m1)) return e;
    if (int e = trsm_update(c, r0 + m1, m2, r0, m1)) return e;
    return trsm_rec(c, r0 + m1, m2);
  }
  if (int e = trsm_rec(c, r0 + m1, m2)) return e;
  if (int e = trsm_update(c, r0, m1, r0 + m1, m2)) return e;
  return trsm_rec(c, r0, m1);
}

int dtrsm_impl(bool ft, char side, char uplo, char transa, char diag, int64_t m, int64_t n, double alpha,
               const double *A, int64_t lda, double *B, int64_t ldb, ftblas_err_report_t *err) {
  std::vector<ftblas_fault_t> faults = take_armed();
  if (reject_armed_cs()) return 3;  // checksum-lane faults: ftblas_dgemm only
  const bool right = side == 'R' || side == 'r';
  if (!right && side != 'L' && side != 'l') return -1;
  const bool lower = uplo == 'L' || uplo == 'l';
  if (!lower && uplo != 'U' && uplo != 'u') return -2;
  if (!is_n(transa) && !is_t(transa)) return -3;
  const bool unit = diag == 'U' || diag == 'u';
  if (!unit && diag != 'N' && diag != 'n') return -4;
  if (m < 0) return -5;
  if (n < 0) return -6;
  const int64_t na = right ? n : m;  // order of op(A)
  if (m > 0 && n > 0 && alpha != 0.0 && A == nullptr) return -8;
  if (lda < std::max<int64_t>(1, na)) return -9;
  if (m > 0 && n > 0 && B == nullptr) return -10;
  if (ldb < std::max<int64_t>(1, m)) return -11;
  zero_report(err, na);
  if (err) { err->unit_k = 0; }
  if (m == 0 || n == 0) return 0;
  if (int e = ensure_device_init()) return e;
  cudaStream_t st = tl_stream;
  const bool trans = is_t(transa);
  // Substitution order along the solve: side L runs over rows and goes forward when op(A) is
  // lower; side R runs over columns and goes forward when op(A) is upper.
  const bool fwd = right ? lower == trans : lower != trans;
  for (const auto &f : faults) {
    const int64_t e = right ? f.j : f.i;
    if (f.i < 0 || f.i >= m || f.j < 0 || f.j >= n || f.step < 0 || f.step >= na || (fwd ? f.step >= e : f.step <= e))
      return 3;
  }
  if (alpha != 1.0) {
    const int blocks = (int)std::min<int64_t>((m * n + 255) / 256, (int64_t)num_sms() * 16);
    ftt::scale_b_kernel<<<blocks, 256, 0, st>>>(m, n, alpha, B, ldb);
    ++tl_launches;
    CUDA_TRY(cudaGetLastError());
    if (alpha == 0.0) return 0;
  }
  const int64_t ev_cap = ft ? std::max<int64_t>(err ? err->events_capacity : 0, 1024) : 0;
  Cleanup cl(st);
  char *rep = nullptr;
  CUDA_TRY(cl.alloc(&rep, 256 + sizeof(ftk::EventDev) * (size_t)std::max<int64_t>(ev_cap, 1)));
  CUDA_TRY(cudaMemsetAsync(rep, 0, 256, st));
  ReportSink sink{reinterpret_cast<unsigned long long *>(rep), reinterpret_cast<ftk::EventDev *>(rep + 256), ev_cap, 0, 0};
  std::vector<ftblas_fault_t> none;
  DmrScratch lsc;
  if (int e = dmr_prepare(false, none, 1, 0, lsc, st)) return e;  // leaf counters only
  cl.mem.push_back(lsc.base);
  TrsmCtx c{ft, fwd, trans, unit, right, (int64_t)ftt::LEAF, A, lda, B, ldb, right ? m : n, &faults, &sink, &lsc, st};
  int r = trsm_rec(c, 0, na);
  if (r == 0 && err && ft) {
    r = finish_report(err, sink.counters, sink.events, ev_cap, sink.units, st);
    unsigned long long lc[ftd::D_N];
    if (r == 0 && cudaMemcpy(lc, lsc.cnt, sizeof lc, cudaMemcpyDeviceToHost) == cudaSuccess) {
      err->detected += (int64_t)lc[ftd::D_DETECTED];
      err->corrected += (int64_t)lc[ftd::D_CORRECTED];
      err->recomputed += (int64_t)lc[ftd::D_UNCORRECTABLE];
    }
  }
  return r;
}

uint64_t splitmix_next(uint64_t &state) {
  state += 0x9E3779B97F4A7C15ull;
  uint64_t z = state;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
double splitmix_uniform(uint64_t &state) { return (double)(splitmix_next(state) >> 11) * 0x1p-53; }

}  // namespace

extern "C" {

int ftblas_dgemm(char transA, char transB, int64_t m, int64_t n, int64_t k, double alpha,
                 const double *A, int64_t lda, const double *B, int64_t ldb, double beta, double *C,
                 int64_t ldc, ftblas_err_report_t *err) {
  return dgemm_impl(true, transA, transB, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, err);
}

int ftblas_dgemm_noft(char transA, char transB, int64_t m, int64_t n, int64_t k, double alpha,
                      const double *A, int64_t lda, const double *B, int64_t ldb, double beta,
                      double *C, int64_t ldc) {
  return dgemm_impl(false, transA, transB, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, nullptr);
}

int ftblas_dgemm_unfused(char transA, char transB, int64_t m, int64_t n, int64_t k, double alpha,
                         const double *A, int64_t lda, const double *B, int64_t ldb, double beta, double *C,
                         int64_t ldc, ftblas_err_report_t *err) {
  return unfused_impl(transA, transB, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, err);
}

int ftblas_dscal(int64_t n, double alpha, double *x, int64_t incx, ftblas_dmr_report_t *rep) {
  return dscal_impl(true, n, alpha, x, incx, rep);
}
int ftblas_dscal_noft(int64_t n, double alpha, double *x, int64_t incx) {
  return dscal_impl(false, n, alpha, x, incx, nullptr);
}
int ftblas_daxpy(int64_t n, double alpha, const double *x, int64_t incx, double *y, int64_t incy,
                 ftblas_dmr_report_t *rep) {
  return daxpy_impl(true, n, alpha, x, incx, y, incy, rep);
}
int ftblas_daxpy_noft(int64_t n, double alpha, const double *x, int64_t incx, double *y, int64_t incy) {
  return daxpy_impl(false, n, alpha, x, incx, y, incy, nullptr);
}
int ftblas_dgemv(char trans, int64_t m, int64_t n, double alpha, const double *A, int64_t lda, const double *x,
                 int64_t incx, double beta, double *y, int64_t incy, ftblas_dmr_report_t *rep) {
  return dgemv_impl(true, trans, m, n, alpha, A, lda, x, incx, beta, y, incy, rep);
}
int ftblas_dgemv_noft(char trans, int64_t m, int64_t n, double alpha, const double *A, int64_t lda,
                      const double *x, int64_t incx, double beta, double *y, int64_t incy) {
  return dgemv_impl(false, trans, m, n, alpha, A, lda, x, incx, beta, y, incy, nullptr);
}

int ftblas_dtrsm(char side, char uplo, char transa, char diag, int64_t m, int64_t n, double alpha, const double *A,
                 int64_t lda, double *B, int64_t ldb, ftblas_err_report_t *err) {
  return dtrsm_impl(true, side, uplo, transa, diag, m, n, alpha, A, lda, B, ldb, err);
}
int ftblas_dtrsm_noft(char side, char uplo, char transa, char diag, int64_t m, int64_t n, double alpha,
                      const double *A, int64_t lda, double *B, int64_t ldb) {
  return dtrsm_impl(false, side, uplo, transa, diag, m, n, alpha, A, lda, B, ldb, nullptr);
}

int ftblas_dgemm_host(char transA, char transB, int64_t m, int64_t n, int64_t k, double alpha,
                      const double *A, int64_t lda, const double *B, int64_t ldb, double beta,
                      double *C, int64_t ldc, ftblas_err_report_t *err) {
  return dgemm_host_impl(true, transA, transB, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, err);
}

int ftblas_dgemm_noft_host(char transA, char transB, int64_t m, int64_t n, int64_t k, double alpha,
                           const double *A, int64_t lda, const double *B, int64_t ldb, double beta,
                           double *C, int64_t ldc) {
  return dgemm_host_impl(false, transA, transB, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, nullptr);
}

int ftblas_inject_arm(const ftblas_fault_t *faults, int64_t n) {
  if (n < 0 || (n > 0 && faults == nullptr)) return 3;
  tl_armed.assign(faults, faults + n);
  tl_have_armed = true;
  return 0;
}

int ftblas_inject_disarm(void) {
  tl_armed.clear();
  tl_have_armed = false;
  tl_armed_cs.clear();
  return 0;
}
int ftblas_inject_arm_checksum(const ftblas_fault_t *faults, const int32_t *lanes, int64_t n) {
  if (n < 0 || (n > 0 && (faults == nullptr || lanes == nullptr))) return 3;
  tl_armed_cs.clear();
  for (int64_t e = 0; e < n; ++e) {
    if (lanes[e] != 1 && lanes[e] != 2) { tl_armed_cs.clear(); return 3; }
    tl_armed_cs.push_back(CsFault{faults[e], lanes[e]});
  }
  return 0;
}

int ftblas_inject_seeded(uint64_t seed, int64_t count, int64_t m, int64_t n, int64_t k,
                         double log10_lo, double log10_hi, ftblas_fault_t *out) {
  if (count < 0 || m <= 0 || n <= 0 || k < 0 || (count > 0 && out == nullptr)) return 3;
  uint64_t st = seed;
  for (int64_t e = 0; e < count; ++e) {
    double u[5];
    for (int q = 0; q < 5; ++q) u[q] = splitmix_uniform(st);
    out[e].i = std::min<int64_t>((int64_t)std::floor(u[0] * (double)m), m - 1);
    out[e].j = std::min<int64_t>((int64_t)std::floor(u[1] * (double)n), n - 1);
    out[e].step = std::min<int64_t>((int64_t)std::floor(u[2] * (double)k), std::max<int64_t>(k - 1, 0));
    const double mag = std::pow(10.0, log10_lo + (log10_hi - log10_lo) * u[3]);
    out[e].delta = u[4] < 0.5 ? -mag : mag;
  }
  return 0;
}

int ftblas_set_stream(void *cuda_stream) {
  tl_stream = static_cast<cudaStream_t>(cuda_stream);
  return 0;
}

int ftblas_set_correction(int mode) {
  if (mode != FTBLAS_CORRECT_RECOMPUTE && mode != FTBLAS_CORRECT_SUBTRACT) return 4;
  tl_correct = mode;
  return 0;
}

int ftblas_set_interval(int64_t kc) {
  if (kc < 0 || kc % ftk::BK != 0) return 4;
  tl_interval = kc;
  return 0;
}

int ftblas_set_encode(int mode) {
  if (mode != FTBLAS_ENCODE_FUSED && mode != FTBLAS_ENCODE_PREPASS && mode != FTBLAS_ENCODE_FUSED_LOCAL &&
      mode != FTBLAS_ENCODE_FUSED_WAIT)
    return 4;
  tl_encode = mode;
  return 0;
}

int ftblas_get_geometry(int32_t *unit_rows, int32_t *unit_cols, int32_t *step_quantum) {
  if (unit_rows) *unit_rows = ftk::TM;
  if (unit_cols) *unit_cols = ftk::TN;
  if (step_quantum) *step_quantum = ftk::BK;
  return 0;
}

int64_t ftblas_take_launch_count(void) {
  const int64_t v = tl_launches;
  tl_launches = 0;
  return v;
}

const char *ftblas_status_string(int status) {
  if (status < 0) {
    static thread_local char buf[64];
    std::snprintf(buf, sizeof buf, "invalid argument %d", -status);
    return buf;
  }
  switch (status) {
    case 0: return "success";
    case 1: return tl_cuda_error.empty() ? "CUDA error" : tl_cuda_error.c_str();
    case 2: return "out of device memory";
    case 3: return "bad fault list";
    case 4: return "bad option value";
    default: return "unknown status";
  }
}

int ftblas_finalize(void) {
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess) return 0;
  std::lock_guard<std::mutex> lk(g_init_mu);
  for (int d = 0; d < ndev && d < 64; ++d) {
    if (!g_init_done[d]) continue;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, d) == cudaSuccess) cudaMemPoolTrimTo(pool, 0);
  }
  return 0;
}

}  // extern "C"
