/*
 * ftblas.h — C ABI of the B200-native online ABFT DGEMM library (libftblas.so).
 *
 * The operation is the paper's Level-3 hot path, FT-BLAS (arXiv 2104.00897):
 *
 *     C = alpha * op(A) * op(B) + beta * C          (DGEMM, §III.C.2)
 *
 * protected online by algorithm-based fault tolerance (ABFT):
 *   - checksum encoding e^T A and B e                        PAPER.md:90   §II.A
 *   - outer-product checksum maintenance (e^T A)B, A(Be)      PAPER.md:93-95 §II.A
 *   - encoding fused into operand loads, reference checksums
 *     fused into the kernel ("purely computational")          PAPER.md:276  §V.B
 *   - verify e^T C / C e against the maintained checksums,
 *     locate the single corrupted C_ij from the intersecting
 *     row and column residuals, correct it in place           PAPER.md:258 §V.A, 445 §VI.C
 *   - one correctable error per verification interval         PAPER.md:95  §II.A
 *
 * Conventions (all entry points):
 *   - Matrices are column-major, BLAS style: element (r, c) of a matrix with leading
 *     dimension ld is at ptr[r + c*ld].  op(A) is m x k, op(B) is k x n, C is m x n.
 *     trans = 'N'/'n' (op(X) = X) or 'T'/'t'/'C'/'c' (op(X) = X^T; real data, so C == T).
 *     A is m x k (lda >= max(1,m)) for 'N' and k x m (lda >= max(1,k)) otherwise;
 *     B is k x n (ldb >= max(1,k)) for 'N' and n x k (ldb >= max(1,n)) otherwise.
 *   - A, B, C are caller-owned DEVICE pointers on the current CUDA device (e.g. the
 *     data_ptr() of torch float64 tensors) unless the function name ends in _host.
 *     C must not alias A or B (BLAS rule; undefined otherwise).  The library never
 *     frees or retains caller pointers.
 *   - beta == 0: C is not read on input (NaN in C is ignored).  alpha == 0 or k == 0:
 *     C = beta*C, no ABFT, no units checked.  m == 0 or n == 0: quick return.
 *   - Work is enqueued on the calling thread's stream (ftblas_set_stream; default: the
 *     legacy default stream 0).
 *   - The library owns lazily allocated per-device scratch (report counters, event ring,
 *     fault lists, host-API staging buffers), stream-ordered from the device's default memory
 *     pool, whose release threshold it sets to a quarter of the device memory (scratch up to
 *     that stays cached between calls); ftblas_finalize() releases it.
 *
 * Status codes (return value of every int function):
 *     0  success — INCLUDING when soft errors were detected and corrected; detection is
 *        reported through the error report, never through the status.
 *    -p  argument p is invalid (LAPACK INFO style): 1 transA, 2 transB, 3 m, 4 n, 5 k,
 *        7 A == NULL, 8 lda, 9 B == NULL, 10 ldb, 12 C == NULL, 13 ldc
 *        (positions in the ftblas_dgemm argument list; NULL checks only when the
 *        operand is read: A and B when alpha != 0 and k > 0, C when m, n > 0).
 *     1  CUDA error (the CUDA error string is kept for ftblas_status_string(1)),
 *     2  out of memory,  3  bad fault list (i outside [0,m), j outside [0,n), step
 *        outside [0,k], or count < 0), 4 bad option value.
 */
#ifndef FTBLAS_H
#define FTBLAS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* One error event (one per flagged verification unit). */
typedef struct {
  int64_t i, j;        /* kind 1: row/column of the corrected element (global, 0-based);
                          kind 2: first row/column of the recomputed unit */
  int32_t kind;        /* 1 = CORRECTED at (i, j); 2 = RECOMPUTED unit (flag pattern other
                          than exactly one row and one column; reading R6/R13) */
  int32_t interval;    /* verification interval index t (0 when Kc == k) */
  double residual_row; /* d_row = (C e)_i - (A(Be))_i at the (first) flagged row, else 0 */
  double residual_col; /* d_col = (e^T C)_j - ((e^T A)B)_j at the (first) flagged col, else 0 */
} ftblas_event_t;

/* Error report of one protected call.  Counters are totals over the call. */
typedef struct {
  int64_t units_checked; /* out: verification units (tile x interval) verified */
  int64_t detected;      /* out: units with any flagged row or column */
  int64_t corrected;     /* out: units with exactly one flagged row and column (fixed in place) */
  int64_t recomputed;    /* out: units recomputed once (any other flag pattern) */
  int64_t n_events;      /* out: events produced (may exceed events_capacity) */
  int32_t unit_rows;     /* out: BM, rows per verification unit */
  int32_t unit_cols;     /* out: BN, columns per verification unit */
  int32_t unit_k;        /* out: Kc, k-length of a verification interval (ftblas_set_interval) */
  int32_t step_quantum;  /* out: BK; an injected fault's step is applied at floor(step/BK)*BK */
  ftblas_event_t *events;  /* in: caller-owned HOST array (may be NULL), filled with the
                              first min(n_events, events_capacity) of ALL the call's events
                              sorted by (interval, i, j) (deterministic: the library keeps
                              one event slot per unit, so nothing is dropped before the
                              sort; FT-DTRSM keeps max(events_capacity, 1024) slots) */
  int64_t events_capacity; /* in */
} ftblas_err_report_t;

/* One injected soft error: after `step` of the k rank-1 updates have been accumulated
 * into acc(i, j) (quantised down to a multiple of step_quantum), add `delta` to it.
 * Models PAPER.md:445 §VI.C: "An element of matrix C is randomly selected for
 * modification when an injection point is reached." */
typedef struct {
  int64_t i, j, step;
  double delta;
} ftblas_fault_t;

/* Protected DGEMM.  Stream-ordered; with err != NULL it returns once the report is complete,
 * i.e. once every result of the call (C, counters, events) has been written: launches of up to
 * 4 waves write the report into mapped pinned host memory themselves (their last CTA, after all
 * others are done) and the call polls it -- the launch may still be retiring when the call
 * returns; longer launches read it back and synchronise the stream.  Consumes (and disarms) any
 * faults armed on this thread. */
int ftblas_dgemm(char transA, char transB, int64_t m, int64_t n, int64_t k, double alpha,
                 const double *A, int64_t lda, const double *B, int64_t ldb, double beta,
                 double *C, int64_t ldc, ftblas_err_report_t *err);

/* Unprotected twin (same mainloop and epilogue, no checksums): the overhead baseline.
 * Fully asynchronous.  Armed faults are also consumed here and injected silently (the
 * negative control: the corruption reaches C undetected). */
int ftblas_dgemm_noft(char transA, char transB, int64_t m, int64_t n, int64_t k, double alpha,
                      const double *A, int64_t lda, const double *B, int64_t ldb, double beta,
                      double *C, int64_t ldc);

/* The UNFUSED ABFT baseline (§V.A): the same
 * protection as ftblas_dgemm built from separate kernels, as in a conventional ABFT library —
 * encode passes e^T A_I, B_J e over A and B (memory-bound), the unprotected GEMM, the
 * carried checksums (e^T A_I) B and A (B_J e) as two skinny GEMMs, reference-sum passes
 * e^T C_IJ, C_IJ e over the product, then verify / locate / correct per unit.  Units are
 * 128 x 128 (err->unit_rows/unit_cols report it).  Same arguments, report, fault injection
 * (faults land in the product GEMM), correction modes and status codes as ftblas_dgemm.
 * When alpha != 1 or beta != 0 the product is verified in library scratch and then combined
 * as C = alpha*T + beta*C.  Library scratch: ~8 (2 m/128 * k + 2 m n/128 ...) bytes. */
int ftblas_dgemm_unfused(char transA, char transB, int64_t m, int64_t n, int64_t k, double alpha,
                         const double *A, int64_t lda, const double *B, int64_t ldb, double beta,
                         double *C, int64_t ldc, ftblas_err_report_t *err);

/* Same as ftblas_dgemm / ftblas_dgemm_noft but A, B, C are HOST pointers (pinned memory
 * recommended).  Copies op inputs host->device, computes, copies C device->host and
 * synchronises the stream before returning.  Device staging is library-owned: all of op(B)
 * plus two row panels of op(A) and C.  Large problems (m >= 16 * 254) run as ~8 row panels
 * (multiples of 254 rows) with copies overlapped with compute on two library streams; the
 * first and last panels run in column chunks (multiples of 254 columns) so compute starts
 * once the first chunk of op(B) has arrived and the last result returns chunk by chunk.
 * When m is small against n (e.g. one rank's row panel of a multi-GPU run) all of op(A) is
 * copied first and op(B) and C stream in column chunks over a single panel instead.
 * Chunk and panel edges are multiples of the verification unit, so the report (units,
 * events with global (i, j)) equals that of one ftblas_dgemm call on the whole problem. */
int ftblas_dgemm_host(char transA, char transB, int64_t m, int64_t n, int64_t k, double alpha,
                      const double *A, int64_t lda, const double *B, int64_t ldb, double beta,
                      double *C, int64_t ldc, ftblas_err_report_t *err);
int ftblas_dgemm_noft_host(char transA, char transB, int64_t m, int64_t n, int64_t k,
                           double alpha, const double *A, int64_t lda, const double *B,
                           int64_t ldb, double beta, double *C, int64_t ldc);

/* Fault injection (test / benchmark hook).  ftblas_inject_arm copies n faults (host
 * array) to this thread's armed list; the next dgemm call on this thread consumes them.
 * Validation against m, n, k happens at that call (status 3). */
int ftblas_inject_arm(const ftblas_fault_t *faults, int64_t n);
int ftblas_inject_disarm(void);

/* Test hook for the checksum lanes themselves (reading R6): perturb a CARRIED checksum of the
 * verification unit that contains C(i, j) instead of a data accumulator -- lanes[e] == 1: the
 * column checksum ((e^T A_I) B_J)_j, lanes[e] == 2: the row checksum (A_I (B_J e))_i -- by
 * delta after `step` rank-1 updates (quantised like data faults).  Such a fault flags one
 * direction only, so its unit is recomputed.  Consumed by the next ftblas_dgemm call on this
 * thread (together with ftblas_inject_arm's list); any other entry point that finds them armed
 * disarms them and returns 3, as does a lane other than 1 or 2. */
int ftblas_inject_arm_checksum(const ftblas_fault_t *faults, const int32_t *lanes, int64_t n);

/* Seeded fault generator: SplitMix64 (Steele, Lea, Flood 2014) seeded with `seed`; per
 * fault draw u0..u4 in [0,1) from the top 53 bits and set i = floor(u0*m),
 * j = floor(u1*n), step = floor(u2*k) (each clamped to the last index),
 * |delta| = 10^(log10_lo + (log10_hi - log10_lo)*u3), sign negative iff u4 < 0.5.
 * Writes `count` entries to the caller-owned `out`. */
int ftblas_inject_seeded(uint64_t seed, int64_t count, int64_t m, int64_t n, int64_t k,
                         double log10_lo, double log10_hi, ftblas_fault_t *out);

/* Thread-local stream for subsequent calls (a cudaStream_t; NULL = legacy stream). */
int ftblas_set_stream(void *cuda_stream);

/* Correction mode for single errors: 0 = recompute C_ij from a fresh k-long dot product
 * (default, reading R4), 1 = subtract the located error magnitude. */
#define FTBLAS_CORRECT_RECOMPUTE 0
#define FTBLAS_CORRECT_SUBTRACT 1
int ftblas_set_correction(int mode);

/* Where ftblas_dgemm forms the checksums e^T A_I and B_J e:
 *   FTBLAS_ENCODE_FUSED (default): in the kernel, from the very tiles staged for the MMA
 *     (the paper's fused encoding, §V.B), each checksum encoded once where the
 *     hardware lets tiles share it: e^T A_I by the tile of tile column 0 and B_J e by the
 *     tile of tile row 0, published per stage through L2 to the other tiles of row I /
 *     column J (a tile whose stage is not published yet encodes it itself: nothing ever
 *     waits; launches of a single wave encode locally).  Library scratch when shared:
 *     8 (m/127 + n/127) k + 4 (m/127 + n/127) ceil(k/16) bytes;
 *   FTBLAS_ENCODE_FUSED_LOCAL: in the kernel, every CTA encodes both of its operand tiles
 *     itself (B_J e split between the two CTAs of a cluster pair);
 *   FTBLAS_ENCODE_PREPASS: two memory-bound passes over A and B before the kernel; the
 *     kernel copies the pre-encoded 16 k-slots into the checksum row of each staged tile.
 *   FTBLAS_ENCODE_FUSED_WAIT: as FUSED, but a tile whose stage is not published yet waits
 *     for its publisher instead of encoding the stage itself, so every checksum is encoded
 *     exactly once (also in single-wave launches).  Relies on the publishing tiles, which
 *     come first in the launch, being resident before the tiles that wait on them (in-order
 *     CTA dispatch); meant for testing the copy paths, not for production use.
 * All feed the same in-kernel carry (C^f) and fused epilogue verification.  FUSED and
 * FUSED_LOCAL produce bitwise-identical checksums (same integer encode of the same data);
 * PREPASS agrees within the threshold (its sums differ only in rounding).
 * Thread-local; returns 4 for an unknown mode. */
#define FTBLAS_ENCODE_FUSED 0
#define FTBLAS_ENCODE_PREPASS 1
#define FTBLAS_ENCODE_FUSED_LOCAL 2
#define FTBLAS_ENCODE_FUSED_WAIT 3
int ftblas_set_encode(int mode);

/* Verification interval Kc of ftblas_dgemm (§II.A,
 * 258 §V.A: verify after every Kc rank-1 updates, one correctable error per interval).
 * 0 (default) means Kc = k: one interval, verified in the epilogue before C is written.
 * With 0 < Kc < k the k-loop is split into T = ceil(k/Kc) intervals; the verification unit is
 * (tile, interval): each interval's increment A_{:,t} B_{t,:} is verified against its own
 * carried checksums (reading R18) and corrected before it is accumulated, and an injected
 * fault belongs to interval floor(step_q / Kc).  err->unit_k reports Kc and
 * err->units_checked counts tiles x intervals.  The increments go through library workspace
 * (interval groups sized to half the free device memory) and a deterministic reduction
 * forms C = alpha * sum_t inc_t + beta * C.  Kc must be a multiple of step_quantum (16);
 * returns 4 otherwise.  Thread-local. */
int ftblas_set_interval(int64_t kc);

/* Verification-unit geometry the kernels use: BM x BN tiles, step quantum BK. */
int ftblas_get_geometry(int32_t *unit_rows, int32_t *unit_cols, int32_t *step_quantum);

/* ---------------------------------------------------------------------------------------
 * Level-1/2 BLAS with dual modular redundancy (DMR; PAPER.md:198-252
 * §IV, 440 §VI.B).  Memory-bound routines are protected by duplicating every computing
 * instruction, not the loads (the paper's sphere of replication): each result
 * is computed twice from the same registers, the two are compared bitwise (a warp vote
 * reduces the verdict), and only verified results are stored (verify-before-store).  On a
 * mismatch a third computation settles it: agreeing with either copy -> corrected, else
 * uncorrectable (the third value is stored and counted).  An armed fault (ftblas_inject_arm)
 * with row index i perturbs the ORIGINAL computation of output i by delta: for DSCAL / DAXPY
 * after the multiply-add, for DGEMV after `step` terms of the dot product (0 <= step <= the
 * dot length); j is ignored.  A fault whose delta does not change the (rounded) original
 * result is not a detection.  Arguments as reference BLAS (x[i*incx] for incx > 0,
 * x[(n-1-i)*|incx|] for incx < 0; incx == 0 is invalid), device pointers, stream-ordered;
 * the call synchronises only when rep != NULL (to fill it).  Status codes as above, with
 * argument positions counted in each function's own list.
 * --------------------------------------------------------------------------------------- */
typedef struct {
  int64_t checked;        /* out: results verified (output elements) */
  int64_t detected;       /* out: results whose two computations disagreed */
  int64_t corrected;      /* out: settled by a third computation agreeing with one copy */
  int64_t uncorrectable;  /* out: all three computations disagreed */
} ftblas_dmr_report_t;

/* x := alpha * x (one rounding per element; PAPER.md:208 DSCAL). */
int ftblas_dscal(int64_t n, double alpha, double *x, int64_t incx, ftblas_dmr_report_t *rep);
/* y := alpha * x + y, computed as fma(alpha, x_i, y_i) (one rounding). */
int ftblas_daxpy(int64_t n, double alpha, const double *x, int64_t incx, double *y, int64_t incy,
                 ftblas_dmr_report_t *rep);
/* y := alpha * op(A) * x + beta * y, A m x n column-major.  Each output is one dot product
 * acc = sum_p fma(op(A)_ip, x_p, acc), p ascending (trans 'N': one thread per row, the exact
 * oracle order; 'T': a warp per column, lane-strided partial sums reduced by a fixed
 * butterfly), then y_i = fma(alpha, acc, beta * y_i) (beta == 0: y not read). */
int ftblas_dgemv(char trans, int64_t m, int64_t n, double alpha, const double *A, int64_t lda,
                 const double *x, int64_t incx, double beta, double *y, int64_t incy,
                 ftblas_dmr_report_t *rep);
/* Unprotected twins (same kernels without duplication): the overhead baselines. */
int ftblas_dscal_noft(int64_t n, double alpha, double *x, int64_t incx);
int ftblas_daxpy_noft(int64_t n, double alpha, const double *x, int64_t incx, double *y, int64_t incy);
int ftblas_dgemv_noft(char trans, int64_t m, int64_t n, double alpha, const double *A, int64_t lda,
                      const double *x, int64_t incx, double beta, double *y, int64_t incy);

/* ---------------------------------------------------------------------------------------
 * FT-DTRSM (§III.C.3, 440, 476): in place (B := X),
 *   side 'L': op(A) X = alpha B (the paper's B = alpha op(A)^-1 B), A m x m;
 *   side 'R': X op(A) = alpha B (B = alpha B op(A)^-1), A n x n;
 * uplo 'L'/'U', transa 'N'/'T'/'C', diag 'N'/'U' (unit diagonal: not read); B m x n; device
 * pointers, column-major.  Recursive blocked algorithm along the solve (B's rows for side L,
 * its columns for side R): a block of len > 128 positions (in substitution order) is split
 * into its first len - u positions, solved first, and its last u positions, updated by the
 * coupling GEMM and then solved: u = 254 j with j = floor((len + 254) / 508) reduced until
 * u < len, or u = 126 when j = 0 (whole 127-row tiles of the protected kernel, even block
 * boundaries); diagonal blocks of <= 128 are solved by
 * a DMR kernel that multiplies by packed reciprocals of the diagonal, the
 * coupling updates (B2 -= op(A)21 X1, or B2 -= X1 op(A)12 on the right) run on the protected
 * DMMA kernel (fused ABFT, this library's ftblas_dgemm path).  err (nullable) sums both: the
 * ABFT units / events of the GEMM updates (event indices global) plus the DMR detections of
 * the diagonal solves (detected/corrected; uncorrectable ones are counted in `recomputed`).
 * An armed fault (i, j, step = p) perturbs the update of B(i, j) by X(p, j) (side L; p must
 * precede i in the substitution order: p < i when op(A) is lower, p > i when upper) or by
 * X(i, p) (side R; p must precede j: p < j when op(A) is upper, p > j when lower); status 3
 * otherwise.  Status codes as ftblas_dgemm with positions in this list. */
int ftblas_dtrsm(char side, char uplo, char transa, char diag, int64_t m, int64_t n, double alpha,
                 const double *A, int64_t lda, double *B, int64_t ldb, ftblas_err_report_t *err);
int ftblas_dtrsm_noft(char side, char uplo, char transa, char diag, int64_t m, int64_t n, double alpha,
                      const double *A, int64_t lda, double *B, int64_t ldb);

/* Number of kernel launches enqueued by this thread since the last call (for the
 * benchmark's launch accounting); resets the counter. */
int64_t ftblas_take_launch_count(void);

const char *ftblas_status_string(int status);

/* Free per-device scratch on every device touched.  Not safe while calls are in flight. */
int ftblas_finalize(void);

#ifdef __cplusplus
}
#endif

#endif /* FTBLAS_H */
