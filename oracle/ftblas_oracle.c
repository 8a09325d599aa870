/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU implementation of online ABFT DGEMM as
 * described in FT-BLAS (arXiv 2104.00897).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load this library.
 * It shares no code, header, table or helper with the CUDA path
 * (paper_2104_00897_b200/csrc); neither side includes or links the other.
 *
 * Arithmetic: IEEE fp64, round-to-nearest, compiled WITHOUT -ffast-math and with
 * -ffp-contract=off so every `x*y + z` below is two roundings, exactly as written.
 *
 * What it computes (citations are PAPER.md line numbers and sections):
 *   - Checksum encoding A^c = [A; e^T A], B^r = [B, B e]        PAPER.md:90 §II.A
 *   - Outer-product maintenance C^f = sum_s A^c(:,s) B^r(s,:)   PAPER.md:93-95 §II.A
 *     restricted to one verification unit (row block I, column block J,
 *     k-interval of length Kc): the carried checksums are (e^T A_I) B_J and A_I (B_J e).
 *   - Reference checksums from the computed C, compare, locate    PAPER.md:258 §V.A
 *   - One error per verification interval, no checkpoint/rollback PAPER.md:95 §II.A
 *   - Correction ("subtracting the error magnitude from the erroneous position")
 *     PAPER.md:445 §VI.C is the optional `subtract` mode; the default `recompute`
 *     mode restores C_ij from a fresh dot product (reading R4).
 *   - Detection threshold: the paper says only "round-off threshold"
 *     (PAPER.md:91); the reading used is the rigorous per-unit bound R1:
 *       tau_col = 2*gamma(kt+bm)*kt*bm*amax*bmax,  tau_row = 2*gamma(kt+bn)*kt*bn*amax*bmax
 *     with gamma(n) = n*u/(1-n*u), u = 2^-53, kt = k accumulated so far, and amax / bmax
 *     the largest |op(A)_ip| / |op(B)_pj| of the unit read so far (exact maxima; a NaN
 *     element is ignored by the max, an infinite one makes it infinite).  tau is then
 *     clamped to the largest finite double (reading R13: non-finite inputs), so a
 *     residual that is NaN or infinite always flags.
 *   - Multi-flag units (out of the paper's one-error model) are recomputed once
 *     without re-verification (reading R6/R13).
 *   - Injected faults: acc_ij += delta after step_q rank-1 updates, with
 *     step_q = floor(step/BK)*BK (reading R8; "an element of matrix C
 *     is randomly selected for modification when an injection point is reached").
 *
 * Parity pins: tests/test_oracle.py (run with -m "not gpu").
 */
#include <float.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

/* lane 0: the data accumulator C_ij; 1: the carried column checksum ((e^T A_I) B_J)_j of the
 * unit containing (i, j); 2: its carried row checksum (A_I (B_J e))_i (reading R6: a fault in a
 * checksum lane). */
typedef struct { int64_t i, j, step; double delta; int64_t lane; } or_fault_t;
typedef struct {
  int64_t i, j;
  int32_t kind;      /* 1 = corrected at (i,j); 2 = recomputed unit with origin (i,j) */
  int32_t interval;  /* verification interval index t */
  double residual_row, residual_col;
} or_event_t;

enum { OR_UNITS_CHECKED = 0, OR_DETECTED, OR_CORRECTED, OR_RECOMPUTED, OR_N_EVENTS, OR_NCOUNTERS };

static const double U = 0x1p-53; /* unit roundoff of binary64 */

/* gamma(n) = n u / (1 - n u)  (standard rounding-error constant; R1). */
double oracle_gamma(int64_t n) {
  double nu = (double)n * U;
  return nu / (1.0 - nu);
}

/* tau = 2 * gamma(kt + len) * kt * len * amax * bmax  (R1), evaluated
 * left to right exactly as written. */
double oracle_tau(int64_t kt, int64_t len, double amax, double bmax) {
  return 2.0 * oracle_gamma(kt + len) * (double)kt * (double)len * amax * bmax;
}

/* op(A)(r, c) for a column-major matrix with leading dimension ld;
 * trans 'N' reads M[r + c*ld], 'T'/'C' reads M[c + r*ld] (real data: C == T). */
static double op_at(const double *M, int64_t ld, int trans, int64_t r, int64_t c) {
  return trans ? M[c + r * ld] : M[r + c * ld];
}

static int is_trans(char t) { return t == 'T' || t == 't' || t == 'C' || t == 'c'; }

/* ---------------------------------------------------------------------------
 * Plain definitions used by the pins (each one a formula written out).
 * ------------------------------------------------------------------------- */

/* Column sums e^T M of an r x c column-major matrix (e^T A). */
void oracle_col_sums(int64_t r, int64_t c, const double *M, int64_t ld, double *out) {
  for (int64_t j = 0; j < c; ++j) {
    double s = 0.0;
    for (int64_t i = 0; i < r; ++i) s += M[i + j * ld];
    out[j] = s;
  }
}

/* Row sums M e of an r x c column-major matrix (B e). */
void oracle_row_sums(int64_t r, int64_t c, const double *M, int64_t ld, double *out) {
  for (int64_t i = 0; i < r; ++i) {
    double s = 0.0;
    for (int64_t j = 0; j < c; ++j) s += M[i + j * ld];
    out[i] = s;
  }
}

/* Plain product C = alpha*op(A)*op(B) + beta*C, triple loop, p ascending,
 * no ABFT (the DGEMM definition; PAPER.md:182 routine).  beta == 0: C0 not read. */
void oracle_gemm_plain(char ta, char tb, int64_t m, int64_t n, int64_t k, double alpha,
                       const double *A, int64_t lda, const double *B, int64_t ldb, double beta,
                       double *C, int64_t ldc) {
  int tA = is_trans(ta), tB = is_trans(tb);
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t j = 0; j < n; ++j) {
    for (int64_t i = 0; i < m; ++i) {
      double acc = 0.0;
      for (int64_t p = 0; p < k; ++p) acc += op_at(A, lda, tA, i, p) * op_at(B, ldb, tB, p, j);
      double out = alpha * acc;
      if (beta != 0.0) out = out + beta * C[i + j * ldc];
      C[i + j * ldc] = out;
    }
  }
}

/* Selected elements of the plain product: out[e] = alpha*sum_p opA(i,p)opB(p,j) + beta*C0[e]
 * (C0 given per element, ignored when beta == 0).  Used for sampled parity at full size. */
void oracle_gemm_elements(char ta, char tb, int64_t k, double alpha, const double *A, int64_t lda,
                          const double *B, int64_t ldb, double beta, int64_t ne, const int64_t *ii,
                          const int64_t *jj, const double *c0, double *out) {
  int tA = is_trans(ta), tB = is_trans(tb);
#pragma omp parallel for schedule(static)
  for (int64_t e = 0; e < ne; ++e) {
    double acc = 0.0;
    for (int64_t p = 0; p < k; ++p) acc += op_at(A, lda, tA, ii[e], p) * op_at(B, ldb, tB, p, jj[e]);
    double o = alpha * acc;
    if (beta != 0.0) o = o + beta * c0[e];
    out[e] = o;
  }
}

/* |C - C_ref| bound helper: S_ij = sum_p |opA(i,p)| |opB(p,j)| for selected elements. */
void oracle_abs_product_elements(char ta, char tb, int64_t k, const double *A, int64_t lda,
                                 const double *B, int64_t ldb, int64_t ne, const int64_t *ii,
                                 const int64_t *jj, double *out) {
  int tA = is_trans(ta), tB = is_trans(tb);
#pragma omp parallel for schedule(static)
  for (int64_t e = 0; e < ne; ++e) {
    double s = 0.0;
    for (int64_t p = 0; p < k; ++p)
      s += fabs(op_at(A, lda, tA, ii[e], p)) * fabs(op_at(B, ldb, tB, p, jj[e]));
    out[e] = s;
  }
}

/* ---------------------------------------------------------------------------
 * One verification unit: rows [i0, i0+bm), columns [j0, j0+bn), all intervals.
 * Follows PAPER.md:93-95 (outer-product maintenance) and 258 (verify/locate),
 * step by step, in the paper's order: for every rank-Kc step, update C, update
 * the checksums, then verify.
 * ------------------------------------------------------------------------- */
typedef struct {
  int tA, tB;
  int64_t k, Kc, BK;
  const double *A, *B;
  int64_t lda, ldb;
  int subtract_mode;
} unit_ctx_t;

typedef struct {
  int64_t detected, corrected, recomputed, checked;
} unit_counts_t;

/* Fresh dot product over p in [0, pe), p ascending. */
static double dot_upto(const unit_ctx_t *x, int64_t i, int64_t j, int64_t pe) {
  double s = 0.0;
  for (int64_t p = 0; p < pe; ++p) s += op_at(x->A, x->lda, x->tA, i, p) * op_at(x->B, x->ldb, x->tB, p, j);
  return s;
}

/* The unit's carried checksums recomputed from scratch over p in [0, pe), fault-free: the same
 * encode and outer-product maintenance as the main loop.  Used when a unit
 * is recomputed (reading R6): its whole C^f block -- data and checksums -- is formed afresh, so a
 * fault that sat in a checksum lane does not outlive the recompute. */
static void carry_fresh(const unit_ctx_t *x, int64_t i0, int64_t bm, int64_t j0, int64_t bn, int64_t pe,
                        double *cs_col, double *cs_row) {
  for (int64_t j = 0; j < bn; ++j) cs_col[j] = 0.0;
  for (int64_t i = 0; i < bm; ++i) cs_row[i] = 0.0;
  for (int64_t p = 0; p < pe; ++p) {
    double a_sum = 0.0, b_sum = 0.0;
    for (int64_t i = 0; i < bm; ++i) a_sum += op_at(x->A, x->lda, x->tA, i0 + i, p);
    for (int64_t j = 0; j < bn; ++j) b_sum += op_at(x->B, x->ldb, x->tB, p, j0 + j);
    for (int64_t j = 0; j < bn; ++j) cs_col[j] += a_sum * op_at(x->B, x->ldb, x->tB, p, j0 + j);
    for (int64_t i = 0; i < bm; ++i) cs_row[i] += op_at(x->A, x->lda, x->tA, i0 + i, p) * b_sum;
  }
}

static void apply_faults_at(double *acc, double *cs_col, double *cs_row, int64_t bm, int64_t i0, int64_t j0,
                            const or_fault_t *f, int64_t nf, int64_t BK, int64_t step_q_wanted) {
  for (int64_t e = 0; e < nf; ++e) {
    int64_t step_q = (f[e].step / BK) * BK; /* reading R8: quantised to BK */
    if (step_q != step_q_wanted) continue;
    if (f[e].lane == 1) cs_col[f[e].j - j0] += f[e].delta;
    else if (f[e].lane == 2) cs_row[f[e].i - i0] += f[e].delta;
    else acc[(f[e].i - i0) + (f[e].j - j0) * bm] += f[e].delta;
  }
}

/* Returns number of events written into ev (at most ev_cap). */
static int64_t verify_unit(const unit_ctx_t *x, int64_t i0, int64_t bm, int64_t j0, int64_t bn,
                           const or_fault_t *f, int64_t nf, double *acc /* bm*bn, out */,
                           or_event_t *ev, int64_t ev_cap, unit_counts_t *cnt) {
  const int64_t k = x->k, Kc = x->Kc;
  const int64_t T = (k + Kc - 1) / Kc;
  double *cs_col = calloc((size_t)bn, sizeof(double)); /* (e^T A_I) B_J, carried */
  double *cs_row = calloc((size_t)bm, sizeof(double)); /* A_I (B_J e), carried   */
  double *r_col = malloc((size_t)bn * sizeof(double));
  double *r_row = malloc((size_t)bm * sizeof(double));
  double *d_col = malloc((size_t)bn * sizeof(double));
  double *d_row = malloc((size_t)bm * sizeof(double));
  double amax = 0.0, bmax = 0.0;
  int64_t nev = 0;
  memset(acc, 0, (size_t)(bm * bn) * sizeof(double));

  for (int64_t t = 0; t < T; ++t) {
    const int64_t ps = t * Kc, pe = (ps + Kc < k) ? ps + Kc : k;
    for (int64_t p = ps; p < pe; ++p) {
      /* Injection point: faults whose quantised step equals p land before update p. */
      apply_faults_at(acc, cs_col, cs_row, bm, i0, j0, f, nf, x->BK, p);

      /* Encode: a_sum = sum_{i in I} opA(i,p)  (e^T A column p),
       *                       b_sum = sum_{j in J} opB(p,j)  (B e row p);
       * running maxima for the threshold (R1). */
      double a_sum = 0.0, b_sum = 0.0;
      for (int64_t i = 0; i < bm; ++i) {
        double a = op_at(x->A, x->lda, x->tA, i0 + i, p);
        a_sum += a;
        if (fabs(a) > amax) amax = fabs(a);
      }
      for (int64_t j = 0; j < bn; ++j) {
        double b = op_at(x->B, x->ldb, x->tB, p, j0 + j);
        b_sum += b;
        if (fabs(b) > bmax) bmax = fabs(b);
      }

      /* Rank-1 update of C (C_s = A(:,s) B(s,:)). */
      for (int64_t j = 0; j < bn; ++j) {
        double b = op_at(x->B, x->ldb, x->tB, p, j0 + j);
        for (int64_t i = 0; i < bm; ++i) acc[i + j * bm] += op_at(x->A, x->lda, x->tA, i0 + i, p) * b;
      }

      /* Checksum maintenance: C^c += (e^T A(:,p)) B(p,:),
       * C^r += A(:,p) (B(p,:) e). */
      for (int64_t j = 0; j < bn; ++j) cs_col[j] += a_sum * op_at(x->B, x->ldb, x->tB, p, j0 + j);
      for (int64_t i = 0; i < bm; ++i) cs_row[i] += op_at(x->A, x->lda, x->tA, i0 + i, p) * b_sum;
    }
    if (t == T - 1) apply_faults_at(acc, cs_col, cs_row, bm, i0, j0, f, nf, x->BK, k); /* step_q == k */

    /* Reference checksums from the computed C: r_col = e^T C_IJ, r_row = C_IJ e. */
    for (int64_t j = 0; j < bn; ++j) {
      double s = 0.0;
      for (int64_t i = 0; i < bm; ++i) s += acc[i + j * bm];
      r_col[j] = s;
    }
    for (int64_t i = 0; i < bm; ++i) {
      double s = 0.0;
      for (int64_t j = 0; j < bn; ++j) s += acc[i + j * bm];
      r_row[i] = s;
    }

    /* Compare against the maintained checksums; flag where not |d| <= tau (R1), tau clamped
     * to the largest finite double so that a NaN or infinite residual flags (R13). */
    double tau_col = oracle_tau(pe, bm, amax, bmax);
    double tau_row = oracle_tau(pe, bn, amax, bmax);
    if (!(tau_col <= DBL_MAX)) tau_col = DBL_MAX;
    if (!(tau_row <= DBL_MAX)) tau_row = DBL_MAX;
    int64_t nfr = 0, nfc = 0, fr = -1, fc = -1;
    for (int64_t i = 0; i < bm; ++i) {
      d_row[i] = r_row[i] - cs_row[i];
      if (!(fabs(d_row[i]) <= tau_row)) { if (fr < 0) fr = i; ++nfr; }
    }
    for (int64_t j = 0; j < bn; ++j) {
      d_col[j] = r_col[j] - cs_col[j];
      if (!(fabs(d_col[j]) <= tau_col)) { if (fc < 0) fc = j; ++nfc; }
    }
    cnt->checked += 1;
    if (nfr == 0 && nfc == 0) continue; /* clean */
    cnt->detected += 1;

    or_event_t e;
    e.interval = (int32_t)t;
    e.residual_row = fr >= 0 ? d_row[fr] : 0.0;
    e.residual_col = fc >= 0 ? d_col[fc] : 0.0;
    if (nfr == 1 && nfc == 1) {
      /* Locate: the single error sits at the intersection, correct it in place. */
      if (x->subtract_mode) acc[fr + fc * bm] -= d_col[fc];
      else acc[fr + fc * bm] = dot_upto(x, i0 + fr, j0 + fc, pe);     /* reading R4 */
      cnt->corrected += 1;
      e.kind = 1; e.i = i0 + fr; e.j = j0 + fc;
    } else {
      /* Out of the one-error model (R6): recompute the whole unit once, no re-verify of this
       * interval; its carried checksums are formed afresh too, so later intervals verify the
       * recomputed block. */
      for (int64_t j = 0; j < bn; ++j)
        for (int64_t i = 0; i < bm; ++i) acc[i + j * bm] = dot_upto(x, i0 + i, j0 + j, pe);
      if (t < T - 1) carry_fresh(x, i0, bm, j0, bn, pe, cs_col, cs_row);
      cnt->recomputed += 1;
      e.kind = 2; e.i = i0; e.j = j0;
    }
    if (nev < ev_cap) ev[nev] = e;
    ++nev;
  }
  free(cs_col); free(cs_row); free(r_col); free(r_row); free(d_col); free(d_row);
  return nev;
}

static int cmp_event(const void *a, const void *b) {
  const or_event_t *x = a, *y = b;
  if (x->interval != y->interval) return x->interval < y->interval ? -1 : 1;
  if (x->i != y->i) return x->i < y->i ? -1 : 1;
  if (x->j != y->j) return x->j < y->j ? -1 : 1;
  return 0;
}

/*
 * ABFT DGEMM over a set of units.  units == NULL means every unit (full oracle);
 * otherwise `units` lists (ti, tj) tile indices (2 entries per unit) and only
 * those units are computed and stored (sampled oracle at full size).
 *
 * C holds C0 on entry (read only when beta != 0) and C_out on exit for the
 * computed units.  counters[OR_NCOUNTERS] out.  events sorted by (interval, i, j).
 * Returns 0, or -1 on bad arguments.
 */
int oracle_dgemm_abft_units(char ta, char tb, int64_t m, int64_t n, int64_t k, double alpha,
                            const double *A, int64_t lda, const double *B, int64_t ldb, double beta,
                            double *C, int64_t ldc, int64_t BM, int64_t BN, int64_t BK, int64_t Kc,
                            int subtract_mode, const or_fault_t *faults, int64_t nfaults,
                            const int64_t *units, int64_t nunits, int64_t *counters,
                            or_event_t *events, int64_t events_cap) {
  for (int c = 0; c < OR_NCOUNTERS; ++c) counters[c] = 0;
  if (m < 0 || n < 0 || k < 0 || BM <= 0 || BN <= 0 || BK <= 0) return -1;
  if (Kc <= 0 || Kc > k) Kc = k;
  if (m == 0 || n == 0) return 0;
  /* alpha == 0 or k == 0: C = beta*C with no ABFT (BLAS semantics). */
  if (alpha == 0.0 || k == 0) {
    if (beta == 1.0) return 0;
    for (int64_t j = 0; j < n; ++j)
      for (int64_t i = 0; i < m; ++i) C[i + j * ldc] = (beta == 0.0) ? 0.0 : beta * C[i + j * ldc];
    return 0;
  }
  const int64_t tm = (m + BM - 1) / BM, tn = (n + BN - 1) / BN;
  const int64_t nu = units ? nunits : tm * tn;
  unit_ctx_t x = {is_trans(ta), is_trans(tb), k, Kc, BK, A, B, lda, ldb, subtract_mode};

  int64_t det = 0, cor = 0, rec = 0, chk = 0, nev_total = 0;
  int64_t ev_used = 0;

#pragma omp parallel for schedule(dynamic, 1) reduction(+ : det, cor, rec, chk)
  for (int64_t u = 0; u < nu; ++u) {
    int64_t ti = units ? units[2 * u] : u % tm;
    int64_t tj = units ? units[2 * u + 1] : u / tm;
    int64_t i0 = ti * BM, j0 = tj * BN;
    int64_t bm = (i0 + BM <= m) ? BM : m - i0;
    int64_t bn = (j0 + BN <= n) ? BN : n - j0;
    /* Faults that fall in this unit (list order preserved). */
    or_fault_t *uf = malloc((size_t)(nfaults > 0 ? nfaults : 1) * sizeof(or_fault_t));
    int64_t nf = 0;
    for (int64_t e = 0; e < nfaults; ++e)
      if (faults[e].i >= i0 && faults[e].i < i0 + bm && faults[e].j >= j0 && faults[e].j < j0 + bn)
        uf[nf++] = faults[e];
    double *acc = malloc((size_t)(bm * bn) * sizeof(double));
    int64_t T = (k + Kc - 1) / Kc;
    or_event_t *ev = malloc((size_t)T * sizeof(or_event_t));
    unit_counts_t cnt = {0, 0, 0, 0};
    int64_t nev = verify_unit(&x, i0, bm, j0, bn, uf, nf, acc, ev, T, &cnt);
    det += cnt.detected; cor += cnt.corrected; rec += cnt.recomputed; chk += cnt.checked;

    /* Output: C = alpha*acc + beta*C0; C0 not read when beta == 0. */
    for (int64_t j = 0; j < bn; ++j)
      for (int64_t i = 0; i < bm; ++i) {
        double o = alpha * acc[i + j * bm];
        if (beta != 0.0) o = o + beta * C[(i0 + i) + (j0 + j) * ldc];
        C[(i0 + i) + (j0 + j) * ldc] = o;
      }
#pragma omp critical
    {
      for (int64_t e = 0; e < nev; ++e) {
        if (ev_used < events_cap) events[ev_used++] = ev[e];
      }
      nev_total += nev;
    }
    free(uf); free(acc); free(ev);
  }
  if (ev_used > 1) qsort(events, (size_t)ev_used, sizeof(or_event_t), cmp_event);
  counters[OR_UNITS_CHECKED] = chk;
  counters[OR_DETECTED] = det;
  counters[OR_CORRECTED] = cor;
  counters[OR_RECOMPUTED] = rec;
  counters[OR_N_EVENTS] = nev_total;
  return 0;
}

/* ---------------------------------------------------------------------------
 * Level-1/2 routines with dual modular redundancy (
 * PAPER.md:198-252 §IV).  Plain definitions plus the DMR bookkeeping: an injected
 * fault perturbs the ORIGINAL computation of one output (PAPER.md:445 injection),
 * the duplicate is fault-free, the mismatch is detected and a third fault-free
 * computation is stored (corrected).  So every output equals its fault-free value;
 * counters = {checked, detected, corrected, uncorrectable}.  For DSCAL / DAXPY an
 * output is detected iff fl(v + D) differs from v bitwise, D the sum of its faults'
 * deltas in list order; for DGEMV iff D != 0 (reading R19: a delta injected inside a
 * dot product is assumed not to be absorbed by rounding).
 * Vectors: element i at v[i*inc] for inc > 0, v[(n-1-i)*(-inc)] for inc < 0.
 * ------------------------------------------------------------------------- */
static int64_t vix(int64_t i, int64_t n, int64_t inc) { return inc > 0 ? i * inc : (n - 1 - i) * (-inc); }

static double fault_sum(const or_fault_t *f, int64_t nf, int64_t index) {
  double d = 0.0;
  for (int64_t e = 0; e < nf; ++e)
    if (f[e].i == index) d += f[e].delta;
  return d;
}

static int fault_any(const or_fault_t *f, int64_t nf, int64_t index) {
  for (int64_t e = 0; e < nf; ++e)
    if (f[e].i == index && f[e].delta != 0.0) return 1;
  return 0;
}

static int bits_differ(double a, double b) {
  uint64_t x, y;
  memcpy(&x, &a, sizeof x);
  memcpy(&y, &b, sizeof y);
  return x != y;
}

/* x := alpha * x  (DSCAL). */
void oracle_dscal(int64_t n, double alpha, double *x, int64_t incx, const or_fault_t *f, int64_t nf,
                  int64_t *counters) {
  int64_t det = 0;
  for (int64_t i = 0; i < n; ++i) {
    double v = alpha * x[vix(i, n, incx)];
    double d = fault_sum(f, nf, i);
    if (d != 0.0 && bits_differ(v + d, v)) ++det;
    x[vix(i, n, incx)] = v;
  }
  counters[0] = n; counters[1] = det; counters[2] = det; counters[3] = 0;
}

/* y := alpha * x + y as one fused multiply-add per element (DAXPY). */
void oracle_daxpy(int64_t n, double alpha, const double *x, int64_t incx, double *y, int64_t incy,
                  const or_fault_t *f, int64_t nf, int64_t *counters) {
  int64_t det = 0;
  for (int64_t i = 0; i < n; ++i) {
    double v = fma(alpha, x[vix(i, n, incx)], y[vix(i, n, incy)]);
    double d = fault_sum(f, nf, i);
    if (d != 0.0 && bits_differ(v + d, v)) ++det;
    y[vix(i, n, incy)] = v;
  }
  counters[0] = n; counters[1] = det; counters[2] = det; counters[3] = 0;
}

/* y := alpha * op(A) * x + beta * y  (DGEMV): acc = sum_p op(A)_ip x_p as an fma chain,
 * p ascending; y_i = fma(alpha, acc, beta * y_i), beta == 0: y not read. */
void oracle_dgemv(char trans, int64_t m, int64_t n, double alpha, const double *A, int64_t lda,
                  const double *x, int64_t incx, double beta, double *y, int64_t incy,
                  const or_fault_t *f, int64_t nf, int64_t *counters) {
  int tr = is_trans(trans);
  int64_t nout = tr ? n : m, len = tr ? m : n, det = 0;
  for (int64_t i = 0; i < nout; ++i) {
    double acc = 0.0;
    if (alpha != 0.0)
      for (int64_t p = 0; p < len; ++p) acc = fma(tr ? A[p + i * lda] : A[i + p * lda], x[vix(p, len, incx)], acc);
    double yb = beta != 0.0 ? beta * y[vix(i, nout, incy)] : 0.0;
    y[vix(i, nout, incy)] = fma(alpha, acc, yb);
    if (fault_any(f, nf, i)) ++det;
  }
  counters[0] = nout; counters[1] = det; counters[2] = det; counters[3] = 0;
}

/* ---------------------------------------------------------------------------
 * DTRSM: op(A) X = alpha B, side 'L', in place,
 * plain column-by-column substitution: forward when op(A) is lower, backward when upper;
 * x_i = (alpha b_i - sum_p op(A)_ip x_p) computed as an fma chain over p in substitution order,
 * then multiplied by the reciprocal 1/op(A)_ii (the paper's packed reciprocal diagonal; unit
 * diagonal: no multiply).  Faults are corrected by the protection (ABFT on the updates, DMR on
 * the diagonal solves), so X is the fault-free solution; which protection reports what is
 * oracle_dtrsm_bookkeeping's (reading R21).
 * ------------------------------------------------------------------------- */
void oracle_dtrsm(char uplo, char transa, char diag, int64_t m, int64_t n, double alpha, const double *A,
                  int64_t lda, double *B, int64_t ldb, int64_t nfaults, int64_t *counters) {
  int lower = (uplo == 'L' || uplo == 'l'), tr = is_trans(transa), unit = (diag == 'U' || diag == 'u');
  int fwd = lower != tr;
#pragma omp parallel for schedule(static)
  for (int64_t j = 0; j < n; ++j) {
    double *b = B + j * ldb;
    for (int64_t i = 0; i < m; ++i) b[i] = alpha * b[i];
    for (int64_t s = 0; s < m; ++s) {
      int64_t i = fwd ? s : m - 1 - s;
      double v = b[i];
      if (!unit) v = v * (1.0 / (tr ? A[i + i * lda] : A[i + i * lda]));
      b[i] = v;
      /* eliminate x_i from the remaining rows */
      if (fwd) {
        for (int64_t p = i + 1; p < m; ++p) b[p] = fma(-(tr ? A[i + p * lda] : A[p + i * lda]), v, b[p]);
      } else {
        for (int64_t p = 0; p < i; ++p) b[p] = fma(-(tr ? A[i + p * lda] : A[p + i * lda]), v, b[p]);
      }
    }
  }
  (void)nfaults; /* the FT bookkeeping is oracle_dtrsm_bookkeeping's */
  counters[0] = counters[1] = counters[2] = counters[3] = 0;
}

/* DTRSM side 'R' (B = alpha B op(A)^-1): X op(A) = alpha B, op(A) n x n, in place,
 * row by row: each row x of X solves x op(A) = alpha b by substitution over the columns of
 * op(A) -- forward (j ascending) when op(A) is upper, backward when lower: x_j = b_j * (1 /
 * op(A)_jj), then b_q -= op(A)_jq x_j for the columns q still to solve (fma, substitution
 * order).  Faults are corrected by the protection, as on the left (reading R21; bookkeeping:
 * oracle_dtrsm_bookkeeping). */
void oracle_dtrsm_right(char uplo, char transa, char diag, int64_t m, int64_t n, double alpha, const double *A,
                        int64_t lda, double *B, int64_t ldb, int64_t nfaults, int64_t *counters) {
  int lower = (uplo == 'L' || uplo == 'l'), tr = is_trans(transa), unit = (diag == 'U' || diag == 'u');
  int fwd = lower == tr; /* op(A) upper -> columns ascending */
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < m; ++r) {
    for (int64_t q = 0; q < n; ++q) B[r + q * ldb] = alpha * B[r + q * ldb];
    for (int64_t s = 0; s < n; ++s) {
      int64_t j = fwd ? s : n - 1 - s;
      double v = B[r + j * ldb];
      if (!unit) v = v * (1.0 / A[j + j * lda]);
      B[r + j * ldb] = v;
      if (fwd) {
        for (int64_t q = j + 1; q < n; ++q) B[r + q * ldb] = fma(-(tr ? A[q + j * lda] : A[j + q * lda]), v, B[r + q * ldb]);
      } else {
        for (int64_t q = 0; q < j; ++q) B[r + q * ldb] = fma(-(tr ? A[q + j * lda] : A[j + q * lda]), v, B[r + q * ldb]);
      }
    }
  }
  (void)nfaults; /* the FT bookkeeping is oracle_dtrsm_bookkeeping's */
  counters[0] = counters[1] = counters[2] = counters[3] = 0;
}

/* ---------------------------------------------------------------------------
 * FT-DTRSM bookkeeping (§III.C.3, 476; reading
 * R21): which protection sees each injected fault, and what it reports.  The blocked solve
 * is the recursion include/ftblas.h documents, written out with its two parameters: the
 * diagonal-block size `leaf` and the GEMM unit size `tm` (blocks of len > leaf positions
 * split off u = 2 tm j positions, j = floor((len + 2 tm) / (4 tm)) reduced until u < len, or
 * u = tm - 1 when j = 0; the part solved first comes first in substitution order).
 *   - A fault (i, j, step p) whose element e (side L: row i; side R: column j) and step p fall
 *     in one diagonal block is seen by that block's DMR solve: one detection and correction per
 *     (block, right-hand side) holding faults, no event (DMR).
 *   - Otherwise it lands in the unique coupling GEMM update whose rows hold e and whose k
 *     range holds p: an ABFT unit (tm x tm, in the update's own coordinates) with one distinct
 *     faulty cell is corrected (event at the global (i, j)); with more cells it is recomputed
 *     (event at the unit's global origin), as in oracle_dgemm_abft (R6).
 *   - units_checked counts the units of every update.
 * counters[5] = {units_checked, detected, corrected, recomputed, n_events}; events sorted by
 * (interval = 0, i, j).  Faults: (i, j, step) triples, n_rhs = m for side R, n for side L. */
typedef struct {
  int right, fwd;
  int64_t leaf, tm, nrhs;
  const or_fault_t *f;
  int64_t nf;
  int64_t cnt[5];
  or_event_t *ev;
  int64_t ev_cap;
} bk_ctx_t;

static int64_t bk_elem(const bk_ctx_t *c, const or_fault_t *f) { return c->right ? f->j : f->i; }
static int64_t bk_rhs(const bk_ctx_t *c, const or_fault_t *f) { return c->right ? f->i : f->j; }

static void bk_event(bk_ctx_t *c, int64_t i, int64_t j, int kind) {
  if (c->cnt[4] < c->ev_cap) {
    or_event_t e = {i, j, kind, 0, 0.0, 0.0};
    c->ev[c->cnt[4]] = e;
  }
  c->cnt[4] += 1;
}

static void bk_leaf(bk_ctx_t *c, int64_t r0, int64_t len) {
  /* one detection per right-hand side with a fault inside this diagonal block */
  for (int64_t rhs = 0; rhs < c->nrhs; ++rhs) {
    int hit = 0;
    for (int64_t e = 0; e < c->nf && !hit; ++e) {
      const int64_t el = bk_elem(c, &c->f[e]);
      hit = bk_rhs(c, &c->f[e]) == rhs && el >= r0 && el < r0 + len && c->f[e].step >= r0 && c->f[e].step < r0 + len;
    }
    if (hit) { c->cnt[1] += 1; c->cnt[2] += 1; }
  }
}

static void bk_gemm(bk_ctx_t *c, int64_t R0, int64_t mr, int64_t K0, int64_t mk) {
  /* update rows (side L) / columns (side R) [R0, R0+mr), k range [K0, K0+mk) */
  const int64_t rows = c->right ? c->nrhs : mr, cols = c->right ? mr : c->nrhs;
  const int64_t tmr = (rows + c->tm - 1) / c->tm, tnc = (cols + c->tm - 1) / c->tm;
  c->cnt[0] += tmr * tnc;
  for (int64_t u = 0; u < tmr * tnc; ++u) {
    const int64_t ti = u % tmr, tj = u / tmr;
    int64_t ncell = 0, ci = -1, cj = -1;
    for (int64_t e = 0; e < c->nf; ++e) {
      const or_fault_t *f = &c->f[e];
      const int64_t el = bk_elem(c, f);
      if (!(el >= R0 && el < R0 + mr && f->step >= K0 && f->step < K0 + mk)) continue;
      const int64_t li = c->right ? f->i : el - R0, lj = c->right ? el - R0 : f->j;  /* update coordinates */
      if (li / c->tm != ti || lj / c->tm != tj) continue;
      if (ncell == 0) { ci = f->i; cj = f->j; ncell = 1; }
      else if (f->i != ci || f->j != cj) ncell = 2;
    }
    if (ncell == 0) continue;
    c->cnt[1] += 1;
    if (ncell == 1) { c->cnt[2] += 1; bk_event(c, ci, cj, 1); }
    else {
      c->cnt[3] += 1;
      bk_event(c, c->right ? ti * c->tm : R0 + ti * c->tm, c->right ? R0 + tj * c->tm : tj * c->tm, 2);
    }
  }
}

static void bk_rec(bk_ctx_t *c, int64_t r0, int64_t len) {
  if (len <= c->leaf) { bk_leaf(c, r0, len); return; }
  int64_t j = (len + 2 * c->tm) / (4 * c->tm);
  while (j > 0 && 2 * c->tm * j >= len) --j;
  const int64_t u = j > 0 ? 2 * c->tm * j : c->tm - 1;
  const int64_t m1 = c->fwd ? len - u : u, m2 = len - m1;
  if (c->fwd) {
    bk_rec(c, r0, m1);
    bk_gemm(c, r0 + m1, m2, r0, m1);
    bk_rec(c, r0 + m1, m2);
  } else {
    bk_rec(c, r0 + m1, m2);
    bk_gemm(c, r0, m1, r0 + m1, m2);
    bk_rec(c, r0, m1);
  }
}

int oracle_dtrsm_bookkeeping(char side, char uplo, char transa, int64_t m, int64_t n, int64_t leaf, int64_t tm,
                             const or_fault_t *faults, int64_t nfaults, int64_t *counters, or_event_t *events,
                             int64_t events_cap) {
  const int right = (side == 'R' || side == 'r'), lower = (uplo == 'L' || uplo == 'l'), tr = is_trans(transa);
  bk_ctx_t c;
  memset(&c, 0, sizeof c);
  c.right = right;
  c.fwd = right ? (lower == tr) : (lower != tr); /* substitution order (ascending when fwd) */
  c.leaf = leaf; c.tm = tm; c.nrhs = right ? m : n;
  c.f = faults; c.nf = nfaults; c.ev = events; c.ev_cap = events_cap;
  if (leaf <= 0 || tm <= 1) return -1;
  if (m > 0 && n > 0) bk_rec(&c, 0, right ? n : m);
  const int64_t ns = c.cnt[4] < events_cap ? c.cnt[4] : events_cap;
  if (ns > 1) qsort(events, (size_t)ns, sizeof(or_event_t), cmp_event);
  for (int q = 0; q < 5; ++q) counters[q] = c.cnt[q];
  return 0;
}

int oracle_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
