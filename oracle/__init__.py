"""ORACLE — TEST INFRASTRUCTURE ONLY.

ctypes front end of ``oracle/ftblas_oracle.c``: a plain, slow CPU implementation of
online ABFT DGEMM (FT-BLAS, arXiv 2104.00897, §II.A, 258 §V.A,
445 §VI.C).  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  It shares no
code with the CUDA path and never imports ``paper_2104_00897_b200``.

Matrices are numpy float64 arrays in column-major (Fortran) order, addressed BLAS
style: element (r, c) of a matrix with leading dimension ``ld`` sits at flat index
``r + c*ld``.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ftblas_oracle.c")
# ORACLE_SANITIZE=1 (tests/test_sanitize.py): the same source under AddressSanitizer and
# UndefinedBehaviorSanitizer, errors fatal; the process must preload libasan.
_SANITIZE = os.environ.get("ORACLE_SANITIZE") == "1"
_LIB = os.path.join(_HERE, "liboracle_san.so" if _SANITIZE else "liboracle.so")

CFLAGS = ["-O2", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", "-std=c11"]
SAN_CFLAGS = ["-g", "-fsanitize=address", "-fsanitize=undefined", "-fno-sanitize-recover=all",
              "-fno-omit-frame-pointer"]


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (no -ffast-math, no FP contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        extra = SAN_CFLAGS if _SANITIZE else []
        subprocess.check_call(["gcc", *CFLAGS, *extra, "-o", _LIB, _SRC, "-lm"])
    return _LIB


class _Fault(ctypes.Structure):
    _fields_ = [("i", ctypes.c_int64), ("j", ctypes.c_int64), ("step", ctypes.c_int64),
                ("delta", ctypes.c_double), ("lane", ctypes.c_int64)]


class _Event(ctypes.Structure):
    _fields_ = [("i", ctypes.c_int64), ("j", ctypes.c_int64), ("kind", ctypes.c_int32),
                ("interval", ctypes.c_int32), ("residual_row", ctypes.c_double),
                ("residual_col", ctypes.c_double)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        d, i64, c = ctypes.c_double, ctypes.c_int64, ctypes.c_char
        P = ctypes.c_void_p
        L.oracle_gamma.restype = d
        L.oracle_gamma.argtypes = [i64]
        L.oracle_tau.restype = d
        L.oracle_tau.argtypes = [i64, i64, d, d]
        L.oracle_col_sums.argtypes = [i64, i64, P, i64, P]
        L.oracle_row_sums.argtypes = [i64, i64, P, i64, P]
        L.oracle_gemm_plain.argtypes = [c, c, i64, i64, i64, d, P, i64, P, i64, d, P, i64]
        L.oracle_gemm_elements.argtypes = [c, c, i64, d, P, i64, P, i64, d, i64, P, P, P, P]
        L.oracle_abs_product_elements.argtypes = [c, c, i64, P, i64, P, i64, i64, P, P, P]
        L.oracle_dgemm_abft_units.restype = ctypes.c_int
        L.oracle_dgemm_abft_units.argtypes = [c, c, i64, i64, i64, d, P, i64, P, i64, d, P, i64,
                                              i64, i64, i64, i64, ctypes.c_int, P, i64, P, i64,
                                              P, P, i64]
        L.oracle_num_threads.restype = ctypes.c_int
        L.oracle_dscal.argtypes = [i64, d, P, i64, P, i64, P]
        L.oracle_daxpy.argtypes = [i64, d, P, i64, P, i64, P, i64, P]
        L.oracle_dgemv.argtypes = [c, i64, i64, d, P, i64, P, i64, d, P, i64, P, i64, P]
        L.oracle_dtrsm.argtypes = [c, c, c, i64, i64, d, P, i64, P, i64, i64, P]
        L.oracle_dtrsm_right.argtypes = [c, c, c, i64, i64, d, P, i64, P, i64, i64, P]
        L.oracle_dtrsm_bookkeeping.restype = ctypes.c_int
        L.oracle_dtrsm_bookkeeping.argtypes = [c, c, c, i64, i64, i64, i64, P, i64, P, P, i64]
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    assert a.dtype == np.float64 or a.dtype == np.int64
    return a.ctypes.data_as(ctypes.c_void_p)


def _flat(a: np.ndarray) -> np.ndarray:
    """Column-major flat view (no copy if already Fortran-contiguous)."""
    a = np.asarray(a, dtype=np.float64)
    if a.ndim == 2:
        a = np.asfortranarray(a).reshape(-1, order="F")
    return np.ascontiguousarray(a)


def gamma(n: int) -> float:
    return lib().oracle_gamma(n)


def tau(kt: int, length: int, amax: float, bmax: float) -> float:
    return lib().oracle_tau(kt, length, amax, bmax)


def col_sums(M: np.ndarray) -> np.ndarray:
    M = np.asfortranarray(M, dtype=np.float64)
    r, c = M.shape
    out = np.zeros(c)
    lib().oracle_col_sums(r, c, _ptr(_flat(M)), max(r, 1), _ptr(out))
    return out


def row_sums(M: np.ndarray) -> np.ndarray:
    M = np.asfortranarray(M, dtype=np.float64)
    r, c = M.shape
    out = np.zeros(r)
    lib().oracle_row_sums(r, c, _ptr(_flat(M)), max(r, 1), _ptr(out))
    return out


def gemm_plain(ta, tb, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc) -> np.ndarray:
    """Plain triple-loop DGEMM; returns a new flat C (input C is not modified)."""
    A, B = _flat(A), _flat(B)
    Cout = _flat(C).copy()
    lib().oracle_gemm_plain(ta.encode(), tb.encode(), m, n, k, alpha, _ptr(A), lda, _ptr(B), ldb,
                            beta, _ptr(Cout), ldc)
    return Cout


def gemm_elements(ta, tb, k, alpha, A, lda, B, ldb, beta, ii, jj, c0=None) -> np.ndarray:
    A, B = _flat(A), _flat(B)
    ii = np.ascontiguousarray(ii, dtype=np.int64)
    jj = np.ascontiguousarray(jj, dtype=np.int64)
    c0 = np.zeros(len(ii)) if c0 is None else np.ascontiguousarray(c0, dtype=np.float64)
    out = np.zeros(len(ii))
    lib().oracle_gemm_elements(ta.encode(), tb.encode(), k, alpha, _ptr(A), lda, _ptr(B), ldb,
                               beta, len(ii), _ptr(ii), _ptr(jj), _ptr(c0), _ptr(out))
    return out


def abs_product_elements(ta, tb, k, A, lda, B, ldb, ii, jj) -> np.ndarray:
    """S_ij = sum_p |opA(i,p)||opB(p,j)| for the parity bound."""
    A, B = _flat(A), _flat(B)
    ii = np.ascontiguousarray(ii, dtype=np.int64)
    jj = np.ascontiguousarray(jj, dtype=np.int64)
    out = np.zeros(len(ii))
    lib().oracle_abs_product_elements(ta.encode(), tb.encode(), k, _ptr(A), lda, _ptr(B), ldb,
                                      len(ii), _ptr(ii), _ptr(jj), _ptr(out))
    return out


@dataclass
class Report:
    units_checked: int
    detected: int
    corrected: int
    recomputed: int
    n_events: int
    events: list  # tuples (interval, i, j, kind, residual_row, residual_col), sorted


def dgemm_abft(ta, tb, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, *, BM, BN, BK, Kc=None,
               faults=(), units=None, subtract=False, events_cap=None):
    """Online ABFT DGEMM oracle.

    ``faults``: iterable of (i, j, step, delta) or (i, j, step, delta, lane): lane 0 the data
    accumulator, 1 the column checksum of column j, 2 the row checksum of row i (reading R6).  ``units``: optional list of (ti, tj)
    tile indices (sampled oracle); C entries outside those units are returned unchanged.
    Returns (C_out_flat, Report).
    """
    A, B = _flat(A), _flat(B)
    Cout = _flat(C).copy()
    faults = list(faults)
    fa = (_Fault * max(len(faults), 1))()
    for e, f in enumerate(faults):
        fa[e] = _Fault(int(f[0]), int(f[1]), int(f[2]), float(f[3]), int(f[4]) if len(f) > 4 else 0)
    if units is not None:
        ua = np.ascontiguousarray(np.asarray(units, dtype=np.int64).reshape(-1))
        uptr, nu = _ptr(ua), len(ua) // 2
    else:
        uptr, nu = None, 0
    if Kc is None or Kc <= 0:
        Kc = k
    if events_cap is None:
        tm = -(-m // BM) if m > 0 else 0
        tn = -(-n // BN) if n > 0 else 0
        nunits = nu if units is not None else tm * tn
        events_cap = max(1, nunits * max(1, -(-k // max(Kc, 1))))
    ev = (_Event * events_cap)()
    counters = np.zeros(5, dtype=np.int64)
    rc = lib().oracle_dgemm_abft_units(ta.encode(), tb.encode(), m, n, k, alpha, _ptr(A), lda,
                                       _ptr(B), ldb, beta, _ptr(Cout), ldc, BM, BN, BK, Kc,
                                       int(subtract), ctypes.cast(fa, ctypes.c_void_p), len(faults),
                                       uptr, nu, _ptr(counters), ctypes.cast(ev, ctypes.c_void_p),
                                       events_cap)
    if rc != 0:
        raise ValueError(f"oracle_dgemm_abft_units rejected arguments (rc={rc})")
    nstored = int(min(counters[4], events_cap))
    events = [(ev[e].interval, ev[e].i, ev[e].j, ev[e].kind, ev[e].residual_row, ev[e].residual_col)
              for e in range(nstored)]
    return Cout, Report(*[int(x) for x in counters], events)


def _faults(faults):
    faults = list(faults)
    fa = (_Fault * max(len(faults), 1))()
    for e, (i, j, s, dlt) in enumerate(faults):
        fa[e] = _Fault(int(i), int(j), int(s), float(dlt), 0)
    return ctypes.cast(fa, ctypes.c_void_p), len(faults), fa


@dataclass
class DmrReport:
    checked: int
    detected: int
    corrected: int
    uncorrectable: int


def dscal(n, alpha, x, incx=1, faults=()):
    """DMR DSCAL oracle (NEXT-4): returns (new x, DmrReport); x is a flat float64 array."""
    xo = np.ascontiguousarray(x, dtype=np.float64).copy()
    fp, nf, _keep = _faults(faults)
    cnt = np.zeros(4, dtype=np.int64)
    lib().oracle_dscal(n, alpha, _ptr(xo), incx, fp, nf, _ptr(cnt))
    return xo, DmrReport(*[int(v) for v in cnt])


def daxpy(n, alpha, x, incx, y, incy, faults=()):
    xo = np.ascontiguousarray(x, dtype=np.float64)
    yo = np.ascontiguousarray(y, dtype=np.float64).copy()
    fp, nf, _keep = _faults(faults)
    cnt = np.zeros(4, dtype=np.int64)
    lib().oracle_daxpy(n, alpha, _ptr(xo), incx, _ptr(yo), incy, fp, nf, _ptr(cnt))
    return yo, DmrReport(*[int(v) for v in cnt])


def dgemv(trans, m, n, alpha, A, lda, x, incx, beta, y, incy, faults=()):
    A = _flat(A)
    xo = np.ascontiguousarray(x, dtype=np.float64)
    yo = np.ascontiguousarray(y, dtype=np.float64).copy()
    fp, nf, _keep = _faults(faults)
    cnt = np.zeros(4, dtype=np.int64)
    lib().oracle_dgemv(trans.encode(), m, n, alpha, _ptr(A), lda, _ptr(xo), incx, beta, _ptr(yo), incy,
                       fp, nf, _ptr(cnt))
    return yo, DmrReport(*[int(v) for v in cnt])


def dtrsm(uplo, transa, diag, m, n, alpha, A, lda, B, ldb, faults=(), side="L"):
    """DTRSM oracle (NEXT-3): solve op(A) X = alpha B (side L, op(A) m x m) or X op(A) = alpha B
    (side R, op(A) n x n); returns (X flat, Report) -- X the fault-free solution (the faults are
    corrected by the protection), the Report the FT bookkeeping of the blocked solve
    (dtrsm_bookkeeping: DMR detections of the diagonal blocks, ABFT units / events of the GEMM
    updates)."""
    A = _flat(A)
    Bo = _flat(B).copy()
    cnt = np.zeros(4, dtype=np.int64)
    fn = lib().oracle_dtrsm if side in ("L", "l") else lib().oracle_dtrsm_right
    fn(uplo.encode(), transa.encode(), diag.encode(), m, n, alpha, _ptr(A), lda, _ptr(Bo), ldb,
       len(list(faults)), _ptr(cnt))
    return Bo, dtrsm_bookkeeping(side, uplo, transa, m, n, faults)


def dtrsm_bookkeeping(side, uplo, transa, m, n, faults, leaf=128, tm=127):
    """FT-DTRSM bookkeeping of the blocked solve (reading R21): which faults the DMR diagonal
    solves settle and which land in the ABFT-protected GEMM updates.  Returns a Report
    (units_checked, detected, corrected, recomputed, n_events, events) with events
    (0, i, j, kind, 0.0, 0.0) sorted by (i, j)."""
    faults = list(faults)
    fa = (_Fault * max(len(faults), 1))()
    for e, (i, j, s_, dlt) in enumerate(faults):
        fa[e] = _Fault(int(i), int(j), int(s_), float(dlt), 0)
    cap = max(1, 2 * len(faults))
    ev = (_Event * cap)()
    cnt = np.zeros(5, dtype=np.int64)
    rc = lib().oracle_dtrsm_bookkeeping(side.encode(), uplo.encode(), transa.encode(), m, n, leaf, tm,
                                        ctypes.cast(fa, ctypes.c_void_p), len(faults), _ptr(cnt),
                                        ctypes.cast(ev, ctypes.c_void_p), cap)
    if rc != 0:
        raise ValueError("oracle_dtrsm_bookkeeping rejected arguments")
    events = [(ev[e].interval, ev[e].i, ev[e].j, ev[e].kind, ev[e].residual_row, ev[e].residual_col)
              for e in range(int(min(cnt[4], cap)))]
    return Report(*[int(x) for x in cnt], events)


def num_threads() -> int:
    return int(lib().oracle_num_threads())
