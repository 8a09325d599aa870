"""Thin Python binding of libftblas.so (include/ftblas.h) — argument marshalling only.

Every step of the ABFT DGEMM runs in the library's CUDA kernels; this module only
converts Python/torch arguments to the C ABI.  It raises loudly when the native
library is missing: there is no CPU fallback.

Function names mirror the C ABI (``ftblas_dgemm``, ``ftblas_dgemm_noft``,
``ftblas_inject_arm`` ...).  Matrix arguments are device pointers: pass a torch
float64 CUDA tensor (its data_ptr() is used) or an int address.  Matrices are
column-major with explicit leading dimensions, exactly as in BLAS.
"""
from __future__ import annotations

import ctypes
import os
import threading
from dataclasses import dataclass, field

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libftblas.so")


class FtblasError(RuntimeError):
    def __init__(self, fn: str, status: int, msg: str):
        super().__init__(f"{fn} returned {status}: {msg}")
        self.status = status


class Event(ctypes.Structure):
    _fields_ = [("i", ctypes.c_int64), ("j", ctypes.c_int64), ("kind", ctypes.c_int32),
                ("interval", ctypes.c_int32), ("residual_row", ctypes.c_double),
                ("residual_col", ctypes.c_double)]


class ErrReport(ctypes.Structure):
    _fields_ = [("units_checked", ctypes.c_int64), ("detected", ctypes.c_int64),
                ("corrected", ctypes.c_int64), ("recomputed", ctypes.c_int64),
                ("n_events", ctypes.c_int64), ("unit_rows", ctypes.c_int32),
                ("unit_cols", ctypes.c_int32), ("unit_k", ctypes.c_int32),
                ("step_quantum", ctypes.c_int32), ("events", ctypes.POINTER(Event)),
                ("events_capacity", ctypes.c_int64)]


class DmrReportC(ctypes.Structure):
    _fields_ = [("checked", ctypes.c_int64), ("detected", ctypes.c_int64),
                ("corrected", ctypes.c_int64), ("uncorrectable", ctypes.c_int64)]


@dataclass
class DmrReport:
    checked: int
    detected: int
    corrected: int
    uncorrectable: int


class Fault(ctypes.Structure):
    _fields_ = [("i", ctypes.c_int64), ("j", ctypes.c_int64), ("step", ctypes.c_int64),
                ("delta", ctypes.c_double)]


@dataclass
class Report:
    units_checked: int
    detected: int
    corrected: int
    recomputed: int
    n_events: int
    unit_rows: int
    unit_cols: int
    unit_k: int
    step_quantum: int
    events: list = field(default_factory=list)  # (interval, i, j, kind, residual_row, residual_col)


_lib = None


def load(path: str | None = None):
    """Load libftblas.so (built by paper_2104_00897_b200.build); raise if absent.  `path`
    selects another build of the same ABI (development tools: libftblas_dev.so)."""
    global _lib
    if _lib is not None:
        return _lib
    path = path or LIB_PATH
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: build it with "
                          "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback)")
    L = ctypes.CDLL(path)
    c, i64, d, P, i32 = ctypes.c_char, ctypes.c_int64, ctypes.c_double, ctypes.c_void_p, ctypes.c_int
    gemm = [c, c, i64, i64, i64, d, P, i64, P, i64, d, P, i64]
    L.ftblas_dgemm.argtypes = gemm + [ctypes.POINTER(ErrReport)]
    L.ftblas_dgemm_unfused.argtypes = gemm + [ctypes.POINTER(ErrReport)]
    L.ftblas_dgemm_noft.argtypes = gemm
    L.ftblas_dgemm_host.argtypes = gemm + [ctypes.POINTER(ErrReport)]
    L.ftblas_dgemm_noft_host.argtypes = gemm
    L.ftblas_inject_arm.argtypes = [ctypes.POINTER(Fault), i64]
    L.ftblas_inject_disarm.argtypes = []
    L.ftblas_inject_arm_checksum.argtypes = [ctypes.POINTER(Fault), ctypes.POINTER(ctypes.c_int32), i64]
    L.ftblas_inject_seeded.argtypes = [ctypes.c_uint64, i64, i64, i64, i64, d, d,
                                       ctypes.POINTER(Fault)]
    L.ftblas_set_stream.argtypes = [P]
    L.ftblas_set_correction.argtypes = [i32]
    L.ftblas_set_encode.argtypes = [i32]
    L.ftblas_set_interval.argtypes = [i64]
    L.ftblas_get_geometry.argtypes = [ctypes.POINTER(ctypes.c_int32)] * 3
    DR = ctypes.POINTER(DmrReportC)
    L.ftblas_dscal.argtypes = [i64, d, P, i64, DR]
    L.ftblas_dscal_noft.argtypes = [i64, d, P, i64]
    L.ftblas_daxpy.argtypes = [i64, d, P, i64, P, i64, DR]
    L.ftblas_daxpy_noft.argtypes = [i64, d, P, i64, P, i64]
    L.ftblas_dgemv.argtypes = [c, i64, i64, d, P, i64, P, i64, d, P, i64, DR]
    L.ftblas_dgemv_noft.argtypes = [c, i64, i64, d, P, i64, P, i64, d, P, i64]
    L.ftblas_dtrsm.argtypes = [c, c, c, c, i64, i64, d, P, i64, P, i64, ctypes.POINTER(ErrReport)]
    L.ftblas_dtrsm_noft.argtypes = [c, c, c, c, i64, i64, d, P, i64, P, i64]
    for fn in ("ftblas_dscal", "ftblas_dscal_noft", "ftblas_daxpy", "ftblas_daxpy_noft",
               "ftblas_dgemv", "ftblas_dgemv_noft", "ftblas_dtrsm", "ftblas_dtrsm_noft"):
        getattr(L, fn).restype = ctypes.c_int
    L.ftblas_take_launch_count.restype = i64
    L.ftblas_take_launch_count.argtypes = []
    L.ftblas_status_string.restype = ctypes.c_char_p
    L.ftblas_status_string.argtypes = [i32]
    L.ftblas_finalize.argtypes = []
    for fn in ("ftblas_dgemm", "ftblas_dgemm_unfused", "ftblas_dgemm_noft", "ftblas_dgemm_host", "ftblas_dgemm_noft_host",
               "ftblas_inject_arm", "ftblas_inject_disarm", "ftblas_inject_seeded", "ftblas_inject_arm_checksum",
               "ftblas_set_stream", "ftblas_set_correction", "ftblas_set_encode",
               "ftblas_set_interval", "ftblas_get_geometry", "ftblas_finalize"):
        getattr(L, fn).restype = ctypes.c_int
    _lib = L
    return L


EXPORTED = ("ftblas_dgemm", "ftblas_dgemm_unfused", "ftblas_dgemm_noft", "ftblas_dgemm_host", "ftblas_dgemm_noft_host",
            "ftblas_inject_arm", "ftblas_inject_disarm", "ftblas_inject_seeded", "ftblas_inject_arm_checksum",
            "ftblas_set_stream", "ftblas_set_correction", "ftblas_set_encode", "ftblas_set_interval",
            "ftblas_get_geometry", "ftblas_take_launch_count", "ftblas_status_string", "ftblas_finalize",
            "ftblas_dscal", "ftblas_dscal_noft", "ftblas_daxpy", "ftblas_daxpy_noft", "ftblas_dgemv",
            "ftblas_dgemv_noft", "ftblas_dtrsm", "ftblas_dtrsm_noft")


def _check(fn, status):
    if status != 0:
        raise FtblasError(fn, status, load().ftblas_status_string(status).decode())


def _ptr(x, where="device"):
    """Address of an operand: a raw int, a float64 torch tensor, or (host entry points) a
    float64 numpy array.  where = "device" (CUDA tensors only) or "host" (numpy or CPU
    tensors).  Marshalling checks only: shapes and leading dimensions are the library's."""
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if hasattr(x, "data_ptr"):  # torch tensor
        if str(x.dtype) != "torch.float64":
            raise TypeError(f"float64 tensor expected, got {x.dtype}")
        if (where == "device") != bool(x.is_cuda):
            raise ValueError(f"{'CUDA' if where == 'device' else 'host'} tensor expected")
        return x.data_ptr()
    if hasattr(x, "ctypes"):  # numpy array
        if where == "device":
            raise ValueError("device entry point: pass a CUDA tensor (or a device address), not a numpy array")
        if str(x.dtype) != "float64":
            raise TypeError(f"float64 array expected, got {x.dtype}")
        return x.ctypes.data
    raise TypeError(type(x))


def _c(t: str) -> bytes:
    return t.encode() if isinstance(t, str) else t


def _report(r: ErrReport, evbuf) -> Report:
    n = min(r.n_events, r.events_capacity)
    ev = [(evbuf[e].interval, evbuf[e].i, evbuf[e].j, evbuf[e].kind, evbuf[e].residual_row,
           evbuf[e].residual_col) for e in range(n)]
    return Report(r.units_checked, r.detected, r.corrected, r.recomputed, r.n_events, r.unit_rows,
                  r.unit_cols, r.unit_k, r.step_quantum, ev)


_tls = threading.local()


def _event_buffer(capacity):
    """Per-thread report buffer of `capacity` events, reused across calls (the Report copies the
    events out; allocating and zeroing a fresh ctypes array cost ~20 us per call)."""
    cache = getattr(_tls, "evbufs", None)
    if cache is None:
        cache = _tls.evbufs = {}
    buf = cache.get(capacity)
    if buf is None:
        buf = cache[capacity] = (Event * capacity)()
    return buf


def _protected(fn, transA, transB, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, report,
               events_capacity, raw_status):
    L = load()
    f = getattr(L, fn)
    if report:
        evbuf = _event_buffer(max(events_capacity, 1))
        r = ErrReport()
        r.events = evbuf
        r.events_capacity = events_capacity
        st = f(_c(transA), _c(transB), m, n, k, alpha, _ptr(A), lda, _ptr(B), ldb, beta, _ptr(C),
               ldc, ctypes.byref(r))
    else:
        st = f(_c(transA), _c(transB), m, n, k, alpha, _ptr(A), lda, _ptr(B), ldb, beta, _ptr(C),
               ldc, None)
    if raw_status:
        return st
    _check(fn, st)
    return _report(r, evbuf) if report else None


def ftblas_dgemm(transA, transB, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, *, report=True,
                 events_capacity=4096, raw_status=False):
    """Protected DGEMM on device pointers.  Returns a Report (synchronises the stream) or,
    with report=False, None (asynchronous)."""
    return _protected("ftblas_dgemm", transA, transB, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc,
                      report, events_capacity, raw_status)


def ftblas_dgemm_unfused(transA, transB, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, *,
                         report=True, events_capacity=4096, raw_status=False):
    """The unfused ABFT baseline (NEXT-2) on device pointers; same contract as ftblas_dgemm,
    128 x 128 verification units."""
    return _protected("ftblas_dgemm_unfused", transA, transB, m, n, k, alpha, A, lda, B, ldb, beta,
                      C, ldc, report, events_capacity, raw_status)


def ftblas_dgemm_noft(transA, transB, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, *,
                      raw_status=False):
    st = load().ftblas_dgemm_noft(_c(transA), _c(transB), m, n, k, alpha, _ptr(A), lda, _ptr(B),
                                  ldb, beta, _ptr(C), ldc)
    if raw_status:
        return st
    _check("ftblas_dgemm_noft", st)


def ftblas_dgemm_host(transA, transB, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, *,
                      report=True, events_capacity=4096):
    """Protected DGEMM on HOST buffers (numpy arrays / host addresses); C updated in place."""
    L = load()
    evbuf = _event_buffer(max(events_capacity, 1))
    r = ErrReport()
    r.events = evbuf
    r.events_capacity = events_capacity
    st = L.ftblas_dgemm_host(_c(transA), _c(transB), m, n, k, alpha, _ptr(A, "host"), lda, _ptr(B, "host"), ldb,
                             beta, _ptr(C, "host"), ldc, ctypes.byref(r) if report else None)
    _check("ftblas_dgemm_host", st)
    return _report(r, evbuf) if report else None


def ftblas_dgemm_noft_host(transA, transB, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc):
    st = load().ftblas_dgemm_noft_host(_c(transA), _c(transB), m, n, k, alpha, _ptr(A, "host"), lda,
                                       _ptr(B, "host"), ldb, beta, _ptr(C, "host"), ldc)
    _check("ftblas_dgemm_noft_host", st)


def _dmr(fn, args, report):
    L = load()
    r = DmrReportC()
    st = getattr(L, fn)(*args, ctypes.byref(r) if report else None)
    _check(fn, st)
    return DmrReport(r.checked, r.detected, r.corrected, r.uncorrectable) if report else None


def ftblas_dscal(n, alpha, x, incx=1, *, report=True):
    """x := alpha*x with DMR (NEXT-4); device vector.  Returns a DmrReport (synchronises)."""
    return _dmr("ftblas_dscal", (n, alpha, _ptr(x), incx), report)


def ftblas_daxpy(n, alpha, x, incx, y, incy, *, report=True):
    """y := fma(alpha, x, y) with DMR."""
    return _dmr("ftblas_daxpy", (n, alpha, _ptr(x), incx, _ptr(y), incy), report)


def ftblas_dgemv(trans, m, n, alpha, A, lda, x, incx, beta, y, incy, *, report=True):
    """y := alpha*op(A)*x + beta*y with DMR."""
    return _dmr("ftblas_dgemv", (_c(trans), m, n, alpha, _ptr(A), lda, _ptr(x), incx, beta, _ptr(y),
                                 incy), report)


def ftblas_dscal_noft(n, alpha, x, incx=1):
    _check("ftblas_dscal_noft", load().ftblas_dscal_noft(n, alpha, _ptr(x), incx))


def ftblas_daxpy_noft(n, alpha, x, incx, y, incy):
    _check("ftblas_daxpy_noft", load().ftblas_daxpy_noft(n, alpha, _ptr(x), incx, _ptr(y), incy))


def ftblas_dgemv_noft(trans, m, n, alpha, A, lda, x, incx, beta, y, incy):
    _check("ftblas_dgemv_noft", load().ftblas_dgemv_noft(_c(trans), m, n, alpha, _ptr(A), lda, _ptr(x),
                                                         incx, beta, _ptr(y), incy))


def ftblas_dtrsm(side, uplo, transa, diag, m, n, alpha, A, lda, B, ldb, *, report=True,
                 events_capacity=4096):
    """FT-DTRSM (NEXT-3): B := alpha op(A)^-1 B (side 'L') or alpha B op(A)^-1 (side 'R') on
    device pointers; returns a Report."""
    L = load()
    evbuf = _event_buffer(max(events_capacity, 1))
    r = ErrReport()
    r.events = evbuf
    r.events_capacity = events_capacity
    st = L.ftblas_dtrsm(_c(side), _c(uplo), _c(transa), _c(diag), m, n, alpha, _ptr(A), lda, _ptr(B),
                        ldb, ctypes.byref(r) if report else None)
    _check("ftblas_dtrsm", st)
    return _report(r, evbuf) if report else None


def ftblas_dtrsm_noft(side, uplo, transa, diag, m, n, alpha, A, lda, B, ldb):
    _check("ftblas_dtrsm_noft", load().ftblas_dtrsm_noft(_c(side), _c(uplo), _c(transa), _c(diag), m, n,
                                                         alpha, _ptr(A), lda, _ptr(B), ldb))


def ftblas_inject_arm(faults):
    faults = list(faults)
    arr = (Fault * max(len(faults), 1))()
    for e, (i, j, s, d) in enumerate(faults):
        arr[e] = Fault(int(i), int(j), int(s), float(d))
    _check("ftblas_inject_arm", load().ftblas_inject_arm(arr, len(faults)))


def ftblas_inject_arm_checksum(faults):
    """Checksum-lane faults (test hook, reading R6): (i, j, step, delta, lane) with lane 1 = the
    column checksum of column j, 2 = the row checksum of row i, of the unit containing (i, j)."""
    faults = list(faults)
    arr = (Fault * max(len(faults), 1))()
    lanes = (ctypes.c_int32 * max(len(faults), 1))()
    for e, (i, j, s, d, lane) in enumerate(faults):
        arr[e] = Fault(int(i), int(j), int(s), float(d))
        lanes[e] = int(lane)
    _check("ftblas_inject_arm_checksum", load().ftblas_inject_arm_checksum(arr, lanes, len(faults)))


def ftblas_inject_disarm():
    _check("ftblas_inject_disarm", load().ftblas_inject_disarm())


def ftblas_inject_seeded(seed, count, m, n, k, log10_lo, log10_hi):
    arr = (Fault * max(count, 1))()
    _check("ftblas_inject_seeded",
           load().ftblas_inject_seeded(seed, count, m, n, k, log10_lo, log10_hi, arr))
    return [(arr[e].i, arr[e].j, arr[e].step, arr[e].delta) for e in range(count)]


def ftblas_set_stream(stream):
    """stream: torch.cuda.Stream, raw cudaStream_t int, or None (legacy default stream)."""
    h = None if stream is None else (stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))
    _check("ftblas_set_stream", load().ftblas_set_stream(h))


def ftblas_set_correction(mode: int):
    _check("ftblas_set_correction", load().ftblas_set_correction(mode))


def ftblas_set_encode(mode: int):
    """ENCODE_FUSED (0, default), ENCODE_PREPASS (1), ENCODE_FUSED_LOCAL (2) or ENCODE_FUSED_WAIT (3);
    thread-local."""
    _check("ftblas_set_encode", load().ftblas_set_encode(mode))


def ftblas_set_interval(kc: int):
    """Verification interval Kc (multiple of 16; 0 = k); thread-local."""
    _check("ftblas_set_interval", load().ftblas_set_interval(int(kc)))


def ftblas_get_geometry():
    a, b, c = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
    _check("ftblas_get_geometry", load().ftblas_get_geometry(ctypes.byref(a), ctypes.byref(b),
                                                            ctypes.byref(c)))
    return a.value, b.value, c.value


def ftblas_take_launch_count() -> int:
    return int(load().ftblas_take_launch_count())


def ftblas_status_string(status: int) -> str:
    return load().ftblas_status_string(status).decode()


def ftblas_finalize():
    _check("ftblas_finalize", load().ftblas_finalize())


ENCODE_FUSED = 0
ENCODE_PREPASS = 1
ENCODE_FUSED_LOCAL = 2
ENCODE_FUSED_WAIT = 3
CORRECT_RECOMPUTE = 0
CORRECT_SUBTRACT = 1
