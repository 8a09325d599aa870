"""Shared test helpers: device upload/download of column-major matrices, the parity bound,
and the comparison of GPU and oracle reports.  No method arithmetic lives here."""
from __future__ import annotations

import contextlib

import numpy as np

U = 2.0 ** -53


def to_dev(X: np.ndarray, ld: int | None = None):
    """Column-major device copy of a 2-D array (flat float64 CUDA tensor), optional padding ld."""
    import torch
    X = np.asfortranarray(X, dtype=np.float64)
    r, c = X.shape
    ld = max(r, 1) if ld is None else ld
    buf = np.zeros((max(c, 1), ld), dtype=np.float64)
    buf[:c, :r] = X.T
    return torch.from_numpy(buf.reshape(-1)).to("cuda")


def from_dev(t, r: int, c: int, ld: int | None = None) -> np.ndarray:
    ld = max(r, 1) if ld is None else ld
    a = t.detach().cpu().numpy().reshape((-1, ld))
    return np.asfortranarray(a[:c, :r].T)


def op(X: np.ndarray, t: str) -> np.ndarray:
    return X.T if t in "TtCc" else X


def bound(case_like, A, B, C0, alpha, beta, ta, tb, k):
    """2 k u (|alpha| (|op(A)||op(B)|) + |beta| |C0|), elementwise (north_star tolerance)."""
    S = np.abs(op(A, ta)) @ np.abs(op(B, tb))
    return 2 * max(k, 1) * U * (abs(alpha) * S + abs(beta) * np.abs(C0))


def unit_tau(A, B, ta, tb, i, j, BM, BN, k):
    """tau_col, tau_row of the unit containing (i, j) (R1, exact maxima), numpy."""
    oA, oB = op(A, ta), op(B, tb)
    I0, J0 = (i // BM) * BM, (j // BN) * BN
    Ia, Jb = oA[I0:I0 + BM, :], oB[:, J0:J0 + BN]
    amax = float(np.nanmax(np.abs(Ia), initial=0.0))
    bmax = float(np.nanmax(np.abs(Jb), initial=0.0))
    bm, bn = Ia.shape[0], Jb.shape[1]
    g = lambda nn: nn * U / (1 - nn * U)  # noqa: E731
    return (2 * g(k + bm) * k * bm * amax * bmax, 2 * g(k + bn) * k * bn * amax * bmax)


def events_key(events):
    return [(int(t), int(i), int(j), int(kind)) for (t, i, j, kind, _, _) in events]


def assert_reports_match(gpu, orc, A=None, B=None, ta="N", tb="N", k=None):
    assert gpu.detected == orc.detected, (gpu, orc)
    assert gpu.corrected == orc.corrected
    assert gpu.recomputed == orc.recomputed
    assert gpu.n_events == orc.n_events
    assert events_key(gpu.events) == events_key(orc.events), (gpu.events, orc.events)
    if A is not None:
        for ge, oe in zip(gpu.events, orc.events):
            tc, tr = unit_tau(A, B, ta, tb, ge[1], ge[2], gpu.unit_rows, gpu.unit_cols, k)
            for gv, ov, tau in ((ge[4], oe[4], tr), (ge[5], oe[5], tc)):
                if np.isfinite(gv) or np.isfinite(ov):
                    assert abs(gv - ov) <= 4 * tau + 8 * U * abs(ov) * k, (ge, oe, tau)


@contextlib.contextmanager
def encode_mode(F, name):
    """Encode mode of ftblas_dgemm for the duration: "fused" (e^T A_I shared along tile rows,
    B_J e along tile columns, as scheduled), "fused_copy" (the same, every tile waiting for the
    published copies: ENCODE_FUSED_WAIT), "fused_local" (every CTA encodes itself) or
    "prepass"."""
    mode = {"fused": F.ENCODE_FUSED, "fused_copy": F.ENCODE_FUSED_WAIT, "fused_local": F.ENCODE_FUSED_LOCAL,
            "prepass": F.ENCODE_PREPASS}[name]
    F.ftblas_set_encode(mode)
    try:
        yield
    finally:
        F.ftblas_set_encode(F.ENCODE_FUSED)
