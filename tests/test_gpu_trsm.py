"""GPU parity of FT-DTRSM: every uplo / trans / diag against the
oracle (well-conditioned systems, max-norm bound 64 m u |X|), bitwise on exact integer
systems, faults in the ABFT-protected GEMM updates and in the DMR diagonal solves all
corrected (integer case: X bitwise equal to the fault-free solution), the unprotected twin
bitwise equal to the protected result when no fault is injected."""
import numpy as np
import pytest

import oracle
from tests.helpers import events_key, from_dev, to_dev

pytestmark = pytest.mark.gpu
U = 2.0 ** -53
F = None


@pytest.fixture(scope="module", autouse=True)
def _lib():
    global F
    from paper_2104_00897_b200 import ftblas
    ftblas.load()
    F = ftblas
    yield


def wellcond(rng, m, uplo):
    A = rng.uniform(-1, 1, (m, m)) / max(m, 1)
    A = (np.tril(A) if uplo == "L" else np.triu(A)) + np.diag(rng.uniform(1, 2, m))
    return np.asfortranarray(A)


@pytest.mark.parametrize("uplo", ["L", "U"])
@pytest.mark.parametrize("tr", ["N", "T"])
@pytest.mark.parametrize("diag", ["N", "U"])
def test_dtrsm_variants_against_oracle(uplo, tr, diag):
    rng = np.random.default_rng(hash((uplo, tr, diag)) % 1000)
    for (m, n) in [(1, 1), (100, 64), (128, 3), (129, 257), (300, 40), (700, 130)]:
        A = wellcond(rng, m, uplo)
        B = np.asfortranarray(rng.uniform(-1, 1, (m, n)))
        dA, dB = to_dev(A), to_dev(B)
        rep = F.ftblas_dtrsm("L", uplo, tr, diag, m, n, 1.25, dA, m, dB, m)
        Xg = from_dev(dB, m, n)
        Xo, _ = oracle.dtrsm(uplo, tr, diag, m, n, 1.25, A, m, B, m)
        Xo = Xo.reshape((n, m)).T
        assert np.max(np.abs(Xg - Xo)) <= 64 * m * U * max(np.max(np.abs(Xo)), 1e-300)
        assert rep.detected == 0


def integer_system(rng, m, n, uplo, tr):
    T = rng.integers(-1, 2, (m, m)).astype(float)
    T = (np.tril(T, -1) if uplo == "L" else np.triu(T, 1)) + np.eye(m)
    X = rng.integers(-3, 4, (m, n)).astype(float)
    B = np.asfortranarray((T.T if tr == "T" else T) @ X)
    return np.asfortranarray(T), B, X


@pytest.mark.parametrize("uplo,tr", [("L", "N"), ("U", "N"), ("L", "T"), ("U", "T")])
def test_dtrsm_integer_exact_with_faults(uplo, tr):
    rng = np.random.default_rng(7)
    m, n = 300, 300
    T, B, X = integer_system(rng, m, n, uplo, tr)
    fwd = (uplo == "L") != (tr == "T")
    # (i, j, p): GEMM-update faults (i and p in different diagonal blocks) and diagonal-block
    # (DMR) faults (same block); p before i in the substitution order; the columns put every
    # fault in its own 127 x 127 unit of whichever update it lands in.
    pairs = [(290, 5, 10), (150, 140, 3), (200, 270, 140), (60, 60, 30), (250, 200, 240)]
    faults = [((i, j, p, 17.0) if fwd else (m - 1 - i, j, m - 1 - p, -9.0)) for (i, j, p) in pairs]
    dB = to_dev(B)
    F.ftblas_inject_arm(faults)
    rep = F.ftblas_dtrsm("L", uplo, tr, "U", m, n, 1.0, to_dev(T), m, dB, m)
    assert np.array_equal(from_dev(dB, m, n), X)
    assert (rep.detected, rep.corrected, rep.recomputed) == (5, 5, 0)
    # the oracle's bookkeeping of the blocked solve (reading R21) decides which faults the GEMM
    # updates' ABFT reports (events with global rows) and which the DMR diagonal solves settle
    bk = oracle.dtrsm_bookkeeping("L", uplo, tr, m, n, faults)
    assert (rep.units_checked, rep.detected, rep.corrected, rep.recomputed) == \
        (bk.units_checked, bk.detected, bk.corrected, bk.recomputed)
    assert events_key(rep.events) == events_key(bk.events) and len(bk.events) >= 2


def test_dtrsm_noft_twin_bitwise_and_alpha():
    rng = np.random.default_rng(9)
    m, n = 520, 77
    A = wellcond(rng, m, "L")
    B = np.asfortranarray(rng.uniform(-1, 1, (m, n)))
    d1, d2 = to_dev(B), to_dev(B)
    F.ftblas_dtrsm("L", "L", "N", "N", m, n, -2.0, to_dev(A), m, d1, m)
    F.ftblas_dtrsm_noft("L", "L", "N", "N", m, n, -2.0, to_dev(A), m, d2, m)
    assert np.array_equal(from_dev(d1, m, n), from_dev(d2, m, n))
    d3 = to_dev(B)
    F.ftblas_dtrsm("L", "U", "T", "N", m, n, 0.0, to_dev(A), m, d3, m)
    assert not from_dev(d3, m, n).any()


def test_dtrsm_argument_errors():
    from paper_2104_00897_b200.ftblas import FtblasError
    A = to_dev(np.eye(4))
    Bd = to_dev(np.ones((4, 2)))
    with pytest.raises(FtblasError):
        F.ftblas_dtrsm("X", "L", "N", "N", 4, 2, 1.0, A, 4, Bd, 4)
    with pytest.raises(FtblasError):  # side R: A is n x n, lda >= n
        F.ftblas_dtrsm("R", "L", "N", "N", 2, 4, 1.0, A, 3, to_dev(np.ones((2, 4))), 2)
    with pytest.raises(FtblasError):
        F.ftblas_dtrsm("L", "X", "N", "N", 4, 2, 1.0, A, 4, Bd, 4)
    F.ftblas_inject_arm([(1, 0, 3, 1.0)])  # forward solve: step must precede the row
    with pytest.raises(FtblasError):
        F.ftblas_dtrsm("L", "L", "N", "N", 4, 2, 1.0, A, 4, Bd, 4)


@pytest.mark.parametrize("uplo", ["L", "U"])
@pytest.mark.parametrize("tr", ["N", "T"])
@pytest.mark.parametrize("diag", ["N", "U"])
def test_dtrsm_right_side_against_oracle(uplo, tr, diag):
    """Side R: X op(A) = alpha B, A n x n, every uplo / trans / diag."""
    rng = np.random.default_rng(hash(("R", uplo, tr, diag)) % 1000)
    for (m, n) in [(1, 1), (64, 100), (3, 128), (257, 129), (40, 300), (130, 700)]:
        A = wellcond(rng, n, uplo)
        B = np.asfortranarray(rng.uniform(-1, 1, (m, n)))
        dB = to_dev(B)
        rep = F.ftblas_dtrsm("R", uplo, tr, diag, m, n, -0.5, to_dev(A), n, dB, m)
        Xg = from_dev(dB, m, n)
        Xo, _ = oracle.dtrsm(uplo, tr, diag, m, n, -0.5, A, n, B, m, side="R")
        Xo = Xo.reshape((n, m)).T
        assert np.max(np.abs(Xg - Xo)) <= 64 * n * U * max(np.max(np.abs(Xo)), 1e-300)
        assert rep.detected == 0


@pytest.mark.parametrize("uplo,tr", [("L", "N"), ("U", "N"), ("L", "T"), ("U", "T")])
def test_dtrsm_right_side_integer_exact_with_faults(uplo, tr):
    rng = np.random.default_rng(17)
    m, n = 260, 300
    T = rng.integers(-1, 2, (n, n)).astype(float)
    T = np.asfortranarray((np.tril(T, -1) if uplo == "L" else np.triu(T, 1)) + np.eye(n))
    X = rng.integers(-3, 4, (m, n)).astype(float)
    B = np.asfortranarray(X @ (T.T if tr == "T" else T))
    fwd = (uplo == "L") == (tr == "T")  # side R: op(A) upper -> columns ascending
    # (i, j, p): row i, column j, step p preceding j in the substitution order; GEMM-update
    # faults (j and p in different diagonal blocks) and diagonal-block (DMR) faults
    pairs = [(5, 290, 10), (140, 150, 3), (250, 200, 140), (60, 60, 30), (200, 250, 240)]
    faults = [((i, j, p, 13.0) if fwd else (i, n - 1 - j, n - 1 - p, -7.0)) for (i, j, p) in pairs]
    dB = to_dev(B)
    F.ftblas_inject_arm(faults)
    rep = F.ftblas_dtrsm("R", uplo, tr, "U", m, n, 1.0, to_dev(T), n, dB, m)
    assert np.array_equal(from_dev(dB, m, n), X)
    assert (rep.detected, rep.corrected, rep.recomputed) == (5, 5, 0)
    bk = oracle.dtrsm_bookkeeping("R", uplo, tr, m, n, faults)
    assert (rep.units_checked, rep.detected, rep.corrected, rep.recomputed) == \
        (bk.units_checked, bk.detected, bk.corrected, bk.recomputed)
    assert events_key(rep.events) == events_key(bk.events) and len(bk.events) >= 2
    d2 = to_dev(B)
    F.ftblas_dtrsm_noft("R", uplo, tr, "U", m, n, 1.0, to_dev(T), n, d2, m)
    assert np.array_equal(from_dev(d2, m, n), X)


@pytest.mark.parametrize("side", ["L", "R"])
def test_dtrsm_multi_fault_units_against_bookkeeping(side):
    """Two cells of one ABFT unit of an update -> recomputed (event at the unit origin), two
    faults of one right-hand side in one diagonal block -> one DMR detection: GPU counters and
    events against the oracle's bookkeeping of the blocked solve (reading R21, R6)."""
    rng = np.random.default_rng(23)
    na, nr = 700, 190
    T = rng.integers(-1, 2, (na, na)).astype(float)
    T = np.asfortranarray(np.tril(T, -1) + np.eye(na))
    X = rng.integers(-3, 4, (na, nr) if side == "L" else (nr, na)).astype(float)
    if side == "L":
        B = np.asfortranarray(T @ X)
        m, n = na, nr
        faults = [(600, 5, 20, 7.0), (601, 6, 30, -3.0), (650, 150, 400, 2.0), (60, 9, 30, 5.0),
                  (20, 9, 5, 1.0), (70, 9, 40, 1.0)]
    else:  # X T = B, T lower -> columns in descending order: step after the column
        B = np.asfortranarray(X @ T)
        m, n = nr, na
        faults = [(5, 20, 600, 7.0), (6, 30, 601, -3.0), (150, 300, 650, 2.0), (9, 640, 660, 5.0),
                  (9, 650, 670, 1.0)]
    dB = to_dev(B)
    F.ftblas_inject_arm(faults)
    rep = F.ftblas_dtrsm(side, "L", "N", "U", m, n, 1.0, to_dev(T), na, dB, m)
    assert np.array_equal(from_dev(dB, m, n), X)
    bk = oracle.dtrsm_bookkeeping(side, "L", "N", m, n, faults)
    assert (rep.units_checked, rep.detected, rep.corrected, rep.recomputed) == \
        (bk.units_checked, bk.detected, bk.corrected, bk.recomputed)
    assert events_key(rep.events) == events_key(bk.events)
    assert bk.recomputed >= 1 and bk.detected > bk.n_events  # ABFT units and DMR blocks
