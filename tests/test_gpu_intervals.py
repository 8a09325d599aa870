"""GPU parity of verification intervals (ftblas_set_interval): the
unit is (tile, interval of Kc rank-1 updates); counters, the sorted (interval, i, j, kind)
events and the values must match the oracle run with the same Kc."""
import numpy as np
import pytest

import oracle
from tests.helpers import assert_reports_match, bound, encode_mode, events_key, from_dev, op, to_dev

pytestmark = pytest.mark.gpu

F = None


@pytest.fixture(scope="module", autouse=True, params=["fused", "fused_copy", "fused_local", "prepass"])
def _lib(request):
    global F
    from paper_2104_00897_b200 import ftblas
    ftblas.load()
    F = ftblas
    with encode_mode(F, request.param):
        yield
    F.ftblas_set_interval(0)
    F.ftblas_set_correction(F.CORRECT_RECOMPUTE)


def rand(rng, r, c, dist="uniform"):
    if dist == "uniform":
        return np.asfortranarray(rng.uniform(-1, 1, (r, c)))
    if dist == "normal":
        return np.asfortranarray(rng.standard_normal((r, c)))
    return np.asfortranarray(rng.integers(-8, 9, (r, c)).astype(float))


def stored(X, t):
    return np.asfortranarray(X.T) if t == "T" else X


def run(A, B, C0, Kc, *, ta="N", tb="N", alpha=1.0, beta=0.0, faults=(), subtract=False):
    m, k = op(A, ta).shape
    n = op(B, tb).shape[1]
    lda, ldb = A.shape[0], B.shape[0]
    dA, dB, dC = to_dev(A), to_dev(B), to_dev(C0)
    F.ftblas_set_interval(Kc)
    F.ftblas_set_correction(F.CORRECT_SUBTRACT if subtract else F.CORRECT_RECOMPUTE)
    try:
        if faults:
            F.ftblas_inject_arm(faults)
        rep = F.ftblas_dgemm(ta, tb, m, n, k, alpha, dA, lda, dB, ldb, beta, dC, m)
    finally:
        F.ftblas_set_interval(0)
        F.ftblas_set_correction(F.CORRECT_RECOMPUTE)
    Cg = from_dev(dC, m, n)
    Co, orep = oracle.dgemm_abft(ta, tb, m, n, k, alpha, A, lda, B, ldb, beta, C0, m,
                                 BM=rep.unit_rows, BN=rep.unit_cols, BK=rep.step_quantum, Kc=Kc,
                                 faults=list(faults), subtract=subtract)
    Co = Co.reshape((n, m)).T
    tol = bound(None, A, B, C0, alpha, beta, ta, tb, k)
    bad = ~(np.abs(Cg - Co) <= tol)
    assert not bad.any(), f"{bad.sum()} out of bound at {np.argwhere(bad)[:3]}"
    assert rep.unit_k == min(Kc, k) and rep.units_checked == orep.units_checked
    return Cg, rep, orep


def test_interval_argument_checked():
    from paper_2104_00897_b200.ftblas import FtblasError
    with pytest.raises(FtblasError):
        F.ftblas_set_interval(10)  # not a multiple of the step quantum
    with pytest.raises(FtblasError):
        F.ftblas_set_interval(-16)


@pytest.mark.parametrize("trans", ["NN", "NT", "TN", "TT"])
@pytest.mark.parametrize("Kc", [16, 48, 64])
def test_intervals_faults_across_intervals(trans, Kc):
    rng = np.random.default_rng(400 + Kc)
    m, n, k = 260, 200, 150  # ragged tiles and a ragged last interval
    A, B, C0 = rand(rng, m, k), rand(rng, k, n), rand(rng, m, n)
    faults = [(3, 4, 0, 5.0),          # interval 0, first update
              (3, 4, k, -7.0),         # same cell, after the last update (last interval)
              (130, 150, 64, 2.5),     # an interval boundary when Kc divides 64
              (200, 10, 100, 1e3), (201, 11, 101, -40.0)]  # same unit, maybe same interval
    _, rep, orep = run(stored(A, trans[0]), stored(B, trans[1]), C0, Kc, ta=trans[0], tb=trans[1],
                       alpha=1.5, beta=-0.5, faults=faults)
    assert_reports_match(rep, orep, stored(A, trans[0]), stored(B, trans[1]), trans[0], trans[1], k)
    assert rep.detected >= 4


def test_intervals_integer_exact_and_per_interval_events():
    rng = np.random.default_rng(410)
    m, n, k = 254, 254, 128
    A, B = rand(rng, m, k, "int"), rand(rng, k, n, "int")
    # one fault per interval in the same cell: every interval reports its own correction
    faults = [(10, 20, 32 * t + 5, float(t + 1)) for t in range(4)]
    Cg, rep, orep = run(A, B, np.zeros((m, n)), 32, faults=faults)
    assert np.array_equal(Cg, A @ B)
    assert events_key(rep.events) == [(t, 10, 20, 1) for t in range(4)] == events_key(orep.events)
    assert [e[4] for e in rep.events] == [1.0, 2.0, 3.0, 4.0]
    assert (rep.corrected, rep.recomputed) == (4, 0)


def test_intervals_no_false_positives_and_subtract():
    rng = np.random.default_rng(411)
    for Kc in (16, 32, 112):
        m, n, k = (int(x) for x in rng.integers(1, 300, 3))
        A, B = rand(rng, m, k, "normal"), rand(rng, k, n, "normal")
        _, rep, _ = run(A, B, np.zeros((m, n)), Kc)
        assert rep.detected == 0
    m, n, k = 200, 150, 96
    A, B = rand(rng, m, k, "int"), rand(rng, k, n, "int")
    Cg, rep, orep = run(A, B, np.zeros((m, n)), 32, faults=[(150, 3, 33, 77.0), (15, 130, 90, -3.0)],
                        subtract=True)
    assert rep.corrected == 2 and np.array_equal(Cg, A @ B)
    assert_reports_match(rep, orep)


@pytest.mark.parametrize("trans", ["NN", "TT"])
def test_intervals_beyond_tau_table(trans):
    """T = 100 intervals (Kc = 16, k = 1600): the kernel forms the tau factors of intervals
    t < 64 before the k-loop and computes the later ones inline at the check (TAU_TAB); events in
    both ranges, a recompute decided at t = 80 (two faults, two rows and two columns) and
    verification of the intervals after it, all equal to the oracle's."""
    rng = np.random.default_rng(420)
    m, n, k, Kc = 200, 190, 1600, 16
    A, B, C0 = rand(rng, m, k), rand(rng, k, n), rand(rng, m, n)
    faults = [(5, 6, 3 * 16 + 2, 4.0),                           # t = 3 (table)
              (150, 20, 70 * 16, -9.0),                          # t = 70 (inline)
              (40, 50, 80 * 16 + 1, 2.0), (41, 60, 80 * 16 + 3, 3.0),  # t = 80: recompute
              (41, 60, 90 * 16, 5.0),                            # t = 90, after the recompute
              (199, 189, k, 1e3)]                                # the last interval (t = 99)
    _, rep, orep = run(stored(A, trans[0]), stored(B, trans[1]), C0, Kc, ta=trans[0], tb=trans[1],
                       alpha=1.0, beta=0.5, faults=faults)
    assert_reports_match(rep, orep, stored(A, trans[0]), stored(B, trans[1]), trans[0], trans[1], k)
    assert rep.units_checked == 4 * 100 and rep.recomputed == 1 and rep.corrected == 4
