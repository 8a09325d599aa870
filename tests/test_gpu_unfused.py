"""GPU parity of the UNFUSED ABFT baseline (ftblas_dgemm_unfused)
against the CPU oracle run with the same 128 x 128 unit geometry: values within
2 k u (|alpha||A||B| + |beta||C0|), identical counters and sorted (interval, i, j, kind)
events, residuals within 4 tau."""
import numpy as np
import pytest

import oracle
from tests.helpers import assert_reports_match, bound, events_key, from_dev, op, to_dev

pytestmark = pytest.mark.gpu

F = None


@pytest.fixture(scope="module", autouse=True)
def _lib():
    global F
    from paper_2104_00897_b200 import ftblas
    ftblas.load()
    F = ftblas
    yield
    F.ftblas_set_correction(F.CORRECT_RECOMPUTE)


def rand(rng, r, c, dist="uniform"):
    if dist == "uniform":
        return np.asfortranarray(rng.uniform(-1, 1, (r, c)))
    if dist == "normal":
        return np.asfortranarray(rng.standard_normal((r, c)))
    return np.asfortranarray(rng.integers(-8, 9, (r, c)).astype(float))


def stored(X, t):
    return np.asfortranarray(X.T) if t == "T" else X


def run_unfused(A, B, C0, *, ta="N", tb="N", alpha=1.0, beta=0.0, faults=(), subtract=False,
                check_values=True, Kc=0):
    m, k = op(A, ta).shape
    n = op(B, tb).shape[1]
    lda, ldb = max(A.shape[0], 1), max(B.shape[0], 1)
    dA, dB, dC = to_dev(A), to_dev(B), to_dev(C0)
    F.ftblas_set_correction(F.CORRECT_SUBTRACT if subtract else F.CORRECT_RECOMPUTE)
    F.ftblas_set_interval(Kc)
    try:
        if faults:
            F.ftblas_inject_arm(faults)
        rep = F.ftblas_dgemm_unfused(ta, tb, m, n, k, alpha, dA, lda, dB, ldb, beta, dC, max(m, 1))
    finally:
        F.ftblas_set_correction(F.CORRECT_RECOMPUTE)
        F.ftblas_set_interval(0)
    assert (rep.unit_rows, rep.unit_cols) == (128, 128)
    Cg = from_dev(dC, m, n)
    Co, orep = oracle.dgemm_abft(ta, tb, m, n, k, alpha, A, lda, B, ldb, beta, C0, max(m, 1),
                                 BM=128, BN=128, BK=rep.step_quantum, faults=list(faults),
                                 subtract=subtract, Kc=Kc or None)
    Co = Co.reshape((n, m)).T
    if check_values:
        tol = bound(None, A, B, C0, alpha, beta, ta, tb, k)
        bad = ~(np.abs(Cg - Co) <= tol)
        assert not bad.any(), f"{bad.sum()} elements out of bound at {np.argwhere(bad)[:3]}"
    return Cg, Co, rep, orep


@pytest.mark.parametrize("trans", ["NN", "NT", "TN", "TT"])
def test_unfused_shapes_and_faults(trans):
    rng = np.random.default_rng(300)
    for (m, n, k) in [(1, 1, 1), (7, 5, 3), (128, 128, 16), (129, 130, 17), (300, 260, 100),
                      (257, 65, 33)]:
        A, B, C0 = rand(rng, m, k), rand(rng, k, n), rand(rng, m, n)
        faults = [(int(rng.integers(0, m)), int(rng.integers(0, n)), int(rng.integers(0, k + 1)),
                   float(rng.choice([-1, 1]) * 10.0 ** rng.uniform(-2, 4)))]
        _, _, rep, orep = run_unfused(stored(A, trans[0]), stored(B, trans[1]), C0, ta=trans[0],
                                      tb=trans[1], faults=faults)
        assert rep.units_checked == orep.units_checked
        assert_reports_match(rep, orep, stored(A, trans[0]), stored(B, trans[1]), trans[0],
                             trans[1], k)
        assert rep.corrected == 1


def test_unfused_integer_residuals_exact_and_bitwise():
    rng = np.random.default_rng(301)
    m, n, k = 256, 384, 96
    A, B = rand(rng, m, k, "int"), rand(rng, k, n, "int")
    for _ in range(40):
        i, j = int(rng.integers(0, m)), int(rng.integers(0, n))
        step = int(rng.integers(0, k + 1))
        delta = float(rng.integers(1, 10000)) * (1 if rng.random() < 0.5 else -1)
        Cg, _, rep, _ = run_unfused(A, B, np.zeros((m, n)), faults=[(i, j, step, delta)])
        (t, ei, ej, kind, rr, rc), = rep.events
        assert (t, ei, ej, kind) == (0, i, j, 1) and rr == delta and rc == delta
        assert np.array_equal(Cg, A @ B)


def test_unfused_alpha_beta_scratch_path_and_multi():
    rng = np.random.default_rng(302)
    m, n, k = 300, 260, 120
    A, B, C0 = rand(rng, m, k, "normal"), rand(rng, k, n, "normal"), rand(rng, m, n)
    faults = [(5, 6, 10, 3.0), (70, 100, 50, -2.0), (200, 200, 119, 50.0), (290, 10, 120, 1e4)]
    _, _, rep, orep = run_unfused(A, B, C0, alpha=1.5, beta=0.5, faults=faults)
    assert_reports_match(rep, orep, A, B, "N", "N", k)
    assert rep.recomputed == 1 and rep.corrected == 2


def test_unfused_subtract_mode_and_no_false_positives():
    rng = np.random.default_rng(303)
    m, n, k = 200, 150, 70
    A, B = rand(rng, m, k, "int"), rand(rng, k, n, "int")
    Cg, _, rep, orep = run_unfused(A, B, np.zeros((m, n)), faults=[(150, 3, 33, 77.0)],
                                   subtract=True)
    assert rep.corrected == 1 and np.array_equal(Cg, A @ B)
    assert_reports_match(rep, orep)
    for r in range(6):
        m, n, k = (int(x) for x in rng.integers(1, 400, 3))
        A, B = rand(rng, m, k, ["uniform", "normal"][r % 2]), rand(rng, k, n)
        _, _, rep, _ = run_unfused(A, B, np.zeros((m, n)))
        assert rep.detected == 0


def test_unfused_nan_input_recomputed():
    rng = np.random.default_rng(304)
    m, n, k = 150, 140, 40
    A, B, C0 = rand(rng, m, k), rand(rng, k, n), rand(rng, m, n)
    A[10, 5] = np.nan
    Cg, _, rep, orep = run_unfused(A, B, C0, check_values=False)
    assert rep.recomputed == orep.recomputed >= 1
    assert events_key(rep.events) == events_key(orep.events)
    assert np.isnan(Cg[10]).all() and not np.isnan(np.delete(Cg, 10, axis=0)).any()


@pytest.mark.parametrize("trans", ["NN", "TT"])
@pytest.mark.parametrize("Kc", [16, 48, 64])
def test_unfused_intervals_match_oracle(trans, Kc):
    """The unfused baseline verifying every Kc updates: per interval the slice
    GEMM, the skinny checksum GEMMs, C e first and e^T C only on a mismatch; counters and the
    sorted (interval, i, j, kind) events equal the oracle's with the same Kc, including a unit
    recomputed in interval 0 that verifies clean (and then corrects a new fault) later (R6')."""
    rng = np.random.default_rng(310 + Kc)
    m, n, k = 260, 200, 150
    A, B, C0 = rand(rng, m, k), rand(rng, k, n), rand(rng, m, n)
    faults = [(3, 4, 0, 5.0), (3, 4, k, -7.0), (130, 70, Kc, 2.5), (131, 71, Kc + 1, 9.0),
              (10, 150, 2 * Kc, -1e3), (250, 199, k - 1, 0.125), (140, 60, 140, 3.0)]
    _, _, rep, orep = run_unfused(stored(A, trans[0]), stored(B, trans[1]), C0, ta=trans[0],
                                  tb=trans[1], faults=faults, Kc=Kc, alpha=1.25, beta=-0.5)
    assert rep.unit_k == Kc and rep.units_checked == orep.units_checked == 3 * 2 * -(-k // Kc)
    assert_reports_match(rep, orep, stored(A, trans[0]), stored(B, trans[1]), trans[0], trans[1], k)
    assert rep.recomputed >= 1 and rep.corrected >= 3
