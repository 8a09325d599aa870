"""GPU edge cases of the method against the oracle (through the C ABI):

  - faults in the checksum lanes themselves (reading R6: one-direction flags -> recompute);
  - the detection threshold: the kernel's tau is the oracle's R1 tau widened only by its
    rounded-up maxima and fixed-point encode term (R1', R17): probed with faults just below and
    just above tau on data whose clean residuals are exactly zero;
  - data whose magnitudes take the encoder's rare paths: max|x| < 2^-972 (the exact
    subnormal-aware fixed-point pass) and |x| >= 2^1017 (the exact integer maximum);
  - infinite inputs (reading R13: every unit that reads one is recomputed; IEEE results).
"""
import numpy as np
import pytest

import oracle
from tests.helpers import U, assert_reports_match, bound, events_key, from_dev, op, to_dev

pytestmark = pytest.mark.gpu
F = None


@pytest.fixture(scope="module", autouse=True)
def _lib():
    global F
    from paper_2104_00897_b200 import ftblas
    ftblas.load()
    F = ftblas
    F.ftblas_set_encode(F.ENCODE_FUSED)
    F.ftblas_set_correction(F.CORRECT_RECOMPUTE)
    yield


def both(A, B, *, ta="N", tb="N", faults=(), cs_faults=(), alpha=1.0, beta=0.0, C0=None):
    m, k = op(A, ta).shape
    n = op(B, tb).shape[1]
    C0 = np.zeros((m, n)) if C0 is None else C0
    dA, dB, dC = to_dev(A), to_dev(B), to_dev(C0)
    if faults:
        F.ftblas_inject_arm(faults)
    if cs_faults:
        F.ftblas_inject_arm_checksum(cs_faults)
    rep = F.ftblas_dgemm(ta, tb, m, n, k, alpha, dA, A.shape[0], dB, B.shape[0], beta, dC, m)
    Cg = from_dev(dC, m, n)
    BM, BN, BK = F.ftblas_get_geometry()
    Co, orep = oracle.dgemm_abft(ta, tb, m, n, k, alpha, A, A.shape[0], B, B.shape[0], beta, C0, m,
                                 BM=BM, BN=BN, BK=BK, faults=list(faults) + list(cs_faults))
    return Cg, Co.reshape((n, m)).T, rep, orep


def rnd(rng, r, c):
    return np.asfortranarray(rng.uniform(-1, 1, (r, c)))


@pytest.mark.parametrize("trans", ["NN", "NT", "TN", "TT"])
def test_checksum_lane_faults(trans):
    """A fault in a carried checksum flags one column (lane 1) or one row (lane 2) and nothing
    in the other direction: the unit is recomputed (R6); C stays within the bound, events and
    residuals match the oracle.  Full tiles, odd tiles (checksum row 0) and a ragged edge."""
    rng = np.random.default_rng(51)
    m, n, k = 300, 280, 200
    A, B = rnd(rng, m, k), rnd(rng, k, n)
    As = np.asfortranarray(A.T) if trans[0] == "T" else A
    Bs = np.asfortranarray(B.T) if trans[1] == "T" else B
    cs = [(5, 9, 32, 2.0, 1), (140, 200, 0, -7.5, 2), (299, 279, 200, 1e3, 1), (130, 3, 100, 0.5, 2)]
    data = [(20, 150, 64, 4.0)]  # a data fault in another unit, corrected as usual
    Cg, Co, rep, orep = both(As, Bs, ta=trans[0], tb=trans[1], faults=data, cs_faults=cs)
    assert (rep.detected, rep.corrected, rep.recomputed) == (5, 1, 4)
    assert_reports_match(rep, orep, As, Bs, trans[0], trans[1], k)
    assert np.all(np.abs(Cg - Co) <= bound(None, As, Bs, np.zeros((m, n)), 1.0, 0.0, trans[0], trans[1], k))
    for e in rep.events:
        if e[3] == 2:
            assert (e[4] == 0.0) != (e[5] == 0.0)  # one direction only


def test_checksum_lane_faults_rejected_elsewhere():
    """Checksum-lane faults belong to ftblas_dgemm: the unprotected twin returns 3 (and
    disarms), an unknown lane is refused when armed."""
    import torch
    d = torch.zeros(64 * 64, dtype=torch.float64, device="cuda")
    F.ftblas_inject_arm_checksum([(1, 1, 0, 1.0, 1)])
    assert F.ftblas_dgemm_noft("N", "N", 64, 64, 64, 1.0, d, 64, d, 64, 0.0, d, 64, raw_status=True) == 3
    assert F.ftblas_dgemm("N", "N", 64, 64, 64, 1.0, d, 64, d, 64, 0.0, d, 64).detected == 0  # disarmed
    with pytest.raises(Exception):
        F.ftblas_inject_arm_checksum([(1, 1, 0, 1.0, 3)])


@pytest.mark.parametrize("k", [256, 1024])
def test_threshold_probe_kernel_tau_just_above_oracle_tau(k):
    """Data whose clean product, sums and carried checksums are exactly zero (rows of A sum to
    0, columns of B constant, integers): a fault at step = k gives residuals exactly delta.
    With tau_o the oracle's R1 threshold (exact maxima), delta = 0.999 tau_o must not flag and
    delta = w tau_o must flag on the GPU, w = 1.0001 (1 + 4/(k+len)) (1+2^-20)^2: the kernel's
    tau lies in [tau_o, w tau_o) -- its R1' rounded-up maxima and R17 encode term (8u per
    element against the 2 gamma(k+len) ~ 2 (k+len) u of R1) widen tau by no more than that."""
    rng = np.random.default_rng(k)
    m = n = 254
    A = rng.integers(-3, 4, (m, k)).astype(float)
    A[:, -1] = -A[:, :-1].sum(axis=1)
    A = np.asfortranarray(A)
    B = np.asfortranarray(np.tile(rng.integers(-5, 6, (1, n)).astype(float), (k, 1)))
    BM, BN, _ = F.ftblas_get_geometry()
    amax, bmax = np.abs(A[:BM]).max(), np.abs(B[:, :BN]).max()
    g = (k + BM) * U / (1 - (k + BM) * U)
    tau_o = 2 * g * k * BM * amax * bmax
    assert tau_o == oracle.tau(k, BM, amax, bmax)
    w = 1.0001 * (1 + 4 / (k + BM)) * (1 + 2.0 ** -20) ** 2
    for scale, flagged in ((0.999, False), (w, True)):
        Cg, Co, rep, orep = both(A, B, faults=[(30, 40, k, scale * tau_o)])
        assert rep.detected == orep.detected == int(flagged), (scale, rep, orep)
        if flagged:
            assert events_key(rep.events) == events_key(orep.events) == [(0, 30, 40, 1)]
            assert rep.events[0][4] == rep.events[0][5] == scale * tau_o  # exact residuals
        assert np.array_equal(Cg, Co)


@pytest.mark.parametrize("scale_a,scale_b", [(2.0 ** -1000, 2.0 ** 60), (2.0 ** 1018, 2.0 ** -1000)])
def test_extreme_magnitudes_take_the_exact_encode_paths(scale_a, scale_b):
    """max|A| < 2^-972 (the encoder's exact fixed-point pass, subnormal-aware; some entries are
    subnormal) and |A| >= 2^1017 (pass 1's float view overflows: the exact integer maximum).
    Products stay normal, so the bound applies; faults are located as by the oracle."""
    rng = np.random.default_rng(61)
    m, n, k = 260, 140, 96
    A = rnd(rng, m, k) * scale_a
    if scale_a < 1:
        A[::7, ::5] *= 2.0 ** -60  # subnormal entries (< 2^-1022)
        assert np.any((A != 0) & (np.abs(A) < 2.0 ** -1022))
    B = rnd(rng, k, n) * scale_b
    unit = scale_a * scale_b * k
    faults = [(3, 4, 48, 50.0 * unit), (200, 130, 96, -20.0 * unit), (140, 10, 0, 5.0 * unit)]
    Cg, Co, rep, orep = both(A, B, faults=faults)
    assert (rep.detected, rep.corrected) == (3, 3)
    assert_reports_match(rep, orep, A, B, "N", "N", k)
    assert np.all(np.abs(Cg - Co) <= bound(None, A, B, np.zeros((m, n)), 1.0, 0.0, "N", "N", k))


def test_infinite_inputs_recompute_their_units():
    """An infinite element of A (B) makes every unit of its tile row (column) flag through its
    non-finite residuals (tau is finite, R13) and be recomputed; the IEEE results (+-Inf, NaN)
    are order-independent, so GPU and oracle agree element by element; all other units are
    within the bound and clean."""
    rng = np.random.default_rng(71)
    m, n, k = 300, 260, 64
    A, B = rnd(rng, m, k), rnd(rng, k, n)
    A[150, 10] = np.inf
    B[20, 5] = -np.inf
    Cg, Co, rep, orep = both(A, B, faults=[(10, 200, 32, 9.0)])
    assert events_key(rep.events) == events_key(orep.events)
    assert rep.recomputed == orep.recomputed >= 3 and rep.corrected == orep.corrected == 1
    assert np.array_equal(np.isnan(Cg), np.isnan(Co))
    inf = np.isinf(Co)
    assert np.array_equal(np.isinf(Cg), inf) and np.array_equal(np.sign(Cg[inf]), np.sign(Co[inf]))
    fin = np.isfinite(Co)
    S = np.abs(A) @ np.abs(B)
    with np.errstate(invalid="ignore"):
        assert np.all(np.abs(Cg - Co)[fin] <= (2 * k * U * S)[fin])
