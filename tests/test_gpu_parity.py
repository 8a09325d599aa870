"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the same seeded
inputs.  Values within 2 k u (|alpha||A||B| + |beta||C0|) elementwise; counters and the
sorted (interval, i, j, kind) event lists identical; residuals within 4 tau."""
import numpy as np
import pytest

import oracle
import synth
from tests.helpers import (U, assert_reports_match, bound, encode_mode, events_key, from_dev, op,
                           to_dev)

pytestmark = pytest.mark.gpu

F = None


@pytest.fixture(scope="module", autouse=True, params=["fused", "fused_copy", "fused_local", "prepass"])
def _lib(request):
    """Every parity test runs under each encode mode of ftblas_dgemm: in-kernel fused encode
    with e^T A_I shared along tile rows (as scheduled, and with every tile forced to take the
    published copy: dev mode 256), every CTA encoding itself, and the pre-encoded checksums
    copied into the staged tiles."""
    global F
    from paper_2104_00897_b200 import ftblas
    ftblas.load()
    F = ftblas
    with encode_mode(F, request.param):
        yield
    F.ftblas_set_correction(F.CORRECT_RECOMPUTE)


def geometry():
    return F.ftblas_get_geometry()


def run_both(A, B, C0, *, ta="N", tb="N", alpha=1.0, beta=0.0, faults=(), lda=None, ldb=None,
             ldc=None, subtract=False, noft=False, check_values=True):
    m = op(A, ta).shape[0]
    k = op(A, ta).shape[1]
    n = op(B, tb).shape[1]
    lda = lda or max(A.shape[0], 1)
    ldb = ldb or max(B.shape[0], 1)
    ldc = ldc or max(m, 1)
    dA, dB, dC = to_dev(A, lda), to_dev(B, ldb), to_dev(C0, ldc)
    F.ftblas_set_correction(F.CORRECT_SUBTRACT if subtract else F.CORRECT_RECOMPUTE)
    if faults:
        F.ftblas_inject_arm(faults)
    if noft:
        F.ftblas_dgemm_noft(ta, tb, m, n, k, alpha, dA, lda, dB, ldb, beta, dC, ldc)
        import torch
        torch.cuda.synchronize()
        rep = None
    else:
        rep = F.ftblas_dgemm(ta, tb, m, n, k, alpha, dA, lda, dB, ldb, beta, dC, ldc)
    Cg = from_dev(dC, m, n, ldc)
    BM, BN, BK = geometry()
    Co, orep = oracle.dgemm_abft(ta, tb, m, n, k, alpha, A, A.shape[0] or 1, B, B.shape[0] or 1,
                                 beta, C0, max(m, 1), BM=BM, BN=BN, BK=BK,
                                 faults=[] if noft else faults, subtract=subtract)
    Co = Co.reshape((n, m)).T if m * n else np.zeros((m, n))
    if check_values and m * n:
        tol = bound(None, A, B, C0, alpha, beta, ta, tb, k)
        err = np.abs(Cg - Co)
        bad = ~(err <= tol)
        assert not bad.any(), f"{bad.sum()} elements out of bound, worst {err[bad].max()} at {np.argwhere(bad)[:3]}"
    return Cg, Co, rep, orep


def rand(rng, r, c, dist="uniform"):
    if dist == "uniform":
        return np.asfortranarray(rng.uniform(-1, 1, (r, c)))
    if dist == "normal":
        return np.asfortranarray(rng.standard_normal((r, c)))
    return np.asfortranarray(rng.integers(-8, 9, (r, c)).astype(float))


def stored(X, t):
    return np.asfortranarray(X.T) if t == "T" else X


@pytest.mark.parametrize("trans", ["NN", "NT", "TN", "TT"])
def test_brute_force_shapes(trans):
    rng = np.random.default_rng(100)
    shapes = [(1, 1, 1), (7, 5, 3), (64, 64, 64), (65, 127, 257), (129, 130, 17), (257, 65, 33),
              (128, 128, 16), (300, 200, 100)]
    shapes += [tuple(int(x) for x in rng.integers(1, 65, 3)) for _ in range(6)]
    for (m, n, k) in shapes:
        A, B = rand(rng, m, k), rand(rng, k, n)
        C0 = rand(rng, m, n)
        _, _, rep, orep = run_both(stored(A, trans[0]), stored(B, trans[1]), C0, ta=trans[0],
                                   tb=trans[1], alpha=1.5, beta=0.5)
        assert rep.detected == 0 and orep.detected == 0
        assert rep.units_checked == orep.units_checked


@pytest.mark.parametrize("trans", ["NN", "TT"])
def test_integer_exact_bitwise(trans):
    """Integer inputs within the exactness window: GPU C is bit-identical to the exact product."""
    rng = np.random.default_rng(101)
    for (m, n, k) in [(64, 64, 64), (130, 257, 64), (33, 17, 200)]:
        A, B = rand(rng, m, k, "int"), rand(rng, k, n, "int")
        Cg, Co, rep, _ = run_both(stored(A, trans[0]), stored(B, trans[1]), np.zeros((m, n)),
                                  ta=trans[0], tb=trans[1])
        assert np.array_equal(Cg, A @ B) and np.array_equal(Co, A @ B)


def test_unaligned_leading_dimensions_v8_path():
    rng = np.random.default_rng(102)
    m, n, k = 131, 77, 45
    A, B, C0 = rand(rng, m, k), rand(rng, k, n), rand(rng, m, n)
    # odd lda/ldb force the 8-byte cp.async path; padded ldc
    run_both(A, B, C0, alpha=-2.0, beta=0.25, lda=m + 1 if m % 2 == 0 else m, ldb=k + 2, ldc=m + 3)
    run_both(stored(A, "T"), stored(B, "T"), C0, ta="T", tb="T", lda=k, ldb=n)


def test_c1_config_single_error_detect_correct():
    c = synth.config("C1")
    Cg, Co, rep, orep = run_both(c.A, c.B, c.C0, faults=c.faults)
    assert (rep.detected, rep.corrected, rep.recomputed) == (1, 1, 0)
    assert events_key(rep.events) == [(0, 17, 203, 1)]
    assert_reports_match(rep, orep, c.A, c.B, "N", "N", c.k)
    clean = c.A @ c.B
    assert np.all(np.abs(Cg - clean) <= bound(None, c.A, c.B, c.C0, 1.0, 0.0, "N", "N", c.k))


def test_c2_config_full():
    c = synth.config("C2")
    Cg, Co, rep, orep = run_both(c.A, c.B, c.C0, alpha=c.alpha, beta=c.beta)
    assert rep.detected == 0 and orep.detected == 0
    assert rep.units_checked == orep.units_checked == -(-2048 // rep.unit_rows) * -(-2048 // rep.unit_cols)


def test_single_injection_campaign_integer_exact():
    """>= 500 single injections over several shapes/trans: exact (i, j), residuals exactly
    delta, corrected C bitwise equal to the fault-free product."""
    rng = np.random.default_rng(103)
    done = 0
    for trans in ["NN", "NT", "TN", "TT"]:
        m, n, k = 256, 384, 96
        A, B = rand(rng, m, k, "int"), rand(rng, k, n, "int")
        exact = A @ B
        dA, dB = to_dev(stored(A, trans[0])), to_dev(stored(B, trans[1]))
        lda, ldb = (k if trans[0] == "T" else m), (n if trans[1] == "T" else k)
        dC = to_dev(np.zeros((m, n)))
        for _ in range(130):
            i, j = int(rng.integers(0, m)), int(rng.integers(0, n))
            step = int(rng.integers(0, k + 1))
            delta = float(rng.integers(1, 10000)) * (1 if rng.random() < 0.5 else -1)
            F.ftblas_inject_arm([(i, j, step, delta)])
            rep = F.ftblas_dgemm(trans[0], trans[1], m, n, k, 1.0, dA, lda, dB, ldb, 0.0, dC, m)
            assert (rep.detected, rep.corrected, rep.recomputed) == (1, 1, 0)
            (t, ei, ej, kind, rr, rc), = rep.events
            assert (t, ei, ej, kind) == (0, i, j, 1)
            assert rr == delta and rc == delta
            done += 1
        assert np.array_equal(from_dev(dC, m, n), exact)
    assert done >= 500


def test_subtract_mode_integer_exact():
    rng = np.random.default_rng(104)
    m, n, k = 200, 150, 70
    A, B = rand(rng, m, k, "int"), rand(rng, k, n, "int")
    Cg, Co, rep, orep = run_both(A, B, np.zeros((m, n)), faults=[(150, 3, 33, 77.0)], subtract=True)
    assert rep.corrected == 1 and np.array_equal(Cg, A @ B)
    assert_reports_match(rep, orep)


def test_multi_error_units_match_oracle():
    rng = np.random.default_rng(105)
    m, n, k = 300, 260, 120
    A, B, C0 = rand(rng, m, k, "normal"), rand(rng, k, n, "normal"), rand(rng, m, n)
    BM, BN, BK = geometry()
    faults = [(5, 6, 10, 3.0), (70, 100, 50, -2.0),          # two cells, same unit -> recompute
              (200, 200, 119, 50.0), (200, 200, 3, 1.5),     # same cell twice -> corrected
              (290, 10, 120, 1e4), (129, 10, 0, 0.5)]
    Cg, Co, rep, orep = run_both(A, B, C0, alpha=1.0, beta=1.0, faults=faults)
    assert_reports_match(rep, orep, A, B, "N", "N", k)
    assert rep.recomputed == 1 and rep.corrected == 3


def test_fault_free_no_false_positives():
    rng = np.random.default_rng(106)
    for r in range(12):
        m, n, k = (int(x) for x in rng.integers(1, 400, 3))
        dist = ["uniform", "normal"][r % 2]
        A, B = rand(rng, m, k, dist), rand(rng, k, n, dist)
        if r % 3 == 2:
            A *= 10.0 ** rng.integers(-6, 6, A.shape)
        _, _, rep, _ = run_both(A, B, np.zeros((m, n)))
        assert rep.detected == 0


def test_negative_control_noft_silent():
    """The unprotected twin applies the same fault and nobody notices: C_ij is off by delta."""
    rng = np.random.default_rng(107)
    m, n, k = 140, 90, 64
    A, B = rand(rng, m, k, "int"), rand(rng, k, n, "int")
    Cg, Co, _, _ = run_both(A, B, np.zeros((m, n)), faults=[(17, 80, 30, 5.0)], noft=True,
                            check_values=False)
    diff = Cg - A @ B
    assert diff[17, 80] == 5.0 and np.count_nonzero(diff) == 1


def test_nan_input_is_recomputed_and_beta_zero_ignores_nan():
    rng = np.random.default_rng(108)
    m, n, k = 150, 140, 40
    A, B = rand(rng, m, k), rand(rng, k, n)
    A[10, 5] = np.nan
    C0 = rand(rng, m, n)
    C0[3, 3] = np.nan
    Cg, Co, rep, orep = run_both(A, B, C0, check_values=False)
    assert rep.recomputed == orep.recomputed >= 1
    assert events_key(rep.events) == events_key(orep.events)
    assert np.isnan(Cg[10]).all() and not np.isnan(np.delete(Cg, 10, axis=0)).any()


def test_quick_returns_on_device():
    import torch
    rng = np.random.default_rng(109)
    m, n = 50, 40
    C0 = rand(rng, m, n)
    dC = to_dev(C0)
    rep = F.ftblas_dgemm("N", "N", m, n, 0, 1.0, None, m, None, 1, 2.0, dC, m)
    assert rep.units_checked == 0 and np.array_equal(from_dev(dC, m, n), 2.0 * C0)
    F.ftblas_dgemm("N", "N", m, n, 5, 0.0, None, m, None, 5, 0.0, dC, m)
    assert not from_dev(dC, m, n).any()
    torch.cuda.synchronize()


def test_host_buffer_api_matches():
    rng = np.random.default_rng(110)
    m, n, k = 190, 170, 150
    A, B, C0 = rand(rng, m, k), rand(rng, k, n), rand(rng, m, n)
    C = np.asfortranarray(C0.copy())
    F.ftblas_inject_arm([(100, 100, 75, 10.0)])
    rep = F.ftblas_dgemm_host("N", "N", m, n, k, 1.5, A, m, B, k, 0.5, C, m)
    Co, orep = oracle.dgemm_abft("N", "N", m, n, k, 1.5, A, m, B, k, 0.5, C0, m,
                                 BM=rep.unit_rows, BN=rep.unit_cols, BK=rep.step_quantum,
                                 faults=[(100, 100, 75, 10.0)])
    assert_reports_match(rep, orep)
    assert np.all(np.abs(C - Co.reshape((n, m)).T) <= bound(None, A, B, C0, 1.5, 0.5, "N", "N", k))


@pytest.mark.parametrize("trans", ["NN", "NT", "TT"])
def test_host_buffer_pipeline_row_panels(trans):
    """m large enough for the row-panel pipeline of the host-buffer API (panels of a multiple
    of 254 rows, copies overlapped with compute; the first and last panels in column chunks of
    a multiple of 254 columns): faults in several panels and chunks, events with global rows
    and columns, counters summed over the pieces, values within the bound."""
    ta, tb = trans
    rng = np.random.default_rng(112)
    m, n, k = 4600, 300, 140
    A, B, C0 = rand(rng, m, k), rand(rng, k, n), rand(rng, m, n)
    As, Bs = stored(A, ta), stored(B, tb)
    lda, ldb = As.shape[0], Bs.shape[0]
    faults = [(5, 7, 10, 3.0), (10, 290, 20, 6.0), (1200, 100, 70, -2.0), (2541, 255, 139, 9.0),
              (4599, 0, 0, 1.5), (4598, 1, 5, 4.0), (4590, 280, 100, -3.0)]
    C = np.asfortranarray(C0.copy())
    F.ftblas_inject_arm(faults)
    rep = F.ftblas_dgemm_host(ta, tb, m, n, k, 1.25, As, lda, Bs, ldb, -0.5, C, m)
    Co, orep = oracle.dgemm_abft(ta, tb, m, n, k, 1.25, As, lda, Bs, ldb, -0.5, C0, m,
                                 BM=rep.unit_rows, BN=rep.unit_cols, BK=rep.step_quantum, faults=faults)
    assert rep.units_checked == orep.units_checked
    assert_reports_match(rep, orep, As, Bs, ta, tb, k)
    assert rep.detected == 6  # two faults share a unit
    assert np.all(np.abs(C - Co.reshape((n, m)).T) <= bound(None, A, B, C0, 1.25, -0.5, "N", "N", k))
    Ct = np.asfortranarray(np.zeros((m, n)))
    F.ftblas_dgemm_noft_host(ta, tb, m, n, k, 1.0, As, lda, Bs, ldb, 0.0, Ct, m)
    assert np.all(np.abs(Ct - A @ B) <= bound(None, A, B, np.zeros((m, n)), 1.0, 0.0, "N", "N", k))


@pytest.mark.parametrize("trans", ["NN", "TT"])
def test_host_buffer_pipeline_column_mode(trans):
    """m small against n: the host-buffer pipeline copies all of op(A), then streams op(B) and
    the result in column chunks over one panel (column mode).  Faults in several chunks;
    report and values as one call on the whole problem."""
    ta, tb = trans
    rng = np.random.default_rng(113)
    m, n, k = 4100, 8000, 300
    A, B, C0 = rand(rng, m, k), rand(rng, k, n), rand(rng, m, n)
    As, Bs = stored(A, ta), stored(B, tb)
    lda, ldb = As.shape[0], Bs.shape[0]
    faults = [(5, 7, 10, 3.0), (4099, 7999, 299, -4.0), (2000, 3500, 150, 2.0), (100, 6000, 0, 8.0),
              (3000, 1200, 300, -1.5)]
    C = np.asfortranarray(C0.copy())
    F.ftblas_inject_arm(faults)
    rep = F.ftblas_dgemm_host(ta, tb, m, n, k, 0.5, As, lda, Bs, ldb, 1.0, C, m)
    Co, orep = oracle.dgemm_abft(ta, tb, m, n, k, 0.5, As, lda, Bs, ldb, 1.0, C0, m,
                                 BM=rep.unit_rows, BN=rep.unit_cols, BK=rep.step_quantum, faults=faults)
    assert rep.units_checked == orep.units_checked
    assert_reports_match(rep, orep, As, Bs, ta, tb, k)
    assert rep.detected == 5 and rep.corrected == 5
    assert np.all(np.abs(C - Co.reshape((n, m)).T) <= bound(None, A, B, C0, 0.5, 1.0, "N", "N", k))


def test_nondefault_stream():
    import torch
    rng = np.random.default_rng(111)
    m, n, k = 256, 256, 256
    A, B = rand(rng, m, k), rand(rng, k, n)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        dA, dB, dC = to_dev(A), to_dev(B), to_dev(np.zeros((m, n)))
    F.ftblas_set_stream(s)
    try:
        F.ftblas_dgemm_noft("N", "N", m, n, k, 1.0, dA, m, dB, k, 0.0, dC, m)
        s.synchronize()
    finally:
        F.ftblas_set_stream(None)
    Co = oracle.gemm_plain("N", "N", m, n, k, 1.0, A, m, B, k, 0.0, np.zeros((m, n)), m)
    assert np.all(np.abs(from_dev(dC, m, n) - Co.reshape((n, m)).T) <=
                  bound(None, A, B, np.zeros((m, n)), 1.0, 0.0, "N", "N", k))
