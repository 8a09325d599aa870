"""Pins for the CPU oracle (-m "not gpu").

Each test checks the oracle against something other than itself: hand-worked
examples (tests/golden, cited), exact integer arithmetic (numpy int64 matmul),
closed forms (identity / diagonal), a library routine within the rounding bound
(numpy float64 matmul), invariants of the checksum algebra, and
analytic predictions of the classification.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")
U = 2.0 ** -53


def F(x):
    return np.asfortranarray(np.asarray(x, dtype=np.float64))


def int_mats(rng, m, n, k, bound=8):
    A = F(rng.integers(-bound, bound + 1, size=(m, k)))
    B = F(rng.integers(-bound, bound + 1, size=(k, n)))
    return A, B


def run(A, B, *, ta="N", tb="N", alpha=1.0, beta=0.0, C0=None, BM=32, BN=32, BK=8, Kc=None,
        faults=(), subtract=False, units=None):
    A, B = F(A), F(B)
    m = A.shape[1] if ta == "T" else A.shape[0]
    k = A.shape[0] if ta == "T" else A.shape[1]
    n = B.shape[0] if tb == "T" else B.shape[1]
    if C0 is None:
        C0 = np.zeros((m, n), order="F")
    Cf, rep = oracle.dgemm_abft(ta, tb, m, n, k, alpha, A, max(A.shape[0], 1), B,
                                max(B.shape[0], 1), beta, F(C0), max(m, 1), BM=BM, BN=BN, BK=BK,
                                Kc=Kc, faults=faults, subtract=subtract, units=units)
    return Cf.reshape((n, m)).T if m * n else np.zeros((m, n)), rep


# ---------------------------------------------------------------------------- golden
def test_encode_worked_examples():
    g = json.load(open(os.path.join(GOLD, "worked_examples.json")))
    for ex in g["encode"]:
        M = np.array(ex["M"], dtype=float)
        assert oracle.row_sums(M).tolist() == ex["row_sums"]
        assert oracle.col_sums(M).tolist() == ex["col_sums"]


def test_rank_k_update_worked_examples():
    """Carried checksums after the rank-k update equal the worked values."""
    g = json.load(open(os.path.join(GOLD, "worked_examples.json")))
    for ex in g["rank_k_update"]:
        A, B = np.array(ex["A"], float), np.array(ex["B"], float)
        C, rep = run(A, B, BM=8, BN=8, BK=1)
        assert rep.detected == 0
        # the maintained sums equal the reference sums of the exact product
        assert oracle.row_sums(C).tolist() == ex["row_sums"]
        assert oracle.col_sums(C).tolist() == ex["col_sums"]


def test_verify_locate_correct_worked_example():
    """C(0,1) corrupted 22 -> 25 is located at (0,1) with magnitude 3 and restored to 22
    (PAPER.md:258 locate, 445 correct)."""
    g = json.load(open(os.path.join(GOLD, "worked_examples.json")))["verify"]
    A, B = np.array(g["A"], float), np.array(g["B"], float)
    C_ok, rep0 = run(A, B, BM=2, BN=2, BK=1)
    assert C_ok.tolist() == g["C"]
    assert oracle.row_sums(C_ok).tolist() == g["maintained_row_sums"]
    assert oracle.col_sums(C_ok).tolist() == g["maintained_col_sums"]
    c = g["corrupt"]
    delta = c["value"] - g["C"][c["i"]][c["j"]]
    for subtract in (False, True):
        C, rep = run(A, B, BM=2, BN=2, BK=1, faults=[(c["i"], c["j"], 2, delta)], subtract=subtract)
        assert (rep.detected, rep.corrected, rep.recomputed) == (1, 1, 0)
        (t, i, j, kind, rr, rc), = rep.events
        e = g["expect_single_error"]
        assert (i, j, kind) == (e["i"], e["j"], 1)
        assert rr == e["magnitude"] and rc == e["magnitude"]
        assert C[c["i"], c["j"]] == g["corrected_value"]
        assert C.tolist() == g["C"]


def test_two_corruptions_different_rows_is_out_of_model():
    """Two corruptions in different rows -> not a single error -> recomputed once."""
    A = np.array([[1, 2], [3, 4]], float)
    B = np.array([[5, 6], [7, 8]], float)
    C, rep = run(A, B, BM=2, BN=2, BK=1, faults=[(0, 1, 2, 3.0), (1, 0, 2, -5.0)])
    assert (rep.detected, rep.corrected, rep.recomputed) == (1, 0, 1)
    assert rep.events[0][3] == 2 and rep.events[0][1:3] == (0, 0)
    assert C.tolist() == [[19, 22], [43, 50]]


def test_hand_multiply():
    A = np.array([[1, 2], [3, 4]], float)
    B = np.array([[5, 6], [7, 8]], float)
    C = oracle.gemm_plain("N", "N", 2, 2, 2, 1.0, A, 2, B, 2, 0.0, np.zeros((2, 2)), 2)
    assert C.reshape(2, 2, order="F").tolist() == [[19, 22], [43, 50]]


def test_splitmix64_reference_vector():
    g = json.load(open(os.path.join(GOLD, "splitmix64.json")))
    s = synth.SplitMix64(g["seed"])
    assert [format(s.next_u64(), "016x") for _ in g["outputs_hex"]] == g["outputs_hex"]


def test_fault_generator_properties():
    f = synth.seeded_faults(7, 1000, 300, 200, 100, -2.0, 4.0)
    assert f == synth.seeded_faults(7, 1000, 300, 200, 100, -2.0, 4.0)  # determinism
    i, j, s, d = (np.array(c) for c in zip(*f))
    assert i.min() >= 0 and i.max() < 300 and j.min() >= 0 and j.max() < 200
    assert s.min() >= 0 and s.max() < 100
    assert np.all(np.abs(d) >= 1e-2) and np.all(np.abs(d) <= 1e4)
    assert 0.4 < np.mean(d < 0) < 0.6
    assert f != synth.seeded_faults(8, 1000, 300, 200, 100, -2.0, 4.0)


# ----------------------------------------------------------------- exact / closed forms
@pytest.mark.parametrize("trans", ["NN", "NT", "TN", "TT"])
def test_brute_force_integer_exact(trans):
    """Integer inputs |x| <= 8, m,n,k <= 64: every partial sum < 2^53, so the oracle's
    product must equal the exact integer product (numpy int64 matmul) bit for bit."""
    rng = np.random.default_rng(11)
    for _ in range(40):
        m, n, k = (int(x) for x in rng.integers(1, 65, 3))
        A, B = int_mats(rng, m, n, k)
        exact = (A.astype(np.int64) @ B.astype(np.int64)).astype(float)
        As = F(A.T) if trans[0] == "T" else A
        Bs = F(B.T) if trans[1] == "T" else B
        C, rep = run(As, Bs, ta=trans[0], tb=trans[1], BM=16, BN=8, BK=4)
        assert np.array_equal(C, exact)
        assert rep.detected == 0
        assert rep.units_checked == math.ceil(m / 16) * math.ceil(n / 8)
        Cp = oracle.gemm_plain(trans[0], trans[1], m, n, k, 1.0, As, As.shape[0], Bs, Bs.shape[0],
                               0.0, np.zeros((m, n)), m).reshape((n, m)).T
        assert np.array_equal(Cp, exact)


def test_checksum_invariant_integers():
    """e^T(AB) = (e^T A)B and (AB)e = A(Be), exact on integers."""
    rng = np.random.default_rng(3)
    for _ in range(30):
        m, n, k = (int(x) for x in rng.integers(1, 50, 3))
        A, B = int_mats(rng, m, n, k)
        C, _ = run(A, B)
        assert np.array_equal(oracle.col_sums(C), oracle.col_sums(A) @ B)
        assert np.array_equal(oracle.row_sums(C), A @ oracle.row_sums(B))


def test_identity_and_diagonal_closed_forms():
    rng = np.random.default_rng(5)
    for m, n in [(1, 1), (7, 13), (64, 33), (130, 70)]:
        B = F(rng.uniform(-1, 1, (m, n)))
        C, rep = run(np.eye(m), B, BM=32, BN=16, BK=8)
        assert np.array_equal(C, B) and rep.detected == 0          # A = I: C = B bitwise
        d = rng.uniform(-2, 2, m)
        C, rep = run(np.diag(d), B, BM=32, BN=16, BK=8)
        assert np.array_equal(C, d[:, None] * B) and rep.detected == 0  # one rounding each


def test_identity_alpha_beta():
    rng = np.random.default_rng(6)
    m, n = 40, 24
    B = F(rng.uniform(-1, 1, (m, n)))
    C0 = F(rng.uniform(-1, 1, (m, n)))
    C, _ = run(np.eye(m), B, alpha=1.5, beta=-0.25, C0=C0)
    assert np.array_equal(C, 1.5 * B + (-0.25) * C0)


@pytest.mark.parametrize("trans", ["NN", "NT", "TN", "TT"])
def test_against_numpy_within_bound(trans):
    """|C - C_np| <= 2 k u (|alpha||A||B| + |beta||C0|) elementwise (gamma_k bound)."""
    rng = np.random.default_rng(17)
    for m, n, k in [(65, 127, 257), (200, 31, 90), (128, 128, 300)]:
        A = F(rng.standard_normal((m, k)))
        B = F(rng.standard_normal((k, n)))
        C0 = F(rng.uniform(-1, 1, (m, n)))
        As = F(A.T) if trans[0] == "T" else A
        Bs = F(B.T) if trans[1] == "T" else B
        C, rep = run(As, Bs, ta=trans[0], tb=trans[1], alpha=1.5, beta=0.5, C0=C0, BM=64, BN=32)
        ref = 1.5 * (A @ B) + 0.5 * C0
        bound = 2 * k * U * (1.5 * (np.abs(A) @ np.abs(B)) + 0.5 * np.abs(C0))
        assert np.all(np.abs(C - ref) <= bound)
        assert rep.detected == 0


def test_quick_returns_and_beta_zero_nan():
    rng = np.random.default_rng(8)
    A = F(rng.uniform(-1, 1, (9, 5)))
    B = F(rng.uniform(-1, 1, (5, 7)))
    C0 = F(rng.uniform(-1, 1, (9, 7)))
    C, rep = run(A, B, alpha=0.0, beta=2.0, C0=C0)
    assert np.array_equal(C, 2.0 * C0) and rep.units_checked == 0
    C, rep = run(A, B, alpha=0.0, beta=0.0, C0=C0)
    assert np.array_equal(C, np.zeros_like(C0))
    C, rep = run(np.zeros((9, 0)), np.zeros((0, 7)), beta=1.0, C0=C0)
    assert np.array_equal(C, C0) and rep.units_checked == 0
    Cn = C0.copy()
    Cn[3, 4] = np.nan
    C, rep = run(A, B, beta=0.0, C0=Cn)
    assert not np.isnan(C).any()


def test_nonfinite_input_flags_and_recomputes():
    """NaN in op(A) -> residuals NaN -> flagged (not |d| <= tau) -> recomputed once (R13)."""
    rng = np.random.default_rng(9)
    A = F(rng.uniform(-1, 1, (20, 10)))
    A[3, 2] = np.nan
    B = F(rng.uniform(-1, 1, (10, 12)))
    C, rep = run(A, B, BM=16, BN=16)
    assert rep.detected == 1 and rep.recomputed == 1
    assert rep.units_checked == 2


# ---------------------------------------------------------------- detection/correction
def test_single_injection_campaign_integer_exact():
    """>= 500 single injections on integer-exact inputs: (i, j) exact, residuals exactly
    delta, corrected C bitwise equal to the fault-free C (SPEC.md:143 / PAPER.md:445)."""
    rng = np.random.default_rng(21)
    trials = 0
    while trials < 520:
        m, n, k = (int(x) for x in rng.integers(1, 65, 3))
        A, B = int_mats(rng, m, n, k)
        clean, _ = run(A, B, BM=16, BN=16, BK=4)
        i, j = int(rng.integers(0, m)), int(rng.integers(0, n))
        step = int(rng.integers(0, k + 1))
        delta = float(rng.integers(1, 1000)) * (1 if rng.random() < 0.5 else -1)
        for subtract in (False, True):
            C, rep = run(A, B, BM=16, BN=16, BK=4, faults=[(i, j, step, delta)], subtract=subtract)
            assert (rep.detected, rep.corrected, rep.recomputed) == (1, 1, 0)
            (t, ei, ej, kind, rr, rc), = rep.events
            assert (ei, ej, kind, t) == (i, j, 1, 0)
            assert rr == delta and rc == delta
            assert np.array_equal(C, clean)
        trials += 1


def test_no_false_positives_float_inputs():
    """Fault-free float inputs: the rigorous tau never flags (R1), >= 500 runs."""
    rng = np.random.default_rng(22)
    for r in range(520):
        m, n, k = (int(x) for x in rng.integers(1, 70, 3))
        dist = r % 3
        if dist == 0:
            A, B = F(rng.uniform(-1, 1, (m, k))), F(rng.uniform(-1, 1, (k, n)))
        elif dist == 1:
            A, B = F(rng.standard_normal((m, k))), F(rng.standard_normal((k, n)))
        else:  # wide dynamic range
            A = F(rng.standard_normal((m, k)) * 10.0 ** rng.integers(-8, 8, (m, k)))
            B = F(rng.standard_normal((k, n)) * 10.0 ** rng.integers(-8, 8, (k, n)))
        _, rep = run(A, B, BM=16, BN=32, BK=8, Kc=int(rng.integers(1, k + 1)))
        assert rep.detected == 0


def test_threshold_boundary_exact_maxima():
    """R1 with exact maxima.  Integer data built so that every partial product, sum and
    carried checksum is exactly 0 (rows of A sum to 0, columns of B constant): a fault applied
    after the last update (step = k) gives residuals exactly delta, so a delta just below
    tau(I, J) is not flagged and one just above is located.  tau uses the unit's own maxima
    max|op(A)_I:| and max|op(B)_:J| (larger values in another row block do not enter it)."""
    rng = np.random.default_rng(29)
    m, n, k = 64, 64, 96
    A = rng.integers(-3, 4, (m, k)).astype(float)
    A[:, -1] = -A[:, :-1].sum(axis=1)
    A[40:, :] *= 1024.0  # row block 1: larger values must not enter unit (0, 0)'s tau
    A = F(A)
    B = F(np.tile(rng.integers(-5, 6, (1, n)).astype(float), (k, 1)))
    g = lambda nn: nn * U / (1 - nn * U)  # noqa: E731
    amax, bmax = np.abs(A[:32]).max(), np.abs(B[:, :32]).max()
    tau = 2 * g(k + 32) * k * 32 * amax * bmax  # tau_col == tau_row: 32 x 32 unit
    for scale, flagged in ((0.999, False), (1.001, True)):
        _, rep = run(A, B, BM=32, BN=32, BK=4, faults=[(5, 7, k, scale * tau)])
        assert (rep.detected == 1) == flagged, (scale, rep)
        if flagged:
            assert rep.events[0][1:4] == (5, 7, 1)
            assert rep.events[0][4] == rep.events[0][5] == scale * tau


def test_nonfinite_residual_always_flags():
    """R13: tau is clamped to the largest finite double, so a unit with an infinite input (tau
    would be infinite) is still flagged by its non-finite residuals and recomputed."""
    rng = np.random.default_rng(31)
    m, n, k = 40, 40, 24
    A, B = F(rng.uniform(-1, 1, (m, k))), F(rng.uniform(-1, 1, (k, n)))
    A[3, 5] = np.inf
    C, rep = run(A, B, BM=32, BN=32, BK=4)
    assert rep.detected >= 1 and rep.corrected + rep.recomputed == rep.detected
    assert all(e[3] == 2 for e in rep.events if e[1] == 0)


def test_threshold_closed_form_and_detection_edge():
    assert oracle.gamma(1) == U / (1 - U)
    assert oracle.gamma(0) == 0.0
    assert oracle.tau(10, 4, 2.0, 3.0) == 2.0 * (14 * U / (1 - 14 * U)) * 10 * 4 * 2.0 * 3.0
    rng = np.random.default_rng(23)
    m, n, k = 48, 40, 100
    A, B = F(rng.uniform(-1, 1, (m, k))), F(rng.uniform(-1, 1, (k, n)))
    amax, bmax = np.abs(A[:32]).max(), np.abs(B[:, :32]).max()
    big = 3.0 * oracle.tau(k, 32, amax, bmax)  # > 2 tau: must be located
    _, rep = run(A, B, BM=32, BN=32, BK=4, faults=[(5, 7, 50, big)])
    assert (rep.corrected, rep.recomputed) == (1, 0) and rep.events[0][1:3] == (5, 7)
    _, rep = run(A, B, BM=32, BN=32, BK=4, faults=[(5, 7, 50, 0.0)])
    assert rep.detected == 0


def analytic_classes(faults, m, n, k, BM, BN, BK, Kc):
    """Group faults by (tile, interval); merge same-cell; one distinct cell -> corrected."""
    T = -(-k // Kc)
    units = {}
    for (i, j, s, d) in faults:
        sq = (s // BK) * BK
        t = min(sq // Kc, T - 1)
        units.setdefault((i // BM, j // BN, t), {}).setdefault((i, j), 0.0)
        units[(i // BM, j // BN, t)][(i, j)] += d
    ev = []
    for (ti, tj, t), cells in units.items():
        cells = {c: v for c, v in cells.items() if v != 0.0}
        if not cells:
            continue
        if len(cells) == 1:
            (i, j), = cells
            ev.append((t, i, j, 1))
        else:
            ev.append((t, ti * BM, tj * BN, 2))
    return sorted(ev)


def test_multi_error_bookkeeping_matches_analytic():
    rng = np.random.default_rng(24)
    for _ in range(60):
        m, n, k = (int(x) for x in rng.integers(8, 90, 3))
        A, B = int_mats(rng, m, n, k)
        clean, _ = run(A, B, BM=16, BN=16, BK=4)
        Kc = int(rng.choice([k, max(4, k // 3)]))
        nf = int(rng.integers(1, 8))
        faults = [(int(rng.integers(0, m)), int(rng.integers(0, n)), int(rng.integers(0, k + 1)),
                   float(rng.integers(1, 500)) * rng.choice([-1, 1])) for _ in range(nf)]
        if rng.random() < 0.3:  # force a same-cell collision
            faults.append((faults[0][0], faults[0][1], int(rng.integers(0, k + 1)), 7.0))
        C, rep = run(A, B, BM=16, BN=16, BK=4, Kc=Kc, faults=faults)
        got = [(t, i, j, kind) for (t, i, j, kind, _, _) in rep.events]
        assert got == analytic_classes(faults, m, n, k, 16, 16, 4, Kc)
        assert rep.detected == rep.corrected + rep.recomputed == len(got)
        assert rep.units_checked == -(-m // 16) * -(-n // 16) * -(-k // Kc)
        assert np.array_equal(C, clean)  # recompute mode restores the exact product


def test_interval_membership_and_step_quantisation():
    """Fault at step 130 with BK=16 is applied after 128 updates (R8) and belongs to
    interval floor(128/Kc); with Kc=64 that is interval 2."""
    rng = np.random.default_rng(25)
    A, B = int_mats(rng, 32, 32, 256)
    _, rep = run(A, B, BM=32, BN=32, BK=16, Kc=64, faults=[(3, 4, 130, 5.0)])
    assert rep.events[0][:4] == (2, 3, 4, 1)
    # two faults in different intervals of one unit are both corrected
    _, rep = run(A, B, BM=32, BN=32, BK=16, Kc=64, faults=[(3, 4, 10, 5.0), (9, 1, 200, 2.0)])
    assert [e[:4] for e in rep.events] == [(0, 3, 4, 1), (3, 9, 1, 1)]
    # step == k lands in the last interval
    _, rep = run(A, B, BM=32, BN=32, BK=16, Kc=64, faults=[(3, 4, 256, 5.0)])
    assert rep.events[0][:4] == (3, 3, 4, 1)


def test_residual_float_within_2tau_of_delta():
    rng = np.random.default_rng(26)
    m = n = k = 96
    A, B = F(rng.standard_normal((m, k))), F(rng.standard_normal((k, n)))
    for d in (1e-2, 3.0, -1e4):
        _, rep = run(A, B, BM=32, BN=32, BK=8, faults=[(40, 70, 33, d)])
        (t, i, j, kind, rr, rc), = rep.events
        amax, bmax = np.abs(A[32:64]).max(), np.abs(B[:, 64:96]).max()
        tau = oracle.tau(k, 32, amax, bmax)
        assert abs(rr - d) <= 2 * tau + 4 * U * abs(d) * k
        assert abs(rc - d) <= 2 * tau + 4 * U * abs(d) * k


def test_sampled_units_equal_full_run():
    rng = np.random.default_rng(27)
    m, n, k = 100, 90, 70
    A, B = F(rng.uniform(-1, 1, (m, k))), F(rng.uniform(-1, 1, (k, n)))
    C0 = F(rng.uniform(-1, 1, (m, n)))
    faults = [(5, 5, 10, 9.0), (70, 80, 60, -3.0)]
    full, rf = run(A, B, alpha=1.5, beta=0.5, C0=C0, faults=faults)
    part, rp = run(A, B, alpha=1.5, beta=0.5, C0=C0, faults=faults, units=[(0, 0), (2, 2)])
    assert np.array_equal(part[:32, :32], full[:32, :32])
    assert np.array_equal(part[64:96, 64:90], full[64:96, 64:90])
    assert np.array_equal(part[40:60, 40:60], C0[40:60, 40:60])  # untouched
    assert [e[:4] for e in rp.events] == [e[:4] for e in rf.events]


def test_gemm_elements_matches_full():
    rng = np.random.default_rng(28)
    m, n, k = 33, 41, 29
    A, B = F(rng.uniform(-1, 1, (k, m))), F(rng.uniform(-1, 1, (n, k)))
    C0 = F(rng.uniform(-1, 1, (m, n)))
    full = oracle.gemm_plain("T", "T", m, n, k, 2.0, A, k, B, n, -1.0, C0, m).reshape((n, m)).T
    ii = rng.integers(0, m, 50)
    jj = rng.integers(0, n, 50)
    el = oracle.gemm_elements("T", "T", k, 2.0, A, k, B, n, -1.0, ii, jj, C0[ii, jj])
    assert np.array_equal(el, full[ii, jj])
    S = oracle.abs_product_elements("T", "T", k, A, k, B, n, ii, jj)
    assert np.allclose(S, (np.abs(A.T) @ np.abs(B.T))[ii, jj], rtol=1e-13)


def test_checksum_lane_fault_flags_one_direction_and_recomputes():
    """Reading R6: a fault in a CARRIED checksum (lane 1: the column checksum of column j, lane 2:
    the row checksum of row i) flags that one column (row) and no row (column): out of the
    one-error pattern, so the unit is recomputed; on integer data the residual is exactly -delta
    and C equals the exact product."""
    rng = np.random.default_rng(37)
    m, n, k = 70, 50, 40
    A, B = int_mats(rng, m, n, k)
    exact = A.astype(np.int64) @ B.astype(np.int64)
    for lane, (i, j) in ((1, (5, 9)), (2, (40, 33))):
        C, rep = run(A, B, BM=32, BN=32, BK=8, faults=[(i, j, 16, 3.0, lane)])
        assert (rep.detected, rep.corrected, rep.recomputed) == (1, 0, 1)
        (t, ei, ej, kind, rr, rc), = rep.events
        assert kind == 2 and (ei, ej) == ((i // 32) * 32, (j // 32) * 32)
        assert (rr, rc) == ((0.0, -3.0) if lane == 1 else (-3.0, 0.0))
        assert np.array_equal(C, exact)


def test_recomputed_unit_gets_fresh_checksums_for_later_intervals():
    """Reading R6 with intervals: a unit recomputed at the end of interval t is re-formed as a
    whole C^f block (data AND carried checksums), so a checksum-lane fault of interval 0 is
    reported once (interval 0, recomputed) and interval 1 of the same unit verifies clean;
    a data fault in interval 1 of that unit is then corrected as usual."""
    rng = np.random.default_rng(43)
    m, n, k = 40, 40, 64
    A, B = int_mats(rng, m, n, k)
    exact = A.astype(np.int64) @ B.astype(np.int64)
    C, rep = run(A, B, BM=32, BN=32, BK=8, Kc=32, faults=[(3, 4, 8, 5.0, 1)])
    assert [(e[0], e[3]) for e in rep.events] == [(0, 2)] and rep.units_checked == 4 * 2
    assert np.array_equal(C, exact)
    C, rep = run(A, B, BM=32, BN=32, BK=8, Kc=32, faults=[(3, 4, 8, 5.0, 1), (6, 7, 40, 2.0)])
    assert [(e[0], e[1], e[2], e[3]) for e in rep.events] == [(0, 0, 0, 2), (1, 6, 7, 1)]
    assert np.array_equal(C, exact)
