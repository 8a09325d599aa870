"""Pins of the DTRSM oracle: closed forms (unit
identity, diagonal with the packed reciprocal), exact integer solves for every uplo/trans,
and scipy's triangular solver within the rounding bound."""
import numpy as np
import scipy.linalg as sla

import oracle

U = 2.0 ** -53


def test_identity_and_diagonal_closed_forms():
    rng = np.random.default_rng(0)
    m, n = 50, 7
    B = np.asfortranarray(rng.uniform(-1, 1, (m, n)))
    X, _ = oracle.dtrsm("L", "N", "U", m, n, 2.5, np.asfortranarray(rng.uniform(-1, 1, (m, m))) * 0, m, B, m)
    assert np.array_equal(X.reshape((n, m)).T, 2.5 * B)  # unit diagonal, zero off-diagonal: X = alpha B
    d = rng.uniform(1, 2, m)
    A = np.asfortranarray(np.diag(d))
    for uplo in "LU":
        for tr in "NT":
            X, _ = oracle.dtrsm(uplo, tr, "N", m, n, 1.5, A, m, B, m)
            assert np.array_equal(X.reshape((n, m)).T, (1.5 * B) * (1.0 / d)[:, None])  # reciprocal multiply


def test_integer_exact_all_variants():
    rng = np.random.default_rng(1)
    m, n = 120, 9
    for uplo in "LU":
        T = rng.integers(-1, 2, (m, m)).astype(float)
        T = np.tril(T, -1) if uplo == "L" else np.triu(T, 1)
        T += np.eye(m)
        for tr in "NT":
            opT = T.T if tr == "T" else T
            X = rng.integers(-3, 4, (m, n)).astype(float)
            B = np.asfortranarray(opT @ X)
            Xo, _ = oracle.dtrsm(uplo, tr, "U", m, n, 1.0, np.asfortranarray(T), m, B, m)
            assert np.array_equal(Xo.reshape((n, m)).T, X)


def test_against_scipy_within_bound():
    rng = np.random.default_rng(2)
    m, n = 200, 13
    for uplo in "LU":
        A = rng.uniform(-1, 1, (m, m)) / m
        A = (np.tril(A) if uplo == "L" else np.triu(A)) + np.diag(rng.uniform(1, 2, m))
        A = np.asfortranarray(A)
        B = np.asfortranarray(rng.uniform(-1, 1, (m, n)))
        for tr in "NT":
            Xo, det = oracle.dtrsm(uplo, tr, "N", m, n, -0.75, A, m, B, m, faults=[(1, 0, 0, 1.0)])
            Xs = sla.solve_triangular(A, -0.75 * B, lower=(uplo == "L"), trans=(1 if tr == "T" else 0))
            Xo = Xo.reshape((n, m)).T
            assert np.max(np.abs(Xo - Xs)) <= 64 * m * U * np.max(np.abs(Xs))
            # faults are corrected by the protection (X fault-free); (1, 0, 0) sits in the one
            # diagonal block: a DMR detection and correction, no ABFT event
            assert (det.detected, det.corrected, det.n_events) == (1, 1, 0)


def test_right_side_closed_forms_integer_and_scipy():
    """Side R (X op(A) = alpha B): diagonal closed form with the packed reciprocal,
    exact integer solves for every uplo / trans, and scipy within the rounding bound."""
    rng = np.random.default_rng(3)
    m, n = 11, 60
    B = np.asfortranarray(rng.uniform(-1, 1, (m, n)))
    d = rng.uniform(1, 2, n)
    for uplo in "LU":
        for tr in "NT":
            X, _ = oracle.dtrsm(uplo, tr, "N", m, n, 1.5, np.asfortranarray(np.diag(d)), n, B, m, side="R")
            assert np.array_equal(X.reshape((n, m)).T, (1.5 * B) * (1.0 / d)[None, :])
    m, n = 9, 110
    for uplo in "LU":
        T = rng.integers(-1, 2, (n, n)).astype(float)
        T = (np.tril(T, -1) if uplo == "L" else np.triu(T, 1)) + np.eye(n)
        for tr in "NT":
            opT = T.T if tr == "T" else T
            X = rng.integers(-3, 4, (m, n)).astype(float)
            Bi = np.asfortranarray(X @ opT)
            Xo, _ = oracle.dtrsm(uplo, tr, "U", m, n, 1.0, np.asfortranarray(T), n, Bi, m, side="R")
            assert np.array_equal(Xo.reshape((n, m)).T, X)
    m, n = 17, 150
    for uplo in "LU":
        A = rng.uniform(-1, 1, (n, n)) / n
        A = np.asfortranarray((np.tril(A) if uplo == "L" else np.triu(A)) + np.diag(rng.uniform(1, 2, n)))
        Bs = np.asfortranarray(rng.uniform(-1, 1, (m, n)))
        for tr in "NT":
            Xo, _ = oracle.dtrsm(uplo, tr, "N", m, n, 0.5, A, n, Bs, m, side="R")
            opA = A.T if tr == "T" else A
            # X op(A) = 0.5 B  <=>  op(A)^T X^T = 0.5 B^T
            Xs = sla.solve_triangular(opA.T, 0.5 * Bs.T, lower=not ((uplo == "L") != (tr == "T"))).T
            Xo = Xo.reshape((n, m)).T
            assert np.max(np.abs(Xo - Xs)) <= 64 * n * U * np.max(np.abs(Xs))


def test_dtrsm_bookkeeping_hand_derived_split():
    """FT-DTRSM bookkeeping (reading R21) against the split worked out by hand for 300
    positions (leaf 128, units 127; include/ftblas.h): forward order solves [0, 46) (leaf),
    updates rows [46, 300) with k in [0, 46), then splits [46, 300) into the leaf [46, 174),
    the update rows [174, 300) with k in [46, 174) and the leaf [174, 300).  Units of the
    first update: 2 x 3, of the second 1 x 3 (n = 300 right-hand sides)."""
    bk = oracle.dtrsm_bookkeeping
    r = bk("L", "L", "N", 300, 300, [(200, 5, 10, 1.0)])  # row 200, step 10: first update
    assert (r.units_checked, r.detected, r.corrected, r.recomputed) == (9, 1, 1, 0)
    assert [e[:4] for e in r.events] == [(0, 200, 5, 1)]
    r = bk("L", "L", "N", 300, 300, [(100, 5, 60, 1.0)])  # both in the leaf [46, 174): DMR
    assert (r.detected, r.corrected, r.n_events) == (1, 1, 0)
    # two cells of one unit of the second update (rows 174.., k 46..174): recomputed, origin (174, 0)
    r = bk("L", "L", "N", 300, 300, [(180, 7, 100, 1.0), (185, 8, 50, 2.0), (181, 200, 60, 3.0)])
    assert (r.detected, r.corrected, r.recomputed) == (2, 1, 1)
    assert [e[:4] for e in r.events] == [(0, 174, 0, 2), (0, 181, 200, 1)]
    # two faults in one leaf block, same right-hand side: one DMR detection (per column)
    r = bk("L", "L", "N", 300, 300, [(100, 5, 60, 1.0), (120, 5, 50, 1.0), (120, 6, 50, 1.0)])
    assert (r.detected, r.corrected, r.n_events) == (2, 2, 0)
    # backward order (lower, transposed): leaf [254, 300) first, then rows [0, 254) with k in
    # [254, 300); row 10, step 280 -> that update, unit (0, 0)
    r = bk("L", "L", "T", 300, 300, [(10, 3, 280, 1.0)])
    assert [e[:4] for e in r.events] == [(0, 10, 3, 1)] and r.units_checked == 2 * 3 + 1 * 3
    # side R, forward (upper, not transposed): the same split over B's 300 columns; row i is the
    # right-hand side: (i 5, column 200, step 10) -> first update, unit (0, (200 - 46) // 127)
    r = bk("R", "U", "N", 260, 300, [(5, 200, 10, 1.0)])
    assert [e[:4] for e in r.events] == [(0, 5, 200, 1)] and r.units_checked == 3 * 2 + 3 * 1
