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
            assert det == (1, 1)  # faults are corrected by the protection: counted, X fault-free


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
