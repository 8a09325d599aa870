"""Pins of the DMR Level-1/2 oracle: closed forms,
exact integer arithmetic, numpy within the rounding bound, reverse increments, and the DMR
bookkeeping (a fault perturbs the original copy only: detected and corrected, the stored
value is the fault-free one; a delta below half an ulp is not a detection)."""
import numpy as np

import oracle

U = 2.0 ** -53


def test_dscal_power_of_two_exact_and_numpy_bitwise():
    rng = np.random.default_rng(0)
    x = rng.standard_normal(1000)
    xo, rep = oracle.dscal(1000, 0.25, x)
    assert np.array_equal(xo, x / 4.0)  # scaling by 2^-2 is exact
    xo, _ = oracle.dscal(1000, 1.7, x)
    assert np.array_equal(xo, 1.7 * x)  # one IEEE multiplication each
    assert (rep.checked, rep.detected, rep.corrected, rep.uncorrectable) == (1000, 0, 0, 0)


def test_dscal_strided_and_reverse_increment():
    x = np.arange(12.0)
    xo, _ = oracle.dscal(4, 3.0, x, incx=3)
    expect = x.copy()
    expect[::3] *= 3.0
    assert np.array_equal(xo, expect)
    xo, _ = oracle.dscal(4, 3.0, x, incx=-3)  # same elements, visited backwards
    assert np.array_equal(xo, expect)


def test_daxpy_integer_exact_and_reverse():
    rng = np.random.default_rng(1)
    x = rng.integers(-50, 50, 777).astype(float)
    y = rng.integers(-50, 50, 777).astype(float)
    yo, _ = oracle.daxpy(777, 3.0, x, 1, y, 1)
    assert np.array_equal(yo, 3.0 * x + y)
    yo, _ = oracle.daxpy(777, 3.0, x, -1, y, 1)  # x read backwards (BLAS negative increment)
    assert np.array_equal(yo, 3.0 * x[::-1] + y)


def test_dgemv_closed_forms_and_numpy_bound():
    rng = np.random.default_rng(2)
    m, n = 37, 23
    A = np.asfortranarray(rng.uniform(-1, 1, (m, n)))
    x = rng.uniform(-1, 1, n)
    y0 = rng.uniform(-1, 1, m)
    yo, rep = oracle.dgemv("N", m, n, 1.5, A, m, x, 1, -0.5, y0, 1)
    ref = 1.5 * (A @ x) - 0.5 * y0
    tol = 2 * n * U * (1.5 * (np.abs(A) @ np.abs(x)) + 0.5 * np.abs(y0)) + 4 * U * np.abs(ref)
    assert np.all(np.abs(yo - ref) <= tol) and rep.checked == m
    xt = rng.uniform(-1, 1, m)
    yt = rng.uniform(-1, 1, n)
    yo, rep = oracle.dgemv("T", m, n, 2.0, A, m, xt, 1, 0.0, yt + np.nan, 1)  # beta == 0: y not read
    ref = 2.0 * (A.T @ xt)
    assert np.all(np.abs(yo - ref) <= 2 * m * U * 2.0 * (np.abs(A.T) @ np.abs(xt)) + 4 * U * np.abs(ref))
    assert rep.checked == n
    I = np.asfortranarray(np.eye(9))
    v = rng.integers(-9, 9, 9).astype(float)
    w = rng.integers(-9, 9, 9).astype(float)
    yo, _ = oracle.dgemv("N", 9, 9, 3.0, I, 9, v, 1, 2.0, w, 1)
    assert np.array_equal(yo, 3.0 * v + 2.0 * w)  # identity closed form, integers exact


def test_dgemv_integer_exact_all_trans_and_increments():
    rng = np.random.default_rng(3)
    m, n = 40, 31
    A = np.asfortranarray(rng.integers(-8, 9, (m, n)).astype(float))
    for tr, (nx, ny) in (("N", (n, m)), ("T", (m, n))):
        x = rng.integers(-8, 9, 2 * nx).astype(float)
        y = rng.integers(-8, 9, ny).astype(float)
        yo, _ = oracle.dgemv(tr, m, n, 1.0, A, m, x, 2, 1.0, y, 1)
        opA = A if tr == "N" else A.T
        assert np.array_equal(yo, opA @ x[::2] + y)


def test_dmr_fault_bookkeeping():
    x = np.linspace(-1, 1, 64)
    faults = [(3, 0, 0, 5.0), (3, 0, 0, -1.0), (10, 0, 0, 1e-30), (40, 0, 0, 0.25)]
    xo, rep = oracle.dscal(64, 2.0, x, 1, faults)
    assert np.array_equal(xo, 2.0 * x)            # stored values are the fault-free ones
    assert (rep.detected, rep.corrected) == (2, 2)  # index 10: 1e-30 is absorbed, not a detection
    y = np.zeros(64)
    yo, rep = oracle.daxpy(64, -1.0, x, 1, y, 1, [(0, 0, 0, 1.0), (63, 0, 0, 2.0)])
    assert np.array_equal(yo, -x) and rep.detected == 2
    A = np.asfortranarray(np.ones((8, 5)))
    yo, rep = oracle.dgemv("N", 8, 5, 1.0, A, 8, np.ones(5), 1, 0.0, np.zeros(8), 1,
                           [(2, 0, 3, 7.0), (2, 0, 5, 1.0), (7, 0, 0, -3.0)])
    assert np.array_equal(yo, np.full(8, 5.0)) and (rep.detected, rep.checked) == (2, 8)
