"""GPU parity of the DMR Level-1/2 routines against the oracle:
DSCAL / DAXPY bitwise (one rounding per element on both sides), DGEMV within
2 n u (|alpha| |op(A)||x| + |beta||y|) (different summation order), identical DMR counters
under injected faults, and the unprotected twins for the negative control."""
import numpy as np
import pytest

import oracle

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


def dev(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to("cuda")


def host(t):
    return t.detach().cpu().numpy()


@pytest.mark.parametrize("n,inc", [(1, 1), (1000, 1), (100003, 1), (4097, 3), (513, -2)])
def test_dscal_bitwise_with_faults(n, inc):
    rng = np.random.default_rng(n)
    x = rng.standard_normal(n * abs(inc))
    faults = [(int(i), 0, 0, float(rng.choice([-1, 1]) * 10 ** rng.uniform(-2, 3)))
              for i in rng.choice(n, size=min(5, n), replace=False)]
    dx = dev(x)
    F.ftblas_inject_arm(faults)
    rep = F.ftblas_dscal(n, 1.3, dx, inc)
    xo, orep = oracle.dscal(n, 1.3, x, inc, faults)
    assert np.array_equal(host(dx), xo)
    assert (rep.checked, rep.detected, rep.corrected, rep.uncorrectable) == \
           (orep.checked, orep.detected, orep.corrected, orep.uncorrectable)


@pytest.mark.parametrize("n,incx,incy", [(777, 1, 1), (100000, 1, 1), (999, 2, -1), (64, -1, 3)])
def test_daxpy_bitwise_with_faults(n, incx, incy):
    rng = np.random.default_rng(n + 7)
    x = rng.uniform(-1, 1, n * abs(incx))
    y = rng.uniform(-1, 1, n * abs(incy))
    faults = [(0, 0, 0, 1.0), (n - 1, 0, 0, -2.5), (n // 2, 0, 0, 1e-30)]
    dx, dy = dev(x), dev(y)
    F.ftblas_inject_arm(faults)
    rep = F.ftblas_daxpy(n, -0.7, dx, incx, dy, incy)
    yo, orep = oracle.daxpy(n, -0.7, x, incx, y, incy, faults)
    assert np.array_equal(host(dy), yo)
    assert (rep.checked, rep.detected, rep.corrected) == (orep.checked, orep.detected, orep.corrected)


@pytest.mark.parametrize("trans", ["N", "T"])
@pytest.mark.parametrize("m,n", [(1, 1), (33, 17), (300, 257), (1025, 64), (64, 2049)])
def test_dgemv_parity_with_faults(trans, m, n):
    rng = np.random.default_rng(m * 31 + n)
    A = np.asfortranarray(rng.uniform(-1, 1, (m, n)))
    lda = m + 3
    Ap = np.zeros((lda, n))
    Ap[:m] = A
    nx, ny = (n, m) if trans == "N" else (m, n)
    x = rng.uniform(-1, 1, nx)
    y = rng.uniform(-1, 1, ny)
    faults = [(int(rng.integers(0, ny)), 0, int(rng.integers(0, nx + 1)), 3.0),
              (ny - 1, 0, nx, -1.5)]
    dA, dx, dy = dev(Ap.reshape(-1, order="F")), dev(x), dev(y)
    F.ftblas_inject_arm(faults)
    rep = F.ftblas_dgemv(trans, m, n, 0.9, dA, lda, dx, 1, -0.3, dy, 1)
    yo, orep = oracle.dgemv(trans, m, n, 0.9, Ap, lda, x, 1, -0.3, y, 1, faults)
    opA = A if trans == "N" else A.T
    tol = 2 * nx * U * (0.9 * (np.abs(opA) @ np.abs(x)) + 0.3 * np.abs(y)) + 4 * U * np.abs(yo)
    assert np.all(np.abs(host(dy) - yo) <= tol)
    assert (rep.checked, rep.detected, rep.corrected) == (orep.checked, orep.detected, orep.corrected)
    assert rep.detected == len({f[0] for f in faults})


def test_dgemv_integer_exact_and_beta_zero():
    rng = np.random.default_rng(9)
    m, n = 200, 150
    A = np.asfortranarray(rng.integers(-8, 9, (m, n)).astype(float))
    for trans in "NT":
        nx, ny = (n, m) if trans == "N" else (m, n)
        x = rng.integers(-8, 9, nx).astype(float)
        dy = dev(np.full(ny, np.nan))
        F.ftblas_dgemv(trans, m, n, 1.0, dev(A.reshape(-1, order="F")), m, dev(x), 1, 0.0, dy, 1)
        assert np.array_equal(host(dy), (A if trans == "N" else A.T) @ x)


def test_noft_twins_are_silent_negative_control():
    rng = np.random.default_rng(11)
    n = 5000
    x = rng.uniform(-1, 1, n)
    dx = dev(x)
    F.ftblas_inject_arm([(17, 0, 0, 4.0)])
    F.ftblas_dscal_noft(n, 2.0, dx, 1)  # the twin has no DMR and does not inject
    assert np.array_equal(host(dx), 2.0 * x)
    F.ftblas_inject_disarm()


def test_argument_errors():
    from paper_2104_00897_b200.ftblas import FtblasError
    with pytest.raises(FtblasError):
        F.ftblas_dscal(-1, 1.0, None, 1)
    with pytest.raises(FtblasError):
        F.ftblas_daxpy(4, 1.0, dev(np.ones(4)), 0, dev(np.ones(4)), 1)
    with pytest.raises(FtblasError):
        F.ftblas_dgemv("X", 2, 2, 1.0, dev(np.ones(4)), 2, dev(np.ones(2)), 1, 0.0, dev(np.ones(2)), 1)
    F.ftblas_inject_arm([(10, 0, 0, 1.0)])
    with pytest.raises(FtblasError):  # fault index outside the 4 outputs
        F.ftblas_dscal(4, 1.0, dev(np.ones(4)), 1)


@pytest.mark.parametrize("m", [512, 2048 + 37, 5000])
def test_dgemv_t_fast_path_faults_settle_bitwise(m):
    """DGEMV 'T' on the unit-stride 16-byte aligned fast path (m >= 512): a fault in the
    original computation is settled by a third computation with the SAME lane partition and
    order, so every faulted column is counted corrected (never uncorrectable) and the stored y
    is bitwise the fault-free result of the unprotected twin.  Faults land in the vectorised
    blocks (both elements of a lane's pair) and in the remainder."""
    rng = np.random.default_rng(m)
    n = 96
    A = np.asfortranarray(rng.standard_normal((m, n)))
    x, y = rng.standard_normal(m), rng.standard_normal(n)
    steps = [0, 1, 63, 64, 511, m - 1, (m // 512) * 512 + 5 if m % 512 > 5 else 2]
    faults = [(j, 0, steps[j % len(steps)], float(rng.choice([-1, 1]) * 10 ** rng.uniform(-3, 3)))
              for j in range(0, n, 3)]
    dA, dx = dev(A.reshape(-1, order="F")), dev(x)
    dy, dy0 = dev(y), dev(y)
    F.ftblas_inject_arm(faults)
    rep = F.ftblas_dgemv("T", m, n, 0.75, dA, m, dx, 1, -0.5, dy, 1)
    F.ftblas_dgemv_noft("T", m, n, 0.75, dA, m, dx, 1, -0.5, dy0, 1)
    assert rep.detected == len(faults) and rep.corrected == len(faults) and rep.uncorrectable == 0
    assert np.array_equal(host(dy), host(dy0))
