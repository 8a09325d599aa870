"""Seeded randomised parity sweep over the protected DGEMM's configuration space: shapes with
ragged tiles, all trans combinations, alpha / beta, 0-4 faults (same-unit collisions included),
every encode mode, intervals Kc < k, and both entry points (device buffers and the host-buffer
pipeline).  Every case must match the oracle run with the same geometry: values within
2 k u (|alpha||A||B| + |beta||C0|), identical counters and sorted (interval, i, j, kind) events."""
import numpy as np
import pytest

import oracle
from tests.helpers import assert_reports_match, bound, encode_mode, from_dev, op, to_dev

pytestmark = pytest.mark.gpu

MODES = ["fused", "fused_copy", "fused_local", "prepass"]


def stored(X, t):
    return np.asfortranarray(X.T) if t == "T" else X


def case(seed):
    rng = np.random.default_rng(seed)
    hi = 1400 if seed % 8 == 7 else 520  # every eighth case spans several waves of tiles
    m, n, k = (int(x) for x in rng.integers(1, hi, 3))
    ta, tb = rng.choice(["N", "T"], 2)
    alpha = float(rng.choice([1.0, -0.75, 2.5]))
    beta = float(rng.choice([0.0, 1.0, 0.5]))
    nf = int(rng.integers(0, 5))
    faults = [(int(rng.integers(0, m)), int(rng.integers(0, n)), int(rng.integers(0, k + 1)),
               float(rng.choice([-1, 1]) * 10 ** rng.uniform(0, 3))) for _ in range(nf)]
    if nf >= 2 and rng.random() < 0.5:  # two faults in one unit
        i, j, s, d = faults[0]
        faults[1] = (min(m - 1, i + 1), j, s, -d)
    kc = int(rng.choice([0, 0, 16 * int(rng.integers(1, 12))]))
    mode = MODES[(seed // 8 + seed) % len(MODES)]  # every mode meets every shape class
    host = bool(rng.random() < 0.25)
    return m, n, k, str(ta), str(tb), alpha, beta, faults, kc, mode, host, rng


@pytest.mark.parametrize("seed", range(120))
def test_fuzz_against_oracle(seed):
    from paper_2104_00897_b200 import ftblas as F
    F.load()
    m, n, k, ta, tb, alpha, beta, faults, kc, mode, host, rng = case(seed)
    A = np.asfortranarray(rng.uniform(-1, 1, (m, k)))
    B = np.asfortranarray(rng.standard_normal((k, n)))
    C0 = np.asfortranarray(rng.uniform(-1, 1, (m, n)))
    As, Bs = stored(A, ta), stored(B, tb)
    # leading dimensions: tight, or padded (odd pads take the library's aligned-repack path)
    pad_a, pad_b = (int(x) for x in rng.choice([0, 0, 1, 3], 2))
    lda, ldb = As.shape[0] + pad_a, Bs.shape[0] + pad_b
    F.ftblas_set_interval(kc)
    try:
        with encode_mode(F, mode):
            F.ftblas_inject_arm(faults)
            if host:
                Cg = np.asfortranarray(C0.copy())
                Ap = np.zeros((lda, As.shape[1]), order="F"); Ap[:As.shape[0]] = As
                Bp = np.zeros((ldb, Bs.shape[1]), order="F"); Bp[:Bs.shape[0]] = Bs
                rep = F.ftblas_dgemm_host(ta, tb, m, n, k, alpha, Ap, lda, Bp, ldb, beta, Cg, m)
            else:
                dC = to_dev(C0)
                rep = F.ftblas_dgemm(ta, tb, m, n, k, alpha, to_dev(As, lda), lda, to_dev(Bs, ldb), ldb, beta, dC, m)
                Cg = from_dev(dC, m, n)
    finally:
        F.ftblas_set_interval(0)
    Co, orep = oracle.dgemm_abft(ta, tb, m, n, k, alpha, As, As.shape[0], Bs, Bs.shape[0], beta, C0, m,
                                 BM=rep.unit_rows, BN=rep.unit_cols, BK=rep.step_quantum,
                                 Kc=rep.unit_k, faults=faults)
    Co = Co.reshape((n, m)).T
    tol = bound(None, A, B, C0, alpha, beta, "N", "N", k)
    bad = ~(np.abs(Cg - Co) <= tol)
    assert not bad.any(), (seed, m, n, k, ta, tb, mode, kc, host, np.argwhere(bad)[:3])
    assert rep.units_checked == orep.units_checked
    assert_reports_match(rep, orep, As, Bs, ta, tb, k)
    assert op(As, ta).shape == (m, k)
