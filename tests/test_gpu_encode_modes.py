"""The in-kernel encode modes of ftblas_dgemm agree bitwise: e^T A_I shared along tile rows
and B_J e along tile columns (published by tile column 0 / tile row 0 and copied by the
others -- forced with dev modes 256 | 512, and as scheduled) and every CTA encoding itself run
the same integer fixed-point encode on the same staged data (R17, R22), so C, the
counters and every event's residuals must be identical to the last bit."""
import numpy as np
import pytest

from tests.helpers import encode_mode, from_dev, to_dev

pytestmark = pytest.mark.gpu


def stored(X, t):
    return np.asfortranarray(X.T) if t == "T" else X


@pytest.mark.parametrize("trans", ["NN", "NT", "TN", "TT"])
def test_row_shared_encode_bitwise_equals_local(trans):
    from paper_2104_00897_b200 import ftblas as F
    F.load()
    ta, tb = trans
    rng = np.random.default_rng(900 + hash(trans) % 100)
    m, n, k = 700, 900, 530  # 6 x 8 tiles, ragged edges and a ragged last stage
    A, B, C0 = rng.standard_normal((m, k)), rng.uniform(-1, 1, (k, n)), rng.uniform(-1, 1, (m, n))
    As, Bs = stored(A, ta), stored(B, tb)
    faults = [(3, 500, 100, 7.5), (650, 10, 529, -3.0), (200, 300, 0, 1e3), (201, 301, 17, 2.0)]
    out = {}
    for name in ("fused_local", "fused_copy", "fused"):
        with encode_mode(F, name):
            dC = to_dev(C0)
            F.ftblas_inject_arm(faults)
            rep = F.ftblas_dgemm(ta, tb, m, n, k, 0.75, to_dev(As), As.shape[0], to_dev(Bs), Bs.shape[0],
                                 -1.5, dC, m)
            out[name] = (from_dev(dC, m, n), rep)
    C_ref, r_ref = out["fused_local"]
    assert r_ref.detected == 3 and r_ref.corrected == 2 and r_ref.recomputed == 1
    for name in ("fused_copy", "fused"):
        C, r = out[name]
        assert np.array_equal(C.view(np.int64), C_ref.view(np.int64)), name
        assert (r.units_checked, r.detected, r.corrected, r.recomputed) == \
            (r_ref.units_checked, r_ref.detected, r_ref.corrected, r_ref.recomputed)
        assert [tuple(e) for e in r.events] == [tuple(e) for e in r_ref.events], name


def test_row_shared_encode_multi_wave_bitwise():
    """Several waves of tiles: later waves find e^T A_I / B_J e published by earlier tiles and copy
    them, the first wave races its producers; either way the result is bitwise the local encode."""
    from paper_2104_00897_b200 import ftblas as F
    F.load()
    rng = np.random.default_rng(990)
    m, n, k = 3000, 2600, 200  # 24 x 21 tiles: 3.4 waves of 148 CTAs
    A, B = rng.uniform(-1, 1, (m, k)), rng.standard_normal((k, n))
    faults = [(int(i), int(j), int(s), float(d)) for i, j, s, d in
              zip(rng.integers(0, m, 12), rng.integers(0, n, 12), rng.integers(0, k, 12), rng.uniform(1, 9, 12))]
    out = {}
    for name in ("fused_local", "fused"):
        with encode_mode(F, name):
            dC = to_dev(np.zeros((m, n)))
            F.ftblas_inject_arm(faults)
            rep = F.ftblas_dgemm("N", "N", m, n, k, 1.0, to_dev(A), m, to_dev(B), k, 0.0, dC, m)
            out[name] = (from_dev(dC, m, n), rep)
    (C0, r0), (C1, r1) = out["fused_local"], out["fused"]
    assert np.array_equal(C0.view(np.int64), C1.view(np.int64))
    assert r0.detected == r1.detected >= 11 and r0.corrected == r1.corrected
    assert [tuple(e) for e in r0.events] == [tuple(e) for e in r1.events]
    assert np.allclose(C1, A @ B, rtol=0, atol=4 * k * 2.0 ** -53 * (np.abs(A) @ np.abs(B)).max())
