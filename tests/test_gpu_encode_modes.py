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
