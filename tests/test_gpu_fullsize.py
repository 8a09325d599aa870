"""GPU parity at the BASELINE.json configurations themselves (C3 in all four trans
combinations, C4a, C4b), in the launch configuration bench.py times: the same seeded inputs
(synth.config) and fault lists, the default encode mode, full size.

The oracle cannot run 10^12-FLOP problems in seconds, so it runs on a sample of verification
units -- every unit holding a fault plus 64 seeded random units -- through the same oracle
entry point (oracle.dgemm_abft(..., units=...)); the paper itself checks every injected run
against a reference result (§VI.C).  Checked:
  - every element of every sampled unit within 2 k u (|alpha||op(A)||op(B)| + |beta||C0|);
  - identical counters and identical sorted (interval, i, j, kind) events (every fault unit is
    sampled, and a flag outside them would show up as an extra GPU event), residuals within
    4 tau;
  - every element of the whole C against cuBLAS (torch.matmul, a library routine) within twice
    the bound (both are within the bound of the exact product): a property that holds at any
    size and covers the units the oracle did not sample.
"""
import zlib

import numpy as np
import pytest

import oracle
import synth
from tests.helpers import U, assert_reports_match, events_key, op

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


def sampled_units(faults, m, n, BM, BN, seed, extra=64):
    """Every unit holding a fault, the ragged last tile row / column and corner, then `extra`
    seeded random units."""
    units = []
    for (i, j, _, _) in faults:
        if (i // BM, j // BN) not in units:
            units.append((i // BM, j // BN))
    tm, tn = -(-m // BM), -(-n // BN)
    for u in [(tm - 1, 0), (0, tn - 1), (tm - 1, tn - 1)]:
        if u not in units:
            units.append(u)
    want = min(len(units) + extra, tm * tn)
    rng = np.random.default_rng(seed)
    while len(units) < want:
        u = (int(rng.integers(0, tm)), int(rng.integers(0, tn)))
        if u not in units:
            units.append(u)
    return units


def op_views(dA, dB, c):
    """op(A) (m x k) and op(B) (k x n) as strided views of the column-major device buffers."""
    m, n, k = c.m, c.n, c.k
    Aop = dA.view(k, m).t() if c.ta == "N" else dA.view(m, k)
    Bop = dB.view(n, k).t() if c.tb == "N" else dB.view(k, n)
    return Aop, Bop


def run_config(c, extra_units=64):
    import torch
    m, n, k = c.m, c.n, c.k
    dA = torch.from_numpy(c.A.reshape(-1, order="F")).to("cuda")
    dB = torch.from_numpy(c.B.reshape(-1, order="F")).to("cuda")
    dC = torch.from_numpy(c.C0.reshape(-1, order="F")).to("cuda")
    F.ftblas_inject_arm(c.faults)
    rep = F.ftblas_dgemm(c.ta, c.tb, m, n, k, c.alpha, dA, c.lda, dB, c.ldb, c.beta, dC, c.ldc,
                         events_capacity=4096)
    BM, BN, BK = rep.unit_rows, rep.unit_cols, rep.step_quantum

    # (1) the whole C against cuBLAS within twice the bound
    Aop, Bop = op_views(dA, dB, c)
    ref = torch.matmul(Aop, Bop)
    S = torch.matmul(Aop.abs(), Bop.abs())
    Cg_t = dC.view(n, m).t()
    tol = 2.0 * (2 * k * U) * (abs(c.alpha) * S)
    if c.beta != 0.0:
        C0 = torch.from_numpy(c.C0.reshape(-1, order="F")).to("cuda").view(n, m).t()
        ref = c.alpha * ref + c.beta * C0
        tol = tol + 2.0 * (2 * k * U) * abs(c.beta) * C0.abs()
    else:
        ref = c.alpha * ref
    bad = ~((Cg_t - ref).abs() <= tol)
    assert int(bad.sum()) == 0, f"{int(bad.sum())} elements differ from cuBLAS beyond 2x the bound"
    del ref, S, bad, tol

    # (2) the sampled oracle: all fault units + seeded units
    units = sampled_units(c.faults, m, n, BM, BN, seed=zlib.crc32(c.name.encode()), extra=extra_units)
    Co, orep = oracle.dgemm_abft(c.ta, c.tb, m, n, k, c.alpha, c.A, c.lda, c.B, c.ldb, c.beta, c.C0,
                                 c.ldc, BM=BM, BN=BN, BK=BK, faults=c.faults, units=units)
    Co = Co.reshape((n, m)).T
    Cg = Cg_t.cpu().numpy()
    oA, oB = op(c.A, c.ta), op(c.B, c.tb)
    worst = 0.0
    for (ti, tj) in units:
        I = slice(ti * BM, min((ti + 1) * BM, m))
        J = slice(tj * BN, min((tj + 1) * BN, n))
        Sb = np.abs(oA[I, :]) @ np.abs(oB[:, J])
        bound = 2 * k * U * (abs(c.alpha) * Sb + abs(c.beta) * np.abs(c.C0[I, J]))
        err = np.abs(Cg[I, J] - Co[I, J])
        assert np.all(err <= bound), (c.name, ti, tj, float((err / np.maximum(bound, 1e-300)).max()))
        worst = max(worst, float((err / np.maximum(bound, 1e-300)).max()))
    assert orep.units_checked == len(units)
    assert rep.units_checked == -(-m // BM) * -(-n // BN)
    assert_reports_match(rep, orep, c.A, c.B, c.ta, c.tb, k)
    return rep, orep, worst


@pytest.mark.parametrize("trans", ["NN", "NT", "TN", "TT"])
def test_c3_full_size_parity(trans):
    """C3: 8192^3, N(0,1), 20 seeded single errors of magnitude 10^U(-2,4)."""
    c = synth.config("C3", trans=trans)
    rep, orep, worst = run_config(c)
    assert rep.detected == len({(i // rep.unit_rows, j // rep.unit_cols) for (i, j, _, _) in c.faults})
    assert rep.corrected + rep.recomputed == rep.detected


@pytest.mark.parametrize("name", ["C4a", "C4b"])
def test_c4_full_size_parity(name):
    """C4a 16384 x 16384 x 1024 and C4b 16384 x 512 x 16384, U[-1,1], errors at 1 per 10^11
    FLOPs (reading R10)."""
    c = synth.config(name)
    rep, orep, worst = run_config(c)
    assert rep.detected >= 1


def test_many_events_both_readbacks_and_capacity():
    """More than 200 faults in distinct units: both report read-backs (the first 32 events ride
    with the counters, the rest in a second copy) carry every event; a small events_capacity
    returns the FIRST events of the full sorted list (deterministic), n_events stays the total."""
    import torch
    m = n = 4064  # 32 x 32 units of 127
    k = 256
    rng = np.random.default_rng(77)
    A = np.asfortranarray(rng.uniform(-1, 1, (m, k)))
    B = np.asfortranarray(rng.uniform(-1, 1, (k, n)))
    cells = rng.choice(32 * 32, size=300, replace=False)
    faults = [(int(u % 32) * 127 + int(rng.integers(0, 127)), int(u // 32) * 127 + int(rng.integers(0, 127)),
               int(rng.integers(0, k + 1)), float(rng.choice([-1, 1]) * 10 ** rng.uniform(-2, 4))) for u in cells]
    dA = torch.from_numpy(A.reshape(-1, order="F")).to("cuda")
    dB = torch.from_numpy(B.reshape(-1, order="F")).to("cuda")
    dC = torch.zeros(m * n, dtype=torch.float64, device="cuda")
    F.ftblas_inject_arm(faults)
    rep = F.ftblas_dgemm("N", "N", m, n, k, 1.0, dA, m, dB, k, 0.0, dC, m, events_capacity=1000)
    Co, orep = oracle.dgemm_abft("N", "N", m, n, k, 1.0, A, m, B, k, 0.0, np.zeros((m, n)), m,
                                 BM=rep.unit_rows, BN=rep.unit_cols, BK=rep.step_quantum, faults=faults)
    assert rep.n_events == orep.n_events == 300 and len(rep.events) == 300
    assert_reports_match(rep, orep, A, B, "N", "N", k)
    Cg = dC.view(n, m).t().cpu().numpy()
    S = np.abs(A) @ np.abs(B)
    assert np.all(np.abs(Cg - Co.reshape((n, m)).T) <= 2 * k * U * S)
    # capacity 50: the first 50 events of the sorted list
    F.ftblas_inject_arm(faults)
    rep2 = F.ftblas_dgemm("N", "N", m, n, k, 1.0, dA, m, dB, k, 0.0, dC, m, events_capacity=50)
    assert rep2.n_events == 300 and events_key(rep2.events) == events_key(orep.events)[:50]


@pytest.mark.parametrize("trans", ["NN", "TT"])
def test_few_wave_ksplit_parity(trans):
    """A launch the host splits in k (wave_ksplit: 156 tiles on 148 SMs, k = 2048 -> 2 splits
    of 64 stages, 312 CTAs in 3 rounds instead of 2 full-length ones), with faults in both
    splits' k-ranges, after the last update (step = k: the owner adds it to the summed block)
    and a two-fault unit (recomputed unsplit by the tile's owner), beta != 0: values within the
    bound and events / counters equal to the oracle's on every fault unit + seeded units."""
    m, n, k = 12 * 127, 13 * 127, 2048
    faults = [(10, 20, 0, 3.0),                          # split 0, first update
              (400, 700, 1000, -50.0),                   # split 0 (stages 0..63)
              (900, 1200, 1500, 7.5),                    # split 1 (stages 64..127)
              (1523, 1650, k, 1e3),                      # after the last update, corner unit
              (3 * 127 + 5, 4 * 127 + 6, 300, 2.0),      # two faults in one unit: recompute
              (3 * 127 + 60, 4 * 127 + 90, 1800, -4.0)]
    c = synth.make_case("fewwave_" + trans, trans[0], trans[1], m, n, k, alpha=1.5, beta=0.5,
                        seed=77, faults=faults)
    rep, orep, _ = run_config(c, extra_units=12)
    assert (rep.detected, rep.corrected, rep.recomputed) == (5, 4, 1)


@pytest.mark.parametrize("trans", ["NN", "TN"])
def test_encoder_head_ctas_parity(trans):
    """A two-wave protected launch (289 tiles, k = 512): encoder CTAs at the head of the grid
    publish every tile row's e^T A_I and tile column's B_J e, and every tile -- those of tile
    row / column 0 included -- copies them (R22).  Faults in tile row 0, tile column 0, the
    corner and the interior, a two-fault unit, beta != 0: values, counters and events equal to
    the oracle's on every fault unit + seeded units."""
    m = n = 2048
    k = 512
    faults = [(3, 500, 100, 5.0),                        # tile row 0
              (700, 2, 300, -3.0),                       # tile column 0
              (0, 0, 0, 11.0),                           # tile (0, 0), first update
              (2047, 2047, k, 1e3),                      # corner sliver, after the last update
              (1000, 1000, 256, 2.5), (1001, 1010, 400, -6.0)]  # two faults in one unit
    c = synth.make_case("enchead_" + trans, trans[0], trans[1], m, n, k, alpha=1.0, beta=0.5,
                        seed=91, faults=faults)
    rep, orep, _ = run_config(c, extra_units=12)
    assert (rep.detected, rep.corrected, rep.recomputed) == (5, 4, 1)
