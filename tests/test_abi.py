"""C-ABI boundary tests that need no GPU: the library loads, exports every symbol the
header declares, validates arguments (BLAS INFO convention) before touching the device,
and its seeded fault generator agrees with the independent one in synth/."""
import ctypes
import os
import re

import pytest

import synth
from paper_2104_00897_b200 import ftblas as F
from paper_2104_00897_b200.perfmodel import predict_unfused_overhead

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "ftblas.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(ftblas_[a-z_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    L = F.load()
    syms = header_symbols()
    assert len(syms) >= 13
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(F.EXPORTED)


def test_argument_checks_lapack_info_style():
    A = B = C = 0x1000  # never dereferenced: checks fail before any device work
    g = lambda *a: F.ftblas_dgemm(*a, report=False, raw_status=True)  # noqa: E731
    assert g("X", "N", 4, 4, 4, 1.0, A, 4, B, 4, 0.0, C, 4) == -1
    assert g("N", "Q", 4, 4, 4, 1.0, A, 4, B, 4, 0.0, C, 4) == -2
    assert g("N", "N", -1, 4, 4, 1.0, A, 4, B, 4, 0.0, C, 4) == -3
    assert g("N", "N", 4, -1, 4, 1.0, A, 4, B, 4, 0.0, C, 4) == -4
    assert g("N", "N", 4, 4, -1, 1.0, A, 4, B, 4, 0.0, C, 4) == -5
    assert g("N", "N", 4, 4, 4, 1.0, None, 4, B, 4, 0.0, C, 4) == -7
    assert g("N", "N", 4, 4, 4, 1.0, A, 3, B, 4, 0.0, C, 4) == -8
    assert g("T", "N", 4, 4, 6, 1.0, A, 4, B, 6, 0.0, C, 4) == -8   # lda >= k for 'T'
    assert g("N", "N", 4, 4, 4, 1.0, A, 4, None, 4, 0.0, C, 4) == -9
    assert g("N", "N", 4, 4, 4, 1.0, A, 4, B, 3, 0.0, C, 4) == -10
    assert g("N", "T", 4, 5, 4, 1.0, A, 4, B, 4, 0.0, C, 4) == -10  # ldb >= n for 'T'
    assert g("N", "N", 4, 4, 4, 1.0, A, 4, B, 4, 0.0, None, 4) == -12
    assert g("N", "N", 4, 4, 4, 1.0, A, 4, B, 4, 0.0, C, 3) == -13
    assert F.ftblas_dgemm_noft("N", "N", 4, 4, 4, 1.0, A, 4, B, 4, 0.0, C, 2, raw_status=True) == -13
    # 'C' means transpose for real data; lowercase accepted
    assert g("c", "t", 0, 4, 4, 1.0, A, 4, B, 4, 0.0, C, 1) == 0
    # quick return m == 0 / n == 0 touches nothing
    assert g("N", "N", 0, 4, 4, 1.0, A, 1, B, 4, 0.0, C, 1) == 0
    assert g("N", "N", 4, 0, 4, 1.0, A, 4, B, 4, 0.0, None, 4) == 0
    assert "argument 8" in F.ftblas_status_string(-8)


def test_report_geometry_on_quick_return():
    r = F.ErrReport()
    st = F.load().ftblas_dgemm(b"N", b"N", 0, 5, 7, 1.0, None, 1, None, 7, 0.0, None, 1,
                               ctypes.byref(r))
    assert st == 0 and r.units_checked == 0 and r.detected == 0
    BM, BN, BK = F.ftblas_get_geometry()
    assert (r.unit_rows, r.unit_cols, r.unit_k, r.step_quantum) == (BM, BN, 7, BK)
    assert BM > 0 and BN > 0 and BK > 0


def test_inject_seeded_matches_independent_generator():
    for seed, cnt, m, n, k in [(1, 20, 8192, 8192, 8192), (99, 100, 32768, 32768, 32768),
                               (7, 5, 3, 2, 1)]:
        lib = F.ftblas_inject_seeded(seed, cnt, m, n, k, -2.0, 4.0)
        ref = synth.seeded_faults(seed, cnt, m, n, k, -2.0, 4.0)
        assert [f[:3] for f in lib] == [f[:3] for f in ref]
        for a, b in zip(lib, ref):  # pow() in C and Python: same libm, allow 1 ulp anyway
            assert abs(a[3] - b[3]) <= abs(b[3]) * 2.0 ** -52


def test_inject_arm_validation_and_options():
    assert F.load().ftblas_inject_arm(None, -1) == 3
    F.ftblas_inject_arm([(0, 0, 0, 1.0)])
    F.ftblas_inject_disarm()
    assert F.load().ftblas_set_correction(7) == 4
    F.ftblas_set_correction(F.CORRECT_SUBTRACT)
    F.ftblas_set_correction(F.CORRECT_RECOMPUTE)
    assert F.ftblas_take_launch_count() >= 0


def test_paper_overhead_model_closed_form():
    """(6 + 2K/Kc) P_mm / (n P_mv): worked value and linearity."""
    assert predict_unfused_overhead(1000, 1000, 250, 35.0, 1.0) == pytest.approx(0.49, abs=1e-15)
    r35 = predict_unfused_overhead(4096, 4096, 256, 35.0, 1.0)
    r5 = predict_unfused_overhead(4096, 4096, 256, 5.0, 1.0)
    assert r35 == pytest.approx(7 * r5, rel=1e-15)
    assert predict_unfused_overhead(14, 14, 14, 1.0, 1.0) == pytest.approx(8 / 14)
    with pytest.raises(ValueError):
        predict_unfused_overhead(10, 10, 20, 1.0, 1.0)


def test_release_library_reads_no_environment():
    """The release library has no development switches: no FTBLAS_DEV_* environment names are
    referenced by libftblas.so (they exist only in the -DFTBLAS_DEV build)."""
    data = open(F.LIB_PATH, "rb").read()
    for name in (b"FTBLAS_DEV_MODE", b"FTBLAS_DEV_PROF", b"FTBLAS_DEV_E2E"):
        assert name not in data, name


def test_option_setters_validate_without_a_gpu():
    """Thread-local options: encode modes FUSED / PREPASS / FUSED_LOCAL / FUSED_WAIT accepted,
    others -> 4; the interval must be a non-negative multiple of the step quantum."""
    L = F.load()
    for mode in (F.ENCODE_FUSED, F.ENCODE_PREPASS, F.ENCODE_FUSED_LOCAL, F.ENCODE_FUSED_WAIT):
        assert L.ftblas_set_encode(mode) == 0
    assert L.ftblas_set_encode(4) == 4 and L.ftblas_set_encode(-1) == 4
    assert L.ftblas_set_encode(F.ENCODE_FUSED) == 0
    assert L.ftblas_set_interval(32) == 0 and L.ftblas_set_interval(0) == 0
    assert L.ftblas_set_interval(20) == 4 and L.ftblas_set_interval(-16) == 4
    assert L.ftblas_set_correction(1) == 0 and L.ftblas_set_correction(0) == 0
    assert L.ftblas_set_correction(2) == 4


def test_binding_rejects_wrong_operand_kinds():
    """Marshalling checks of the binding (no GPU needed): device entry points take CUDA
    tensors or raw addresses, host entry points numpy arrays or CPU tensors, float64 only."""
    import numpy as np
    import torch
    a64 = np.zeros((4, 4))
    with pytest.raises(ValueError):
        F.ftblas_dgemm("N", "N", 4, 4, 4, 1.0, a64, 4, a64, 4, 0.0, a64, 4)
    with pytest.raises(ValueError):
        F.ftblas_dgemm_noft("N", "N", 4, 4, 4, 1.0, torch.zeros(16, dtype=torch.float64), 4, 0x1000, 4, 0.0, 0x1000, 4)
    with pytest.raises(TypeError):
        F.ftblas_dgemm_host("N", "N", 4, 4, 4, 1.0, a64.astype(np.float32), 4, a64, 4, 0.0, a64, 4)
    with pytest.raises(TypeError):
        F.ftblas_dscal(16, 2.0, torch.zeros(16, dtype=torch.float32), 1)
