import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")
    config.addinivalue_line("markers", "slow: long-running")


def pytest_sessionstart(session):
    # FTBLAS_TEST_LIB: run the suite on another build of the same ABI -- libftblas_checked.so
    # (device bounds assertions, host ASan/UBSan; tests/test_sanitize.py, tools/gpu_checked.sh).
    lib = os.environ.get("FTBLAS_TEST_LIB")
    if lib:
        from paper_2104_00897_b200 import ftblas
        ftblas.load(os.path.join(ROOT, "paper_2104_00897_b200", lib))


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        have_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        have_gpu = False
    if have_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)
