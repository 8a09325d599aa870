"""Sanitizer runs (race detection / sanitizers; compute-sanitizer is closed on this
pool).  The oracle's pins run against the oracle built under AddressSanitizer and
UndefinedBehaviorSanitizer (errors fatal), and the host-side ABI tests run against
libftblas_checked.so (host ASan/UBSan + the device bounds assertions of -DFTBLAS_CHECKED; its
GPU half runs on the B200 through tools/gpu_checked.sh).  Each run is a subprocess with libasan
preloaded, since the interpreter itself is not instrumented."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _asan_runtime():
    p = subprocess.run(["gcc", "-print-file-name=libasan.so"], capture_output=True, text=True).stdout.strip()
    return p if os.path.isabs(p) and os.path.exists(p) else None


def _run(tests, extra_env):
    asan = _asan_runtime()
    if asan is None:
        pytest.skip("gcc has no libasan runtime")
    env = dict(os.environ, LD_PRELOAD=asan,
               ASAN_OPTIONS="detect_leaks=0:protect_shadow_gap=0:alloc_dealloc_mismatch=0:"
                            "detect_odr_violation=0:abort_on_error=1",
               UBSAN_OPTIONS="halt_on_error=1:print_stacktrace=1", **extra_env)
    # the instrumented builds are the ones the child process maps
    probe = ("import conftest, oracle; from paper_2104_00897_b200 import ftblas as F; oracle.lib(); "
             "conftest.pytest_sessionstart(None); F.load(); print(open('/proc/self/maps').read())")
    pr = subprocess.run([sys.executable, "-c", probe], cwd=os.path.join(ROOT, "tests"), env=env,
                        capture_output=True, text=True, timeout=300)
    maps = pr.stdout
    assert "libasan" in maps, pr.stderr[-3000:]
    assert ("liboracle_san.so" in maps) == (extra_env.get("ORACLE_SANITIZE") == "1")
    assert ("libftblas_checked.so" in maps) == ("FTBLAS_TEST_LIB" in extra_env)
    r = subprocess.run([sys.executable, "-m", "pytest", *tests, "-q", "-m", "not gpu", "-p", "no:cacheprovider",
                        "-p", "no:randomly"], cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert "ERROR: AddressSanitizer" not in out and "runtime error:" not in out, out[-4000:]
    return out


def test_oracle_under_asan_ubsan():
    out = _run(["tests/test_oracle.py", "tests/test_oracle_trsm.py", "tests/test_oracle_dmr.py"],
               {"ORACLE_SANITIZE": "1"})
    assert "passed" in out


def test_host_library_under_asan_ubsan():
    from paper_2104_00897_b200 import build
    build.build(checked=True)
    out = _run(["tests/test_abi.py"], {"FTBLAS_TEST_LIB": "libftblas_checked.so"})
    assert "passed" in out
