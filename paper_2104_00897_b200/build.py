"""Build libftblas.so in-tree with nvcc for sm_100a (no JIT cache: the .so travels with the repo)."""
from __future__ import annotations

import glob
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libftblas.so")
LIB_DEV = os.path.join(HERE, "libftblas_dev.so")
LIB_WATCH = os.path.join(HERE, "libftblas_watch.so")
LIB_CHECKED = os.path.join(HERE, "libftblas_checked.so")
LIB_TIMELINE = os.path.join(HERE, "libftblas_tl.so")

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-warn-spills"]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cuh"))
                  + [os.path.join(ROOT, "include", "ftblas.h")])


def build(force: bool = False, verbose: bool = False, dev: bool = False, watchdog: bool = False,
          checked: bool = False, timeline: bool = False) -> str:
    """libftblas.so (release).  dev=True: libftblas_dev.so, the same sources with -DFTBLAS_DEV
    (the development switches of tools/dev_*.py; never loaded by the product or the tests);
    watchdog=True: libftblas_watch.so, dev + -DFTBLAS_WATCHDOG (mbarrier-wait watchdog of
    tools/hang_probe.py); checked=True: libftblas_checked.so, the release sources with the
    device bounds assertions of -DFTBLAS_CHECKED and the host code under AddressSanitizer and
    UndefinedBehaviorSanitizer (tools/gpu_checked.sh runs the GPU suite on it); timeline=True:
    libftblas_tl.so, the release sources plus the per-CTA clock timeline of -DFTBLAS_DEV_TIMELINE
    (tools/dev_timeline.py; no other development switch, so its kernels time like the release)."""
    lib = LIB_CHECKED if checked else (LIB_WATCH if watchdog else (LIB_DEV if dev else (LIB_TIMELINE if timeline else LIB)))
    dev = dev or watchdog
    newest = max(os.path.getmtime(s) for s in sources())
    if not force and os.path.exists(lib) and os.path.getmtime(lib) >= newest:
        return lib
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    flags = (["-DFTBLAS_DEV"] if dev else []) + (["-DFTBLAS_WATCHDOG"] if watchdog else []) + \
        (["-DFTBLAS_DEV_TIMELINE"] if timeline else [])
    if checked:
        flags += ["-DFTBLAS_CHECKED", "-lasan", "-lubsan"]
        for f in ("-fsanitize=address", "-fsanitize=undefined", "-fno-sanitize-recover=all", "-fno-omit-frame-pointer"):
            flags += ["-Xcompiler", f]
    cmd = [nvcc, *NVCC_FLAGS, *flags, "-o", lib, os.path.join(CSRC, "ftblas.cu")]
    if verbose:
        print(" ".join(cmd))
    subprocess.check_call(cmd)
    return lib


if __name__ == "__main__":
    print(build(force=True, verbose=True))
