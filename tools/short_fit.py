"""Dev: fixed vs per-k cost of a tile on short shapes.  Times the protected kernel, the
unprotected kernel and cuBLAS over a k sweep at a few m = n, and fits t = t0 + t1 * k per
kernel (t0: the per-launch + per-wave fixed cost, t1: the k-loop).
usage: python tools/short_fit.py [MN ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2104_00897_b200 import ftblas as F

F.load()
REPS = int(os.environ.get("REPS", "20"))


def timed(fn):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * REPS)]
    for r in range(REPS):
        ev[2 * r].record()
        fn()
        ev[2 * r + 1].record()
    torch.cuda.synchronize()
    return float(np.median([ev[2 * r].elapsed_time(ev[2 * r + 1]) for r in range(REPS)])) * 1e3  # us


mns = [int(a) for a in sys.argv[1:]] or [2048, 1524, 1016]
ks = [256, 512, 1024, 2048, 4096, 8192]
st = torch.cuda.current_stream()
F.ftblas_set_stream(st.cuda_stream)
for mn in mns:
    rows = {"ft": [], "noft": [], "cublas": []}
    for k in ks:
        g = torch.Generator(device="cuda").manual_seed(k)
        A = torch.rand(mn * k, dtype=torch.float64, device="cuda", generator=g)
        B = torch.rand(k * mn, dtype=torch.float64, device="cuda", generator=g)
        C = torch.zeros(mn * mn, dtype=torch.float64, device="cuda")
        A2, B2 = A.view(k, mn).t(), B.view(mn, k).t()
        rows["ft"].append(timed(lambda: F.ftblas_dgemm("N", "N", mn, mn, k, 1.0, A, mn, B, k, 0.0, C, mn, report=False)))
        rows["noft"].append(timed(lambda: F.ftblas_dgemm_noft("N", "N", mn, mn, k, 1.0, A, mn, B, k, 0.0, C, mn)))
        rows["cublas"].append(timed(lambda: torch.mm(A2, B2)))
    for name, t in rows.items():
        t1, t0 = np.polyfit(ks, t, 1)
        tf = [2.0 * mn * mn * k / (x * 1e-6) / 1e12 for k, x in zip(ks, t)]
        print(f"{mn} {name:7s} t0 {t0:7.1f} us  t1 {t1 * 1e3:7.1f} ns/k  "
              + " ".join(f"k{k}:{x:.0f}us/{f:.1f}TF" for k, x, f in zip(ks, t, tf)), flush=True)
