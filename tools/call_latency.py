"""Dev: per-call wall time of the protected and unprotected DGEMM at N^3 (argv[1], default 256):
asynchronous unprotected, unprotected + sync, protected without report + sync, protected with
report (synchronous by contract), protected with report + one fault."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2104_00897_b200 import ftblas as F
m = n = k = int(sys.argv[1]) if len(sys.argv) > 1 else 256
A = torch.rand(m * k, dtype=torch.float64, device="cuda"); B = torch.rand(k * n, dtype=torch.float64, device="cuda")
C = torch.zeros(m * n, dtype=torch.float64, device="cuda")
def wall(fn, r=100):
    for _ in range(10): fn()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(r): fn()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / r * 1e6
print(f"N={m}")
print("noft async          %.1f us" % wall(lambda: F.ftblas_dgemm_noft("N", "N", m, n, k, 1.0, A, m, B, k, 0.0, C, m)))
print("noft + sync         %.1f us" % wall(lambda: (F.ftblas_dgemm_noft("N", "N", m, n, k, 1.0, A, m, B, k, 0.0, C, m), torch.cuda.synchronize())))
print("ft no report + sync %.1f us" % wall(lambda: (F.ftblas_dgemm("N", "N", m, n, k, 1.0, A, m, B, k, 0.0, C, m, report=False), torch.cuda.synchronize())))
print("ft report           %.1f us" % wall(lambda: F.ftblas_dgemm("N", "N", m, n, k, 1.0, A, m, B, k, 0.0, C, m)))
print("ft report cap 1024  %.1f us" % wall(lambda: F.ftblas_dgemm("N", "N", m, n, k, 1.0, A, m, B, k, 0.0, C, m, events_capacity=1024)))
def ftf():
    F.ftblas_inject_arm([(17, 203, 128, 1e3)])
    F.ftblas_dgemm("N", "N", m, n, k, 1.0, A, m, B, k, 0.0, C, m)
print("ft report + fault   %.1f us" % wall(ftf))
# host-side cost of one call (the time the Python call itself takes; the GPU runs behind)
def host(fn, r=200):
    for _ in range(10): fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(r):
        t0 = time.perf_counter(); fn(); ts.append(time.perf_counter() - t0)
    torch.cuda.synchronize()
    ts.sort()
    return ts[len(ts) // 2] * 1e6
import ctypes
L = F.load()
pA, pB, pC = A.data_ptr(), B.data_ptr(), C.data_ptr()
print("host: noft binding       %.1f us" % host(lambda: F.ftblas_dgemm_noft("N", "N", m, n, k, 1.0, A, m, B, k, 0.0, C, m)))
print("host: noft raw ctypes    %.1f us" % host(lambda: L.ftblas_dgemm_noft(b"N", b"N", m, n, k, 1.0, pA, m, pB, k, 0.0, pC, m)))
print("host: ft no report       %.1f us" % host(lambda: F.ftblas_dgemm("N", "N", m, n, k, 1.0, A, m, B, k, 0.0, C, m, report=False)))
print("host: ft raw no report   %.1f us" % host(lambda: L.ftblas_dgemm(b"N", b"N", m, n, k, 1.0, pA, m, pB, k, 0.0, pC, m, None)))
