import time, torch, sys, os
sys.path.insert(0, os.getcwd())
from paper_2104_00897_b200 import ftblas as F
m = n = k = 256
A = torch.rand(m*k, dtype=torch.float64, device="cuda"); B = torch.rand(k*n, dtype=torch.float64, device="cuda"); C = torch.zeros(m*n, dtype=torch.float64, device="cuda")
def wall(fn, r=200):
    for _ in range(20): fn()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(r): fn()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / r * 1e6
print("noft async   %.1f us" % wall(lambda: F.ftblas_dgemm_noft("N","N",m,n,k,1.0,A,m,B,k,0.0,C,m)))
print("noft + sync  %.1f us" % wall(lambda: (F.ftblas_dgemm_noft("N","N",m,n,k,1.0,A,m,B,k,0.0,C,m), torch.cuda.synchronize())))
print("ft no report + sync %.1f us" % wall(lambda: (F.ftblas_dgemm("N","N",m,n,k,1.0,A,m,B,k,0.0,C,m, report=False), torch.cuda.synchronize())))
print("ft report    %.1f us" % wall(lambda: F.ftblas_dgemm("N","N",m,n,k,1.0,A,m,B,k,0.0,C,m)))
def ftf():
    F.ftblas_inject_arm([(17, 203, 128, 1e3)]); F.ftblas_dgemm("N","N",m,n,k,1.0,A,m,B,k,0.0,C,m)
print("ft report + fault  %.1f us" % wall(ftf))
