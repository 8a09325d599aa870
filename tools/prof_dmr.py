"""Profiling target: one protected and one unprotected launch of each DMR routine (DSCAL,
DAXPY on 2^27 elements, DGEMV 'N' and 'T' on 8192^2), unit stride."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2104_00897_b200 import ftblas as F
n = 1 << 27
x = torch.rand(n, dtype=torch.float64, device="cuda")
y = torch.rand(n, dtype=torch.float64, device="cuda")
F.ftblas_dscal_noft(n, 1.0000001, x, 1)
F.ftblas_dscal(n, 1.0000001, x, 1, report=False)
F.ftblas_daxpy_noft(n, 1e-9, x, 1, y, 1)
F.ftblas_daxpy(n, 1e-9, x, 1, y, 1, report=False)
m = 8192
A = torch.rand(m * m, dtype=torch.float64, device="cuda")
v = torch.rand(m, dtype=torch.float64, device="cuda")
w = torch.rand(m, dtype=torch.float64, device="cuda")
for tr in "NT":
    F.ftblas_dgemv_noft(tr, m, m, 1.0, A, m, v, 1, 0.5, w, 1)
    F.ftblas_dgemv(tr, m, m, 1.0, A, m, v, 1, 0.5, w, 1, report=False)
torch.cuda.synchronize()
print("ok")
