"""Profiling target: one unprotected and one protected DTRSM at m = n = 8192."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2104_00897_b200 import ftblas as F
m = n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
A = torch.rand(m, m, dtype=torch.float64, device="cuda") / m
A = torch.tril(A) + torch.diag(1 + torch.rand(m, dtype=torch.float64, device="cuda"))
Acm = A.t().contiguous()
B = torch.rand(n, m, dtype=torch.float64, device="cuda")
F.ftblas_dtrsm_noft("L", "L", "N", "N", m, n, 1.0, Acm, m, B, m)
F.ftblas_dtrsm("L", "L", "N", "N", m, n, 1.0, Acm, m, B, m, report=False)
torch.cuda.synchronize()
print("ok")
