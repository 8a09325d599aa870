"""Profiling target: one noft and one ft launch at m=n=k=N (default 4096), NN."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2104_00897_b200 import ftblas as F
N = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
ta = sys.argv[2] if len(sys.argv) > 2 else "NN"
g = torch.Generator(device="cuda").manual_seed(0)
A = torch.rand(N * N, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
B = torch.rand(N * N, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
C = torch.zeros(N * N, dtype=torch.float64, device="cuda")
F.ftblas_dgemm_noft(ta[0], ta[1], N, N, N, 1.0, A, N, B, N, 0.0, C, N)
F.ftblas_dgemm(ta[0], ta[1], N, N, N, 1.0, A, N, B, N, 0.0, C, N, report=False)
torch.cuda.synchronize()
print("ok")
