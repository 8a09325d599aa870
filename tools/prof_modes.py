"""Dev profiling target: one protected launch at N^3 NN per encode mode (FUSED, FUSED_LOCAL, PREPASS)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2104_00897_b200 import ftblas as F
N = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
A = torch.rand(N * N, dtype=torch.float64, device="cuda") * 2 - 1
B = torch.rand(N * N, dtype=torch.float64, device="cuda") * 2 - 1
C = torch.zeros(N * N, dtype=torch.float64, device="cuda")
for mode in (F.ENCODE_FUSED, F.ENCODE_FUSED_LOCAL, F.ENCODE_PREPASS):
    F.ftblas_set_encode(mode)
    F.ftblas_dgemm("N", "N", N, N, N, 1.0, A, N, B, N, 0.0, C, N, report=False)
torch.cuda.synchronize()
