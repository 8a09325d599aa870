"""Profiling target: one protected launch with verification every KC updates (NN, M x N x K)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2104_00897_b200 import ftblas as F

M, N, K, KC = (int(x) for x in (sys.argv[1:5] if len(sys.argv) > 4 else (4096, 4096, 8192, 512)))
g = torch.Generator(device="cuda").manual_seed(0)
A = torch.rand(M * K, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
B = torch.rand(K * N, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
C = torch.zeros(M * N, dtype=torch.float64, device="cuda")
F.ftblas_set_interval(KC)
F.ftblas_dgemm("N", "N", M, N, K, 1.0, A, M, B, K, 0.0, C, M, report=False)
torch.cuda.synchronize()
print("ok")
