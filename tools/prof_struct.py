"""Dev profiling target (dev build): the unprotected kernel on the protected kernel's 127-row
grid and the protected kernel without encode / flags / proxy fence / interval maxima
(FTBLAS_DEV_MODE=6182 = 32 | 2 | 4 | 2048 | 4096): the structural difference of the two.
usage: FTBLAS_DEV_MODE=6182 python tools/prof_struct.py [M N K]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2104_00897_b200 import build as _build, ftblas as F

F.load(_build.build(dev=True))
M, N, K = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (32766, 32766, 4096)))
A = torch.rand(M * K, dtype=torch.float64, device="cuda") * 2 - 1
B = torch.rand(K * N, dtype=torch.float64, device="cuda") * 2 - 1
C = torch.zeros(M * N, dtype=torch.float64, device="cuda")
F.ftblas_dgemm_noft("N", "N", M, N, K, 1.0, A, M, B, K, 0.0, C, M)
F.ftblas_dgemm("N", "N", M, N, K, 1.0, A, M, B, K, 0.0, C, M, report=False)
torch.cuda.synchronize()
print("ok")
