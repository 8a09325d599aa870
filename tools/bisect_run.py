import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_00897_b200.ftblas as F
F.LIB_PATH = sys.argv[1]
import torch
m = n = k = 256
A = torch.rand(m * k, dtype=torch.float64, device="cuda"); B = torch.rand(k * n, dtype=torch.float64, device="cuda")
C = torch.zeros(m * n, dtype=torch.float64, device="cuda")
try:
    rep = F.ftblas_dgemm("N", "N", m, n, k, 1.0, A, m, B, k, 0.0, C, m)
    print(os.path.basename(sys.argv[1]), "OK", rep.detected, rep.recomputed)
except Exception as e:
    print(os.path.basename(sys.argv[1]), "ERR", e)
try:
    F.ftblas_dgemm_noft("N", "N", m, n, k, 1.0, A, m, B, k, 0.0, C, m); torch.cuda.synchronize()
    print(os.path.basename(sys.argv[1]), "noft OK")
except Exception as e:
    print(os.path.basename(sys.argv[1]), "noft ERR", e)
