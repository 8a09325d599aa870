import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_00897_b200.ftblas as F
F.LIB_PATH = sys.argv[1]
which = sys.argv[2]
tr = sys.argv[4] if len(sys.argv) > 4 else "NN"
import torch
m = n = k = int(sys.argv[3]) if len(sys.argv) > 3 else 256
A = torch.rand(m * k, dtype=torch.float64, device="cuda"); B = torch.rand(k * n, dtype=torch.float64, device="cuda")
C = torch.zeros(m * n, dtype=torch.float64, device="cuda")
try:
    if which == "noft":
        F.ftblas_dgemm_noft("N", "N", m, n, k, 1.0, A, m, B, k, 0.0, C, m); torch.cuda.synchronize(); r = ""
    else:
        r = F.ftblas_dgemm(tr[0], tr[1], m, n, k, 1.0, A, m, B, k, 0.0, C, m)
    Am = A.view(k, m).t() if tr[0] == "N" else A.view(m, k)
    Bm = B.view(n, k).t() if tr[1] == "N" else B.view(k, n)
    ref = Am @ Bm
    print(os.path.basename(sys.argv[1]), which, m, tr, "OK err", (C.view(n, m).t() - ref).abs().max().item(), r if not r else (r.detected, r.recomputed))
except Exception as e:
    print(os.path.basename(sys.argv[1]), which, m, "ERR", e)
