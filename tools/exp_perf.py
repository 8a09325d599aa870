"""Dev: ft vs noft timing at 8192^3 NN for an alternative build (argv[1] = .so)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_00897_b200.ftblas as F
if len(sys.argv) > 1: F.LIB_PATH = sys.argv[1]
import torch
N = 8192
A = torch.rand(N * N, dtype=torch.float64, device="cuda"); B = torch.rand(N * N, dtype=torch.float64, device="cuda")
C = torch.zeros(N * N, dtype=torch.float64, device="cuda")
def t(ft):
    ts = []
    for r in range(4):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        if ft: F.ftblas_dgemm("N", "N", N, N, N, 1.0, A, N, B, N, 0.0, C, N, report=False)
        else: F.ftblas_dgemm_noft("N", "N", N, N, N, 1.0, A, N, B, N, 0.0, C, N)
        e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    return min(ts[1:])
a, b = t(False), t(True)
rep = F.ftblas_dgemm("N", "N", N, N, N, 1.0, A, N, B, N, 0.0, C, N)
print(os.path.basename(F.LIB_PATH), f"noft {a:.2f} ms ft {b:.2f} ms overhead {100*(b-a)/a:.1f}%  det {rep.detected}")
