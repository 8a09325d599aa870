"""Dev: protected / unprotected time at M N K (env) for the default and an alternative library build."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2104_00897_b200 import ftblas as F
if len(sys.argv) > 1:
    F.LIB_PATH = sys.argv[1]
N = int(os.environ.get("N", "16384")); M, K = int(os.environ.get("M", N)), int(os.environ.get("K", N))
A = torch.rand(M * K, dtype=torch.float64, device="cuda") * 2 - 1
B = torch.rand(K * N, dtype=torch.float64, device="cuda") * 2 - 1
C = torch.zeros(M * N, dtype=torch.float64, device="cuda")
def t(fn, r=3):
    fn(); torch.cuda.synchronize(); ts = []
    for _ in range(r):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True); e0.record(); fn(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    return min(ts)
no = t(lambda: F.ftblas_dgemm_noft("N", "N", M, N, K, 1.0, A, M, B, K, 0.0, C, M))
ft = t(lambda: F.ftblas_dgemm("N", "N", M, N, K, 1.0, A, M, B, K, 0.0, C, M, report=False))
print(json.dumps({"lib": sys.argv[1] if len(sys.argv) > 1 else "default", "MNK": [M, N, K], "noft_ms": round(no, 3),
                  "ft_ms": round(ft, 3), "overhead_pct": round(100 * (ft - no) / no, 2)}), flush=True)
