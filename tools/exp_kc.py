"""Dev: protected time at verification intervals Kc (0 = k) and the unprotected time, for the
default or an alternative library build: python tools/exp_kc.py [LIB]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2104_00897_b200 import ftblas as F
if len(sys.argv) > 1:
    F.LIB_PATH = sys.argv[1]
M, N, K = (int(os.environ.get(x, d)) for x, d in (("M", 16384), ("N", 16384), ("K", 8192)))
A = torch.rand(M * K, dtype=torch.float64, device="cuda") * 2 - 1
B = torch.rand(K * N, dtype=torch.float64, device="cuda") * 2 - 1
C = torch.zeros(M * N, dtype=torch.float64, device="cuda")
def t(fn, r=3):
    fn(); torch.cuda.synchronize(); ts = []
    for _ in range(r):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True); e0.record(); fn(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    return min(ts)
out = {"lib": sys.argv[1] if len(sys.argv) > 1 else "default", "MNK": [M, N, K]}
out["noft_ms"] = t(lambda: F.ftblas_dgemm_noft("N", "N", M, N, K, 1.0, A, M, B, K, 0.0, C, M))
for kc in (0, 2048, 512):
    F.ftblas_set_interval(kc)
    out[f"ft_ms_Kc{kc}"] = t(lambda: F.ftblas_dgemm("N", "N", M, N, K, 1.0, A, M, B, K, 0.0, C, M, report=False))
F.ftblas_set_interval(0)
print(json.dumps({k: (round(v, 3) if isinstance(v, float) else v) for k, v in out.items()}), flush=True)
