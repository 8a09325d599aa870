"""Dev: protected time with intervals Kc (argv) at M N K (env), per encode mode."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2104_00897_b200 import ftblas as F
M, N, K = int(os.environ.get("M", 16384)), int(os.environ.get("N", 512)), int(os.environ.get("K", 16384))
A = torch.rand(M * K, dtype=torch.float64, device="cuda") * 2 - 1
B = torch.rand(K * N, dtype=torch.float64, device="cuda") * 2 - 1
C = torch.zeros(M * N, dtype=torch.float64, device="cuda")
def t(fn, r=3):
    fn(); torch.cuda.synchronize(); ts = []
    for _ in range(r):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True); e0.record(); fn(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    return min(ts)
no = t(lambda: F.ftblas_dgemm_noft("N", "N", M, N, K, 1.0, A, M, B, K, 0.0, C, M))
for kc in [int(x) for x in sys.argv[1:]]:
    for name, mode in (("fused", F.ENCODE_FUSED), ("local", F.ENCODE_FUSED_LOCAL)):
        F.ftblas_set_encode(mode); F.ftblas_set_interval(kc)
        ft = t(lambda: F.ftblas_dgemm("N", "N", M, N, K, 1.0, A, M, B, K, 0.0, C, M, report=False))
        print(json.dumps({"MNK": [M, N, K], "Kc": kc, "mode": name, "ovh": round(100 * (ft - no) / no, 2)}), flush=True)
F.ftblas_set_interval(0); F.ftblas_set_encode(F.ENCODE_FUSED)
