"""Dev: FT overhead per encode mode (FUSED row-shared, FUSED_LOCAL, PREPASS) at M N K (env)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2104_00897_b200 import ftblas as F
N = int(os.environ.get("N", "8192")); M, K = int(os.environ.get("M", N)), int(os.environ.get("K", N))
g = torch.Generator(device="cuda").manual_seed(0)
A = torch.rand(M * K, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
B = torch.rand(K * N, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
C = torch.zeros(M * N, dtype=torch.float64, device="cuda")
def t(fn, r=4):
    fn(); torch.cuda.synchronize(); ts = []
    for _ in range(r):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True); e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return min(ts)
noft = t(lambda: F.ftblas_dgemm_noft("N", "N", M, N, K, 1.0, A, M, B, K, 0.0, C, M))
res = {"MNK": [M, N, K], "noft_ms": noft}
for name, mode in (("fused", F.ENCODE_FUSED), ("fused_local", F.ENCODE_FUSED_LOCAL), ("prepass", F.ENCODE_PREPASS)):
    F.ftblas_set_encode(mode)
    ms = t(lambda: F.ftblas_dgemm("N", "N", M, N, K, 1.0, A, M, B, K, 0.0, C, M, report=False))
    res[name] = round(100 * (ms - noft) / noft, 2)
F.ftblas_set_encode(F.ENCODE_FUSED)
print(json.dumps(res), flush=True)
