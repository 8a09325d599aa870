"""Dev: unprotected / protected time for each trans combination at N^3 (env N), optional alt lib."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2104_00897_b200 import ftblas as F
if len(sys.argv) > 1:
    F.LIB_PATH = sys.argv[1]
N = int(os.environ.get("N", "8192"))
A = torch.rand(N * N, dtype=torch.float64, device="cuda"); B = torch.rand(N * N, dtype=torch.float64, device="cuda")
C = torch.zeros(N * N, dtype=torch.float64, device="cuda")
def t(fn, r=3):
    fn(); torch.cuda.synchronize(); ts = []
    for _ in range(r):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True); e0.record(); fn(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    return min(ts)
res = {}
for tr in ("NN", "NT", "TN", "TT"):
    no = t(lambda: F.ftblas_dgemm_noft(tr[0], tr[1], N, N, N, 1.0, A, N, B, N, 0.0, C, N))
    ft = t(lambda: F.ftblas_dgemm(tr[0], tr[1], N, N, N, 1.0, A, N, B, N, 0.0, C, N, report=False))
    res[tr] = [round(2 * N ** 3 / no / 1e9, 2), round(2 * N ** 3 / ft / 1e9, 2)]
print(json.dumps(res), flush=True)
