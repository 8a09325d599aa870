"""Dev: DGEMV protected / unprotected / torch (cuBLAS) GB/s at several square sizes."""
import sys, os, torch, json
sys.path.insert(0, os.getcwd())
from paper_2104_00897_b200 import ftblas as F
for m in (2048, 4096, 8192, 16384):
    k = m
    A = torch.rand(m * k, dtype=torch.float64, device="cuda"); v = torch.rand(k, dtype=torch.float64, device="cuda"); w = torch.rand(m, dtype=torch.float64, device="cuda")
    def t(fn):
        for _ in range(3): fn()
        torch.cuda.synchronize(); best = 1e9
        for _ in range(10):
            a, b = torch.cuda.Event(True), torch.cuda.Event(True); a.record(); fn(); b.record(); torch.cuda.synchronize(); best = min(best, a.elapsed_time(b))
        return best
    by = 8 * (m * k + 2 * m + k)
    res = {}
    for tr in "NT":
        t1 = t(lambda: F.ftblas_dgemv(tr, m, k, 1.0, A, m, v, 1, 0.5, w, 1, report=False))
        t0 = t(lambda: F.ftblas_dgemv_noft(tr, m, k, 1.0, A, m, v, 1, 0.5, w, 1))
        Am = A.view(k, m).t(); op = Am if tr == "N" else Am.t()
        tt = t(lambda: torch.addmv(w if tr == "N" else w, op, v, beta=0.5, alpha=1.0, out=w))
        res[tr] = [round(by / t1 / 1e6), round(by / t0 / 1e6), round(by / tt / 1e6)]
    print(m, res, flush=True)
