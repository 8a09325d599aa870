"""Dev: cost of the online intermediate checks (dev build, FTBLAS_DEV_PROF): per check, the
clocks from the first MMA thread's arrival to the end of the first staging round (arrival skew
of the 8 MMA warps + staging) and the clocks of the reductions and the decision; and the
protected / unprotected times at Kc = k and Kc = KC.  usage: python tools/dev_check_cost.py M N K KC"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

M, N, K, KC = (int(x) for x in (sys.argv[1:5] if len(sys.argv) > 4 else (8192, 8192, 32768, 2048)))
ntiles = ((M + 126) // 127) * ((N + 126) // 127)
prof = torch.zeros(ntiles * 12 * 2 + 64, dtype=torch.int64, device="cuda")
os.environ["FTBLAS_DEV_PROF"] = str(prof.data_ptr())
from paper_2104_00897_b200 import build as _build, ftblas as F  # noqa: E402
F.load(_build.build(dev=True))
g = torch.Generator(device="cuda").manual_seed(0)
A = torch.rand(M * K, dtype=torch.float64, device="cuda", generator=g)
B = torch.rand(K * N, dtype=torch.float64, device="cuda", generator=g)
C = torch.zeros(M * N, dtype=torch.float64, device="cuda")


def t(fn):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


noft = t(lambda: F.ftblas_dgemm_noft("N", "N", M, N, K, 1.0, A, M, B, K, 0.0, C, M))
F.ftblas_set_interval(0)
ft = t(lambda: F.ftblas_dgemm("N", "N", M, N, K, 1.0, A, M, B, K, 0.0, C, M, report=False))
prof.zero_()
F.ftblas_set_interval(KC)
ftk = t(lambda: F.ftblas_dgemm("N", "N", M, N, K, 1.0, A, M, B, K, 0.0, C, M, report=False))
F.ftblas_set_interval(0)
p = prof[: ntiles * 24].view(ntiles, 12, 2)[:, 8:12, :].reshape(ntiles, 8).double()
calls = p[:, 2].sum().item()
print(f"{M}x{N}x{K}: noft {noft:.2f} ms, ft {ft:.2f} ms ({100 * (ft - noft) / noft:.2f}%), "
      f"ft Kc={KC} {ftk:.2f} ms ({100 * (ftk - noft) / noft:.2f}%)", flush=True)
print(f"intermediate checks: {calls:.0f} (2 timed runs); per check clk: skew+stage "
      f"{p[:, 0].sum().item() / calls:.0f}, reductions {p[:, 1].sum().item() / calls:.0f}, "
      f"decision {p[:, 3].sum().item() / calls:.0f}; of the first: arrival skew (first barrier) "
      f"{p[:, 4].sum().item() / calls:.0f}, drain of the warp's DMMA stream {p[:, 5].sum().item() / calls:.0f}", flush=True)
