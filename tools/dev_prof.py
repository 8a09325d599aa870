"""Dev: per-warp wait/work clock split for the FT kernel (FTBLAS_DEV_PROF)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
N = 4096
ntiles = (N // 128) ** 2
prof = torch.zeros(ntiles * 12 * 2, dtype=torch.int64, device="cuda")
os.environ["FTBLAS_DEV_PROF"] = str(prof.data_ptr())
from paper_2104_00897_b200 import ftblas as F
g = torch.Generator(device="cuda").manual_seed(0)
A = torch.rand(N * N, dtype=torch.float64, device="cuda", generator=g)
B = torch.rand(N * N, dtype=torch.float64, device="cuda", generator=g)
C = torch.zeros(N * N, dtype=torch.float64, device="cuda")
for mode in sys.argv[1:] or ["0"]:
    os.environ["FTBLAS_DEV_CS"] = mode
    prof.zero_()
    F.ftblas_dgemm("N", "N", N, N, N, 1.0, A, N, B, N, 0.0, C, N, report=False)
    torch.cuda.synchronize()
    p = prof.view(ntiles, 12, 2).double().mean(0) / (N // 16)  # per stage
    print("mode", mode, "per-stage clk [wait, work] by warp:",
          " ".join(f"w{w}:{p[w,0]:.0f}/{p[w,1]:.0f}" for w in range(12)), flush=True)
