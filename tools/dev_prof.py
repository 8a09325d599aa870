"""Dev: per-warp wait/work clock split of the FT kernel (FTBLAS_DEV_PROF; encoder warps only).
Prints the per-job averages of encoder warps 1..3: clocks waiting for the TMA bytes and
clocks spent encoding one stage."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
N = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
ntiles = ((N + 126) // 127) ** 2
prof = torch.zeros(ntiles * 12 * 2, dtype=torch.int64, device="cuda")
os.environ["FTBLAS_DEV_PROF"] = str(prof.data_ptr())
from paper_2104_00897_b200 import build as _build, ftblas as F
F.load(_build.build(dev=True))  # development switches: libftblas_dev.so (-DFTBLAS_DEV)
g = torch.Generator(device="cuda").manual_seed(0)
A = torch.rand(N * N, dtype=torch.float64, device="cuda", generator=g)
B = torch.rand(N * N, dtype=torch.float64, device="cuda", generator=g)
C = torch.zeros(N * N, dtype=torch.float64, device="cuda")
F.ftblas_dgemm("N", "N", N, N, N, 1.0, A, N, B, N, 0.0, C, N, report=False)
torch.cuda.synchronize()
jobs = (N // 16) / 4.0
p = prof.view(ntiles, 12, 2).double().mean(0) / jobs
print("per-job clk [wait TMA, encode] by encoder warp:",
      " ".join(f"w{w}:{p[w,0]:.0f}/{p[w,1]:.0f}" for w in range(0, 4)), flush=True)
