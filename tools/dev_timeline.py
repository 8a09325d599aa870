"""Dev: per-CTA timeline of MMA warp 0 in the protected kernel (build with -DFTBLAS_DEV_TIMELINE):
clocks from the k-loop start to the first encoded stage, the k-loop, and the verify epilogue.
usage: python tools/dev_timeline.py LIB.so M N K [noft]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
lib, M, N, K = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
ntiles = ((M + 126) // 127) * ((N + 126) // 127) + 1
prof = torch.zeros(ntiles * 12 * 2, dtype=torch.int64, device="cuda")
os.environ["FTBLAS_DEV_PROF"] = str(prof.data_ptr())
from paper_2104_00897_b200 import build as _build, ftblas as F
F.load(_build.build(dev=True))  # development switches: libftblas_dev.so (-DFTBLAS_DEV)
F.LIB_PATH = lib
g = torch.Generator(device="cuda").manual_seed(0)
A = torch.rand(M * K, dtype=torch.float64, device="cuda", generator=g)
B = torch.rand(K * N, dtype=torch.float64, device="cuda", generator=g)
C = torch.zeros(M * N, dtype=torch.float64, device="cuda")
noft = len(sys.argv) > 5 and sys.argv[5] == "noft"
if noft:
    F.ftblas_dgemm_noft("N", "N", M, N, K, 1.0, A, M, B, K, 0.0, C, M)
else:
    F.ftblas_dgemm("N", "N", M, N, K, 1.0, A, M, B, K, 0.0, C, M, report=False)
torch.cuda.synchronize()
p = prof.view(ntiles, 12, 2)[:, 4:6, :].reshape(ntiles, 4)[:, :3].double()
p = p[p[:, 1] > 0]
m = p.mean(0)
print(f"{'noft' if noft else 'ft'} {M}x{N}x{K}: CTAs {p.shape[0]}  first-stage wait {m[0]:.0f} clk, k-loop {m[1]:.0f} clk "
      f"({m[1] / max(1, (K + 15) // 16):.0f}/stage), verify {m[2]:.0f} clk", flush=True)
