"""Dev: encoder warps' per-job [wait, work] clocks (FTBLAS_DEV_PROF) for the publishing tiles and
the others, and the first-stage wait of each group.  usage: python tools/dev_encoder_jobs.py M N K"""
import sys, os
sys.path.insert(0, "/root/repo")
import torch
M, N, K = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
ntiles = ((M + 126) // 127) * ((N + 126) // 127)
prof = torch.zeros(ntiles * 12 * 2, dtype=torch.int64, device="cuda")
os.environ["FTBLAS_DEV_PROF"] = str(prof.data_ptr())
from paper_2104_00897_b200 import build as _build, ftblas as F
F.load(_build.build(dev=True))
g = torch.Generator(device="cuda").manual_seed(0)
A = torch.rand(M * K, dtype=torch.float64, device="cuda", generator=g)
B = torch.rand(K * N, dtype=torch.float64, device="cuda", generator=g)
C = torch.zeros(M * N, dtype=torch.float64, device="cuda")
F.ftblas_dgemm("N", "N", M, N, K, 1.0, A, M, B, K, 0.0, C, M, report=False)
torch.cuda.synchronize(); prof.zero_()
F.ftblas_dgemm("N", "N", M, N, K, 1.0, A, M, B, K, 0.0, C, M, report=False)
torch.cuda.synchronize()
p = prof.view(ntiles, 12, 2).double()
nk = (K + 15) // 16
jobs = nk / 4.0
# encoder warps 0..3: [wait, work] sums; per job
for name, sel in (("publishers", slice(0, N // 127 + M // 127)), ("others", slice(N // 127 + M // 127 + 1, None)), ("all", slice(None))):
    q = p[sel].mean(0) / jobs
    print(name, "per-job clk [wait, work]:", " ".join(f"w{w}:{q[w,0]:.0f}/{q[w,1]:.0f}" for w in range(4)))
t = p[:, 10:12, :].reshape(ntiles, 4)
print("first-ready clk by CTA group: publishers %.0f others %.0f" % (t[:N // 127 + M // 127, 1].mean(), t[N // 127 + M // 127 + 1:, 1].mean()))
