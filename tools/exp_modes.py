"""Dev: FT overhead (NN, m x n x k from env M N K, default 8192^3) under FTBLAS_DEV_MODE variants
(1 skip pass 2, 2 skip encode, 4 never flag, 32 noft on the 127 grid, 128 no clusters, 1024 skip
the last check)."""
import sys, os, json, subprocess
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r'''
import sys, os, json
sys.path.insert(0, %r)
import torch
from paper_2104_00897_b200 import build as _build, ftblas as F
F.load(_build.build(dev=True))  # development switches: libftblas_dev.so (-DFTBLAS_DEV)
N = int(os.environ.get("N", "8192"))
M, K = int(os.environ.get("M", N)), int(os.environ.get("K", N))
g = torch.Generator(device="cuda").manual_seed(0)
A = torch.rand(M * K, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
B = torch.rand(K * N, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
C = torch.zeros(M * N, dtype=torch.float64, device="cuda")
F.ftblas_set_encode(int(os.environ.get("ENC", "0")))
res = {}
for name in ["noft", "ft", "noft", "ft"]:
    ts = []
    for r in range(int(os.environ.get("REPS", "4"))):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        if name == "ft": F.ftblas_dgemm("N", "N", M, N, K, 1.0, A, M, B, K, 0.0, C, M, report=False)
        else: F.ftblas_dgemm_noft("N", "N", M, N, K, 1.0, A, M, B, K, 0.0, C, M)
        e1.record(); torch.cuda.synchronize()
        if r: ts.append(e0.elapsed_time(e1))
    res[name] = min(ts)
print(json.dumps({"mode": os.environ.get("FTBLAS_DEV_MODE", "0"), "enc": os.environ.get("ENC", "0"), "MNK": [M, N, K], "noft_ms": res["noft"], "ft_ms": res["ft"],
                  "overhead_pct": 100 * (res["ft"] - res["noft"]) / res["noft"]}), flush=True)
''' % ROOT
for mode in (sys.argv[1:] or ["0", "5", "6"]):
    env = dict(os.environ, FTBLAS_DEV_MODE=mode)
    subprocess.run([sys.executable, "-c", code], env=env)
