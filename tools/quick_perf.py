"""Dev timing: ft vs noft DGEMM TFLOP/s at a few sizes (CUDA events, inputs > L2 or flushed)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2104_00897_b200 import ftblas as F

def run(m, n, k, ta="N", tb="N", reps=5):
    g = torch.Generator(device="cuda").manual_seed(0)
    lda = k if ta == "T" else m
    ldb = n if tb == "T" else k
    A = torch.rand(m * k, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    B = torch.rand(k * n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    C = torch.rand(m * n, dtype=torch.float64, device="cuda", generator=g)
    beta = float(os.environ.get("BETA", "0"))  # beta != 0: the epilogue reads C0
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
    res = {}
    for name in ["noft", "ft", "noft", "ft"]:
        ts = []
        for r in range(reps + 1):
            flush.zero_()
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            if name == "ft":
                F.ftblas_dgemm(ta, tb, m, n, k, 1.0, A, lda, B, ldb, beta, C, m, report=False)
            else:
                F.ftblas_dgemm_noft(ta, tb, m, n, k, 1.0, A, lda, B, ldb, beta, C, m)
            e1.record(); torch.cuda.synchronize()
            if r: ts.append(e0.elapsed_time(e1))
        res[name] = min(ts)
    fl = 2.0 * m * n * k
    out = {"shape": [m, n, k, ta + tb], "beta": beta, "noft_ms": res["noft"], "ft_ms": res["ft"],
           "noft_tflops": fl / res["noft"] / 1e9, "ft_tflops": fl / res["ft"] / 1e9,
           "overhead_pct": 100 * (res["ft"] - res["noft"]) / res["noft"]}
    print(json.dumps(out), flush=True)

shapes = [(2048, 2048, 2048, "N", "N"), (8192, 8192, 8192, "N", "N"), (8192, 8192, 8192, "T", "N"),
          (8192, 8192, 8192, "N", "T"), (8192, 8192, 8192, "T", "T"), (16384, 16384, 1024, "N", "N"),
          (16384, 512, 16384, "N", "N")]
if os.environ.get("C5"):
    shapes.append((32768, 32768, 32768, "N", "N"))
if os.environ.get("SHAPES"):  # e.g. SHAPES=2048x2048x2048NN,16384x16384x1024NN
    shapes = [(int(x.split("x")[0]), int(x.split("x")[1]), int(x.split("x")[2][:-2]), x[-2], x[-1])
              for x in os.environ["SHAPES"].split(",")]
for shp in shapes:
    run(*shp, reps=int(os.environ.get("REPS", "5")) if shp[0] < 32768 else 2)
