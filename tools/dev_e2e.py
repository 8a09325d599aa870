"""Dev: stream-event timeline of ftblas_dgemm_host at M N K (FTBLAS_DEV_E2E), plus pinned copy rates."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
os.environ["FTBLAS_DEV_E2E"] = "1"
from paper_2104_00897_b200 import build as _build, ftblas as F
F.load(_build.build(dev=True))  # development switches: libftblas_dev.so (-DFTBLAS_DEV)
M, N, K = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (32768, 32768, 32768)))
h = torch.empty(1 << 27, dtype=torch.float64, pin_memory=True); d = torch.empty_like(h, device="cuda")
for name, fn in (("H2D", lambda: d.copy_(h, non_blocking=True)), ("D2H", lambda: h.copy_(d, non_blocking=True))):
    fn(); torch.cuda.synchronize(); t0 = time.perf_counter(); fn(); torch.cuda.synchronize()
    print(f"{name} pinned 1 GiB: {(1 << 30) / (time.perf_counter() - t0) / 1e9:.1f} GB/s", flush=True)
A = torch.rand(M * K, dtype=torch.float64, pin_memory=True)
B = torch.rand(K * N, dtype=torch.float64, pin_memory=True)
C = torch.empty(M * N, dtype=torch.float64, pin_memory=True)
for it in range(2):
    t0 = time.perf_counter()
    F.ftblas_dgemm_host("N", "N", M, N, K, 1.0, A, M, B, K, 0.0, C, M, report=True)
    print(f"call {it}: {1e3 * (time.perf_counter() - t0):.1f} ms wall", flush=True)
