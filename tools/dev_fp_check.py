"""Dev: count detections on fault-free inputs across k (false-positive hunt)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2104_00897_b200 import ftblas as F
for (m, n, k) in [(256, 256, 256), (256, 256, 1024), (256, 256, 4096), (1024, 1024, 8192), (2048, 2048, 2048), (8192, 8192, 8192)]:
    g = torch.Generator(device="cuda").manual_seed(0)
    A = torch.rand(m * k, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    B = torch.rand(k * n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    C = torch.zeros(m * n, dtype=torch.float64, device="cuda")
    rep = F.ftblas_dgemm("N", "N", m, n, k, 1.0, A, m, B, k, 0.0, C, m, events_capacity=8)
    Cref = (A.view(k, m).t() @ B.view(n, k).t())
    err = (C.view(n, m).t() - Cref).abs().max().item()
    print(m, n, k, "units", rep.units_checked, "detected", rep.detected, "recomputed", rep.recomputed,
          "maxerr", err, "ev", rep.events[:2], flush=True)
