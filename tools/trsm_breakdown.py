"""Dev: device time of one protected and one unprotected DTRSM (side L, lower, N) by kernel,
from the torch profiler (CUPTI).  argv[1] = m = n (default 8192), argv[2] = library (optional)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import profile, ProfilerActivity
from paper_2104_00897_b200 import ftblas as F
if len(sys.argv) > 2:
    F.LIB_PATH = sys.argv[2]

m = n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
A = torch.rand(m, m, dtype=torch.float64, device="cuda") / m
A = torch.tril(A) + torch.diag(1 + torch.rand(m, dtype=torch.float64, device="cuda"))
Acm = A.t().contiguous()
B0 = torch.rand(n, m, dtype=torch.float64, device="cuda")
for name, fn in (("noft", F.ftblas_dtrsm_noft), ("ft", lambda *a: F.ftblas_dtrsm(*a, report=False))):
    B = B0.clone()
    fn("L", "L", "N", "N", m, n, 1.0, Acm, m, B, m)
    torch.cuda.synchronize()
    B = B0.clone()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        fn("L", "L", "N", "N", m, n, 1.0, Acm, m, B, m)
        torch.cuda.synchronize()
    agg = {}
    for ev in prof.events():
        if ev.device_type == torch.autograd.DeviceType.CUDA:
            key = ev.name.split("(")[0][:70]
            c, t = agg.get(key, (0, 0.0))
            agg[key] = (c + 1, t + ev.device_time_total)
    tot = sum(t for _, t in agg.values())
    print(f"== {name} {m}: device busy {tot / 1e3:.2f} ms")
    for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:12]:
        print(f"   {c:5d} x  {t / 1e3:8.3f} ms  {k}")
