"""Dev: where the time of a small protected call goes (C1, 256^3 by default): device activity
(kernels, memsets, copies) per call from the torch profiler (CUPTI), next to the wall time of the
call.  argv[1] = N."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import profile, ProfilerActivity
from paper_2104_00897_b200 import ftblas as F

m = n = k = int(sys.argv[1]) if len(sys.argv) > 1 else 256
A = torch.rand(m * k, dtype=torch.float64, device="cuda"); B = torch.rand(k * n, dtype=torch.float64, device="cuda")
C = torch.zeros(m * n, dtype=torch.float64, device="cuda")
R = 20

calls = {
    "noft": lambda: F.ftblas_dgemm_noft("N", "N", m, n, k, 1.0, A, m, B, k, 0.0, C, m),
    "ft_noreport": lambda: F.ftblas_dgemm("N", "N", m, n, k, 1.0, A, m, B, k, 0.0, C, m, report=False),
    "ft_report": lambda: F.ftblas_dgemm("N", "N", m, n, k, 1.0, A, m, B, k, 0.0, C, m),
    "ft_report_fault": lambda: (F.ftblas_inject_arm([(17, 203, 128, 1e3)]),
                                F.ftblas_dgemm("N", "N", m, n, k, 1.0, A, m, B, k, 0.0, C, m)),
}
for name, fn in calls.items():
    for _ in range(10): fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(R): fn(); torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / R * 1e6
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        for _ in range(R): fn(); torch.cuda.synchronize()
    dev = {}
    for ev in prof.events():
        if ev.device_type == torch.autograd.DeviceType.CUDA:
            dev.setdefault(ev.name, []).append(ev.device_time_total if hasattr(ev, "device_time_total") else ev.cuda_time_total)
    print(f"== {name}: wall {wall:.1f} us per call (with sync)")
    for kname, ts in sorted(dev.items(), key=lambda kv: -sum(kv[1])):
        print(f"   {len(ts) / R:4.1f}/call  {sum(ts) / len(ts):8.1f} us  {kname[:90]}")
    # host API time per call (cudaLaunchKernel, cudaMemcpyAsync, cudaStreamSynchronize, ...)
    host = {}
    for ev in prof.events():
        if ev.device_type == torch.autograd.DeviceType.CPU and ev.name.startswith("cuda"):
            host.setdefault(ev.name, []).append(ev.cpu_time_total)
    for hname, ts in sorted(host.items(), key=lambda kv: -sum(kv[1])):
        print(f"   host {len(ts) / R:4.1f}/call  {sum(ts) / len(ts):8.1f} us  {hname}")
