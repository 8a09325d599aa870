"""cuBLAS FP64 DGEMM via torch.matmul — a measuring stick only (never in the product path)."""
import json, torch
n = 8192
a = torch.randn(n, n, dtype=torch.float64, device="cuda")
b = torch.randn(n, n, dtype=torch.float64, device="cuda")
for _ in range(3):
    c = a @ b
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ts = []
for _ in range(10):
    e0.record(); c = a @ b; e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
best = min(ts); mean = sum(ts) / len(ts)
print(json.dumps({"cublas_dgemm_n": n, "best_ms": best, "mean_ms": mean,
                  "best_tflops": 2 * n**3 / best / 1e9, "mean_tflops": 2 * n**3 / mean / 1e9}))
