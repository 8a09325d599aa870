"""FT-DTRSM benchmark: protected and unprotected TFLOP/s (m^2 n FLOPs,
side L), overhead %, under 20 injected faults (as the paper's Fig. 8), and torch's float64
solve_triangular (cuBLAS) as a measuring stick.  CUDA events, best of R after warm-up."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2104_00897_b200 import ftblas as F  # noqa: E402

if len(sys.argv) > 1:  # alternative build of the library
    F.LIB_PATH = sys.argv[1]

R = 5


def timed(fn, reset):
    for _ in range(2):
        reset()
        fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(R):
        reset()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


def main():
    for m in (8192, 16384):
        n = m
        g = torch.Generator(device="cuda").manual_seed(0)
        A = torch.rand(m, m, dtype=torch.float64, device="cuda", generator=g) / m
        A = torch.tril(A) + torch.diag(1 + torch.rand(m, dtype=torch.float64, device="cuda", generator=g))
        Acm = A.t().contiguous()  # column-major storage of A
        B0 = torch.rand(n, m, dtype=torch.float64, device="cuda", generator=g)  # column-major m x n
        B = torch.empty_like(B0)
        reset = lambda: B.copy_(B0)  # noqa: E731
        flops = float(m) * m * n
        faults = []
        for q in range(20):  # cross-block faults spread over the updates
            i = int((q + 1) * (m - 1) / 21)
            faults.append((i, (q * 977) % n, max(0, i - 300 - 37 * q), 1.0 + q))
        t_ft = timed(lambda: F.ftblas_dtrsm("L", "L", "N", "N", m, n, 1.0, Acm, m, B, m, report=False), reset)
        t_no = timed(lambda: F.ftblas_dtrsm_noft("L", "L", "N", "N", m, n, 1.0, Acm, m, B, m), reset)

        def inj():
            F.ftblas_inject_arm(faults)
            F.ftblas_dtrsm("L", "L", "N", "N", m, n, 1.0, Acm, m, B, m, report=False)
        t_inj = timed(inj, reset)
        reset()
        F.ftblas_inject_arm(faults)
        rep = F.ftblas_dtrsm("L", "L", "N", "N", m, n, 1.0, Acm, m, B, m)
        Bt = B0.t()  # m x n row-major view for torch
        t_ref = timed(lambda: torch.linalg.solve_triangular(A, Bt, upper=False), lambda: None)
        print(json.dumps({"routine": "dtrsm L L N N", "m": m, "n": n, "ms_ft": t_ft, "ms_noft": t_no,
                          "ms_ft_20faults": t_inj, "tflops_ft": flops / t_ft / 1e9, "tflops_noft": flops / t_no / 1e9,
                          "tflops_ft_20faults": flops / t_inj / 1e9, "overhead_pct": 100 * (t_ft - t_no) / t_no,
                          "overhead_20faults_pct": 100 * (t_inj - t_no) / t_no,
                          "torch_solve_triangular_tflops": flops / t_ref / 1e9,
                          "faults_report": {"detected": rep.detected, "corrected": rep.corrected,
                                            "recomputed": rep.recomputed, "units": rep.units_checked}}), flush=True)
        # side R on the same sizes: X op(A) = B with op(A) = A^T (upper), every row an RHS
        t_ftr = timed(lambda: F.ftblas_dtrsm("R", "L", "T", "N", m, n, 1.0, Acm, m, B, m, report=False), reset)
        t_nor = timed(lambda: F.ftblas_dtrsm_noft("R", "L", "T", "N", m, n, 1.0, Acm, m, B, m), reset)
        t_refr = timed(lambda: torch.linalg.solve_triangular(A.t(), Bt, upper=True, left=False), lambda: None)
        print(json.dumps({"routine": "dtrsm R L T N", "m": m, "n": n, "ms_ft": t_ftr, "ms_noft": t_nor,
                          "tflops_ft": flops / t_ftr / 1e9, "tflops_noft": flops / t_nor / 1e9,
                          "overhead_pct": 100 * (t_ftr - t_nor) / t_nor,
                          "torch_solve_triangular_tflops": flops / t_refr / 1e9}), flush=True)
        del A, Acm, B0, B, Bt


if __name__ == "__main__":
    main()
