"""DMR Level-1/2 benchmark: achieved HBM bandwidth of the protected
routines and their unprotected twins, DMR overhead %, with and without injected faults, and
the same operation through torch (cuBLAS / torch elementwise kernels) as a measuring stick.
CUDA events on the launch stream, best of R after warm-up; inputs larger than L2.
Prints one JSON object per routine."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2104_00897_b200 import ftblas as F  # noqa: E402

R = 10
PEAK = 6549.8  # MEASURED_PEAKS.json hbm_gbs (copy bandwidth, read + write)


def timed(fn):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(R):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


def line(name, nbytes, t_ft, t_noft, t_inj, rep, t_torch):
    print(json.dumps({"routine": name, "bytes": nbytes, "ms_dmr": t_ft, "ms_noft": t_noft, "ms_dmr_faults": t_inj,
                      "gbs_dmr": nbytes / t_ft / 1e6, "gbs_noft": nbytes / t_noft / 1e6,
                      "gbs_torch": nbytes / t_torch / 1e6,
                      "frac_hbm_dmr": nbytes / t_ft / 1e6 / PEAK, "overhead_pct": 100 * (t_ft - t_noft) / t_noft,
                      "faults_report": rep.__dict__ if rep else None}), flush=True)


def main():
    g = torch.Generator(device="cuda").manual_seed(0)
    n = 1 << 28  # 2 GiB per vector
    x = torch.rand(n, dtype=torch.float64, device="cuda", generator=g)
    y = torch.rand(n, dtype=torch.float64, device="cuda", generator=g)
    faults = [(int(i), 0, 0, 1.0) for i in torch.randint(0, n, (16,), generator=g, device="cuda").tolist()]

    def inj(call):
        def f():
            F.ftblas_inject_arm(faults)
            call()
        return f
    t1 = timed(lambda: F.ftblas_dscal(n, 1.0000001, x, 1, report=False))
    t0 = timed(lambda: F.ftblas_dscal_noft(n, 1.0000001, x, 1))
    ti = timed(inj(lambda: F.ftblas_dscal(n, 1.0000001, x, 1, report=False)))
    F.ftblas_inject_arm(faults)
    line("dscal", 16 * n, t1, t0, ti, F.ftblas_dscal(n, 1.0, x, 1), timed(lambda: x.mul_(1.0000001)))
    t1 = timed(lambda: F.ftblas_daxpy(n, 1e-9, x, 1, y, 1, report=False))
    t0 = timed(lambda: F.ftblas_daxpy_noft(n, 1e-9, x, 1, y, 1))
    ti = timed(inj(lambda: F.ftblas_daxpy(n, 1e-9, x, 1, y, 1, report=False)))
    F.ftblas_inject_arm(faults)
    line("daxpy", 24 * n, t1, t0, ti, F.ftblas_daxpy(n, 0.0, x, 1, y, 1), timed(lambda: y.add_(x, alpha=1e-9)))
    del x, y
    m = k = 16384
    A = torch.rand(m * k, dtype=torch.float64, device="cuda", generator=g)
    v = torch.rand(max(m, k), dtype=torch.float64, device="cuda", generator=g)
    w = torch.rand(max(m, k), dtype=torch.float64, device="cuda", generator=g)
    gf = [(int(i), 0, int(s), 1.0) for i, s in zip(torch.randint(0, m, (16,), generator=g, device="cuda").tolist(),
                                                    torch.randint(0, k, (16,), generator=g, device="cuda").tolist())]
    for tr in "NT":
        call = lambda: F.ftblas_dgemv(tr, m, k, 1.0, A, m, v, 1, 0.5, w, 1, report=False)  # noqa: E731
        t1 = timed(call)
        t0 = timed(lambda: F.ftblas_dgemv_noft(tr, m, k, 1.0, A, m, v, 1, 0.5, w, 1))

        def ci():
            F.ftblas_inject_arm(gf)
            call()
        ti = timed(ci)
        F.ftblas_inject_arm(gf)
        Am = A.view(k, m).t()  # the column-major m x k matrix as a torch view
        op = Am if tr == "N" else Am.t()
        xin, yout = (v[:k], w[:m]) if tr == "N" else (v[:m], w[:k])
        t_t = timed(lambda: torch.addmv(yout, op, xin, beta=0.5, alpha=1.0, out=yout))
        line(f"dgemv_{tr}", 8 * (m * k + 2 * m + k), t1, t0, ti,
             F.ftblas_dgemv(tr, m, k, 1.0, A, m, v, 1, 0.5, w, 1), t_t)


if __name__ == "__main__":
    main()
