"""bench.py — protected (ABFT) FP64 DGEMM throughput on B200, BASELINE.json metric.

Default workload: config C5 (m = n = k = 32768, NN, U[-1,1], 100 injected errors in
total, C row panels over the ranks, error counters all-reduced over NCCL), which is the
configuration the metric is quoted on ("at 1/2/4/8 B200") and fits one GPU.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5|C4a|C4b|C3|C2|C1]
    torchrun --nproc-per-node N bench.py --gpus N ...      (N > 1)
    python bench.py --impl reference ...                   (the CPU oracle arm)

One step = one protected DGEMM of the whole workload (every §8(a) row: staging, fused
encode, DMMA update, carry, fault hook, verify/locate/correct, store, report) plus the
NCCL all-reduce of the error counters.  Inputs are resident in HBM before timing; they
are larger than L2 (8.6 GB per operand), so no flush is needed.  Device time is taken
with CUDA events on the launch stream, barrier + synchronize on both sides, max over
ranks.  The unprotected twin is timed the same way for the overhead; the end-to-end
number goes through ftblas_dgemm_host (pinned host buffers, H2D + D2H in the region).
"""
from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ABFT-DGEMM FP64 TFLOP/s and % of FP64 peak; ABFT overhead % at 1/2/4/8 B200"
# FP64 ceiling measured on this pool's B200 by microbench/fp64_peak.cu (DMMA.8x8x4,
# 148 SMs, 1965 MHz; profiles/fp64_peak.json): MEASURED_PEAKS.json has no FP64 entry.
FP64_PEAK_TFLOPS = 37.0
FP64_NOMINAL_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="C5")
    p.add_argument("--size", type=int, default=0, help="override C5 size (dev only)")
    p.add_argument("--seed", type=int, default=1234)
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-unfused", action="store_true", help="skip the comparison timings (PREPASS encode, unfused baseline, no-fault protected, cuBLAS)")
    p.add_argument("--interval", type=int, default=0,
                   help="verification interval Kc (multiple of 16; 0 = k): ftblas_set_interval")
    p.add_argument("--cpu-sample-units", type=int, default=0)
    return p.parse_args()


# ------------------------------------------------------------------ workload description
def workload(cfg: str, size: int, seed: int):
    """Problem shape, trans, alpha/beta, fault list (global indices), distribution."""
    import synth
    if cfg == "C5":
        n = size or synth.C5_N
        return dict(name=f"C5 NN {n}^3 row-panels", m=n, n=n, k=n, ta="N", tb="N", alpha=1.0,
                    beta=0.0, dist="uniform", faults=synth.c5_faults(seed, size=n))
    c = {"C1": (256, 256, 256), "C2": (2048, 2048, 2048), "C3": (8192, 8192, 8192),
         "C4a": (16384, 16384, 1024), "C4b": (16384, 512, 16384)}[cfg[:2] if cfg.startswith("C3") else cfg]
    m, n, k = c
    alpha, beta = (1.5, 0.5) if cfg == "C2" else (1.0, 0.0)
    tr = cfg[2:] if cfg.startswith("C3") and len(cfg) == 4 else "NN"  # C3 / C3NT / C3TN / C3TT
    if cfg == "C1":
        faults = [(17, 203, 128, 1e3)]
    elif cfg.startswith("C3"):
        faults = synth.seeded_faults(seed + 1, 20, m, n, k, *synth.FAULT_LOG10)
    elif cfg in ("C4a", "C4b"):
        faults = synth.seeded_faults(seed + 1, round(2 * m * n * k / 1e11), m, n, k, *synth.FAULT_LOG10)
    else:
        faults = []
    return dict(name=f"{cfg} {tr} {m}x{n}x{k}", m=m, n=n, k=k, ta=tr[0], tb=tr[1], alpha=alpha,
                beta=beta, dist="normal" if cfg.startswith("C3") else "uniform", faults=faults)


def gen_panel(torch, rows, cols, seed, tag, idx, dist, device):
    """Seeded device-side generation of a rows x cols column-major panel (flat tensor)."""
    g = torch.Generator(device=device)
    g.manual_seed((seed * 1000003 + tag * 7919 + idx) & 0x7FFFFFFFFFFFFFFF)
    if dist == "normal":
        return torch.randn(rows * cols, dtype=torch.float64, device=device, generator=g)
    return torch.rand(rows * cols, dtype=torch.float64, device=device, generator=g).mul_(2).sub_(1)


# ------------------------------------------------------------------ clocks sampler
class Clocks:
    def __init__(self, index: int):
        self.samples, self.proc, self.index = [], None, index

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,power.draw,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # nvidia-smi's start-up (process spawn, NVML init) must not overlap the timed region
            # of a short workload: wait for its first sample (bounded).
            t_end = time.time() + 5.0
            while not self.samples and time.time() < t_end and self.proc.poll() is None:
                time.sleep(0.01)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 3 + i and s[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "power_w_max": max(float(s[2]) for s in self.samples if s[2].replace(".", "").isdigit())
                if self.samples else None, "samples": len(self.samples)}


# ------------------------------------------------------------------ CPU oracle arm
def oracle_sample(W, rank_rows, seed, units_wanted, torch, A_dev, B_dev, lda, ldb, BM, BN, BK):
    """Run the oracle (as it stands) on a bounded sample of units of this workload:
    the units containing faults first, then seeded random units.  Returns
    (tflops, seconds, units, threads)."""
    import numpy as np
    import oracle
    m, n, k = rank_rows, W["n"], W["k"]
    faults = W["local_faults"]
    units = []
    for (i, j, s, d) in faults:
        u = (i // BM, j // BN)
        if u not in units:
            units.append(u)
    units = units[:16]
    rng = np.random.default_rng(seed)
    tm, tn = -(-m // BM), -(-n // BN)
    # Extra units are drawn from the same tile rows/columns (bounded host copies), topped up
    # with seeded random tile rows/columns when there are too few faults.
    rset = sorted({u[0] for u in units} | {int(x) for x in rng.integers(0, tm, max(0, 4 - len(units)))})
    cset = sorted({u[1] for u in units} | {int(x) for x in rng.integers(0, tn, max(0, 4 - len(units)))})
    cand = [(a, b) for a in rset for b in cset if (a, b) not in units]
    rng.shuffle(cand)
    units += cand[:max(0, units_wanted - len(units))]
    # Host copies of just the rows / columns the sampled units read (column-major, 'N').
    rows = sorted({ti for ti, _ in units})
    cols = sorted({tj for _, tj in units})
    Ah = A_dev.view(k, lda)  # [p][i]
    Bh = B_dev.view(n, ldb)  # [j][p]
    Asub = np.concatenate([Ah[:, r * BM:(r + 1) * BM].cpu().numpy() for r in rows], axis=1)
    Bsub = np.concatenate([Bh[c * BN:(c + 1) * BN, :].cpu().numpy() for c in cols], axis=0)
    ms, ns = Asub.shape[1], Bsub.shape[0]
    A_f = np.ascontiguousarray(Asub.reshape(-1))      # (ms x k) column-major, ld = ms
    B_f = np.ascontiguousarray(Bsub.reshape(-1))      # (k x ns) column-major, ld = k
    rmap = {r: q for q, r in enumerate(rows)}
    cmap = {c: q for q, c in enumerate(cols)}
    sub_units = [(rmap[ti], cmap[tj]) for ti, tj in units]
    sub_faults = [(rmap[i // BM] * BM + i % BM, cmap[j // BN] * BN + j % BN, s, d)
                  for (i, j, s, d) in faults if (i // BM, j // BN) in units]
    C0 = np.zeros(ms * ns)
    t0 = time.perf_counter()
    _, rep = oracle.dgemm_abft("N", "N", ms, ns, k, W["alpha"], A_f, ms, B_f, k, 0.0, C0, ms,
                               BM=BM, BN=BN, BK=BK, faults=sub_faults, units=sub_units)
    dt = time.perf_counter() - t0
    flops = 2.0 * BM * BN * k * len(units)
    return flops / dt / 1e12, dt, len(units), oracle.num_threads(), rep


def unit_geometry():
    """(BM, BN, BK) of the library's verification units (header constants; no GPU needed)."""
    try:
        from paper_2104_00897_b200 import ftblas as F
        return F.ftblas_get_geometry()
    except Exception:  # library not built: the documented constants
        return 127, 127, 16


def reference_arm(args):
    """--impl reference: the CPU oracle, as it stands, on the box's host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import numpy as np
    import oracle
    import synth
    W = workload(args.config, args.size, args.seed)
    k = W["k"]
    BM, BN, BK = unit_geometry()
    threads = oracle.num_threads()
    units_per_step = max(2, min(threads, 64))
    rng = np.random.default_rng(args.seed)
    # A bounded sample per step: `units_per_step` verification units of the workload, with
    # their operand rows/columns drawn with the workload's recipe.
    Arows = synth.matrix(args.seed, "refA", BM * units_per_step, k, W["dist"]) if k <= 8192 else None
    times = []
    for step in range(args.warmup + args.steps):
        if Arows is None:
            Arows = synth.matrix(args.seed, "refA", BM * units_per_step, k, W["dist"])
        B = synth.matrix(args.seed, "refB", k, BN, W["dist"])
        units = [(u, 0) for u in range(units_per_step)]
        fl = [(int(rng.integers(0, BM)), int(rng.integers(0, BN)), int(rng.integers(0, k)), 10.0)]
        t0 = time.perf_counter()
        oracle.dgemm_abft("N", "N", BM * units_per_step, BN, k, W["alpha"], Arows,
                          BM * units_per_step, B, k, 0.0, np.zeros((BM * units_per_step, BN)),
                          BM * units_per_step, BM=BM, BN=BN, BK=BK, faults=fl, units=units)
        if step >= args.warmup:
            times.append(time.perf_counter() - t0)
    t = sum(times) / len(times)
    v = 2.0 * BM * BN * k * units_per_step / t / 1e12
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "TFLOP/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": W["name"], "m": W["m"], "n": W["n"], "k": k},
            "cpu_baseline": {"value": v, "unit": "TFLOP/s", "cores": threads, "kind": "oracle",
                             "sample": f"{units_per_step} verification units ({BM}x{BN}, k={k}) "
                                       "of the workload per step, one injected error"},
            "e2e": {"value": v, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our arm
def main():
    args = parse()
    if args.impl == "reference":
        reference_arm(args)
        return
    import torch
    import torch.distributed as dist

    from paper_2104_00897_b200 import ftblas as F
    from paper_2104_00897_b200.parallel import RowPanelPartitioner

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    F.load()

    W = workload(args.config, args.size, args.seed)
    part = RowPanelPartitioner(W["m"], world, unit_rows=F.ftblas_get_geometry()[0])
    r0, r1 = part.rows(rank)
    mloc, n, k = r1 - r0, W["n"], W["k"]
    W["local_faults"] = part.route_faults(W["faults"], rank)
    ta, tb, alpha, beta = W["ta"], W["tb"], W["alpha"], W["beta"]
    lda = k if ta == "T" else mloc
    ldb = n if tb == "T" else k

    # Inputs: A panel(s) drawn per 128-row block group so the data is identical for every P.
    A = torch.empty(mloc * k, dtype=torch.float64, device=dev)
    Av = A.view(k, mloc) if ta == "N" else A.view(mloc, k)
    panel = part.gen_block_rows
    for (g0, g1) in panel(r0, r1):
        blk = gen_panel(torch, g1 - g0, k, args.seed, 1, g0 // panel.block, W["dist"], dev)
        if ta == "N":
            Av[:, g0 - r0:g1 - r0] = blk.view(k, g1 - g0)
        else:
            Av[g0 - r0:g1 - r0, :] = blk.view(g1 - g0, k)
        del blk
    B = gen_panel(torch, k, n, args.seed, 2, 0, W["dist"], dev)
    C = torch.zeros(mloc * n, dtype=torch.float64, device=dev)
    C0 = gen_panel(torch, mloc, n, args.seed, 3, rank, "uniform", dev) if beta != 0.0 else None
    torch.cuda.synchronize()

    stream = torch.cuda.current_stream(dev)
    F.ftblas_set_stream(stream)
    F.ftblas_set_interval(args.interval)
    counters = torch.zeros(5, dtype=torch.int64, device=dev)

    def step(ft=True):
        """ft: True = the fused protected kernel, False = the unprotected twin,
        "unfused" = the unfused ABFT baseline (NEXT-2), same faults and report,
        "clean" = the fused protected kernel with no fault armed,
        "async" = the fused protected kernel with its faults, no report (no host synchronisation)."""
        if beta != 0.0:
            C.copy_(C0)
        if ft:
            if ft != "clean":
                F.ftblas_inject_arm(W["local_faults"])
            call = F.ftblas_dgemm_unfused if ft == "unfused" else F.ftblas_dgemm
            if ft == "async":
                call(ta, tb, mloc, n, k, alpha, A, lda, B, ldb, beta, C, mloc, report=False)
                return None
            rep = call(ta, tb, mloc, n, k, alpha, A, lda, B, ldb, beta, C, mloc, events_capacity=1024)
            if world > 1:
                counters.copy_(torch.tensor([rep.units_checked, rep.detected, rep.corrected,
                                             rep.recomputed, rep.n_events], dtype=torch.int64))
                dist.all_reduce(counters)  # NCCL over NVLink: the only collective
            return rep
        F.ftblas_dgemm_noft(ta, tb, mloc, n, k, alpha, A, lda, B, ldb, beta, C, mloc)
        return None

    def timed(ft, steps, warmup, label=None):
        # Collect before the warm-up (a collection between warm-up and timed region leaves the
        # GPU idle for milliseconds, and the first timed step of a short workload then pays the
        # ramp back up), and no collector pause inside the timed region.
        gc.collect()
        gc.disable()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
        for e in ev:  # create the CUDA events outside the timed region
            e.record(stream)
        for _ in range(warmup):
            step(ft)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        F.ftblas_take_launch_count()
        ev[0].record(stream)
        reps = []
        for i in range(steps):
            reps.append(step(ft))
            ev[i + 1].record(stream)
        torch.cuda.synchronize()
        gc.enable()
        launches = F.ftblas_take_launch_count()
        ms = ev[0].elapsed_time(ev[-1])
        per = [ev[i].elapsed_time(ev[i + 1]) for i in range(steps)]
        if world > 1:
            t = torch.tensor([ms] + per, dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms, per = float(t[0].item()), [float(x) for x in t[1:].tolist()]
            dist.barrier()
        timed.min_ms[label if label is not None else ft] = min(per)
        timed.per[label if label is not None else ft] = per
        return ms, launches, reps
    timed.min_ms = {}
    timed.per = {}

    # Kernel-only time of the dominant kernel for the roofline: same launches, events
    # bracketing only the ftblas_dgemm call (report copy excluded) on the launch stream.
    with Clocks(local) as clk:
        ms_ft, launches, reps = timed(True, args.steps, args.warmup)
    if world == 1:
        r_ = reps[-1]
        counters.copy_(torch.tensor([r_.units_checked, r_.detected, r_.corrected, r_.recomputed, r_.n_events],
                                    dtype=torch.int64))
    cnt = counters.cpu().tolist()  # all-reduced counters of the last protected step
    ms_noft, _, _ = timed(False, args.steps, max(1, args.warmup // 2))
    pre = None
    if not args.no_unfused:
        F.ftblas_set_encode(F.ENCODE_PREPASS)
        try:
            ms_pre, _, reps_pre = timed(True, args.steps, max(1, args.warmup // 2), label="prepass")
        finally:
            F.ftblas_set_encode(F.ENCODE_FUSED)
        rp = reps_pre[-1]
        pre = {"tflops": 2.0 * W["m"] * n * k * args.steps / (ms_pre * 1e-3) / 1e12,
               "overhead_pct": 100.0 * (ms_pre - ms_noft) / ms_noft, "units_checked": rp.units_checked,
               "detected": rp.detected, "corrected": rp.corrected, "recomputed": rp.recomputed}
    unf = None
    if not args.no_unfused:
        ms_unf, _, reps_unf = timed("unfused", args.steps, max(1, args.warmup // 2))
        ru = reps_unf[-1]
        unf = {"tflops": 2.0 * W["m"] * n * k * args.steps / (ms_unf * 1e-3) / 1e12,
               "overhead_pct": 100.0 * (ms_unf - ms_noft) / ms_noft, "unit": "128x128",
               "units_checked": ru.units_checked, "detected": ru.detected, "corrected": ru.corrected,
               "recomputed": ru.recomputed}
    ms_clean = ms_async = None
    if not args.no_unfused:
        ms_clean, _, _ = timed("clean", args.steps, 1)
        ms_async, _, _ = timed("async", args.steps, 1)
    # cuBLAS DGEMM (torch.matmul on float64) on the same operands: a measuring stick, not a target.
    ms_cublas = None
    if not args.no_unfused:
        Aop = A.view(k, mloc).t() if ta == "N" else A.view(mloc, k)
        Bop = B.view(n, k).t() if tb == "N" else B.view(k, n)
        torch.matmul(Aop, Bop)
        torch.cuda.synchronize()
        cb = []
        for _ in range(2):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            Ct = torch.matmul(Aop, Bop)
            e1.record(stream)
            torch.cuda.synchronize()
            cb.append(e0.elapsed_time(e1))
            del Ct
        ms_cublas = min(cb)
        if world > 1:
            t = torch.tensor([ms_cublas], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms_cublas = float(t.item())
    kern = []
    for _ in range(max(2, min(args.steps, 3))):
        F.ftblas_inject_arm(W["local_faults"])
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        F.ftblas_dgemm(ta, tb, mloc, n, k, alpha, A, lda, B, ldb, beta, C, mloc, report=False)
        e1.record(stream)
        torch.cuda.synchronize()
        kern.append(e0.elapsed_time(e1))
    kern_ms = statistics.mean(kern)

    flops_total = 2.0 * W["m"] * n * k
    tflops = flops_total * args.steps / (ms_ft * 1e-3) / 1e12
    tflops_noft = flops_total * args.steps / (ms_noft * 1e-3) / 1e12
    rep = reps[-1]

    # End to end through the public host-buffer API (pinned host memory, H2D + D2H inside).
    e2e = None
    if not args.no_e2e:
        Ah = torch.empty(A.numel(), dtype=torch.float64, pin_memory=True)
        Bh = torch.empty(B.numel(), dtype=torch.float64, pin_memory=True)
        Ch = torch.empty(C.numel(), dtype=torch.float64, pin_memory=True)
        Ah.copy_(A)
        Bh.copy_(B)
        if C0 is not None:
            Ch.copy_(C0)
        torch.cuda.synchronize()
        ts = []
        for it in range(1 + max(1, min(args.steps, 3))):
            if world > 1:
                dist.barrier()
            F.ftblas_inject_arm(W["local_faults"])
            t0 = time.perf_counter()
            F.ftblas_dgemm_host(ta, tb, mloc, n, k, alpha, Ah, lda, Bh, ldb, beta, Ch, mloc,
                                report=True, events_capacity=1024)
            dt = time.perf_counter() - t0
            if it:
                ts.append(dt)
        dt = statistics.mean(ts)
        if world > 1:
            t = torch.tensor([dt], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t.item())
        h2d = 8 * (A.numel() + B.numel() + (C.numel() if beta != 0.0 else 0)) * world
        e2e = {"value": flops_total / dt / 1e12, "unit": "TFLOP/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": 8 * W["m"] * n, "ms_per_step": dt * 1e3}
        del Ah, Bh, Ch

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import oracle
        nthreads = oracle.num_threads()
        # ~10-30 s of host work: every unit holding a fault plus seeded random units.
        BM, BN, BK = F.ftblas_get_geometry()
        per_unit = 2.0 * BM * BN * k
        want = args.cpu_sample_units or int(max(len({(i // BM, j // BN) for i, j, _, _ in W["local_faults"]}),
                                                min(4096, 1.5e10 * nthreads / per_unit)))
        v, dt, nu, thr, orep = oracle_sample(W, mloc, args.seed, want, torch, A, B, lda, ldb, BM, BN, BK)
        cpu = {"value": v, "unit": "TFLOP/s", "cores": thr, "kind": "oracle",
               "sample": f"{nu} verification units ({BM}x{BN}, k={k}) of the workload incl. every "
                         f"unit holding a fault; {dt:.1f} s; oracle found {orep.detected} flagged units"}

    achieved = flops_total / world / (kern_ms * 1e-3) / 1e12
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        traffic = json.load(open(tp)).get(f"{args.config}:{W['m']}:{world}")
    line = {
        "metric": METRIC, "value": tflops, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_ft / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": W["name"], "m": W["m"], "n": n, "k": k, "trans": ta + tb,
                   "alpha": alpha, "beta": beta, "dist": W["dist"], "faults_per_step": len(W["faults"]),
                   "parallelism": f"row-panels x{world}", "l2": "inputs larger than L2 (no flush)",
                   "interval_Kc": args.interval or k},
        "abft": {"tflops_protected": tflops, "tflops_unprotected": tflops_noft,
                 "overhead_pct": 100.0 * (ms_ft - ms_noft) / ms_noft,
                 "pct_of_fp64_peak": 100.0 * tflops / (world * FP64_PEAK_TFLOPS),
                 "units_checked": cnt[0], "detected": cnt[1], "corrected": cnt[2],
                 "recomputed": cnt[3], "events": cnt[4],
                 "prepass_encode": pre, "unfused_baseline": unf,
                 "ms_per_step_min": {"protected": timed.min_ms.get(True), "unprotected": timed.min_ms.get(False)},
                 "ms_per_step_all": {"protected": timed.per.get(True), "unprotected": timed.per.get(False)},
                 "tflops_protected_no_faults": (flops_total * args.steps / (ms_clean * 1e-3) / 1e12
                                                if ms_clean else None),
                 # the protected call without a report (asynchronous, like the unprotected one):
                 # the computational overhead without the report's host round trip per call
                 "async_no_report": ({"tflops": flops_total * args.steps / (ms_async * 1e-3) / 1e12,
                                      "overhead_pct": 100.0 * (ms_async - ms_noft) / ms_noft}
                                     if ms_async else None),
                 "cublas_dgemm_tflops": flops_total / (ms_cublas * 1e-3) / 1e12 if ms_cublas else None},
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": FP64_PEAK_TFLOPS,
                     "unit": "TFLOP/s", "frac": achieved / FP64_PEAK_TFLOPS, "traffic": traffic,
                     "kernel": "dgemm_abft_kernel (FT)", "kernel_ms": kern_ms,
                     "peak_source": "measured FP64 DMMA microbenchmark (profiles/fp64_peak.json); "
                                    f"nominal {FP64_NOMINAL_TFLOPS:.1f}"},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
