"""bench.py — protected (ABFT) FP64 DGEMM throughput on B200, BASELINE.json metric.

Default workload: config C5 (m = n = k = 32768, NN, U[-1,1], 100 injected errors in
total, C row panels over the ranks, error counters all-reduced over NCCL), which is the
configuration the metric is quoted on ("at 1/2/4/8 B200") and fits one GPU.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5|C4a|C4b|C3|C2|C1]
    torchrun --nproc-per-node N bench.py --gpus N ...      (N > 1)
    python bench.py --impl reference ...                   (the CPU oracle arm)

One step = one protected DGEMM of the whole workload (every §8(a) row: staging, fused
encode, DMMA update, carry, fault hook, verify/locate/correct, store, report) plus the
all-reduce of the error counters.  Inputs are resident in HBM before timing; they are larger
than L2 (8.6 GB per operand), so no flush is needed.  Device time is taken with CUDA events
on the launch stream, barrier + synchronize on both sides, max over ranks.

Beside the contract's K timed steps the line carries:
  abft        the ABFT overhead from K interleaved (protected, unprotected) pairs, the PREPASS
              encode and the unfused baseline (NEXT-2), cuBLAS DGEMM as a measuring stick;
  roofline    the protected kernel's FP64 throughput against the measured DMMA peak;
  e2e         the same metric through ftblas_dgemm_host (pinned host buffers, H2D + D2H inside);
  cpu_baseline + parity   (rank 0, N = 1) the oracle on a bounded sample of the workload's
              verification units -- every unit holding a fault plus seeded units -- timed on
              the host cores and compared with the GPU result: values, counters, events;
  per_config  (N = 1) short interleaved protected / unprotected runs of C1-C4b.
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
# The library's verification-unit geometry as documented in include/ftblas.h (127 x 127 data
# rows / columns of the 128 x 128 C^f tile, step quantum 16).  The reference arm uses these
# constants so that it never loads libftblas.so; our arm reads them from the library.
DOC_GEOMETRY = (127, 127, 16)
U = 2.0 ** -53


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="C5")
    p.add_argument("--size", type=int, default=0, help="override C5 size (dev only)")
    p.add_argument("--seed", type=int, default=1234)
    p.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                   help="process-group backend for N > 1 (gloo: host-side test of the multi-rank path)")
    p.add_argument("--one-device", action="store_true",
                   help="every rank on cuda:0 (test of the multi-rank code path on one GPU; ranks never wait on each other's kernels)")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-per-config", action="store_true")
    p.add_argument("--no-unfused", action="store_true",
                   help="skip the comparison timings (PREPASS encode, unfused baseline, cuBLAS)")
    p.add_argument("--interval", type=int, default=0,
                   help="verification interval Kc (multiple of 16; 0 = k): ftblas_set_interval")
    p.add_argument("--cpu-sample-units", type=int, default=0)
    p.add_argument("--no-sweep", action="store_true",
                   help="skip the verification-interval sweep (fused vs unfused at Kc, overhead model)")
    return p.parse_args()


# ------------------------------------------------------------------ workload description
def workload(cfg: str, size: int, seed: int):
    """Problem shape, trans, alpha/beta, fault list (global indices), distribution."""
    import synth
    if cfg == "C5":
        n = size or synth.C5_N
        return dict(name=f"C5 NN {n}^3 row-panels", cfg="C5", m=n, n=n, k=n, ta="N", tb="N", alpha=1.0,
                    beta=0.0, dist="uniform", faults=synth.c5_faults(seed, size=n))
    base = cfg[:2] if cfg.startswith("C3") else cfg
    m, n, k = {"C1": (256, 256, 256), "C2": (2048, 2048, 2048), "C3": (8192, 8192, 8192),
               "C4a": (16384, 16384, 1024), "C4b": (16384, 512, 16384)}[base]
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
    return dict(name=f"{cfg} {tr} {m}x{n}x{k}", cfg=cfg, m=m, n=n, k=k, ta=tr[0], tb=tr[1], alpha=alpha,
                beta=beta, dist="normal" if cfg.startswith("C3") else "uniform", faults=faults)


def config_dict(W, world, args):
    return {"workload": W["name"], "m": W["m"], "n": W["n"], "k": W["k"], "trans": W["ta"] + W["tb"],
            "alpha": W["alpha"], "beta": W["beta"], "dist": W["dist"], "faults_per_step": len(W["faults"]),
            "parallelism": f"row-panels x{world}", "l2": "inputs larger than L2 (no flush)",
            "interval_Kc": args.interval or W["k"]}


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
            # nvidia-smi's start-up must not overlap the timed region of a short workload: wait
            # for its first sample (bounded).
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
        pw = [float(s[2]) for s in self.samples if s[2].replace(".", "").isdigit()]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "power_w_max": max(pw) if pw else None, "samples": len(self.samples)}


# ------------------------------------------------------------------ CPU oracle arm
def reference_arm(args):
    """--impl reference: the CPU oracle, as it stands, on the box's host cores, on a bounded
    sample of the workload's verification units per step.  Never loads libftblas.so."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import numpy as np
    import oracle
    import synth
    world = int(os.environ.get("WORLD_SIZE", "1"))
    W = workload(args.config, args.size, args.seed)
    k = W["k"]
    BM, BN, BK = DOC_GEOMETRY
    threads = oracle.num_threads()
    units_per_step = max(2, min(threads, 64))
    rng = np.random.default_rng(args.seed)
    # A bounded sample per step: `units_per_step` verification units of the workload, with
    # their operand rows / columns drawn with the workload's recipe and one injected error.
    Arows = synth.matrix(args.seed, "refA", BM * units_per_step, k, W["dist"])
    B = synth.matrix(args.seed, "refB", k, BN, W["dist"])
    times = []
    for step in range(args.warmup + args.steps):
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
            "data": "synthetic", "config": config_dict(W, world, args),
            "cpu_baseline": {"value": v, "unit": "TFLOP/s", "cores": threads, "kind": "oracle",
                             "sample": f"{units_per_step} verification units ({BM}x{BN}, k={k}) "
                                       "of the workload per step, one injected error"},
            "e2e": {"value": v, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ oracle sample + parity
def oracle_parity(W, torch, A_dev, B_dev, C_dev, rep, BM, BN, BK, units_wanted, seed):
    """The oracle (as it stands) on a bounded sample of this workload's verification units:
    EVERY unit holding a fault, then seeded units drawn from the same tile rows / columns (so
    the host copies stay bounded).  Timed on the host cores (cpu_baseline), then compared with
    the GPU result of the same call: every element of every sampled unit within
    2 k u |op(A)||op(B)| (alpha = 1, beta = 0 at C5), the GPU's counters and sorted events
    equal to the oracle's (every fault unit is sampled)."""
    import numpy as np
    import oracle
    m, n, k = W["m"], W["n"], W["k"]
    faults = W["faults"]
    units = []
    for (i, j, s, d) in faults:
        if (i // BM, j // BN) not in units:
            units.append((i // BM, j // BN))
    n_fault_units = len(units)
    rng = np.random.default_rng(seed)
    tm, tn = -(-m // BM), -(-n // BN)
    rset = sorted({u[0] for u in units} | {int(x) for x in rng.integers(0, tm, max(0, 4 - len(units)))})
    cset = sorted({u[1] for u in units} | {int(x) for x in rng.integers(0, tn, max(0, 4 - len(units)))})
    cand = [(a, b) for a in rset for b in cset if (a, b) not in units]
    rng.shuffle(cand)
    units += cand[:max(0, units_wanted - len(units))]
    rows = sorted({ti for ti, _ in units})
    cols = sorted({tj for _, tj in units})
    Ah = A_dev.view(k, m)   # [p][i]  (op(A) = A, 'N')
    Bh = B_dev.view(n, k)   # [j][p]
    Asub = torch.cat([Ah[:, r * BM:(r + 1) * BM] for r in rows], dim=1).cpu().numpy()
    Bsub = torch.cat([Bh[c * BN:(c + 1) * BN, :] for c in cols], dim=0).cpu().numpy()
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
    Co, orep = oracle.dgemm_abft("N", "N", ms, ns, k, W["alpha"], A_f, ms, B_f, k, 0.0, C0, ms,
                                 BM=BM, BN=BN, BK=BK, faults=sub_faults, units=sub_units)
    dt = time.perf_counter() - t0
    Co = Co.reshape((ns, ms)).T
    # values: every element of every sampled unit, bound from |op(A)||op(B)| on the device
    Cg = C_dev.view(n, m)  # [j][i]
    worst = 0.0
    for (ti, tj) in units:
        i0, i1 = ti * BM, min((ti + 1) * BM, m)
        j0, j1 = tj * BN, min((tj + 1) * BN, n)
        S = torch.matmul(Ah[:, i0:i1].t().abs(), Bh[j0:j1, :].t().abs())  # (bm x bn)
        g = Cg[j0:j1, i0:i1].t()
        si, sj = rmap[ti] * BM, cmap[tj] * BN
        o = torch.from_numpy(np.ascontiguousarray(Co[si:si + (i1 - i0), sj:sj + (j1 - j0)])).to(g.device)
        r = ((g - o).abs() / (2 * k * U * abs(W["alpha"]) * S).clamp_min(1e-300)).max().item()
        worst = max(worst, r)
    # events: the oracle's (sub coordinates -> global) against the GPU's, sorted
    def glob(i, j):
        return rows[i // BM] * BM + i % BM, cols[j // BN] * BN + j % BN
    oev = sorted((t, *glob(i, j), kind) for (t, i, j, kind, _, _) in orep.events)
    gev = sorted((t, i, j, kind) for (t, i, j, kind, _, _) in rep.events)
    counters_match = (rep.detected, rep.corrected, rep.recomputed, rep.n_events) == \
                     (orep.detected, orep.corrected, orep.recomputed, orep.n_events)
    parity = {"units": len(units), "fault_units": n_fault_units, "max_err_over_bound": worst,
              "values_within_bound": worst <= 1.0, "events_match": oev == gev, "counters_match": counters_match,
              "gpu": {"detected": rep.detected, "corrected": rep.corrected, "recomputed": rep.recomputed},
              "oracle": {"detected": orep.detected, "corrected": orep.corrected, "recomputed": orep.recomputed}}
    flops = 2.0 * BM * BN * k * len(units)
    cpu = {"value": flops / dt / 1e12, "unit": "TFLOP/s", "cores": oracle.num_threads(), "kind": "oracle",
           "sample": f"{len(units)} verification units ({BM}x{BN}, k={k}) of the workload: all "
                     f"{n_fault_units} units holding a fault + seeded units of the same tile rows / columns; "
                     f"{dt:.1f} s"}
    return cpu, parity


# ------------------------------------------------------------------ per-config lines (N = 1)
def per_config_runs(torch, F, stream, dev, seed, steps=8, warmup=1, reps=3):
    """Short interleaved protected / unprotected runs of the other BASELINE configs: per kind,
    blocks of `steps` back-to-back calls timed with CUDA events, the kinds interleaved block by
    block, the median block reported.  The protected call carries its report (a host
    synchronisation per call); `async_tflops` is the protected call without a report."""
    out = {}
    for cfg in ("C1", "C2", "C3", "C3NT", "C3TN", "C3TT", "C4a", "C4b"):
        W = workload(cfg, 0, seed)
        m, n, k, ta, tb = W["m"], W["n"], W["k"], W["ta"], W["tb"]
        A = gen_panel(torch, m, k, seed, 11, 0, W["dist"], dev)
        B = gen_panel(torch, k, n, seed, 12, 0, W["dist"], dev)
        C0 = gen_panel(torch, m, n, seed, 13, 0, "uniform", dev) if W["beta"] != 0.0 else None
        # beta != 0 (C2): one C buffer per call of a block, refilled from C0 outside the timed
        # region (DGEMM overwrites C; restoring it is not part of the operation)
        Cs = [torch.zeros(m * n, dtype=torch.float64, device=dev) for _ in range(steps if C0 is not None else 1)]
        lda = k if ta == "T" else m
        ldb = n if tb == "T" else k

        def refill():
            if C0 is not None:
                for Cb in Cs:
                    Cb.copy_(C0)

        def call(kind, i):
            C = Cs[i % len(Cs)]
            if kind == "noft":
                F.ftblas_dgemm_noft(ta, tb, m, n, k, W["alpha"], A, lda, B, ldb, W["beta"], C, m)
                return None
            F.ftblas_inject_arm(W["faults"])
            return F.ftblas_dgemm(ta, tb, m, n, k, W["alpha"], A, lda, B, ldb, W["beta"], C, m,
                                  report=(kind == "ft"))

        # Blocks of `steps` back-to-back calls per kind, the kinds interleaved block by block
        # (a call's host-side issue overlaps the previous call's kernel, as in a loop of calls;
        # the protected call with its report synchronises inside every call).
        times = {"ft": [], "noft": [], "async": []}
        rep = None
        for it in range(warmup + reps):
            for kind in ("ft", "noft", "async"):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                refill()
                torch.cuda.synchronize()
                e0.record(stream)
                for i in range(steps):
                    r = call(kind, i)
                e1.record(stream)
                torch.cuda.synchronize()
                if it >= warmup:
                    times[kind].append(e0.elapsed_time(e1) / steps)
                if r is not None:
                    rep = r
        Aop = A.view(k, m).t() if ta == "N" else A.view(m, k)
        Bop = B.view(n, k).t() if tb == "N" else B.view(k, n)
        cb = []
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            if C0 is not None:  # the same alpha / beta update through cuBLAS (addmm)
                torch.addmm(C0.view(n, m).t(), Aop, Bop, beta=W["beta"], alpha=W["alpha"])
            else:
                torch.matmul(Aop, Bop)
            e1.record(stream)
            torch.cuda.synchronize()
            cb.append(e0.elapsed_time(e1))
        fl = 2.0 * m * n * k
        t_ft, t_no, t_as = (statistics.median(times[x]) for x in ("ft", "noft", "async"))
        out[cfg] = {"shape": f"{ta}{tb} {m}x{n}x{k}", "faults": len(W["faults"]),
                    "tflops_protected": fl / t_ft / 1e9, "tflops_unprotected": fl / t_no / 1e9,
                    "overhead_pct": 100.0 * (t_ft - t_no) / t_no,
                    "async_tflops": fl / t_as / 1e9, "async_overhead_pct": 100.0 * (t_as - t_no) / t_no,
                    "cublas_tflops": fl / min(cb) / 1e9, "ms": {"protected": t_ft, "unprotected": t_no},
                    "detected": rep.detected, "corrected": rep.corrected, "recomputed": rep.recomputed,
                    "calls_per_block": steps, "blocks": reps}
        del A, B, Cs, C0
        torch.cuda.empty_cache()
    return out


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
    if args.one_device and world > 1 and args.backend != "gloo":
        raise SystemExit("--one-device needs --backend gloo (NCCL runs one rank per device)")
    local = 0 if args.one_device else int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
    cdev = dev if (world == 1 or args.backend == "nccl") else torch.device("cpu")  # collective tensors
    F.load()

    W = workload(args.config, args.size, args.seed)
    BM, BN, BK = F.ftblas_get_geometry()
    if world > 1:  # the unit partition must be the same on every rank (SURVEY §8(e) invariant)
        geo = [None] * world
        dist.all_gather_object(geo, (BM, BN, BK))
        assert all(g == (BM, BN, BK) for g in geo), geo
    part = RowPanelPartitioner(W["m"], world, unit_rows=BM)
    r0, r1 = part.rows(rank)
    mloc, n, k = r1 - r0, W["n"], W["k"]
    W["local_faults"] = part.route_faults(W["faults"], rank)
    ta, tb, alpha, beta = W["ta"], W["tb"], W["alpha"], W["beta"]
    lda = k if ta == "T" else mloc
    ldb = n if tb == "T" else k

    # Inputs: A panel(s) drawn per unit-height row block so the data is identical for every P.
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
    counters = torch.zeros(5, dtype=torch.int64, device=cdev)

    def step(kind="ft"):
        """ft: the fused protected kernel with the workload's faults and its report, counters
        all-reduced; noft: the unprotected twin; unfused: the unfused ABFT baseline (NEXT-2)."""
        if beta != 0.0:
            C.copy_(C0)
        if kind == "noft":
            F.ftblas_dgemm_noft(ta, tb, mloc, n, k, alpha, A, lda, B, ldb, beta, C, mloc)
            return None
        F.ftblas_inject_arm(W["local_faults"])
        call = F.ftblas_dgemm_unfused if kind == "unfused" else F.ftblas_dgemm
        rep = call(ta, tb, mloc, n, k, alpha, A, lda, B, ldb, beta, C, mloc, events_capacity=4096)
        if world > 1:
            counters.copy_(torch.tensor([rep.units_checked, rep.detected, rep.corrected,
                                         rep.recomputed, rep.n_events], dtype=torch.int64))
            dist.all_reduce(counters)  # the only collective of the data path
        return rep

    def sync_all():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    def max_over_ranks(vals):
        if world == 1:
            return vals
        t = torch.tensor(vals, dtype=torch.float64, device=cdev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return [float(x) for x in t.tolist()]

    # 1. the contract: W untimed warm-up steps, K timed protected steps
    gc.collect()
    gc.disable()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    for e in ev:  # created (and recorded once) outside the timed region
        e.record(stream)
    for _ in range(args.warmup):
        step("ft")
    sync_all()
    F.ftblas_take_launch_count()
    with Clocks(local) as clk:
        ev[0].record(stream)
        reps = []
        for i in range(args.steps):
            reps.append(step("ft"))
            ev[i + 1].record(stream)
        torch.cuda.synchronize()
    launches = F.ftblas_take_launch_count()
    gc.enable()
    ms_all = [ev[0].elapsed_time(ev[-1])] + [ev[i].elapsed_time(ev[i + 1]) for i in range(args.steps)]
    ms_all = max_over_ranks(ms_all)
    if world > 1:
        dist.barrier()
    ms_ft, per_ft = ms_all[0], ms_all[1:]
    rep = reps[-1]
    if world == 1:
        counters.copy_(torch.tensor([rep.units_checked, rep.detected, rep.corrected, rep.recomputed,
                                     rep.n_events], dtype=torch.int64))
    cnt = counters.cpu().tolist()  # all-reduced counters of the last protected step
    # global events on rank 0 (host gather; not part of the timed path)
    events_global = [(t, i + r0, j, kind) for (t, i, j, kind, _, _) in rep.events]
    if world > 1:
        allev = [None] * world
        dist.all_gather_object(allev, events_global)
        events_global = sorted(e for evs in allev for e in evs)

    # 2. the overhead: K interleaved (protected, unprotected) pairs, each call timed on its own
    pairs = {"ft": [], "noft": []}
    for it in range(args.steps + 1):
        for kind in ("ft", "noft"):
            sync_all()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            step(kind)
            e1.record(stream)
            torch.cuda.synchronize()
            if it > 0:  # the first pair warms the unprotected kernel
                pairs[kind].append(e0.elapsed_time(e1))
    pairs["ft"], pairs["noft"] = max_over_ranks(pairs["ft"]), max_over_ranks(pairs["noft"])
    t_pft, t_pno = statistics.mean(pairs["ft"]), statistics.mean(pairs["noft"])

    # 3. comparisons: PREPASS encode, the unfused baseline (NEXT-2), cuBLAS (measuring stick)
    flops_total = 2.0 * W["m"] * n * k
    ncmp = max(2, args.steps // 4)

    def short(kind, encode=None):
        if encode is not None:
            F.ftblas_set_encode(encode)
        try:
            step(kind)
            sync_all()
            ts, r = [], None
            for _ in range(ncmp):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                r = step(kind)
                e1.record(stream)
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
        finally:
            F.ftblas_set_encode(F.ENCODE_FUSED)
        t = statistics.mean(max_over_ranks(ts))
        return {"tflops": flops_total / (t * 1e-3) / 1e12, "overhead_pct": 100.0 * (t - t_pno) / t_pno,
                "units_checked": r.units_checked, "detected": r.detected, "corrected": r.corrected,
                "recomputed": r.recomputed, "steps": ncmp}
    pre = unf = None
    ms_cublas = None
    if not args.no_unfused:
        pre = short("ft", F.ENCODE_PREPASS)
        unf = short("unfused")
        unf["unit"] = "128x128"
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
        ms_cublas = max_over_ranks([min(cb)])[0]

    # 3b. verification every Kc updates (NEXT-1 fused online check vs the NEXT-2 unfused scheme)
    #     and the paper's overhead model of unfused ABFT:
    #     T_ovhd / T_gemm = (6 + 2K/Kc) P_mm / (n P_mv), with P_mm the unprotected DGEMM rate
    #     and P_mv the DGEMV rate measured here on the same operands.
    sweep = None
    if not args.no_sweep and world == 1 and args.interval == 0:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        xv = torch.ones(k, dtype=torch.float64, device=dev)
        yv = torch.zeros(mloc, dtype=torch.float64, device=dev)

        def gemv():  # y = op(A) x over the resident op(A) (the unprotected DGEMV, NEXT-4 twin)
            if ta == "N":
                F.ftblas_dgemv_noft("N", mloc, k, 1.0, A, mloc, xv, 1, 0.0, yv, 1)
            else:
                F.ftblas_dgemv_noft("T", k, mloc, 1.0, A, k, xv, 1, 0.0, yv, 1)
        gemv()
        torch.cuda.synchronize()
        gemv_ms = []
        for _ in range(3):
            e0.record(stream)
            gemv()
            e1.record(stream)
            torch.cuda.synchronize()
            gemv_ms.append(e0.elapsed_time(e1))
        p_mv = 2.0 * mloc * k / (min(gemv_ms) * 1e-3) / 1e12
        p_mm = flops_total / (t_pno * 1e-3) / 1e12
        rows = []
        for kc in [k, 8192, 2048, 512]:
            if kc > k or kc % 16:
                continue
            F.ftblas_set_interval(0 if kc == k else kc)
            try:
                tt = {}
                for kind in ("ft", "unfused"):
                    ts_ = []
                    for _ in range(max(1, ncmp // 2)):
                        e0.record(stream)
                        r_ = step(kind)
                        e1.record(stream)
                        torch.cuda.synchronize()
                        ts_.append(e0.elapsed_time(e1))
                    tt[kind] = (min(ts_), r_)
            finally:
                F.ftblas_set_interval(0)
            T_ = -(-k // kc)
            rows.append({"Kc": kc, "intervals": T_,
                         "fused_overhead_pct": 100.0 * (tt["ft"][0] - t_pno) / t_pno,
                         "unfused_overhead_pct": 100.0 * (tt["unfused"][0] - t_pno) / t_pno,
                         "model_unfused_pct": 100.0 * (6 + 2 * T_) * p_mm / (n * p_mv),
                         "fused_events": tt["ft"][1].n_events, "unfused_events": tt["unfused"][1].n_events,
                         "fused_units": tt["ft"][1].units_checked, "unfused_units": tt["unfused"][1].units_checked})
        sweep = {"p_mm_tflops": p_mm, "p_mv_tflops": p_mv, "p_mm_over_p_mv": p_mm / p_mv, "n": n,
                 "model": "(6 + 2K/Kc) P_mm / (n P_mv) (PAPER.md:261-265)", "rows": rows}

    # 4. the dominant kernel alone (roofline): events bracketing only the protected launch
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

    # 5. rank 0, N = 1: the oracle on a bounded sample (cpu_baseline) and parity with the GPU
    #    result of one protected call of the workload
    cpu = parity = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and args.interval == 0 \
            and ta == "N" and tb == "N" and beta == 0.0:
        import oracle
        nthreads = oracle.num_threads()
        per_unit = 2.0 * BM * BN * k
        nfu = len({(i // BM, j // BN) for i, j, _, _ in W["faults"]})
        want = args.cpu_sample_units or int(max(nfu + 16, min(4096, 1.5e10 * nthreads / per_unit)))
        F.ftblas_inject_arm(W["faults"])
        prep = F.ftblas_dgemm(ta, tb, mloc, n, k, alpha, A, lda, B, ldb, beta, C, mloc, events_capacity=1 << 16)
        cpu, parity = oracle_parity(W, torch, A, B, C, prep, BM, BN, BK, want, args.seed)

    # 6. end to end through the public host-buffer API (pinned host memory, H2D + D2H inside)
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
                                report=True, events_capacity=4096)
            dt = time.perf_counter() - t0
            if it:
                ts.append(dt)
        dt = max_over_ranks([statistics.mean(ts)])[0]
        h2d = 8 * (A.numel() + B.numel() + (C.numel() if beta != 0.0 else 0)) * world
        e2e = {"value": flops_total / dt / 1e12, "unit": "TFLOP/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": 8 * W["m"] * n, "ms_per_step": dt * 1e3}
        del Ah, Bh, Ch

    # 7. the other configurations (N = 1)
    per_config = None
    if world == 1 and not args.no_per_config and args.config == "C5" and not args.size:
        del A, B, C, C0
        torch.cuda.empty_cache()
        per_config = per_config_runs(torch, F, stream, dev, args.seed)

    achieved = flops_total / world / (kern_ms * 1e-3) / 1e12
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        traffic = json.load(open(tp)).get(f"{args.config}:{W['m']}:{world}")
    tflops = flops_total * args.steps / (ms_ft * 1e-3) / 1e12
    line = {
        "metric": METRIC, "value": tflops, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_ft / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(W, world, args),
        "abft": {"tflops_protected": tflops,
                 "tflops_unprotected": flops_total / (t_pno * 1e-3) / 1e12,
                 "overhead_pct": 100.0 * (t_pft - t_pno) / t_pno,
                 "overhead_method": f"{args.steps} interleaved (protected, unprotected) pairs, mean of each",
                 "tflops_protected_interleaved": flops_total / (t_pft * 1e-3) / 1e12,
                 "pct_of_fp64_peak": 100.0 * tflops / (world * FP64_PEAK_TFLOPS),
                 "units_checked": cnt[0], "detected": cnt[1], "corrected": cnt[2],
                 "recomputed": cnt[3], "events": cnt[4], "events_global": len(events_global),
                 "prepass_encode": pre, "unfused_baseline": unf,
                 "ms_per_step_all": {"protected": per_ft, "pairs_protected": pairs["ft"],
                                     "pairs_unprotected": pairs["noft"]},
                 "cublas_dgemm_tflops": flops_total / (ms_cublas * 1e-3) / 1e12 if ms_cublas else None,
                 "interval_sweep": sweep},
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": FP64_PEAK_TFLOPS,
                     "unit": "TFLOP/s", "frac": achieved / FP64_PEAK_TFLOPS, "traffic": traffic,
                     "kernel": "dgemm_abft_kernel (FT)", "kernel_ms": kern_ms,
                     "peak_source": "measured FP64 DMMA microbenchmark (profiles/fp64_peak.json); "
                                    f"nominal {FP64_NOMINAL_TFLOPS:.1f}"},
        "cpu_baseline": cpu,
        "parity": parity,
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "per_config": per_config,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
