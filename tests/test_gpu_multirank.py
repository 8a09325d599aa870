"""The multi-rank path of SURVEY.md §8(e) run for real on one GPU: world-size-2 process groups
(gloo) whose ranks each call libftblas on their own C row panel on cuda:0.  The ranks never
wait on each other's kernels (their only exchange is the host-side counter all-reduce and the
event gather), so running them on one device tests the code path, not any overlap.  The
all-reduced counters, the gathered global events and the assembled C must equal one
single-process call on the whole problem (the row panels are aligned to the unit height, so
the set of verification units is the same), and bench.py's torchrun branch must report the
single-process counters."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem():
    rng = np.random.default_rng(41)
    m, n, k = 1016, 900, 384  # 8 x 8 units of 127 (the last column ragged)
    A = np.asfortranarray(rng.uniform(-1, 1, (m, k)))
    B = np.asfortranarray(rng.uniform(-1, 1, (k, n)))
    faults = [(5, 7, 100, 40.0), (300, 899, 0, -3.0), (508, 127, 384, 1e3), (1015, 450, 200, 0.5),
              (700, 10, 16, 2.0), (701, 11, 32, 2.0)]  # the last two share a unit: recomputed
    return m, n, k, A, B, faults


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    from paper_2104_00897_b200 import ftblas as F
    from paper_2104_00897_b200.parallel import RowPanelPartitioner, allreduce_counters
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    F.load()
    m, n, k, A, B, faults = _problem()
    BM = F.ftblas_get_geometry()[0]
    part = RowPanelPartitioner(m, world, BM)
    r0, r1 = part.rows(rank)
    dA = torch.from_numpy(np.asfortranarray(A[r0:r1]).reshape(-1, order="F")).to("cuda")
    dB = torch.from_numpy(B.reshape(-1, order="F")).to("cuda")
    dC = torch.zeros((r1 - r0) * n, dtype=torch.float64, device="cuda")
    F.ftblas_inject_arm(part.route_faults(faults, rank))
    rep = F.ftblas_dgemm("N", "N", r1 - r0, n, k, 1.0, dA, r1 - r0, dB, k, 0.0, dC, r1 - r0)
    cnt = allreduce_counters([rep.units_checked, rep.detected, rep.corrected, rep.recomputed,
                              rep.n_events], dist, "cpu")
    gathered = [None] * world
    dist.all_gather_object(gathered, (r0, r1, dC.view(n, r1 - r0).t().cpu().numpy(),
                                      part.to_global_events(rep.events, rank),
                                      (rep.unit_rows, rep.unit_cols, rep.step_quantum)))
    if rank == 0:
        C = np.zeros((m, n))
        ev = []
        for (a0, a1, Cp, e, geo) in gathered:
            C[a0:a1] = Cp
            ev += e
        q.put((cnt, sorted(ev), C, [g[4] for g in gathered]))
    dist.barrier()
    dist.destroy_process_group()


def test_world2_panels_on_one_gpu_match_single_call():
    import torch
    from paper_2104_00897_b200 import ftblas as F
    F.load()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    cnt, ev, C, geos = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert geos[0] == geos[1]
    m, n, k, A, B, faults = _problem()
    dA = torch.from_numpy(A.reshape(-1, order="F")).to("cuda")
    dB = torch.from_numpy(B.reshape(-1, order="F")).to("cuda")
    dC = torch.zeros(m * n, dtype=torch.float64, device="cuda")
    F.ftblas_inject_arm(faults)
    rep = F.ftblas_dgemm("N", "N", m, n, k, 1.0, dA, m, dB, k, 0.0, dC, m)
    assert cnt == [rep.units_checked, rep.detected, rep.corrected, rep.recomputed, rep.n_events]
    assert (rep.corrected, rep.recomputed) == (4, 1)
    assert [e[:4] for e in ev] == [e[:4] for e in rep.events]
    # Values: the single call (64 tiles) and the panels (32 each) split k differently
    # (single-wave k-split: 2 and 4 splits), so they agree within the parity bound, not bitwise.
    Cs = dC.view(n, m).t().cpu().numpy()
    assert np.all(np.abs(C - Cs) <= 2 * (2 * k * 2.0 ** -53) * (np.abs(A) @ np.abs(B)))


def test_bench_torchrun_gloo_one_device():
    """bench.py's multi-rank branch (torchrun, 2 ranks, gloo, both on cuda:0) on a small C5:
    its all-reduced counters equal the single-process line's."""
    common = ["--size", "1016", "--steps", "2", "--warmup", "1", "--no-e2e", "--no-per-config",
              "--no-unfused", "--no-cpu-baseline"]
    env = dict(os.environ, MASTER_ADDR="127.0.0.1")
    one = subprocess.run([sys.executable, "bench.py", *common], cwd=ROOT, capture_output=True, text=True,
                         timeout=600, env=env)
    assert one.returncode == 0, one.stderr[-3000:]
    l1 = json.loads(one.stdout.strip().splitlines()[-1])
    two = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py",
                          "--gpus", "2", "--backend", "gloo", "--one-device", *common],
                         cwd=ROOT, capture_output=True, text=True, timeout=600, env=env)
    assert two.returncode == 0, two.stderr[-3000:]
    l2 = json.loads([x for x in two.stdout.strip().splitlines() if x.startswith("{")][-1])
    assert l2["n_gpus"] == 2 and l1["n_gpus"] == 1
    keys = ("units_checked", "detected", "corrected", "recomputed", "events", "events_global")
    assert [l1["abft"][x] for x in keys] == [l2["abft"][x] for x in keys]
    assert l1["abft"]["detected"] > 30  # 100 faults over 64 units: ~51 distinct units
