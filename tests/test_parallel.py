"""Row-panel partitioner + counter all-reduce (host logic of the multi-GPU path), run on
CPU with world_size-2 gloo process groups.  Each rank computes its panel with the CPU
oracle standing in for the device (no GPU here); the all-reduced counters and the
gathered global events must equal the single-process run (SURVEY.md §8(e) invariant)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle
from paper_2104_00897_b200.parallel import RowPanelPartitioner, allreduce_counters


def test_partition_rows_cover_and_align():
    for unit in (127, 128):
        for m in [1, 127, 128, 300, 1000, 32768]:
            for P in [1, 2, 3, 4, 8]:
                part = RowPanelPartitioner(m, P, unit)
                spans = [part.rows(r) for r in range(P)]
                assert spans[0][0] == 0 and spans[-1][1] == m
                for (a0, a1), (b0, b1) in zip(spans, spans[1:]):
                    assert a1 == b0
                for (r0, r1) in spans:
                    assert r0 % unit == 0
                # units split as evenly as whole units allow (at most one unit apart)
                nu = [-(-(r1 - r0) // unit) for (r0, r1) in spans]
                assert max(nu) - min(nu) <= 1
    # C5 on the library's 127-row units: 259 unit rows over 8 ranks -> 32 or 33 each
    part = RowPanelPartitioner(32768, 8, 127)
    assert sorted({(r1 - r0 + 126) // 127 for (r0, r1) in (part.rows(r) for r in range(8))}) == [32, 33]
    part = RowPanelPartitioner(32768, 8, 128)
    assert [part.rows(r) for r in range(8)] == [(4096 * r, 4096 * (r + 1)) for r in range(8)]
    faults = [(5000, 3, 7, 1.0), (100, 4, 0, 2.0), (32767, 0, 9, 3.0)]
    assert part.route_faults(faults, 1) == [(904, 3, 7, 1.0)]
    assert part.route_faults(faults, 7) == [(4095, 0, 9, 3.0)]
    assert part.owner(5000) == 1
    blocks = list(part.gen_block_rows(4096, 4500))
    assert blocks[0] == (4096, 4224) and blocks[-1] == (4480, 4500)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, m, n, k, faults, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(5)
    A = np.asfortranarray(rng.integers(-8, 9, (m, k)).astype(float))
    B = np.asfortranarray(rng.integers(-8, 9, (k, n)).astype(float))
    part = RowPanelPartitioner(m, world, 32)
    r0, r1 = part.rows(rank)
    Ap = np.asfortranarray(A[r0:r1])
    Cp, rep = oracle.dgemm_abft("N", "N", r1 - r0, n, k, 1.0, Ap, max(r1 - r0, 1), B, k, 0.0,
                                np.zeros((r1 - r0, n)), max(r1 - r0, 1), BM=32, BN=32, BK=4,
                                faults=part.route_faults(faults, rank))
    cnt = allreduce_counters([rep.units_checked, rep.detected, rep.corrected, rep.recomputed,
                              rep.n_events], dist, "cpu")
    evs = part.to_global_events(rep.events, rank)
    gathered = [None] * world
    dist.all_gather_object(gathered, (r0, r1, Cp.reshape((n, r1 - r0)).T, evs))
    if rank == 0:
        C = np.zeros((m, n))
        allev = []
        for (a0, a1, Cpart, e) in gathered:
            C[a0:a1] = Cpart
            allev += e
        q.put((cnt, sorted(allev), C))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_world2_matches_single_process(world):
    m, n, k = 200, 96, 40
    faults = [(10, 10, 5, 3.0), (150, 40, 39, 2.0), (150, 41, 0, 1.0), (199, 95, 40, 7.0)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, m, n, k, faults, q)) for r in range(world)]
    for p in procs:
        p.start()
    cnt, ev, C = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rng = np.random.default_rng(5)
    A = np.asfortranarray(rng.integers(-8, 9, (m, k)).astype(float))
    B = np.asfortranarray(rng.integers(-8, 9, (k, n)).astype(float))
    C1, rep1 = oracle.dgemm_abft("N", "N", m, n, k, 1.0, A, m, B, k, 0.0, np.zeros((m, n)), m,
                                 BM=32, BN=32, BK=4, faults=faults)
    assert cnt == [rep1.units_checked, rep1.detected, rep1.corrected, rep1.recomputed, rep1.n_events]
    assert [e[:4] for e in ev] == [e[:4] for e in rep1.events]
    assert np.array_equal(C, C1.reshape((n, m)).T) and np.array_equal(C, A @ B)
