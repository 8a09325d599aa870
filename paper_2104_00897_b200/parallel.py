"""Multi-GPU row-panel partitioner (BASELINE config C5).

C is split into row panels: rank r owns rows [r0, r1) of C and of op(A), holds a full
replica of op(B), and runs the protected DGEMM on its panel independently.  Panel
boundaries are aligned to the verification-unit height so that the set of units (and so
every counter and every event) is identical for every world size.  The only collective
is the sum all-reduce of the int64 error counters (NCCL over NVLink on GPUs, gloo in
CPU tests).
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass
class RowPanelPartitioner:
    m: int
    world: int
    unit_rows: int = 128

    def rows(self, rank: int):
        """[r0, r1) rows of rank `rank`: units split as evenly as possible, in order."""
        if not 0 <= rank < self.world:
            raise ValueError("rank out of range")
        nu = -(-self.m // self.unit_rows)
        u0 = (rank * nu) // self.world
        u1 = ((rank + 1) * nu) // self.world
        return min(u0 * self.unit_rows, self.m), min(u1 * self.unit_rows, self.m)

    def owner(self, i: int) -> int:
        for r in range(self.world):
            r0, r1 = self.rows(r)
            if r0 <= i < r1:
                return r
        raise ValueError("row out of range")

    def route_faults(self, faults, rank: int):
        """Faults (global i, j, step, delta) owned by `rank`, shifted to local rows."""
        r0, r1 = self.rows(rank)
        return [(i - r0, j, s, d) for (i, j, s, d) in faults if r0 <= i < r1]

    def to_global_events(self, events, rank: int):
        """Translate a rank's events (interval, i, j, kind, rr, rc) back to global rows."""
        r0, _ = self.rows(rank)
        return [(t, i + r0, j, kind, rr, rc) for (t, i, j, kind, rr, rc) in events]

    @property
    def gen_block_rows(self):
        """Generation blocks: unit-height row blocks, each drawn from its own seed stream so
        that a rank's data does not depend on the world size."""
        part = self

        class _Blocks:
            block = part.unit_rows

            def __call__(self, r0, r1):
                b = part.unit_rows
                g = (r0 // b) * b
                while g < r1:
                    yield (max(g, r0), min(g + b, r1))
                    g += b

        return _Blocks()


COUNTER_FIELDS = ("units_checked", "detected", "corrected", "recomputed", "n_events")


def allreduce_counters(report_counts, dist, device):
    """Sum the five int64 counters over the process group; returns a list of ints."""
    import torch
    t = torch.tensor([int(x) for x in report_counts], dtype=torch.int64, device=device)
    dist.all_reduce(t)
    return [int(x) for x in t.tolist()]
