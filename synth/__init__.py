"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NONE of the method's arithmetic: it only draws random operands
(numpy PCG64, column-major float64) and the random fault list the paper's
injection protocol calls for (§VI.C: "An element of matrix C is
randomly selected for modification when an injection point is reached").
The fault list is drawn with SplitMix64 (Steele, Lea, Flood 2014) in the order
specified by SURVEY.md §8(b); the C library's ``ftblas_inject_seeded`` is an
independent implementation of the same generator and tests check the two agree.

Configurations follow BASELINE.json ``configs`` (C1..C5); the recipes and the
readings R9-R12 that fill unstated details are listed in DESIGN.md.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

MASK64 = (1 << 64) - 1


class SplitMix64:
    """SplitMix64: state += golden gamma; mix with two xor-shift-multiply rounds."""

    def __init__(self, seed: int):
        self.state = seed & MASK64

    def next_u64(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & MASK64
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
        return z ^ (z >> 31)

    def uniform(self) -> float:
        """Top 53 bits -> [0, 1)."""
        return (self.next_u64() >> 11) * (1.0 / 9007199254740992.0)


def seeded_faults(seed: int, count: int, m: int, n: int, k: int, log10_lo: float,
                  log10_hi: float):
    """Fault list [(i, j, step, delta)], 5 uniforms per fault in the order u0..u4:
    i = floor(u0*m), j = floor(u1*n), step = floor(u2*k) (each clamped to the last index),
    |delta| = 10**(lo + (hi-lo)*u3), sign negative iff u4 < 0.5."""
    g = SplitMix64(seed)
    out = []
    for _ in range(count):
        u0, u1, u2, u3, u4 = (g.uniform() for _ in range(5))
        i = min(int(math.floor(u0 * m)), m - 1)
        j = min(int(math.floor(u1 * n)), n - 1)
        s = min(int(math.floor(u2 * k)), max(k - 1, 0))
        mag = math.pow(10.0, log10_lo + (log10_hi - log10_lo) * u3)
        out.append((i, j, s, -mag if u4 < 0.5 else mag))
    return out


def _rng(seed: int, tag: str, idx: int = 0) -> np.random.Generator:
    return np.random.default_rng([seed, sum(ord(c) << (8 * q) for q, c in enumerate(tag)), idx])


def matrix(seed: int, tag: str, rows: int, cols: int, dist: str = "uniform", idx: int = 0,
           integer_bound: int = 8) -> np.ndarray:
    """rows x cols Fortran-ordered float64 matrix.
    dist: 'uniform' U[-1,1], 'normal' N(0,1), 'int' integers in [-integer_bound, integer_bound]."""
    g = _rng(seed, tag, idx)
    if dist == "uniform":
        x = g.uniform(-1.0, 1.0, size=(cols, rows))
    elif dist == "normal":
        x = g.standard_normal(size=(cols, rows))
    elif dist == "int":
        x = g.integers(-integer_bound, integer_bound + 1, size=(cols, rows)).astype(np.float64)
    else:
        raise ValueError(dist)
    return x.T  # C-order (cols, rows) transposed == Fortran-order (rows, cols)


@dataclass
class Case:
    name: str
    ta: str
    tb: str
    m: int
    n: int
    k: int
    alpha: float
    beta: float
    A: np.ndarray          # stored matrix (k x m if ta == 'T'), Fortran order
    B: np.ndarray          # stored matrix (n x k if tb == 'T'), Fortran order
    C0: np.ndarray         # m x n, Fortran order
    faults: list = field(default_factory=list)
    seed: int = 0

    @property
    def lda(self):
        return max(1, self.A.shape[0])

    @property
    def ldb(self):
        return max(1, self.B.shape[0])

    @property
    def ldc(self):
        return max(1, self.m)

    @property
    def flops(self):
        return 2.0 * self.m * self.n * self.k


def make_case(name: str, ta: str, tb: str, m: int, n: int, k: int, *, alpha=1.0, beta=0.0,
              dist="uniform", seed=0, faults=(), c0=None) -> Case:
    A = matrix(seed, "A", k if ta == "T" else m, m if ta == "T" else k, dist)
    B = matrix(seed, "B", n if tb == "T" else k, k if tb == "T" else n, dist)
    if c0 is None:
        C0 = matrix(seed, "C", m, n, "uniform") if beta != 0.0 else np.zeros((m, n), order="F")
    else:
        C0 = c0
    return Case(name, ta, tb, m, n, k, alpha, beta, A, B, C0, list(faults), seed)


# ---------------------------------------------------------------------------------------
# BASELINE.json configs.  DESIGN.md readings: R9 |delta| = 10^U(-2,4) with random sign
# for C3/C4/C5, R10 count = round(2mnk/1e11) for C4, R11 C[17][203] = (i=17, j=203),
# R12 alpha=1, beta=0 where unstated.
# ---------------------------------------------------------------------------------------
FAULT_LOG10 = (-2.0, 4.0)


def config(name: str, seed: int = 1234, trans: str = "NN", fault_seed: int | None = None) -> Case:
    fs = seed + 1 if fault_seed is None else fault_seed
    ta, tb = trans[0], trans[1]
    if name == "C1":
        return make_case("C1", "N", "N", 256, 256, 256, alpha=1.0, beta=0.0, seed=seed,
                         faults=[(17, 203, 128, 1e3)])
    if name == "C2":
        return make_case("C2", "N", "N", 2048, 2048, 2048, alpha=1.5, beta=0.5, seed=seed)
    if name == "C3":
        f = seeded_faults(fs, 20, 8192, 8192, 8192, *FAULT_LOG10)
        return make_case("C3" + trans, ta, tb, 8192, 8192, 8192, dist="normal", seed=seed, faults=f)
    if name == "C4a":
        cnt = round(2 * 16384 * 16384 * 1024 / 1e11)
        f = seeded_faults(fs, cnt, 16384, 16384, 1024, *FAULT_LOG10)
        return make_case("C4a", "N", "N", 16384, 16384, 1024, seed=seed, faults=f)
    if name == "C4b":
        cnt = round(2 * 16384 * 512 * 16384 / 1e11)
        f = seeded_faults(fs, cnt, 16384, 512, 16384, *FAULT_LOG10)
        return make_case("C4b", "N", "N", 16384, 512, 16384, seed=seed, faults=f)
    raise ValueError(name)


# C5: 32768^3, C row panels over P in {1,2,4,8}.  A is drawn as 8 fixed row panels of
# 4096 rows so that the data (and therefore every counter and event) is identical for
# every P (SURVEY.md §8(e) invariant).
C5_N = 32768
C5_PANELS = 8
C5_FAULTS = 100


def c5_faults(seed: int = 1234, fault_seed: int | None = None, size: int = C5_N):
    fs = seed + 1 if fault_seed is None else fault_seed
    return seeded_faults(fs, C5_FAULTS, size, size, size, *FAULT_LOG10)


def c5_A_panel(seed: int, q: int, size: int = C5_N) -> np.ndarray:
    """Row panel q (size/8 rows x size cols) of op(A) = A ('N')."""
    rows = size // C5_PANELS
    return matrix(seed, "A5", rows, size, "uniform", idx=q)


def c5_B(seed: int, size: int = C5_N) -> np.ndarray:
    return matrix(seed, "B5", size, size, "uniform")


def rank_rows(m: int, P: int, r: int):
    """Rows [r*m/P, (r+1)*m/P) owned by rank r."""
    return (r * m) // P, ((r + 1) * m) // P


def route_faults(faults, r0: int, r1: int):
    """Faults whose row falls in [r0, r1), shifted to local row indices."""
    return [(i - r0, j, s, d) for (i, j, s, d) in faults if r0 <= i < r1]
