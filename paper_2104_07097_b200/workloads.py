"""Seeded synthetic polytopes for the BASELINE.json configurations.

BASELINE.json names no public dataset: configs 1-2 are the closed-form bodies
of the paper (polytope.cpp:192-208) and configs 3-5 are
random polytopes whose inequality rows are iid N(0, I) normalised to unit
L2 norm with b = 1 (so the unit ball is inside and x0 = 0 is interior).
Each generator is deterministic in its seed so the GPU engine and the CPU
oracle see the same bytes.
"""
from __future__ import annotations

import dataclasses

import numpy as np

from . import Polytope, make_hypercube, make_simplex


@dataclasses.dataclass
class Workload:
    name: str
    polytope: Polytope
    x0: np.ndarray
    z: int
    iterations: int
    description: str


def unit_rows(m: int, n: int, seed: int) -> np.ndarray:
    """m x n column-major matrix of unit-norm Gaussian rows."""
    rng = np.random.default_rng(seed)
    a = rng.standard_normal((n, m)).T  # Fortran-ordered (m, n) view, no copy
    a /= np.sqrt(np.einsum("ij,ij->i", a, a))[:, None]
    return a


def random_polytope(n: int, m: int, seed: int = 2021) -> Polytope:
    return Polytope(unit_rows(m, n, seed), np.ones(m))


def config(idx: int, z: int | None = None, seed: int = 2021) -> Workload:
    """BASELINE.json configs[idx - 1] (1-based like the survey tables)."""
    if idx == 1:
        p = make_hypercube(10)
        return Workload("hypercube n=10", p, np.zeros(10), z or 100, 2000,
                        "A_I=[I;-I], z=100, 1000 burn-in + 1000 kept")
    if idx == 2:
        p = make_simplex(100)
        return Workload("simplex n=100", p, np.full(100, 0.01), z or 1000, 5000,
                        "A_E=1', A_I=-I, x0=1/n, z=1000, 5000 iterations")
    if idx == 3:
        return Workload("random n=500 m_I=20000", random_polytope(500, 20000, seed), np.zeros(500),
                        z or 4096, 1000, "unit-norm Gaussian rows, b=1, x0=0, z=4096")
    if idx == 4:
        n, m_rand, me = 1000, 50000, 100
        rng = np.random.default_rng(seed + 4)
        a_eq = np.asfortranarray(rng.standard_normal((me, n)))
        a_in = np.asfortranarray(np.vstack([np.eye(n), -np.eye(n), unit_rows(m_rand, n, seed)]))
        p = Polytope(a_in, np.ones(2 * n + m_rand), a_eq, np.zeros(me))
        return Workload("projected n=1000 m_I=52000 m_E=100", p, np.zeros(n), z or 8192, 1000,
                        "A_E 100x1000 N(0,1), b_E=0; A_I=[I;-I;50000 unit rows], x0=0, z=8192")
    if idx == 5:
        return Workload("random n=2000 m_I=200000", random_polytope(2000, 200000, seed),
                        np.zeros(2000), z or 4096, 1000,
                        "unit-norm Gaussian rows, b=1, x0=0, 4096 walks per GPU, 1000 iterations")
    raise ValueError(idx)
