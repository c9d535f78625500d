"""Loop-only single-walk hit-and-run, restating the reference's independent
test oracle ScalarWalk (proj/tests/oracles.hpp:139-254) and its helpers
(ray_march_chord :114-131, ks_statistic_uniform :505-515, sample_moments
:522-529).  It shares only the RNG streams with the engine under test -- the
point of the reference's z = 1 equivalence test (proj/tests/test_sampler.cpp:413-485).
Test infrastructure only.
"""
from __future__ import annotations

import ctypes
import ctypes.util
import math

import oracle

_libm = ctypes.CDLL(ctypes.util.find_library("m"))
_libm.sincos.argtypes = [ctypes.c_double, ctypes.POINTER(ctypes.c_double),
                         ctypes.POINTER(ctypes.c_double)]
_TWO_PI = 6.283185307179586


def box_muller(u1: float, u2: float):
    """mhar::box_muller (proj/src/rng.cpp:115-124) with glibc sincos."""
    if not (0.0 < u1 <= 1.0) or not (0.0 <= u2 < 1.0):
        raise ValueError("box_muller: u1 must lie in (0,1], u2 in [0,1)")
    r = math.sqrt(-2.0 * math.log(u1))
    s, c = ctypes.c_double(), ctypes.c_double()
    _libm.sincos(_TWO_PI * u2, ctypes.byref(s), ctypes.byref(c))
    return r * c.value, r * s.value


def _dot(row, v):
    s = 0.0
    for a, b in zip(row, v):
        s += a * b
    return s


class ScalarWalk:
    K_EPS_DEGENERATE_WIDTH = 1e-14
    K_MAX_RETRIES = 16
    K_MAX_THETA_REJECTS = 64

    def __init__(self, a_in, b_in, projection=None):
        self.a_in = [list(map(float, row)) for row in a_in]
        self.b_in = list(map(float, b_in))
        self.projection = None if projection is None else [list(map(float, r)) for r in projection]

    def normals(self, s: oracle.Stream, n: int):
        h = [0.0] * n
        for p in range((n + 1) // 2):
            u1 = s.next_uniform_open()
            u2 = s.next_uniform()
            c, sn = box_muller(u1, u2)
            h[2 * p] = c
            if 2 * p + 1 < n:
                h[2 * p + 1] = sn
        return h

    def apply_projection(self, h):
        if self.projection is None:
            return h
        n = len(h)
        return [_dot(self.projection[i], h) for i in range(n)]

    def chord(self, x, d, eps_dir):
        lower, upper = -math.inf, math.inf
        pos = neg = False
        for row, b in zip(self.a_in, self.b_in):
            ax = 0.0
            ad = 0.0
            for a, xj, dj in zip(row, x, d):
                ax += a * xj
                ad += a * dj
            slack = b - ax
            if ad > eps_dir:
                lam = slack / ad
                pos = True
                upper = min(upper, lam)
            elif ad < -eps_dir:
                lam = slack / ad
                neg = True
                lower = max(lower, lam)
        if not pos or not neg:
            return lower, upper, True
        return lower, upper, not (upper - lower > self.K_EPS_DEGENERATE_WIDTH)

    def draw_theta(self, theta_stream, lower, upper):
        for _ in range(self.K_MAX_THETA_REJECTS):
            u = theta_stream.next_uniform()
            t = lower + u * (upper - lower)
            if lower < t < upper:
                return t
        return lower + 0.5 * (upper - lower)

    def _usable(self, d):
        if self.projection is None:
            return True
        return math.sqrt(sum(v * v for v in d)) > 1e-12

    def advance(self, column_stream, theta_stream, x, eps_dir) -> bool:
        n = len(x)
        d = self.apply_projection(self.normals(column_stream, n))
        usable = self._usable(d)
        lo = hi = 0.0
        if usable:
            lo, hi, dg = self.chord(x, d, eps_dir)
            usable = not dg
        attempt = 0
        while not usable and attempt < self.K_MAX_RETRIES:
            attempt += 1
            d = self.apply_projection(self.normals(column_stream, n))
            if not self._usable(d):
                continue
            lo, hi, dg = self.chord(x, d, eps_dir)
            usable = not dg
        if not usable:
            return False
        t = self.draw_theta(theta_stream, lo, hi)
        for j in range(n):
            x[j] += t * d[j]
        return True


def ray_march_chord(a_in, b_in, x, d, resolution):
    def feasible(t):
        p = [xj + t * dj for xj, dj in zip(x, d)]
        return all(sum(a * v for a, v in zip(row, p)) <= b for row, b in zip(a_in, b_in))

    k = 1
    while feasible(k * resolution):
        k += 1
    upper = k * resolution
    k = 1
    while feasible(-k * resolution):
        k += 1
    return -k * resolution, upper


def ks_statistic_uniform(u):
    u = sorted(u)
    n = float(len(u))
    d = 0.0
    for i, v in enumerate(u):
        d = max(d, v - i / n, (i + 1) / n - v)
    return d


def sample_moments(xs):
    xs = list(xs)
    mean = sum(xs) / len(xs)
    var = sum((v - mean) ** 2 for v in xs) / (len(xs) - 1)
    return mean, var
