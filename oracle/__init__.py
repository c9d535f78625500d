"""ctypes binding for the CPU oracle (oracle/mhar_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference arm as the checker.  The product
(paper_2104_07097_b200) never imports this module.

All matrices are numpy float64 arrays in column-major (Fortran) order, the
layout of the reference's Eigen::MatrixXd (proj/include/mhar/linalg.hpp:7-10).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "build", "libmhar_oracle.so")

THETA_STREAM_ID = (1 << 64) - 1  # WalkRng::kThetaStreamId, proj/include/mhar/rng.hpp:53

_dp = C.POINTER(C.c_double)
_u8p = C.POINTER(C.c_uint8)
_u64p = C.POINTER(C.c_uint64)
_i64p = C.POINTER(C.c_int64)
_i64 = C.c_int64


class RunConfig(C.Structure):
    _fields_ = [("z", _i64), ("phi", _i64), ("t_target", _i64), ("burn_in", _i64),
                ("reproject_every", _i64), ("seed", C.c_uint64), ("eps_dir", C.c_double),
                ("eps_feas", C.c_double)]


class FrResult(C.Structure):
    _fields_ = [("cross_edges", _i64), ("expected_cross", C.c_double),
                ("variance_cross", C.c_double), ("z_value", C.c_double),
                ("shared_end_pairs", _i64), ("pooled_size", _i64)]


class RunStats(C.Structure):
    _fields_ = [("windows", _i64), ("iterate_count", _i64), ("redraw_count", _i64),
                ("err_chain", _i64), ("seconds", C.c_double)]


def build() -> str:
    """Compile the oracle with its Makefile (gcc, no GPU needed)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        L.orc_mix64.restype = C.c_uint64
        L.orc_mix64.argtypes = [C.c_uint64]
        L.orc_stream_init.restype = C.c_uint64
        L.orc_stream_init.argtypes = [C.c_uint64, C.c_uint64]
        L.orc_next_u64.restype = C.c_uint64
        L.orc_next_u64.argtypes = [_u64p]
        L.orc_next_uniform.restype = C.c_double
        L.orc_next_uniform.argtypes = [_u64p]
        L.orc_next_uniform_open.restype = C.c_double
        L.orc_next_uniform_open.argtypes = [_u64p]
        L.orc_box_muller.restype = C.c_int
        L.orc_box_muller.argtypes = [C.c_double, C.c_double, _dp, _dp]
        L.orc_fill_standard_normal.argtypes = [_u64p, _dp, _i64]
        L.orc_fill_standard_normal_matrix.argtypes = [_u64p, _i64, _dp, _i64]
        L.orc_vector_math_width.restype = C.c_int
        L.orc_chord_scan.argtypes = [_dp, _dp, _i64, C.c_double, _dp, _dp,
                                     C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.orc_gemm.argtypes = [_i64, _i64, _i64, _dp, _dp, _dp]
        L.orc_set_threads.argtypes = [C.c_int]
        L.orc_get_threads.restype = C.c_int
        L.orc_lambda_intervals.restype = C.c_int
        L.orc_lambda_intervals.argtypes = [_dp, _dp, _i64, _i64, _dp, _dp, _i64, C.c_double,
                                           _dp, _dp, _u8p, _u8p, _i64p]
        L.orc_invert.restype = C.c_int
        L.orc_invert.argtypes = [_dp, _i64, _dp]
        L.orc_compute_projection.restype = C.c_int
        L.orc_compute_projection.argtypes = [_dp, _i64, _i64, _dp, _dp]
        L.orc_reproject.restype = C.c_int
        L.orc_reproject.argtypes = [_dp, _dp, _dp, _i64, _i64, _dp, _i64]
        L.orc_contains.restype = C.c_int
        L.orc_contains.argtypes = [_dp, _dp, _i64, _dp, _dp, _i64, _i64, _dp, C.c_double]
        L.orc_make_hypercube.argtypes = [_i64, _dp, _dp]
        L.orc_make_simplex.argtypes = [_i64, _dp, _dp, _dp, _dp]
        L.orc_step.restype = C.c_int
        L.orc_step.argtypes = [_dp, _dp, _i64, _i64, _dp, C.c_double, _u64p, _u64p, _dp, _i64,
                               _i64p, _i64p]
        L.orc_step_injected.restype = C.c_int
        L.orc_step_injected.argtypes = [_dp, _dp, _i64, _i64, _dp, C.c_double, _dp, _i64, _dp,
                                        _dp, _dp, _dp, _dp, _u8p, _i64p]
        L.orc_run.restype = C.c_int
        L.orc_run.argtypes = [_dp, _dp, _i64, _dp, _dp, _i64, _i64, C.POINTER(RunConfig), _dp,
                              _dp, C.POINTER(RunStats)]
        _u32p = C.POINTER(C.c_uint32)
        L.orc_philox4x32_10.argtypes = [_u32p, _u32p, _u32p]
        L.orc_philox_u64x2.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint64,
                                       C.c_uint32, C.c_uint32, _u64p, _u64p]
        L.orc_philox_normals.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint32, _dp,
                                         _i64]
        L.orc_step_philox.restype = C.c_int
        L.orc_step_philox.argtypes = [_dp, _dp, _i64, _i64, _dp, C.c_double, C.c_uint64, _i64,
                                      C.c_uint64, _dp, _i64, _i64p, _i64p]
        _i32p = C.POINTER(C.c_int32)
        L.orc_minimum_spanning_tree.restype = C.c_int
        L.orc_minimum_spanning_tree.argtypes = [_dp, _i64, _i64, _i32p, _i32p, _dp]
        L.orc_friedman_rafsky.restype = C.c_int
        L.orc_friedman_rafsky.argtypes = [_dp, _i64, _dp, _i64, _i64, C.POINTER(FrResult)]
        _lib = L
    return _lib


def _d(a):
    return None if a is None else a.ctypes.data_as(_dp)


def _f(a):
    """float64 Fortran-ordered copy (or view) of a."""
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


# ---------------------------------------------------------------- streams ---

class Stream:
    """RngStream (proj/include/mhar/rng.hpp:16-33)."""

    def __init__(self, seed: int, stream: int):
        self.state = C.c_uint64(lib().orc_stream_init(seed & (2**64 - 1), stream & (2**64 - 1)))

    def next_u64(self) -> int:
        return lib().orc_next_u64(C.byref(self.state))

    def next_uniform(self) -> float:
        return lib().orc_next_uniform(C.byref(self.state))

    def next_uniform_open(self) -> float:
        return lib().orc_next_uniform_open(C.byref(self.state))

    def fill_standard_normal(self, n: int) -> np.ndarray:
        out = np.empty(n)
        lib().orc_fill_standard_normal(C.byref(self.state), _d(out), n)
        return out


class WalkRng:
    """WalkRng (proj/include/mhar/rng.hpp:42-55): z column streams + theta."""

    def __init__(self, seed: int, z: int):
        L = lib()
        self.cols = np.array([L.orc_stream_init(seed, k) for k in range(z)], dtype=np.uint64)
        self.theta = np.array([L.orc_stream_init(seed, THETA_STREAM_ID)], dtype=np.uint64)

    @property
    def width(self) -> int:
        return len(self.cols)

    def fill_standard_normal_matrix(self, n: int) -> np.ndarray:
        out = np.empty((n, self.width), order="F")
        lib().orc_fill_standard_normal_matrix(self.cols.ctypes.data_as(_u64p), self.width,
                                              _d(out), n)
        return out


def box_muller(u1: float, u2: float):
    c, s = C.c_double(), C.c_double()
    st = lib().orc_box_muller(u1, u2, C.byref(c), C.byref(s))
    if st:
        raise ValueError("box_muller: u1 must lie in (0,1], u2 in [0,1)")
    return c.value, s.value


# ------------------------------------------------------------- polytopes ---

def make_hypercube(n: int):
    A = np.empty((2 * n, n), order="F")
    b = np.empty(2 * n)
    lib().orc_make_hypercube(n, _d(A), _d(b))
    return A, b


def make_simplex(n: int):
    A = np.empty((n, n), order="F")
    b = np.empty(n)
    AE = np.empty((1, n), order="F")
    bE = np.empty(1)
    lib().orc_make_simplex(n, _d(A), _d(b), _d(AE), _d(bE))
    return A, b, AE, bE


# ---------------------------------------------------------------- algebra ---

def gemm(A, B):
    A, B = _f(A), _f(B)
    Cm = np.empty((A.shape[0], B.shape[1]), order="F")
    lib().orc_gemm(A.shape[0], A.shape[1], B.shape[1], _d(A), _d(B), _d(Cm))
    return Cm


def invert(a):
    a = _f(a)
    inv = np.empty_like(a, order="F")
    st = lib().orc_invert(_d(a), a.shape[0], _d(inv))
    return st, inv


def compute_projection(AE):
    AE = _f(AE)
    me, n = AE.shape
    P = np.empty((n, n), order="F")
    G = np.empty((me, me), order="F")
    st = lib().orc_compute_projection(_d(AE), me, n, _d(P), _d(G))
    return st, P, G


def reproject(AE, Ginv, bE, X):
    AE, Ginv, X = _f(AE), _f(Ginv), _f(X).copy(order="F")
    bE = np.ascontiguousarray(bE, dtype=np.float64)
    lib().orc_reproject(_d(AE), _d(Ginv), _d(bE), AE.shape[0], AE.shape[1], _d(X), X.shape[1])
    return X


def contains(A, b, x, eps, AE=None, bE=None):
    A = _f(A)
    x = np.ascontiguousarray(x, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    me = 0 if AE is None else AE.shape[0]
    AEf = None if AE is None else _f(AE)
    bEf = None if bE is None else np.ascontiguousarray(bE, dtype=np.float64)
    return bool(lib().orc_contains(_d(A), _d(b), A.shape[0], _d(AEf), _d(bEf), me, A.shape[1],
                                   _d(x), eps))


def chord_scan(num, den, eps):
    num = np.ascontiguousarray(num, dtype=np.float64)
    den = np.ascontiguousarray(den, dtype=np.float64)
    lo, hi = C.c_double(), C.c_double()
    p, q = C.c_int(), C.c_int()
    lib().orc_chord_scan(_d(num), _d(den), len(num), eps, C.byref(lo), C.byref(hi), C.byref(p),
                         C.byref(q))
    return lo.value, hi.value, bool(p.value), bool(q.value)


def lambda_intervals(A, b, X, D, eps_dir):
    """Returns (status, lower, upper, degenerate, sides, err_chain)."""
    A, X, D = _f(A), _f(X), _f(D)
    b = np.ascontiguousarray(b, dtype=np.float64)
    z = X.shape[1]
    lo, hi = np.zeros(z), np.zeros(z)
    dg, sd = np.zeros(z, np.uint8), np.zeros(z, np.uint8)
    err = C.c_int64(-1)
    st = lib().orc_lambda_intervals(_d(A), _d(b), A.shape[0], A.shape[1], _d(X), _d(D), z,
                                    eps_dir, _d(lo), _d(hi), dg.ctypes.data_as(_u8p),
                                    sd.ctypes.data_as(_u8p), C.byref(err))
    return st, lo, hi, dg, sd, err.value


def step(A, b, P, eps_dir, rng: WalkRng, X):
    """One reference iterate in place on X (Fortran n x z).  Returns
    (status, redraws, err_chain)."""
    A = _f(A)
    b = np.ascontiguousarray(b, dtype=np.float64)
    Pf = None if P is None else _f(P)
    assert X.flags.f_contiguous and X.dtype == np.float64
    red = C.c_int64(0)
    err = C.c_int64(-1)
    st = lib().orc_step(_d(A), _d(b), A.shape[0], A.shape[1], _d(Pf), eps_dir,
                        rng.cols.ctypes.data_as(_u64p), rng.theta.ctypes.data_as(_u64p), _d(X),
                        X.shape[1], C.byref(red), C.byref(err))
    return st, red.value, err.value


def philox4x32_10(ctr, key):
    """Philox4x32-10 of a 4-word counter under a 2-word key (4 uint32)."""
    c = (C.c_uint32 * 4)(*ctr)
    k = (C.c_uint32 * 2)(*key)
    o = (C.c_uint32 * 4)()
    lib().orc_philox4x32_10(c, k, o)
    return list(o)


def philox_normals(seed, walk, iterate, attempt, n):
    out = np.empty(n)
    lib().orc_philox_normals(seed & (2**64 - 1), walk, iterate, attempt, _d(out), n)
    return out


def step_philox(A, b, P, eps_dir, seed, chain_offset, iterate, X):
    """One reference iterate in place on X (Fortran n x z) with the engine's
    Philox draws for (seed, global walk chain_offset + k, iterate).  Returns
    (status, redraws, err_chain)."""
    A = _f(A)
    b = np.ascontiguousarray(b, dtype=np.float64)
    Pf = None if P is None else _f(P)
    assert X.flags.f_contiguous and X.dtype == np.float64
    red = C.c_int64(0)
    err = C.c_int64(-1)
    st = lib().orc_step_philox(_d(A), _d(b), A.shape[0], A.shape[1], _d(Pf), eps_dir,
                               seed & (2**64 - 1), chain_offset, iterate, _d(X), X.shape[1],
                               C.byref(red), C.byref(err))
    return st, red.value, err.value


def step_injected(A, b, P, eps_dir, X, H, U):
    """Injected-draw iterate (test hook semantics).  Returns
    (status, X_new, lower, upper, theta, flags, err_chain)."""
    A, H = _f(A), _f(H)
    X = _f(X).copy(order="F")
    b = np.ascontiguousarray(b, dtype=np.float64)
    U = np.ascontiguousarray(U, dtype=np.float64)
    Pf = None if P is None else _f(P)
    z = X.shape[1]
    lo, hi, th = np.zeros(z), np.zeros(z), np.zeros(z)
    fl = np.zeros(z, np.uint8)
    err = C.c_int64(-1)
    st = lib().orc_step_injected(_d(A), _d(b), A.shape[0], A.shape[1], _d(Pf), eps_dir, _d(X), z,
                                 _d(H), _d(U), _d(lo), _d(hi), _d(th), fl.ctypes.data_as(_u8p),
                                 C.byref(err))
    return st, X, lo, hi, th, fl, err.value


def run(A, b, x0, *, z, phi, t_target, burn_in, reproject_every, seed, eps_dir=1e-11,
        eps_feas=1e-9, AE=None, bE=None, collect=True):
    """Full run with warm start (resolved config).  Returns (status, samples, stats)."""
    A = _f(A)
    b = np.ascontiguousarray(b, dtype=np.float64)
    x0 = np.ascontiguousarray(x0, dtype=np.float64)
    me = 0 if AE is None else AE.shape[0]
    AEf = None if AE is None else _f(AE)
    bEf = None if bE is None else np.ascontiguousarray(bE, dtype=np.float64)
    n = A.shape[1]
    windows = (t_target + z - 1) // z
    samples = np.empty((windows * z, n)) if collect else None
    cfg = RunConfig(z, phi, t_target, burn_in, reproject_every, seed, eps_dir, eps_feas)
    stats = RunStats()
    st = lib().orc_run(_d(A), _d(b), A.shape[0], _d(AEf), _d(bEf), me, n, C.byref(cfg), _d(x0),
                       _d(samples), C.byref(stats))
    return st, samples, stats


# ------------------------------------------------ two-sample tree test ----

def minimum_spanning_tree(points):
    """stats.cpp:50-91 (row points)."""
    P = np.ascontiguousarray(points, dtype=np.float64)
    if P.ndim == 1:
        P = P[:, None]
    N, n = P.shape
    a = np.empty(N - 1, np.int32)
    b = np.empty(N - 1, np.int32)
    w = np.empty(N - 1)
    lib().orc_minimum_spanning_tree(_d(P), N, n, a.ctypes.data_as(C.POINTER(C.c_int32)),
                                    b.ctypes.data_as(C.POINTER(C.c_int32)), _d(w))
    return a, b, w


def friedman_rafsky(sample_a, sample_b):
    """stats.cpp:93-143.  Returns (status, FrResult)."""
    A = np.ascontiguousarray(sample_a, dtype=np.float64)
    B = np.ascontiguousarray(sample_b, dtype=np.float64)
    if A.ndim == 1:
        A, B = A[:, None], B[:, None]
    r = FrResult()
    st = lib().orc_friedman_rafsky(_d(A), A.shape[0], _d(B), B.shape[0], A.shape[1], C.byref(r))
    return st, r
