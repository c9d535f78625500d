"""Two-sample uniformity screening on the GPU: the
reference's stats module (/root/reference/proj/include/mhar/stats.hpp,
src/stats.cpp) -- uniform reference samplers for the box and the simplex,
the Euclidean minimum spanning tree and the Friedman-Rafsky statistic, with
the O(N^2) Prim tree on the device (csrc/stats_kernels.cuh)."""
from __future__ import annotations

import ctypes as C
import dataclasses

import numpy as np

from . import ErrorCode, MharError, _check, lib

kUniformityZThreshold = -1.64  # stats.hpp:45


@dataclasses.dataclass
class MstTestResult:
    """stats.hpp:34-41."""
    cross_edges: int
    expected_cross: float
    variance_cross: float
    z_value: float
    shared_end_pairs: int
    pooled_size: int


def _rows(x):
    x = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    if x.ndim == 1:
        x = x[:, None]
    return x


def minimum_spanning_tree(points, device: int = 0):
    """Prim tree of the row points (stats.cpp:50-91): (a, b, weight) arrays of
    the N - 1 edges in insertion order."""
    P = _rows(points)
    N, n = P.shape
    if N < 2:
        raise MharError(ErrorCode.invalid_argument, "minimum_spanning_tree: need at least two points")
    a = np.empty(N - 1, np.int32)
    b = np.empty(N - 1, np.int32)
    w = np.empty(N - 1)
    _check(lib().mhar_minimum_spanning_tree(P.ctypes.data_as(C.POINTER(C.c_double)), N, n, device,
                                            a.ctypes.data_as(C.POINTER(C.c_int32)),
                                            b.ctypes.data_as(C.POINTER(C.c_int32)),
                                            w.ctypes.data_as(C.POINTER(C.c_double))))
    return a, b, w


def friedman_rafsky(sample_a, sample_b, device: int = 0) -> MstTestResult:
    """stats.cpp:93-143 on the GPU."""
    from . import _FrResult
    A, B = _rows(sample_a), _rows(sample_b)
    if A.shape[1] != B.shape[1]:
        raise MharError(ErrorCode.dimension_mismatch, "friedman_rafsky: samples have different widths")
    r = _FrResult()
    _check(lib().mhar_friedman_rafsky(A.ctypes.data_as(C.POINTER(C.c_double)), A.shape[0],
                                      B.ctypes.data_as(C.POINTER(C.c_double)), B.shape[0],
                                      A.shape[1], device, C.byref(r)))
    return MstTestResult(r.cross_edges, r.expected_cross, r.variance_cross, r.z_value,
                         r.shared_end_pairs, r.pooled_size)


def sample_uniform_hypercube(rng: np.random.Generator, n: int, count: int) -> np.ndarray:
    """count x n points uniform on [-1, 1]^n (stats.cpp:11-20)."""
    if n < 1 or count < 1:
        raise MharError(ErrorCode.invalid_argument, "sample_uniform_hypercube: n and count >= 1")
    return 2.0 * rng.random((count, n)) - 1.0


def sample_uniform_simplex(rng: np.random.Generator, n: int, count: int) -> np.ndarray:
    """count x n points uniform on the standard simplex via normalised
    exponential spacings (stats.cpp:22-48)."""
    if n < 2 or count < 1:
        raise MharError(ErrorCode.invalid_argument, "sample_uniform_simplex: need n >= 2")
    e = -np.log(1.0 - rng.random((count, n)))
    s = e.sum(1, keepdims=True)
    return np.where(s > 0, e / np.where(s > 0, s, 1.0), 1.0 / n)
