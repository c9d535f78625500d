"""B200-native MHAR (Matrix Hit-and-Run) chain-step engine.

Python mirror of the reference sampler interface
(/root/reference/proj/include/mhar/{polytope,sampler,projection,errors}.hpp)
over the engine's C ABI (include/mhar_b200.h, libmhar_b200.so).  Every
computation runs in the CUDA library; there is no CPU fallback -- importing
this package without the built library raises.

    p = make_hypercube(10)
    cfg = resolve(SamplerConfig(z=100, phi=1, t_target=100_000, burn_in=1000), p)
    out = run(p, cfg, x0=np.zeros(10))          # SampleSet, like mhar::run
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import os
from typing import Optional

import numpy as np

__all__ = [
    "MharError", "ErrorCode", "Polytope", "SamplerConfig", "ProjectionOperator", "SampleSet",
    "LambdaIntervals", "Engine", "Group", "WalkState", "resolve", "compute_projection", "run", "step",
    "make_hypercube", "make_simplex", "contains", "library_path", "FLAG_DEGENERATE",
    "FLAG_HAS_UPPER", "FLAG_HAS_LOWER", "FLAG_COLLAPSED", "FLAG_THETA_MIDPOINT",
    "kDegenerateWidth", "kMaxDirectionRetries", "kNearZeroDirection",
]

HERE = os.path.dirname(os.path.abspath(__file__))
# MHAR_LIB selects an alternative in-tree build (tuning experiments only).
_LIB_PATH = os.environ.get("MHAR_LIB") or os.path.join(HERE, "lib", "libmhar_b200.so")

# Constants mirrored from the reference headers.
kDegenerateWidth = 1e-14      # sampler.hpp:40
kMaxDirectionRetries = 16     # sampler.hpp:43
kNearZeroDirection = 1e-12    # projection.hpp:25

FLAG_DEGENERATE = 1
FLAG_HAS_UPPER = 2
FLAG_HAS_LOWER = 4
FLAG_COLLAPSED = 8
FLAG_THETA_MIDPOINT = 16

RNG_PHILOX = 0
RNG_REFERENCE = 1
SLACK_RECOMPUTE = 0
SLACK_INCREMENTAL = 1
F64_DMMA = 0
F64_INT8 = 1


class ErrorCode:
    """mhar::ErrorCode (proj/include/mhar/errors.hpp:10-24); status = 1 + ordinal."""
    invalid_argument = 1
    dimension_mismatch = 2
    singular_matrix = 3
    rank_deficient_eq = 4
    empty_polytope = 5
    no_interior = 6
    unbounded_polytope = 7
    direction_degenerate = 8
    retry_exhausted = 9
    cycle_suspected = 10
    degenerate_test = 11
    numerical_failure = 12
    io_failure = 13
    cuda = 100

    NAMES = {1: "INVALID_ARGUMENT", 2: "DIMENSION_MISMATCH", 3: "SINGULAR_MATRIX",
             4: "RANK_DEFICIENT_EQ", 5: "EMPTY_POLYTOPE", 6: "NO_INTERIOR",
             7: "UNBOUNDED_POLYTOPE", 8: "DIRECTION_DEGENERATE", 9: "RETRY_EXHAUSTED",
             10: "CYCLE_SUSPECTED", 11: "DEGENERATE_TEST", 12: "NUMERICAL_FAILURE",
             13: "IO_FAILURE", 100: "CUDA_ERROR"}


class MharError(RuntimeError):
    """mhar::Error (errors.hpp:30-37): carries the ErrorCode status."""

    def __init__(self, code: int, message: str):
        super().__init__(message)
        self.code = code

    @property
    def name(self) -> str:
        return ErrorCode.NAMES.get(self.code, "UNKNOWN")


# ------------------------------------------------------------ C ABI -------

class _Polytope(C.Structure):
    _fields_ = [("n", C.c_int64), ("m_in", C.c_int64), ("m_eq", C.c_int64),
                ("a_in", C.POINTER(C.c_double)), ("b_in", C.POINTER(C.c_double)),
                ("a_eq", C.POINTER(C.c_double)), ("b_eq", C.POINTER(C.c_double))]


class _Options(C.Structure):
    _fields_ = [("z", C.c_int64), ("chain_offset", C.c_int64), ("seed", C.c_uint64),
                ("eps_dir", C.c_double), ("eps_feas", C.c_double), ("rng", C.c_int),
                ("slack_mode", C.c_int), ("refresh_every", C.c_int64), ("device", C.c_int),
                ("small_path", C.c_int), ("precision", C.c_int), ("fp32_margin", C.c_double),
                ("f64_engine", C.c_int), ("fp32_direction", C.c_int), ("z_plan", C.c_int64)]


class _RunConfig(C.Structure):
    _fields_ = [("phi", C.c_int64), ("windows", C.c_int64), ("burn_in", C.c_int64),
                ("reproject_every", C.c_int64)]


class _RunStats(C.Structure):
    _fields_ = [("iterate_count", C.c_int64), ("windows", C.c_int64),
                ("redraw_count", C.c_int64), ("err_walk", C.c_int64), ("seconds", C.c_double)]


class _CtxStats(C.Structure):
    _fields_ = [("iterations", C.c_int64), ("redraw_count", C.c_int64),
                ("kernel_launches", C.c_int64), ("chord_launches", C.c_int64),
                ("chord_ms", C.c_double), ("chord_timed", C.c_int64),
                ("chord_flops", C.c_double), ("refreshes", C.c_int64),
                ("z", C.c_int64), ("z_padded", C.c_int64), ("m_padded", C.c_int64),
                ("n_padded", C.c_int64), ("chord_kernel", C.c_int64)]


# mhar_chord_kernel (include/mhar_b200.h)
CHORD_KERNELS = {1: "small_kernel", 2: "chord2_kernel", 3: "chord3_kernel",
                 4: "chord_tc32_kernel", 5: "chord_i8_kernel", 6: "diag_chord_kernel"}


def _stats_dict(s: "_CtxStats") -> dict:
    d = {f[0]: getattr(s, f[0]) for f in s._fields_}
    d["chord_kernel"] = CHORD_KERNELS.get(d["chord_kernel"], str(d["chord_kernel"]))
    return d


_dp = C.POINTER(C.c_double)
_u8p = C.POINTER(C.c_uint8)
_i64p = C.POINTER(C.c_int64)

# Every symbol include/mhar_b200.h declares (checked by tests/test_abi_exports.py).
EXPORTED_SYMBOLS = [
    "mhar_default_options", "mhar_ctx_create", "mhar_ctx_destroy", "mhar_set_state",
    "mhar_get_state", "mhar_get_state_rows_device", "mhar_step", "mhar_sync", "mhar_step_timed",
    "mhar_step_injected", "mhar_lambda_intervals", "mhar_check_state", "mhar_run",
    "mhar_compute_projection", "mhar_get_stats", "mhar_set_timing", "mhar_reset_stats",
    "mhar_flops_per_iterate", "mhar_last_error", "mhar_version", "mhar_device_count",
    "mhar_minimum_spanning_tree", "mhar_friedman_rafsky", "mhar_generate_directions",
    "mhar_select_points", "mhar_chebyshev_center", "mhar_debug_last_iterate",
    "mhar_get_iteration", "mhar_set_iteration", "mhar_get_streams", "mhar_set_streams",
    "mhar_request_refresh", "mhar_group_create", "mhar_group_destroy", "mhar_group_info",
    "mhar_group_context", "mhar_group_set_state", "mhar_group_get_state", "mhar_group_step",
    "mhar_group_run",
]


class _FrResult(C.Structure):
    _fields_ = [("cross_edges", C.c_int64), ("expected_cross", C.c_double),
                ("variance_cross", C.c_double), ("z_value", C.c_double),
                ("shared_end_pairs", C.c_int64), ("pooled_size", C.c_int64)]

MHAR_GROUP_MAX_DEV = 16


class _GroupInfo(C.Structure):
    _fields_ = [("ndev", C.c_int), ("uses_nccl", C.c_int), ("z_total", C.c_int64),
                ("devices", C.c_int * MHAR_GROUP_MAX_DEV), ("z", C.c_int64 * MHAR_GROUP_MAX_DEV),
                ("offset", C.c_int64 * MHAR_GROUP_MAX_DEV), ("last_max_violation", C.c_double),
                ("last_redraws", C.c_int64), ("gather", C.c_int)]


# mhar_group_gather (include/mhar_b200.h)
GROUP_GATHER = {0: "copy", 1: "nccl", 2: "direct"}


class _LpStats(C.Structure):
    _fields_ = [("rounds", C.c_int32), ("reserved", C.c_int32), ("pivots", C.c_int64),
                ("working_rows", C.c_int64)]


_lib = None


def library_path() -> str:
    return _LIB_PATH


def lib():
    """Loads libmhar_b200.so.  Raises if it is missing: no fallback path."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        raise ImportError(f"{_LIB_PATH} is missing; build it with "
                          "`python -c 'import __graft_entry__ as g; g.build()'`")
    L = C.CDLL(_LIB_PATH)
    L.mhar_default_options.argtypes = [C.POINTER(_Options)]
    L.mhar_default_options.restype = None
    L.mhar_ctx_create.argtypes = [C.POINTER(_Polytope), _dp, _dp, C.POINTER(_Options),
                                  C.POINTER(C.c_void_p)]
    L.mhar_ctx_destroy.argtypes = [C.c_void_p]
    L.mhar_set_state.argtypes = [C.c_void_p, _dp]
    L.mhar_get_state.argtypes = [C.c_void_p, _dp]
    L.mhar_get_state_rows_device.argtypes = [C.c_void_p, C.c_void_p]
    L.mhar_get_iteration.argtypes = [C.c_void_p, _i64p]
    L.mhar_get_iteration.restype = C.c_int
    L.mhar_set_iteration.argtypes = [C.c_void_p, C.c_int64]
    L.mhar_set_iteration.restype = C.c_int
    _u64p = C.POINTER(C.c_uint64)
    L.mhar_get_streams.argtypes = [C.c_void_p, _u64p, _u64p]
    L.mhar_get_streams.restype = C.c_int
    L.mhar_set_streams.argtypes = [C.c_void_p, _u64p, _u64p]
    L.mhar_set_streams.restype = C.c_int
    L.mhar_request_refresh.argtypes = [C.c_void_p]
    L.mhar_request_refresh.restype = C.c_int
    L.mhar_group_create.argtypes = [C.POINTER(_Polytope), _dp, _dp, C.POINTER(_Options),
                                    C.POINTER(C.c_int), C.c_int, C.POINTER(C.c_void_p)]
    L.mhar_group_create.restype = C.c_int
    L.mhar_group_destroy.argtypes = [C.c_void_p]
    L.mhar_group_destroy.restype = C.c_int
    L.mhar_group_info.argtypes = [C.c_void_p, C.POINTER(_GroupInfo)]
    L.mhar_group_info.restype = C.c_int
    L.mhar_group_context.argtypes = [C.c_void_p, C.c_int]
    L.mhar_group_context.restype = C.c_void_p
    L.mhar_group_set_state.argtypes = [C.c_void_p, _dp]
    L.mhar_group_set_state.restype = C.c_int
    L.mhar_group_get_state.argtypes = [C.c_void_p, _dp]
    L.mhar_group_get_state.restype = C.c_int
    L.mhar_group_step.argtypes = [C.c_void_p, C.c_int64, C.c_int64]
    L.mhar_group_step.restype = C.c_int
    L.mhar_group_run.argtypes = [C.c_void_p, C.POINTER(_RunConfig), _dp, _dp,
                                 C.POINTER(_RunStats)]
    L.mhar_group_run.restype = C.c_int
    L.mhar_debug_last_iterate.argtypes = [C.c_void_p, _dp, _dp, _dp, _dp]
    L.mhar_debug_last_iterate.restype = C.c_int
    L.mhar_step.argtypes = [C.c_void_p, C.c_int64, C.c_int64]
    L.mhar_sync.argtypes = [C.c_void_p]
    L.mhar_step_timed.argtypes = [C.c_void_p, C.c_int64, C.c_int64, _dp]
    L.mhar_step_injected.argtypes = [C.c_void_p, _dp, _dp, _dp, _dp, _dp, _u8p]
    L.mhar_lambda_intervals.argtypes = [C.c_void_p, _dp, _dp, _dp, _dp, _u8p]
    L.mhar_check_state.argtypes = [C.c_void_p, C.c_double, _i64p, _dp, _dp]
    L.mhar_run.argtypes = [C.c_void_p, C.POINTER(_RunConfig), _dp, _dp, C.POINTER(_RunStats)]
    L.mhar_compute_projection.argtypes = [_dp, C.c_int64, C.c_int64, _dp, _dp]
    L.mhar_get_stats.argtypes = [C.c_void_p, C.POINTER(_CtxStats)]
    L.mhar_set_timing.argtypes = [C.c_void_p, C.c_int]
    L.mhar_reset_stats.argtypes = [C.c_void_p]
    L.mhar_flops_per_iterate.argtypes = [C.c_void_p]
    L.mhar_flops_per_iterate.restype = C.c_double
    L.mhar_last_error.restype = C.c_char_p
    L.mhar_version.restype = C.c_char_p
    L.mhar_device_count.argtypes = [C.POINTER(C.c_int)]
    _i32p = C.POINTER(C.c_int32)
    L.mhar_minimum_spanning_tree.argtypes = [_dp, C.c_int64, C.c_int64, C.c_int, _i32p, _i32p, _dp]
    L.mhar_minimum_spanning_tree.restype = C.c_int
    L.mhar_friedman_rafsky.argtypes = [_dp, C.c_int64, _dp, C.c_int64, C.c_int64, C.c_int,
                                       C.POINTER(_FrResult)]
    L.mhar_friedman_rafsky.restype = C.c_int
    L.mhar_generate_directions.argtypes = [C.c_void_p, _dp]
    L.mhar_generate_directions.restype = C.c_int
    L.mhar_select_points.argtypes = [C.c_void_p, _dp, _dp, _dp, _dp, _u8p, _dp]
    L.mhar_select_points.restype = C.c_int
    L.mhar_chebyshev_center.argtypes = [C.POINTER(_Polytope), C.c_int, _dp, _dp,
                                        C.POINTER(_LpStats)]
    L.mhar_chebyshev_center.restype = C.c_int
    for name in ("mhar_ctx_create", "mhar_ctx_destroy", "mhar_set_state", "mhar_get_state",
                 "mhar_get_state_rows_device", "mhar_step", "mhar_sync", "mhar_step_timed",
                 "mhar_step_injected",
                 "mhar_lambda_intervals", "mhar_check_state", "mhar_run",
                 "mhar_compute_projection", "mhar_get_stats", "mhar_set_timing",
                 "mhar_reset_stats", "mhar_device_count"):
        getattr(L, name).restype = C.c_int
    _lib = L
    return L


def _check(status: int):
    if status != 0:
        msg = lib().mhar_last_error().decode(errors="replace")
        raise MharError(status, msg)


def _d(a):
    return None if a is None else a.ctypes.data_as(_dp)


def _f(a):
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


def _sized(what: str, a, shape, dtype=np.float64):
    """a as a contiguous array of exactly `shape` (the C ABI reads that many
    elements from the pointer): DIMENSION_MISMATCH otherwise."""
    a = np.asfortranarray(np.asarray(a, dtype=dtype))
    if a.shape != tuple(shape):
        raise MharError(ErrorCode.dimension_mismatch,
                        f"{what} has shape {a.shape}, expected {tuple(shape)}")
    return a


# -------------------------------------------------------------- types ------

class Polytope:
    """{x : a_in x <= b_in, a_eq x = b_eq} (polytope.hpp:12-25)."""

    def __init__(self, a_in, b_in, a_eq=None, b_eq=None):
        self.a_in = _f(a_in)
        if self.a_in.ndim != 2:
            raise MharError(ErrorCode.dimension_mismatch,
                            f"polytope: a_in must be a matrix, got shape {self.a_in.shape}")
        self.b_in = np.ascontiguousarray(b_in, dtype=np.float64).reshape(-1)
        n = self.a_in.shape[1]
        if a_eq is None or np.asarray(a_eq).size == 0:
            self.a_eq = np.zeros((0, n), order="F")
            self.b_eq = np.zeros(0) if b_eq is None else \
                np.ascontiguousarray(b_eq, dtype=np.float64).reshape(-1)
        else:
            self.a_eq = _f(a_eq)
            self.b_eq = np.ascontiguousarray(b_eq, dtype=np.float64).reshape(-1)
        # the reference constructor's checks (polytope.cpp:16-33, :90-97); the
        # engine reads exactly these extents through the C ABI
        for what, got, want in (("b_in length", self.b_in.size, self.a_in.shape[0]),
                                ("a_eq width", self.a_eq.shape[1] if self.a_eq.ndim == 2 else -1, n),
                                ("b_eq length", self.b_eq.size, self.a_eq.shape[0])):
            if got != want:
                raise MharError(ErrorCode.dimension_mismatch,
                                f"polytope: {what} is {got}, expected {want}")

    def dim(self) -> int:
        return self.a_in.shape[1]

    def num_inequalities(self) -> int:
        return self.a_in.shape[0]

    def num_equalities(self) -> int:
        return self.a_eq.shape[0]


def make_hypercube(n: int) -> Polytope:
    """[-1, 1]^n as 2n rows (polytope.cpp:192-199)."""
    if n < 1:
        raise MharError(ErrorCode.invalid_argument, "make_hypercube: n must be >= 1")
    return Polytope(np.vstack([np.eye(n), -np.eye(n)]), np.ones(2 * n))


def make_simplex(n: int) -> Polytope:
    """{x >= 0, sum x = 1} (polytope.cpp:201-208)."""
    if n < 2:
        raise MharError(ErrorCode.invalid_argument, "make_simplex: n must be >= 2")
    return Polytope(-np.eye(n), np.zeros(n), np.ones((1, n)), np.ones(1))


@dataclasses.dataclass
class SamplerConfig:
    """mhar::SamplerConfig (sampler.hpp:16-25); 0 / -1 sentinels resolve."""
    z: int = 0
    phi: int = 0
    t_target: int = 1
    seed: int = 0
    eps_dir: float = 1e-11
    eps_feas: float = 1e-9
    reproject_every: int = -1
    burn_in: int = -1


def resolve(cfg: SamplerConfig, p: Polytope) -> SamplerConfig:
    """resolve() (sampler.cpp:127-141)."""
    r = dataclasses.replace(cfg)
    n = p.dim()
    walk_dim = n - p.num_equalities()
    if r.z == 0:
        r.z = max(p.num_inequalities(), n) + 1
    if r.phi == 0:
        r.phi = walk_dim ** 3
    if r.burn_in < 0:
        r.burn_in = r.phi
    if r.reproject_every < 0:
        r.reproject_every = r.phi
    if r.z < 1:
        raise MharError(ErrorCode.invalid_argument, "config: z must be >= 1")
    if r.phi < 1:
        raise MharError(ErrorCode.invalid_argument, "config: phi must be >= 1")
    if r.t_target < 1:
        raise MharError(ErrorCode.invalid_argument, "config: t_target must be >= 1")
    if not r.eps_dir > 0.0:
        raise MharError(ErrorCode.invalid_argument, "config: eps_dir must be > 0")
    if not r.eps_feas > 0.0:
        raise MharError(ErrorCode.invalid_argument, "config: eps_feas must be > 0")
    return r


@dataclasses.dataclass
class ProjectionOperator:
    """projection.hpp:11-15."""
    p: np.ndarray
    gram_inverse: np.ndarray
    source_eq: np.ndarray


def compute_projection(a_eq) -> ProjectionOperator:
    """compute_projection (projection.cpp:9-34), host side as in the reference."""
    a_eq = _f(a_eq)
    me, n = a_eq.shape
    if me == 0:
        raise MharError(ErrorCode.invalid_argument,
                        "compute_projection: equality matrix is empty")
    P = np.empty((n, n), order="F")
    G = np.empty((me, me), order="F")
    _check(lib().mhar_compute_projection(_d(a_eq), me, n, _d(P), _d(G)))
    return ProjectionOperator(P, G, a_eq.copy(order="F"))


@dataclasses.dataclass
class LambdaIntervals:
    """sampler.hpp:33-37 (+ the MHAR_FLAG_* bits per walk)."""
    lower: np.ndarray
    upper: np.ndarray
    degenerate: np.ndarray
    flags: np.ndarray


@dataclasses.dataclass
class WalkState:
    """sampler.hpp:69-74."""
    x: np.ndarray
    t: int = 0
    j: int = 0
    redraws: int = 0


@dataclasses.dataclass
class SampleSet:
    """sampler.hpp:82-91."""
    samples: np.ndarray
    config: SamplerConfig
    start: np.ndarray
    start_radius: float
    seconds: float
    iterate_count: int
    windows: int
    redraw_count: int


# ------------------------------------------------------------- engine ------

def _context_args(p, z, seed, projector, eps_dir, eps_feas, rng, slack, refresh_every, device,
                  chain_offset, small_path, precision, fp32_margin, f64_engine, fp32_direction,
                  z_plan=0):
    """(polytope struct, options struct, P, G) for mhar_ctx_create /
    mhar_group_create; the returned arrays back the struct pointers."""
    L = lib()
    poly = _Polytope()
    poly.n = p.dim()
    poly.m_in = p.num_inequalities()
    poly.m_eq = p.num_equalities()
    poly.a_in = _d(p.a_in)
    poly.b_in = _d(p.b_in)
    if poly.m_eq > 0:
        poly.a_eq = _d(p.a_eq)
        poly.b_eq = _d(p.b_eq)
    opt = _Options()
    L.mhar_default_options(C.byref(opt))
    opt.z = int(z)
    opt.chain_offset = int(chain_offset)
    opt.seed = int(seed) & (2**64 - 1)
    opt.eps_dir = eps_dir
    opt.eps_feas = eps_feas
    opt.rng = {"philox": RNG_PHILOX, "reference": RNG_REFERENCE}[rng]
    opt.slack_mode = {"recompute": SLACK_RECOMPUTE, "incremental": SLACK_INCREMENTAL}[slack]
    opt.refresh_every = int(refresh_every)
    opt.device = int(device)
    opt.small_path = 1 if small_path else 0
    opt.precision = int(precision)
    opt.fp32_margin = float(fp32_margin)
    opt.f64_engine = {"dmma": F64_DMMA, "int8": F64_INT8}[f64_engine]
    opt.fp32_direction = {"split": 0, "rounded": 1}[fp32_direction]
    opt.z_plan = int(z_plan)
    P = G = None
    if projector is not None:
        me = p.num_equalities()
        P = _sized("projector: p", projector.p, (p.dim(), p.dim()))
        G = _sized("projector: gram_inverse", projector.gram_inverse, (me, me))
    return poly, opt, P, G


class Engine:
    """One device context: the polytope resident in HBM plus z walks.

    rng: "philox" (default; keyed on global walk ids so shards are
    independent of the GPU count) or "reference" (the reference's SplitMix
    streams: column stream k and the shared theta stream, rng.hpp:42-55).
    slack: "incremental" (default) or "recompute" (one fused A_I[X|D] pass
    per iterate).  small_path: allow the walk-resident kernel for bodies that
    fit in shared memory (Philox only).  f64_engine (precision 64): "dmma"
    (default, fp64 tensor cores) or "int8" (A_I d formed exactly from 53-bit
    fixed-point operands split into int8 slices on the tcgen05 int8 tensor
    cores -- the Ozaki scheme; n <= 4608; refreshes and checks stay DMMA).
    fp32_direction (precision 32): "split" (default; the walk moves along its
    fp64 direction, the tensor cores see it as two operands) or "rounded"
    (the fast form: the direction is rounded to one operand and the walk
    moves along the rounded direction).
    """

    def __init__(self, p: Polytope, z: int, seed: int = 0, projector: Optional[ProjectionOperator] = None,
                 eps_dir: float = 1e-11, eps_feas: float = 1e-9, rng: str = "philox",
                 slack: str = "incremental", refresh_every: int = 128, device: int = 0,
                 chain_offset: int = 0, small_path: bool = True, precision: int = 64,
                 fp32_margin: float = 0.0, f64_engine: str = "dmma",
                 fp32_direction: str = "split", z_plan: int = 0):
        # z_plan: the whole run's walk count when this context is one shard
        # of it (mhar_options.z_plan): every sharding then takes the same
        # kernels, so the samples do not depend on the placement
        L = lib()
        self.p = p
        self.n = p.dim()
        self.z = int(z)
        self._keep = []
        poly, opt, P, G = _context_args(p, z, seed, projector, eps_dir, eps_feas, rng, slack,
                                        refresh_every, device, chain_offset, small_path,
                                        precision, fp32_margin, f64_engine, fp32_direction,
                                        z_plan)
        self.precision = int(precision)
        self.f64_engine = f64_engine
        self.rng = rng
        h = C.c_void_p()
        _check(L.mhar_ctx_create(C.byref(poly), _d(P), _d(G), C.byref(opt), C.byref(h)))
        self._h = h
        self.eps_feas = eps_feas
        self._args = (poly, P, G)  # keep the arrays the structs point to alive

    def close(self):
        if getattr(self, "_h", None):
            lib().mhar_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # state
    def set_state(self, x):
        x = _f(x)
        if x.shape != (self.n, self.z):
            raise MharError(ErrorCode.dimension_mismatch,
                            f"set_state: x is {x.shape}, expected {(self.n, self.z)}")
        _check(lib().mhar_set_state(self._h, _d(x)))

    def get_state(self, out: Optional[np.ndarray] = None) -> np.ndarray:
        x = np.empty((self.n, self.z), order="F") if out is None else out
        if x.shape != (self.n, self.z) or not x.flags.f_contiguous or x.dtype != np.float64:
            raise MharError(ErrorCode.dimension_mismatch, "get_state: out must be n x z F-order")
        _check(lib().mhar_get_state(self._h, _d(x)))
        return x

    def state_rows_to_device(self, dev_ptr: int):
        """Row-major z x n copy of the walks into caller-owned device memory."""
        _check(lib().mhar_get_state_rows_device(self._h, C.c_void_p(dev_ptr)))

    # iterates
    def step(self, iters: int = 1, reproject_every: int = 0, sync: bool = True):
        _check(lib().mhar_step(self._h, int(iters), int(reproject_every)))
        if sync:
            self.sync()

    def sync(self):
        _check(lib().mhar_sync(self._h))

    def request_refresh(self):
        """The next iterate recomputes the incremental slack cache (the
        refresh pass of every refresh_every iterates)."""
        _check(lib().mhar_request_refresh(self._h))

    def step_timed(self, iters: int = 1, reproject_every: int = 0) -> float:
        """Iterates bracketed by CUDA events on the engine's stream; device ms."""
        ms = C.c_double(0.0)
        _check(lib().mhar_step_timed(self._h, int(iters), int(reproject_every), C.byref(ms)))
        return ms.value

    def step_injected(self, H, U):
        """Test hook: returns (lower, upper, theta, flags); moves the state."""
        H = _sized("step_injected: H", H, (self.n, self.z))
        U = _sized("step_injected: U", U, (self.z,))
        lo, hi, th = np.empty(self.z), np.empty(self.z), np.empty(self.z)
        fl = np.empty(self.z, np.uint8)
        _check(lib().mhar_step_injected(self._h, _d(H), _d(U), _d(lo), _d(hi), _d(th),
                                        fl.ctypes.data_as(_u8p)))
        return lo, hi, th, fl

    def generate_directions(self) -> np.ndarray:
        """generate_directions (sampler.cpp:143-148): the next n x z batch of
        standard normals from the walks' streams (advances them)."""
        h = np.empty((self.n, self.z), order="F")
        _check(lib().mhar_generate_directions(self._h, _d(h)))
        return h

    def select_points(self, X, D, intervals: "LambdaIntervals") -> np.ndarray:
        """select_points (sampler.cpp:214-233): x + theta d, theta uniform on
        each open chord from the theta stream; DIRECTION_DEGENERATE on flags."""
        X = _sized("select_points: x", X, (self.n, self.z))
        D = _sized("select_points: d", D, (self.n, self.z))
        lo = _sized("select_points: lower", intervals.lower, (self.z,))
        hi = _sized("select_points: upper", intervals.upper, (self.z,))
        dg = _sized("select_points: degenerate", intervals.degenerate, (self.z,), np.uint8)
        out = np.empty((self.n, self.z), order="F")
        _check(lib().mhar_select_points(self._h, _d(X), _d(D), _d(lo), _d(hi),
                                        dg.ctypes.data_as(_u8p), _d(out)))
        return out

    def lambda_intervals(self, X, D) -> LambdaIntervals:
        X = _sized("compute_lambda_intervals: x", X, (self.n, self.z))
        D = _sized("compute_lambda_intervals: d", D, (self.n, self.z))
        lo, hi = np.empty(self.z), np.empty(self.z)
        fl = np.empty(self.z, np.uint8)
        _check(lib().mhar_lambda_intervals(self._h, _d(X), _d(D), _d(lo), _d(hi),
                                           fl.ctypes.data_as(_u8p)))
        return LambdaIntervals(lo, hi, (fl & FLAG_DEGENERATE).astype(np.uint8), fl)

    @property
    def iteration(self) -> int:
        """Iterates executed (the Philox counter of the next iterate)."""
        v = C.c_int64(0)
        _check(lib().mhar_get_iteration(self._h, C.byref(v)))
        return v.value

    @iteration.setter
    def iteration(self, value: int):
        _check(lib().mhar_set_iteration(self._h, int(value)))

    def get_streams(self):
        """Reference-stream mode: (z column stream states, theta stream state),
        the WalkRng counters (rng.hpp:42-55)."""
        cols = np.empty(self.z, np.uint64)
        th = np.empty(1, np.uint64)
        _u64p = C.POINTER(C.c_uint64)
        _check(lib().mhar_get_streams(self._h, cols.ctypes.data_as(_u64p), th.ctypes.data_as(_u64p)))
        return cols, int(th[0])

    def set_streams(self, cols, theta):
        cols = np.ascontiguousarray(cols, dtype=np.uint64)
        if cols.shape != (self.z,):
            raise MharError(ErrorCode.dimension_mismatch,
                            f"set_streams: {cols.shape[0]} column streams for {self.z} walks")
        th = np.array([theta], dtype=np.uint64)
        _u64p = C.POINTER(C.c_uint64)
        _check(lib().mhar_set_streams(self._h, cols.ctypes.data_as(_u64p), th.ctypes.data_as(_u64p)))

    def checkpoint(self):
        """Everything a walk set needs to resume: (X, iteration) with Philox
        directions, (X, (column streams, theta stream)) on the reference
        streams."""
        if self.rng == "reference":
            return self.get_state(), self.get_streams()
        return self.get_state(), self.iteration

    def restore(self, checkpoint):
        X, key = checkpoint
        self.set_state(X)
        if isinstance(key, tuple):
            self.set_streams(*key)
        else:
            self.iteration = key

    def debug_last_iterate(self):
        """Test hook: (D n x z, lower, upper, theta) of the last iterate."""
        d = np.empty((self.n, self.z), order="F")
        lo, hi, th = np.empty(self.z), np.empty(self.z), np.empty(self.z)
        _check(lib().mhar_debug_last_iterate(self._h, _d(d), _d(lo), _d(hi), _d(th)))
        return d, lo, hi, th

    def check_state(self, eps: float):
        """(first_bad or -1, max_i (A x - b)_i per walk, max |A_E x - b_E| per walk)."""
        fb = C.c_int64(-1)
        mv, me = np.empty(self.z), np.empty(self.z)
        _check(lib().mhar_check_state(self._h, eps, C.byref(fb), _d(mv), _d(me)))
        return fb.value, mv, me

    def run(self, x0, phi: int, windows: int, burn_in: int = 0, reproject_every: int = 0,
            collect: bool = True):
        cfg = _RunConfig(int(phi), int(windows), int(burn_in), int(reproject_every))
        x0 = np.ascontiguousarray(x0, dtype=np.float64)
        if x0.shape != (self.n,):
            # mhar_run reads exactly n doubles from x0
            raise MharError(ErrorCode.dimension_mismatch,
                            f"run: x0 has shape {x0.shape}, expected ({self.n},)")
        samples = np.empty((windows * self.z, self.n)) if collect else None
        st = _RunStats()
        _check(lib().mhar_run(self._h, C.byref(cfg), _d(x0), _d(samples), C.byref(st)))
        return samples, st

    def stats(self) -> dict:
        s = _CtxStats()
        _check(lib().mhar_get_stats(self._h, C.byref(s)))
        return _stats_dict(s)

    def set_timing(self, on: bool):
        _check(lib().mhar_set_timing(self._h, 1 if on else 0))

    def reset_stats(self):
        _check(lib().mhar_reset_stats(self._h))

    def flops_per_iterate(self) -> float:
        return lib().mhar_flops_per_iterate(self._h)


def _prefer_bundled_nccl():
    """Point MHAR_NCCL_LIB (csrc/group.cu) at the NCCL that torch bundles, so
    the group and a later `import torch` share one libnccl.so.2."""
    if os.environ.get("MHAR_NCCL_LIB"):
        return
    import importlib.util
    try:
        spec = importlib.util.find_spec("nvidia.nccl")
    except (ImportError, ValueError):
        return
    for d in (spec.submodule_search_locations or []) if spec else []:
        cand = os.path.join(d, "lib", "libnccl.so.2")
        if os.path.exists(cand):
            os.environ["MHAR_NCCL_LIB"] = cand
            return


class Group:
    """Several GPUs driven from this process (mhar_group_*): z_total walks in
    contiguous shards over `devices` keyed on their global ids (the samples
    do not depend on the device list), the polytope replicated, one host
    thread per device; collection windows gathered to devices[0] with NCCL
    (peer copies when a device is listed twice or NCCL is absent)."""

    def __init__(self, p: Polytope, z_total: int, devices, seed: int = 0,
                 projector: Optional[ProjectionOperator] = None, eps_dir: float = 1e-11,
                 eps_feas: float = 1e-9, slack: str = "incremental", refresh_every: int = 128,
                 chain_offset: int = 0, small_path: bool = True, precision: int = 64,
                 fp32_margin: float = 0.0, f64_engine: str = "dmma",
                 fp32_direction: str = "split", rng: str = "philox"):
        _prefer_bundled_nccl()
        L = lib()
        self.p = p
        self.n = p.dim()
        self.z = int(z_total)
        self.devices = [int(d) for d in devices]
        poly, opt, P, G = _context_args(p, z_total, seed, projector, eps_dir, eps_feas, rng,
                                        slack, refresh_every, self.devices[0], chain_offset,
                                        small_path, precision, fp32_margin, f64_engine,
                                        fp32_direction)
        devs = (C.c_int * len(self.devices))(*self.devices)
        h = C.c_void_p()
        _check(L.mhar_group_create(C.byref(poly), _d(P), _d(G), C.byref(opt), devs,
                                   len(self.devices), C.byref(h)))
        self._h = h
        self._args = (poly, P, G)

    def close(self):
        if getattr(self, "_h", None):
            lib().mhar_group_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def info(self) -> dict:
        gi = _GroupInfo()
        _check(lib().mhar_group_info(self._h, C.byref(gi)))
        nd = gi.ndev
        return {"ndev": nd, "uses_nccl": bool(gi.uses_nccl), "z_total": gi.z_total,
                "devices": list(gi.devices[:nd]), "z": list(gi.z[:nd]),
                "offset": list(gi.offset[:nd]), "last_max_violation": gi.last_max_violation,
                "last_redraws": gi.last_redraws, "gather": GROUP_GATHER.get(gi.gather, "?")}

    def set_state(self, x):
        x = _f(x)
        if x.shape != (self.n, self.z):
            raise MharError(ErrorCode.dimension_mismatch,
                            f"set_state: x is {x.shape}, expected {(self.n, self.z)}")
        _check(lib().mhar_group_set_state(self._h, _d(x)))

    def get_state(self) -> np.ndarray:
        x = np.empty((self.n, self.z), order="F")
        _check(lib().mhar_group_get_state(self._h, _d(x)))
        return x

    def step(self, iters: int = 1, reproject_every: int = 0):
        _check(lib().mhar_group_step(self._h, int(iters), int(reproject_every)))

    def run(self, x0, phi: int, windows: int, burn_in: int = 0, reproject_every: int = 0,
            collect: bool = True):
        x0 = np.ascontiguousarray(x0, dtype=np.float64)
        if x0.shape != (self.n,):
            raise MharError(ErrorCode.dimension_mismatch,
                            f"run: x0 has shape {x0.shape}, expected ({self.n},)")
        cfg = _RunConfig(int(phi), int(windows), int(burn_in), int(reproject_every))
        samples = np.empty((windows * self.z, self.n)) if collect else None
        st = _RunStats()
        _check(lib().mhar_group_run(self._h, C.byref(cfg), _d(x0), _d(samples), C.byref(st)))
        return samples, st

    def context_stats(self, i: int) -> dict:
        """Shard i's single-device counters (mhar_get_stats)."""
        h = lib().mhar_group_context(self._h, int(i))
        if not h:
            raise MharError(ErrorCode.invalid_argument, f"group has no shard {i}")
        s = _CtxStats()
        _check(lib().mhar_get_stats(C.c_void_p(h), C.byref(s)))
        return _stats_dict(s)


# ------------------------------------------------ reference-style calls ----

def step(p: Polytope, projector: Optional[ProjectionOperator], cfg: SamplerConfig,
         engine: Engine, state: WalkState):
    """step() (sampler.hpp:79-80) on an engine holding the walks' RNG:
    state.x is uploaded, advanced one iterate on the device, and read back.
    The engine holds its device copy of the body, so p must be the polytope
    it was built for (the same object or the same arrays)."""
    q = engine.p

    def same(a, b):  # the same array memory (or both empty of one shape)
        return a is b or (a.shape == b.shape and (a.size == 0 or (
            a.strides == b.strides and
            a.__array_interface__["data"][0] == b.__array_interface__["data"][0])))
    if p is not q and not (same(p.a_in, q.a_in) and same(p.b_in, q.b_in)
                           and same(p.a_eq, q.a_eq) and same(p.b_eq, q.b_eq)):
        raise MharError(ErrorCode.invalid_argument,
                        "step: the engine was built for another polytope (build an Engine for p)")
    engine.set_state(state.x)
    before = engine.stats()["redraw_count"]
    engine.step(1)
    state.x = engine.get_state()
    state.j += 1
    state.redraws += engine.stats()["redraw_count"] - before


def contains(p: Polytope, x, eps: float) -> bool:
    """contains() (polytope.cpp:177-190), evaluated on the host for one point
    (API completeness; the engine checks every walk on the device)."""
    x = np.asarray(x, dtype=np.float64)
    if x.shape[0] != p.dim():
        raise MharError(ErrorCode.dimension_mismatch, "contains: dimension mismatch")
    if p.num_inequalities() and (p.a_in @ x - p.b_in).max() > eps:
        return False
    if p.num_equalities() and np.abs(p.a_eq @ x - p.b_eq).max() > eps:
        return False
    return True


@dataclasses.dataclass
class ChebyshevCenter:
    """chebyshev.hpp:8-11 (+ the constraint-generation counters)."""
    x: np.ndarray
    radius: float
    rounds: int = 0
    pivots: int = 0
    working_rows: int = 0


def chebyshev_center(p: Polytope, device: int = 0) -> ChebyshevCenter:
    """chebyshev_center (chebyshev.hpp:22-25): centre and radius of the
    largest inscribed ball, solved on the GPU by constraint generation over a
    device-resident simplex tableau.  Raises EMPTY_POLYTOPE /
    UNBOUNDED_POLYTOPE / NO_INTERIOR / NUMERICAL_FAILURE like the reference."""
    L = lib()
    a_in = np.asfortranarray(p.a_in, dtype=np.float64)
    b_in = np.ascontiguousarray(p.b_in, dtype=np.float64)
    poly = _Polytope()
    poly.n = p.dim()
    poly.m_in = p.num_inequalities()
    poly.m_eq = p.num_equalities()
    poly.a_in = a_in.ctypes.data_as(_dp)
    poly.b_in = b_in.ctypes.data_as(_dp)
    if poly.m_eq > 0:
        a_eq = np.asfortranarray(p.a_eq, dtype=np.float64)
        b_eq = np.ascontiguousarray(p.b_eq, dtype=np.float64)
        poly.a_eq = a_eq.ctypes.data_as(_dp)
        poly.b_eq = b_eq.ctypes.data_as(_dp)
    x = np.zeros(p.dim())
    r = C.c_double(0.0)
    st = _LpStats()
    _check(L.mhar_chebyshev_center(C.byref(poly), int(device), _d(x), C.byref(r), C.byref(st)))
    return ChebyshevCenter(x=x, radius=r.value, rounds=st.rounds, pivots=st.pivots,
                           working_rows=st.working_rows)


def run(p: Polytope, cfg: SamplerConfig, x0=None, rng: str = "philox", slack: str = "incremental",
        device: int = 0, clock=None) -> SampleSet:
    """run() (sampler.cpp:274-335) on one B200.  Without x0 the start is the
    Chebyshev centre (sampler.cpp:276), computed before the clock starts as
    in the reference; with x0 that warm start replaces it (start_radius 0).
    `clock` (the reference's ClockFn, sampler.cpp:278-282; default the host's
    monotonic clock) is read once before the projector is built and once
    after the last collection, so `seconds` spans projector construction,
    the context (polytope upload and packing) and every iterate, as the
    reference's window does (sampler.cpp:284-335)."""
    import time
    rc = resolve(cfg, p)
    radius = 0.0
    if x0 is None:
        center = chebyshev_center(p, device=device)
        x0, radius = center.x, center.radius
    x0 = np.ascontiguousarray(x0, dtype=np.float64)
    if x0.shape != (p.dim(),):
        raise MharError(ErrorCode.dimension_mismatch,
                        f"run: x0 has shape {x0.shape}, expected ({p.dim()},)")
    if clock is None:
        clock = time.perf_counter
    t0 = clock()
    projector = compute_projection(p.a_eq) if p.num_equalities() > 0 else None
    windows = (rc.t_target + rc.z - 1) // rc.z
    with Engine(p, rc.z, seed=rc.seed, projector=projector, eps_dir=rc.eps_dir,
                eps_feas=rc.eps_feas, rng=rng, slack=slack, device=device) as eng:
        samples, st = eng.run(x0, rc.phi, windows, rc.burn_in,
                              rc.reproject_every if projector is not None else 0)
    seconds = clock() - t0
    return SampleSet(samples=samples, config=rc, start=np.asarray(x0, dtype=np.float64),
                     start_radius=radius, seconds=seconds, iterate_count=st.iterate_count,
                     windows=st.windows, redraw_count=st.redraw_count)


from .throughput import (BenchConfig, BenchRecord, bench_csv_string, bench_json_string,  # noqa: E402
                         measure_throughput, sweep_padding, write_bench_csv, write_bench_json)
