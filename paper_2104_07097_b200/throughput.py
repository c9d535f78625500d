"""Throughput harness of the reference (proj/include/mhar/bench.hpp,
proj/src/bench.cpp:9-61): repeated run() calls at a padding z, rates
z * phi * windows / seconds per repetition, and the padding sweep the paper
uses to pick z* (PAPER.md:700-716).  Timing spans projector construction and
the walk loop; centring is excluded (run() centres before reading the clock)."""
from __future__ import annotations

import dataclasses
import math
from typing import Callable, Optional, Sequence

import numpy as np


@dataclasses.dataclass
class BenchConfig:
    """mhar::BenchConfig (bench.hpp:14-20)."""
    phi: int = 1000
    windows: int = 1         # collected batches per run
    repetitions: int = 5
    seed: int = 0            # repetition r runs with seed + r
    burn_in: int = 0


@dataclasses.dataclass
class BenchRecord:
    """mhar::BenchRecord (bench_types.hpp:9-20)."""
    figure: str = ""
    n: int = 0
    z: int = 0
    phi: int = 0
    windows: int = 0
    total_samples: int = 0   # iterates produced per repetition
    run_seconds: list = dataclasses.field(default_factory=list)
    run_sps: list = dataclasses.field(default_factory=list)
    mean_sps: float = 0.0
    std_sps: float = 0.0     # sample standard deviation, 0 for one run


def measure_throughput(p, z: int, cfg: BenchConfig, figure: str,
                       clock: Optional[Callable[[], float]] = None, x0=None,
                       device: int = 0) -> BenchRecord:
    """measure_throughput (bench.cpp:9-47): `repetitions` runs at padding z,
    repetition r seeded seed + r; INVALID_ARGUMENT for non-positive counts,
    NUMERICAL_FAILURE for a non-positive run time."""
    from . import MharError, ErrorCode, SamplerConfig, run
    if z < 1 or cfg.phi < 1 or cfg.windows < 1 or cfg.repetitions < 1 or cfg.burn_in < 0:
        raise MharError(ErrorCode.invalid_argument,
                        "INVALID_ARGUMENT: measure_throughput: all counts must be positive")
    rec = BenchRecord(figure=figure, n=p.dim(), z=int(z), phi=int(cfg.phi),
                      windows=int(cfg.windows),
                      total_samples=int(z) * int(cfg.phi) * int(cfg.windows))
    for rep in range(cfg.repetitions):
        sc = SamplerConfig(z=int(z), phi=int(cfg.phi), t_target=int(z) * int(cfg.windows),
                           burn_in=int(cfg.burn_in), seed=int(cfg.seed) + rep)
        out = run(p, sc, x0=x0, clock=clock, device=device)
        if not out.seconds > 0.0:
            raise MharError(ErrorCode.numerical_failure,
                            "NUMERICAL_FAILURE: measure_throughput: non-positive run time")
        rec.run_seconds.append(out.seconds)
        rec.run_sps.append(float(out.iterate_count) / out.seconds)
    rec.mean_sps = sum(rec.run_sps) / len(rec.run_sps)
    if len(rec.run_sps) > 1:
        sq = sum((v - rec.mean_sps) * (v - rec.mean_sps) for v in rec.run_sps)
        rec.std_sps = math.sqrt(sq / (len(rec.run_sps) - 1))
    return rec


def sweep_padding(p, z_values: Sequence[int], cfg: BenchConfig, figure: str,
                  clock: Optional[Callable[[], float]] = None, x0=None,
                  device: int = 0) -> list:
    """sweep_padding (bench.cpp:49-61): one record per padding value with phi
    and the window count held fixed."""
    from . import MharError, ErrorCode
    if len(z_values) == 0:
        raise MharError(ErrorCode.invalid_argument,
                        "INVALID_ARGUMENT: sweep_padding: z list is empty")
    return [measure_throughput(p, int(z), cfg, figure, clock=clock, x0=x0, device=device)
            for z in z_values]


def _fmt(v: float) -> str:
    """Shortest round-trip decimal (io.hpp:13); integral values without '.0'."""
    r = repr(float(v))
    return r[:-2] if r.endswith(".0") else r


def bench_csv_string(records: Sequence[BenchRecord]) -> str:
    """bench_csv_string (io.hpp): header, then one line per record."""
    s = "figure,n,z,phi,windows,total_samples,mean_sps,std_sps,runs\n"
    for r in records:
        s += (f"{r.figure},{r.n},{r.z},{r.phi},{r.windows},{r.total_samples},"
              f"{_fmt(r.mean_sps)},{_fmt(r.std_sps)},{len(r.run_seconds)}\n")
    return s


def bench_json_string(records: Sequence[BenchRecord]) -> str:
    """bench_json_string (io.hpp): {"format_version": 1, "records": [...]},
    sorted keys, two-space indent, per-run detail kept."""
    import json
    recs = [{"figure": r.figure, "n": r.n, "z": r.z, "phi": r.phi, "windows": r.windows,
             "total_samples": r.total_samples, "mean_sps": float(r.mean_sps),
             "std_sps": float(r.std_sps), "run_seconds": [float(v) for v in r.run_seconds],
             "run_sps": [float(v) for v in r.run_sps]} for r in records]
    return json.dumps({"format_version": 1, "records": recs}, indent=2, sort_keys=True) + "\n"


def write_bench_csv(path: str, records: Sequence[BenchRecord]) -> None:
    _write(path, bench_csv_string(records))


def write_bench_json(path: str, records: Sequence[BenchRecord]) -> None:
    _write(path, bench_json_string(records))


def _write(path: str, text: str) -> None:
    from . import MharError, ErrorCode
    try:
        with open(path, "w") as f:
            f.write(text)
    except OSError as e:
        raise MharError(ErrorCode.io_failure, f"IO_FAILURE: cannot write {path}: {e}") from e
