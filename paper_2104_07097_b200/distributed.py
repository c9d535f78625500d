"""Multi-GPU plumbing: walks are sharded across ranks (one process per GPU);
nothing is exchanged per iterate.

Walks never interact (the reference's per-column loops, proj/src/sampler.cpp
:182-200 and :258-270), and the Philox streams are keyed on the
GLOBAL walk id, so a sample set is identical whatever the GPU count.  The
only collectives are the ones the north star names: gathering collected
samples to rank 0 and reducing diagnostics (NCCL over NVLink on GPUs; gloo on
CPU for the tests).
"""
from __future__ import annotations

import dataclasses
from typing import Optional

import numpy as np


def shard_walks(z_total: int, world: int, rank: int):
    """Contiguous walk range of `rank`: (z_local, global offset).  The first
    z_total % world ranks take one extra walk."""
    if z_total < world:
        raise ValueError(f"{z_total} walks cannot be sharded over {world} ranks")
    base, extra = divmod(z_total, world)
    z_local = base + (1 if rank < extra else 0)
    offset = rank * base + min(rank, extra)
    return z_local, offset


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (device time of a timed region)."""
    import torch
    import torch.distributed as dist
    if not dist.is_initialized():
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


@dataclasses.dataclass
class Diagnostics:
    redraws: int
    max_violation: float
    max_eq_residual: float
    coord_sum: np.ndarray   # per-coordinate sum of collected samples (moment checks)
    coord_sumsq: np.ndarray
    count: int


def reduce_diagnostics(redraws: int, max_violation: float, max_eq: float, rows, device=None
                       ) -> Diagnostics:
    """All-reduce of the per-rank diagnostics: redraw count, worst
    containment slack, and per-coordinate sums for moment checks (<= 2n
    doubles)."""
    import torch
    import torch.distributed as dist
    rows_t = rows if isinstance(rows, torch.Tensor) else torch.as_tensor(np.asarray(rows))
    rows_t = rows_t.to(device=device, dtype=torch.float64)
    n = rows_t.shape[1]
    sums = torch.cat([rows_t.sum(0), (rows_t * rows_t).sum(0),
                      torch.tensor([float(redraws), float(rows_t.shape[0])], dtype=torch.float64,
                                   device=rows_t.device)])
    mx = torch.tensor([float(max_violation), float(max_eq)], dtype=torch.float64,
                      device=rows_t.device)
    if dist.is_initialized():
        dist.all_reduce(sums, op=dist.ReduceOp.SUM)
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    s = sums.cpu().numpy()
    return Diagnostics(redraws=int(round(s[2 * n])), max_violation=float(mx[0]),
                       max_eq_residual=float(mx[1]), coord_sum=s[:n], coord_sumsq=s[n:2 * n],
                       count=int(round(s[2 * n + 1])))


def gather_rows(local_rows, z_counts, dst: int = 0):
    """Gather every rank's (z_local x n) sample rows to rank `dst` in global
    walk order (rank-major = walk-id order, since shards are contiguous).
    A true gather: only `dst` receives (torch's NCCL gather is a grouped
    ncclSend / ncclRecv; gloo has its own), so at 8 ranks and config 5 each
    rank sends its 65.5 MB once instead of receiving 524 MB.  Ragged shards
    are padded to the largest.  Returns the (sum z) x n tensor on dst, None
    elsewhere."""
    import torch
    import torch.distributed as dist
    if not dist.is_initialized():
        return local_rows
    zmax = max(z_counts)
    n = local_rows.shape[1]
    if local_rows.shape[0] == zmax:
        padded = local_rows.contiguous()
    else:
        padded = torch.zeros((zmax, n), dtype=local_rows.dtype, device=local_rows.device)
        padded[: local_rows.shape[0]] = local_rows
    rank = dist.get_rank()
    bufs = None
    if rank == dst:
        bufs = [torch.empty((zmax, n), dtype=local_rows.dtype, device=local_rows.device)
                for _ in z_counts]
    dist.gather(padded, gather_list=bufs, dst=dst)
    if rank != dst:
        return None
    return torch.cat([b[:z] for b, z in zip(bufs, z_counts)], 0)


def first_failure(local_bad: int, offset: int, device=None) -> int:
    """Global id of the lowest walk that failed containment on any rank, or
    -1: the reference's run() raises NUMERICAL_FAILURE naming the first
    failing walk (sampler.cpp:319-324), so every rank learns it."""
    import torch
    import torch.distributed as dist
    big = float(2 ** 62)
    v = float(local_bad + offset) if local_bad >= 0 else big
    if not dist.is_initialized():
        return -1 if v == big else int(v)
    t = torch.tensor([v], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    v = float(t.item())
    return -1 if v == big else int(v)


def _backend_is_device() -> bool:
    """True when the process group's collectives take CUDA tensors (NCCL)."""
    import torch.distributed as dist
    return not dist.is_initialized() or dist.get_backend() != "gloo"


class ShardedSampler:
    """One rank's share of a multi-GPU MHAR run: an Engine over the rank's
    contiguous walk range on its local GPU, collection windows gathered to
    rank 0 over NCCL (device memory to device memory, no host round trip)."""

    def __init__(self, polytope, z_total: int, seed: int, projector=None, rank: int = 0,
                 world: int = 1, local_rank: int = 0, **engine_kw):
        from . import Engine
        self.z_total = z_total
        self.world = world
        self.rank = rank
        self.z, self.offset = shard_walks(z_total, world, rank)
        self.z_counts = [shard_walks(z_total, world, r)[0] for r in range(world)]
        self.n = polytope.dim()
        self.device = local_rank
        engine_kw.setdefault("z_plan", z_total)  # same kernels for every world size
        self.engine = Engine(polytope, self.z, seed=seed, projector=projector, device=local_rank,
                             chain_offset=self.offset, **engine_kw)

    def set_start(self, x0):
        X = np.empty((self.n, self.z), order="F")
        X[:] = np.asarray(x0, dtype=np.float64)[:, None]
        self.engine.set_state(X)

    def window(self, phi: int, reproject_every: int = 0, gather: bool = True):
        """phi iterates on every rank, containment check of every walk, gather
        to rank 0.  Raises MharError(NUMERICAL_FAILURE) on every rank, naming
        the lowest global walk outside the body, like the reference's run()
        (sampler.cpp:319-324), before anything is gathered."""
        import torch
        from . import ErrorCode, MharError
        self.engine.step(phi, reproject_every)
        bad, viol, eqv = self.engine.check_state(self.engine.eps_feas)
        rows = torch.empty((self.z, self.n), dtype=torch.float64, device=f"cuda:{self.device}")
        self.engine.state_rows_to_device(rows.data_ptr())
        dev = rows.device if _backend_is_device() else "cpu"
        failed = first_failure(bad, self.offset, device=dev)
        if failed >= 0:
            raise MharError(ErrorCode.numerical_failure,
                            f"NUMERICAL_FAILURE: walk {failed} left the polytope at a collection")
        diag = reduce_diagnostics(self.engine.stats()["redraw_count"], float(viol.max()),
                                  float(eqv.max()), rows, device=dev)
        full = gather_rows(rows if dev != "cpu" else rows.cpu(), self.z_counts) if gather else None
        return full, diag

    def close(self):
        self.engine.close()
