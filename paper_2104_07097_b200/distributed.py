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
    Uses all_gather (NCCL has no gather): ragged shards are padded to the
    largest.  Returns the (sum z) x n tensor on dst, None elsewhere."""
    import torch
    import torch.distributed as dist
    if not dist.is_initialized():
        return local_rows
    zmax = max(z_counts)
    n = local_rows.shape[1]
    padded = torch.zeros((zmax, n), dtype=local_rows.dtype, device=local_rows.device)
    padded[: local_rows.shape[0]] = local_rows
    out = torch.empty((len(z_counts) * zmax, n), dtype=local_rows.dtype, device=local_rows.device)
    dist.all_gather_into_tensor(out, padded)
    if dist.get_rank() != dst:
        return None
    parts = [out[r * zmax: r * zmax + z] for r, z in enumerate(z_counts)]
    return torch.cat(parts, 0)


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
        self.engine = Engine(polytope, self.z, seed=seed, projector=projector, device=local_rank,
                             chain_offset=self.offset, **engine_kw)

    def set_start(self, x0):
        X = np.empty((self.n, self.z), order="F")
        X[:] = np.asarray(x0, dtype=np.float64)[:, None]
        self.engine.set_state(X)

    def window(self, phi: int, reproject_every: int = 0, gather: bool = True):
        """phi iterates on every rank, containment check, gather to rank 0."""
        import torch
        self.engine.step(phi, reproject_every)
        bad, viol, eqv = self.engine.check_state(self.engine.eps_feas)
        rows = torch.empty((self.z, self.n), dtype=torch.float64, device=f"cuda:{self.device}")
        self.engine.state_rows_to_device(rows.data_ptr())
        diag = reduce_diagnostics(self.engine.stats()["redraw_count"], float(viol.max()),
                                  float(eqv.max()), rows, device=rows.device)
        full = gather_rows(rows, self.z_counts) if gather else None
        return full, diag, bad

    def close(self):
        self.engine.close()
