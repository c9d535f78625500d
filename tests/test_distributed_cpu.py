"""Multi-rank host logic on CPU (gloo, world_size 2): walk sharding, the
rank-0 sample gather in global walk order, diagnostics reduction and the
max-over-ranks timer -- the collectives the GPU path runs over NCCL."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2104_07097_b200.distributed import first_failure, gather_rows, max_over_ranks, \
    reduce_diagnostics, shard_walks


def test_shard_walks_cover_exactly():
    for z, w in [(32768, 8), (4096, 1), (10, 3), (7, 7), (100, 4)]:
        spans = [shard_walks(z, w, r) for r in range(w)]
        assert sum(s[0] for s in spans) == z
        off = 0
        for zl, o in spans:
            assert o == off
            off += zl
    with pytest.raises(ValueError):
        shard_walks(2, 3, 0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, z_total, n, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        z, off = shard_walks(z_total, world, rank)
        counts = [shard_walks(z_total, world, r)[0] for r in range(world)]
        # each walk's row is its global id repeated: the gather must restore order
        rows = torch.arange(off, off + z, dtype=torch.float64)[:, None].repeat(1, n)
        full = gather_rows(rows, counts)
        diag = reduce_diagnostics(redraws=rank + 1, max_violation=-1.0 - rank, max_eq=rank * 1e-12,
                                  rows=rows)
        t = max_over_ranks(1.5 + rank)
        # containment failure: rank 1's local walk 2 is the only one outside
        bad = first_failure(2 if rank == 1 else -1, off)
        none = first_failure(-1, off)
        q.put((rank, None if full is None else full.numpy(), diag.redraws, diag.max_violation,
               diag.max_eq_residual, diag.count, diag.coord_sum.tolist(), t, bad, none, off))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("z_total", [10, 7])
def test_gather_and_reduce_world2(z_total):
    world, n = 2, 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, z_total, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r = q.get(timeout=120)
        res[r[0]] = r
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    full = res[0][1]
    assert full.shape == (z_total, n)
    assert np.array_equal(full[:, 0], np.arange(z_total))
    assert res[1][1] is None
    for r in range(world):
        _, _, red, mv, meq, cnt, csum, t, bad, none, _ = res[r]
        assert red == 3 and mv == -1.0 and meq == 1e-12 and cnt == z_total
        assert csum[0] == sum(range(z_total))
        assert t == 2.5
        # every rank learns the global id of the failing walk (sampler.cpp:319-324)
        assert bad == res[1][10] + 2 and none == -1
