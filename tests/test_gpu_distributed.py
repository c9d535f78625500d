"""The multi-GPU plumbing through real NCCL on the one GPU a test box has:
a world-size-1 process group runs the same collectives (gather of the
collected rows to rank 0 device to device, the containment-failure min, all_reduce of the diagnostics, max of the
timers) the N-GPU bench runs, on rows the engine writes straight into device
memory.  The multi-rank logic itself is covered on gloo
(tests/test_distributed_cpu.py)."""
import socket

import numpy as np
import pytest

import paper_2104_07097_b200 as mh
from paper_2104_07097_b200 import workloads
from paper_2104_07097_b200.distributed import ShardedSampler, max_over_ranks

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_nccl_window_gather_matches_the_engine():
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_port()}", rank=0,
                            world_size=1)
    try:
        p = workloads.random_polytope(40, 400, seed=6)
        z = 300
        sh = ShardedSampler(p, z, seed=5)
        sh.set_start(np.zeros(40))
        full, diag = sh.window(12)
        assert diag.count == z and diag.max_violation <= 1e-9
        got = full.cpu().numpy()
        sh.close()
        with mh.Engine(p, z, seed=5) as eng:
            eng.set_state(np.zeros((40, z)))
            eng.step(12)
            ref = eng.get_state().T
        np.testing.assert_array_equal(got, ref)
        np.testing.assert_allclose(diag.coord_sum, ref.sum(0), rtol=1e-12, atol=1e-12)
        assert max_over_ranks(3.5, device="cuda") == 3.5
    finally:
        dist.destroy_process_group()
