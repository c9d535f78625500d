"""Several devices behind the C ABI (mhar_group_*, csrc/group.cu): one host
process, one thread and stream per device, walks sharded by global id, the
collection windows gathered to devices[0].

A test box has one GPU, so the multi-device logic runs with a device listed
several times (every shard a separate context on GPU 0, the peer-copy
gather) and the NCCL gather / all-reduce at world size 1
(MHAR_GROUP_NCCL=1).  The bar: bit-identical to one context over all walks
-- the sample set of the reference's run() (sampler.cpp:274-335) does not
depend on how the walks are placed."""
import numpy as np
import pytest

import paper_2104_07097_b200 as mh
from paper_2104_07097_b200 import workloads

pytestmark = pytest.mark.gpu


def _single(p, z, seed, steps, op=None, reproject=0, **kw):
    with mh.Engine(p, z, seed=seed, projector=op, **kw) as eng:
        eng.set_state(np.zeros((p.dim(), z)) if op is None else
                      np.repeat(np.full((p.dim(), 1), 1.0 / p.dim()), z, 1))
        eng.step(steps, reproject)
        return eng.get_state()


@pytest.mark.parametrize("gather", ["direct", "copy"])
def test_group_window_gather_modes(monkeypatch, gather):
    # DIRECT (default where every device reaches devices[0]): each shard's
    # check + unpack kernel stores its rows into the root's window buffer;
    # COPY: staged rows and copy-engine peer copies -- the same samples
    monkeypatch.setenv("MHAR_GROUP_GATHER", gather)
    p = workloads.random_polytope(36, 700, seed=12)
    z, seed = 222, 6
    x0 = np.zeros(36)
    with mh.Engine(p, z, seed=seed) as eng:
        ref, rst = eng.run(x0, phi=5, windows=4)
    with mh.Group(p, z, [0, 0, 0], seed=seed) as g:
        assert g.info()["gather"] == gather
        got, st = g.run(x0, phi=5, windows=4)
        info = g.info()
    assert np.array_equal(got, ref)
    assert info["last_redraws"] == rst.redraw_count
    assert info["last_max_violation"] <= 1e-9


@pytest.mark.parametrize("devices", [[0], [0, 0], [0, 0, 0]])
def test_group_step_equals_one_context(devices):
    p = workloads.random_polytope(40, 900, seed=4)
    z, seed = 301, 21  # ragged shards: 301 = 151 + 150, 101 + 100 + 100
    ref = _single(p, z, seed, 12)
    with mh.Group(p, z, devices, seed=seed) as g:
        info = g.info()
        assert info["ndev"] == len(devices) and sum(info["z"]) == z
        assert info["offset"][0] == 0 and not info["uses_nccl"]
        g.set_state(np.zeros((40, z)))
        g.step(12)
        got = g.get_state()
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("devices", [[0, 0], [0, 0, 0, 0]])
def test_group_run_equals_one_context_with_equalities(devices):
    # simplex with a collapsing-free projected walk and the reprojection
    # cadence; samples in global walk order, every window
    p = mh.make_simplex(30)
    op = mh.compute_projection(p.a_eq)
    z, seed = 203, 8
    x0 = np.full(30, 1.0 / 30)
    with mh.Engine(p, z, seed=seed, projector=op) as eng:
        ref, rst = eng.run(x0, phi=7, windows=5, burn_in=10, reproject_every=7)
    with mh.Group(p, z, devices, seed=seed, projector=op) as g:
        got, st = g.run(x0, phi=7, windows=5, burn_in=10, reproject_every=7)
        info = g.info()
    assert np.array_equal(got, ref)
    assert st.iterate_count == rst.iterate_count == z * 7 * 5
    assert st.redraw_count == rst.redraw_count
    assert info["last_max_violation"] <= 1e-9


def test_group_run_large_body_multikernel_path():
    # the tensor-core chord path (incremental slack, refresh cadence) per shard
    p = workloads.random_polytope(300, 6000, seed=5)
    z, seed = 512, 3
    x0 = np.zeros(300)
    with mh.Engine(p, z, seed=seed, refresh_every=16) as eng:
        ref, _ = eng.run(x0, phi=20, windows=3)
    with mh.Group(p, z, [0, 0], seed=seed, refresh_every=16) as g:
        got, st = g.run(x0, phi=20, windows=3)
        assert g.context_stats(0)["chord_launches"] > 0
    assert np.array_equal(got, ref)


def test_group_run_chord3_shards():
    # n_pad >= 384: every shard runs chord3_kernel (128-walk units, ragged
    # shard sizes 151 + 150 pad to 256 each)
    p = workloads.random_polytope(400, 3000, seed=6)
    z, seed = 301, 9
    x0 = np.zeros(400)
    with mh.Engine(p, z, seed=seed, refresh_every=8) as eng:
        assert eng.stats()["chord_kernel"] == "chord3_kernel"
        ref, _ = eng.run(x0, phi=6, windows=3)
    with mh.Group(p, z, [0, 0], seed=seed, refresh_every=8) as g:
        got, _ = g.run(x0, phi=6, windows=3)
        assert g.context_stats(1)["chord_kernel"] == "chord3_kernel"
    assert np.array_equal(got, ref)


def test_group_kernel_choice_follows_the_whole_run():
    # simplex n = 1000: 2000 walks take the kernel chain, a 1000-walk shard
    # alone would take the walk-resident kernel (mhar_options.z_plan): the
    # group's shards plan for the run's 2000 walks, so the samples equal one
    # context's bit for bit
    n, z, seed = 1000, 2000, 5
    p = mh.make_simplex(n)
    op = mh.compute_projection(p.a_eq)
    x0 = np.full(n, 1.0 / n)
    with mh.Engine(p, z, seed=seed, projector=op) as eng:
        assert eng.stats()["chord_kernel"] == "diag_chord_kernel"
        ref, _ = eng.run(x0, phi=4, windows=2, reproject_every=3)
    with mh.Engine(p, z // 2, seed=seed, projector=op) as half:
        assert half.stats()["chord_kernel"] == "small_kernel"  # what a shard would pick alone
    with mh.Group(p, z, [0, 0], seed=seed, projector=op) as g:
        assert g.context_stats(0)["chord_kernel"] == "diag_chord_kernel"
        got, _ = g.run(x0, phi=4, windows=2, reproject_every=3)
    assert np.array_equal(got, ref)


def test_group_nccl_gather_at_world_one(monkeypatch):
    # the NCCL path (grouped send/recv gather + all-reduce of diagnostics)
    # through real NCCL on the one GPU
    monkeypatch.setenv("MHAR_GROUP_NCCL", "1")
    p = workloads.random_polytope(24, 400, seed=9)
    z, seed = 130, 4
    x0 = np.zeros(24)
    with mh.Engine(p, z, seed=seed) as eng:
        ref, rst = eng.run(x0, phi=9, windows=4)
    with mh.Group(p, z, [0], seed=seed) as g:
        assert g.info()["uses_nccl"]
        got, st = g.run(x0, phi=9, windows=4)
        info = g.info()
    assert np.array_equal(got, ref)
    assert info["last_redraws"] == rst.redraw_count
    assert info["last_max_violation"] <= 1e-9


def test_group_errors():
    p = workloads.random_polytope(10, 60, seed=1)
    with pytest.raises(mh.MharError) as e:
        mh.Group(p, 64, [0, 0], rng="reference")
    assert e.value.code == mh.ErrorCode.invalid_argument
    with pytest.raises(mh.MharError) as e:
        mh.Group(p, 1, [0, 0])
    assert e.value.code == mh.ErrorCode.invalid_argument
    with pytest.raises(mh.MharError):
        mh.Group(p, 64, [0, 999])
    # a device-side failure on a shard surfaces with the walk's global id
    quadrant = mh.Polytope(-np.eye(2), np.zeros(2))
    with mh.Group(quadrant, 40, [0, 0], seed=1, small_path=False) as g:
        g.set_state(np.ones((2, 40)))
        with pytest.raises(mh.MharError) as e:
            g.step(1)
    assert e.value.code == mh.ErrorCode.unbounded_polytope
    with mh.Engine(quadrant, 40, seed=1, small_path=False) as eng:
        eng.set_state(np.ones((2, 40)))
        with pytest.raises(mh.MharError) as e1:
            eng.step(1)
    assert str(e.value) == str(e1.value)


def test_group_state_round_trip_and_no_collection():
    p = workloads.random_polytope(30, 500, seed=2)
    z = 97
    X = np.asfortranarray(np.random.default_rng(0).uniform(-0.01, 0.01, (30, z)))
    with mh.Group(p, z, [0, 0, 0], seed=3) as g:
        g.set_state(X)
        assert np.array_equal(g.get_state(), X)
        S, st = g.run(np.zeros(30), phi=5, windows=2, collect=False)
        assert S is None and st.iterate_count == z * 5 * 2
        with pytest.raises(mh.MharError) as e:
            g.set_state(np.zeros((30, z + 1)))
        assert e.value.code == mh.ErrorCode.dimension_mismatch
        with pytest.raises(mh.MharError):
            g.run(np.zeros(29), phi=5, windows=1)


def test_group_reference_streams_single_device():
    # one device may keep the reference's own streams (bit-exact uniforms):
    # the group over [0] equals a context on the same streams
    p = mh.make_hypercube(4)
    with mh.Engine(p, 3, seed=99, rng="reference") as eng:
        ref, _ = eng.run(np.zeros(4), phi=10, windows=3, burn_in=10)
    with mh.Group(p, 3, [0], seed=99, rng="reference") as g:
        got, _ = g.run(np.zeros(4), phi=10, windows=3, burn_in=10)
    assert np.array_equal(got, ref)
