"""Oracle parity of the TIMED path at BASELINE.json shapes.

The bench's headline kernel is the incremental chord pass
(`chord2_kernel<INCREMENTAL>`: A_I D on DMMA plus the streamed slack cache),
and the int8-slice engine's `chord_i8_kernel`; configs 1-2 run the
walk-resident `small_kernel`.  These tests run those kernels exactly as the
bench / run() do -- several iterates, the first one the refresh pass, the
rest incremental -- and compare every iterate's walks with the CPU oracle's
restatement of the reference step (proj/src/sampler.cpp:235-272), including
the redraw counts and the reprojection cadence (sampler.cpp:304-311,
projection.cpp:53-60):

- reference-stream mode (the reference's own SplitMix streams, bit-exact
  uniforms; oracle.step): configs 3, 4 (with equalities, reprojection every
  5 iterates) and 5 on the DMMA and int8 engines;
- production mode (Philox, the bench's mode; oracle.step_philox draws the
  same Philox4x32-10 values, pinned to the published known-answer vectors in
  test_oracle_kats.py): the bench's own config-5 workload at its full 4096
  walks, checked on walk slices (walks never interact, so a slice of the
  oracle is the oracle), and the small kernel on configs 1-2.

Tolerance: 1e-9 x max|x| per walk after every iterate (north star, fp64),
identical redraw counts.  The only differences are summation order in the
dot products and, in Philox mode, CUDA's vs glibc's log/sincos (an ulp or
two in the normals)."""
import numpy as np
import pytest

import oracle
import paper_2104_07097_b200 as mh
from paper_2104_07097_b200 import workloads

pytestmark = pytest.mark.gpu
RTOL = 1e-9
EPS_DIR = 1e-11
ENGINES = ["dmma", "int8"]


@pytest.fixture(scope="module")
def cfg_cache():
    cache = {}

    def get(idx):
        if idx not in cache:
            cache[idx] = workloads.config(idx)
        return cache[idx]
    return get


@pytest.fixture(scope="module", autouse=True)
def oracle_threads():
    import os
    oracle.lib().orc_set_threads(os.cpu_count() or 1)


def _assert_close(Xg, Xr, what):
    scale = np.maximum(np.abs(Xr).max(axis=0), 1e-12)
    err = (np.abs(Xg - Xr).max(axis=0) / scale).max()
    assert err <= RTOL, f"{what}: max relative walk difference {err:.3e}"
    return err


def _reference_stream_trajectory(w, z, iters, engine, reproject_every=0, seed=31):
    p = w.polytope
    n = p.dim()
    op = mh.compute_projection(p.a_eq) if p.num_equalities() else None
    X0 = np.asfortranarray(np.repeat(w.x0[:, None], z, axis=1))
    rng = oracle.WalkRng(seed, z)
    Xr = X0.copy(order="F")
    worst = 0.0
    with mh.Engine(p, z, seed=seed, projector=op, rng="reference", slack="incremental",
                   refresh_every=1000, f64_engine=engine) as eng:
        eng.set_state(X0)
        red_orc = 0
        for it in range(1, iters + 1):
            eng.step(1, reproject_every)
            st, red, _ = oracle.step(p.a_in, p.b_in, None if op is None else op.p, EPS_DIR, rng,
                                     Xr)
            assert st == 0
            red_orc += red
            if op is not None and reproject_every and it % reproject_every == 0:
                Xr = oracle.reproject(p.a_eq, op.gram_inverse, p.b_eq, Xr)
            worst = max(worst, _assert_close(eng.get_state(), Xr, f"iterate {it}"))
        s = eng.stats()
        assert s["redraw_count"] == red_orc
        # one refresh pass (plus one after each reprojection), every other
        # iterate on the incremental kernel
        assert s["refreshes"] == 1 + (iters // reproject_every if reproject_every else 0)
        bad, viol, eqv = eng.check_state(1e-9)
        assert bad == -1
    return worst


@pytest.mark.parametrize("engine", ENGINES)
def test_reference_streams_config3_full_width(cfg_cache, engine):
    # config 3 at its full 4096 walks, 10 iterates (9 incremental)
    _reference_stream_trajectory(cfg_cache(3), 4096, 10, engine)


@pytest.mark.parametrize("engine", ENGINES)
def test_reference_streams_config4_with_reprojection(cfg_cache, engine):
    # config 4 (m_E = 100, dense P, m_I = 52000) on 1024 walks, 12 iterates,
    # reprojection after iterates 5 and 10 against orc_reproject
    _reference_stream_trajectory(cfg_cache(4), 1024, 12, engine, reproject_every=5)


@pytest.mark.parametrize("engine", ENGINES)
def test_reference_streams_config5(cfg_cache, engine):
    # the config-5 polytope (n = 2000, m_I = 2e5) on 512 walks, 5 iterates
    _reference_stream_trajectory(cfg_cache(5), 512, 5, engine)


def _philox_slices(w, z, iters, engine, slices, seed=2021, **kw):
    """The engine in its production mode over all z walks; the oracle on
    walk slices [a, b) with chain_offset a (walks are independent)."""
    p = w.polytope
    n = p.dim()
    op = mh.compute_projection(p.a_eq) if p.num_equalities() else None
    X0 = np.asfortranarray(np.repeat(w.x0[:, None], z, axis=1))
    refs = {sl: X0[:, sl[0]:sl[1]].copy(order="F") for sl in slices}
    with mh.Engine(p, z, seed=seed, projector=op, f64_engine=engine, **kw) as eng:
        eng.set_state(X0)
        for it in range(iters):
            eng.step(1)
            Xg = eng.get_state()
            for (a, b), Xr in refs.items():
                st, red, _ = oracle.step_philox(p.a_in, p.b_in, None if op is None else op.p,
                                                EPS_DIR, seed, a, it, Xr)
                assert st == 0 and red == 0
                _assert_close(Xg[:, a:b], Xr, f"iterate {it}, walks {a}:{b}")
        s = eng.stats()
        assert s["redraw_count"] == 0
        return s


@pytest.mark.parametrize("engine", ENGINES)
def test_philox_bench_workload_config5(cfg_cache, engine):
    # the bench's own workload: config 5, 4096 walks, Philox, incremental
    # slack with the default refresh cadence; iterate 0 is the refresh pass,
    # 1..4 the timed kernel.  Walks 0..127 and 3968..4095 checked.
    s = _philox_slices(cfg_cache(5), 4096, 5, engine, [(0, 128), (3968, 4096)])
    assert s["refreshes"] == 1


def test_philox_config3_full_width(cfg_cache):
    _philox_slices(cfg_cache(3), 4096, 6, "dmma", [(0, 4096)])


@pytest.mark.parametrize("idx", [1, 2])
def test_small_kernel_against_oracle(cfg_cache, idx):
    # configs 1-2 run every iterate of a batch in one walk-resident launch
    # (small_kernel.cuh); one launch of 40 iterates against 40 oracle steps
    # (config 2 reprojects every 10, sampler.cpp:307-310)
    w = cfg_cache(idx)
    p = w.polytope
    z, iters, seed = w.z, 40, 7
    op = mh.compute_projection(p.a_eq) if p.num_equalities() else None
    reproject = 10 if op is not None else 0
    X0 = np.asfortranarray(np.repeat(w.x0[:, None], z, axis=1))
    Xr = X0.copy(order="F")
    with mh.Engine(p, z, seed=seed, projector=op) as eng:
        eng.set_state(X0)
        eng.step(iters, reproject)
        Xg = eng.get_state()
        launches = eng.stats()["kernel_launches"]
    assert launches < iters  # the walk-resident kernel, not a per-iterate chain
    for it in range(iters):
        st, red, _ = oracle.step_philox(p.a_in, p.b_in, None if op is None else op.p, EPS_DIR,
                                        seed, 0, it, Xr)
        assert st == 0
        if op is not None and (it + 1) % reproject == 0:
            Xr = oracle.reproject(p.a_eq, op.gram_inverse, p.b_eq, Xr)
    _assert_close(Xg, Xr, f"config {idx} after {iters} iterates")


def test_philox_normals_match_the_oracle_draws():
    # the direction batch itself: generate_directions on a Philox context
    # returns the oracle's Philox normals to a few ulps (CUDA vs glibc
    # log/sincos), for odd n and walk ids past 2^32
    n, z, seed, off = 37, 65, 99, (1 << 32) + 5
    p = workloads.random_polytope(n, 200, seed=1)
    with mh.Engine(p, z, seed=seed, chain_offset=off, small_path=False) as eng:
        H0 = eng.generate_directions()
        H1 = eng.generate_directions()
    for it, H in enumerate([H0, H1]):
        ref = np.stack([oracle.philox_normals(seed, off + k, it, 0, n) for k in range(z)], 1)
        np.testing.assert_allclose(H, ref, rtol=4e-15, atol=4e-15)
