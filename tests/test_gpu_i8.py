"""The int8-slice fp64 engine (f64_engine="int8", csrc/chord_i8.cuh): the
rates A_I d formed exactly from 53-bit fixed-point operands split into int8
slices on the tcgen05 int8 tensor cores (Ozaki scheme).

The bar is the fp64 one (north star): one iterate with injected normals H and
chord positions U matches the reference step within 1e-9 relative -- the
engine's rates are those of the direction rounded to 53 bits relative to the
walk's largest coordinate, and of A_I rounded to 53 bits relative to each
row's largest entry, so the chord differs from the exact fp64 one by a few
ulps.  A tighter check pins that: the bounds agree with the DMMA engine's to
1e-12 of the chord width."""
import numpy as np
import pytest

import paper_2104_07097_b200 as mh
from paper_2104_07097_b200 import workloads

pytestmark = pytest.mark.gpu
RTOL = 1e-9
EPS_DIR = 1e-11


def _interior(p, z, rng, shrink=0.5):
    X = rng.uniform(-1, 1, (p.dim(), z))
    s = np.max((p.a_in @ X) / p.b_in[:, None], axis=0)
    return np.asfortranarray(X * (shrink / s))


def _compare(p, X, H, U, eng, orc):
    lo, hi, th, fl = eng.step_injected(H, U)
    Xg = eng.get_state()
    st, Xr, lor, hir, thr, flr, _ = orc.step_injected(p.a_in, p.b_in, None, EPS_DIR, X, H, U)
    assert st == 0
    np.testing.assert_array_equal(fl, flr)
    ok = (flr & mh.FLAG_DEGENERATE) == 0
    w = np.where(ok, hir - lor, 1.0)
    assert np.all(np.abs(lo - lor)[ok] <= RTOL * w[ok])
    assert np.all(np.abs(hi - hir)[ok] <= RTOL * w[ok])
    assert np.all(np.abs(th - thr)[ok] <= RTOL * w[ok])
    scale = np.maximum(np.abs(Xr).max(axis=0), 1e-12)
    assert np.all(np.abs(Xg - Xr).max(axis=0) <= RTOL * scale)
    return lo, hi, th


@pytest.mark.parametrize("n,m,z", [(10, 20, 100), (37, 301, 77), (64, 1000, 300), (5, 10, 1),
                                   (129, 4000, 256)])
def test_i8_injected_step_parity(orc, n, m, z):
    rng = np.random.default_rng(n * 13 + m + z)
    p = mh.make_hypercube(n) if m == 2 * n else workloads.random_polytope(n, m, seed=n + m)
    X = _interior(p, z, rng)
    H = np.asfortranarray(rng.standard_normal((n, z)))
    U = rng.uniform(0, 1, z)
    with mh.Engine(p, z, f64_engine="int8") as eng:
        eng.set_state(X)
        _compare(p, X, H, U, eng, orc)


def test_i8_injected_step_config3(orc):
    # config 3 at full polytope size (n = 500, m_I = 20000) on 256 walks
    p = workloads.config(3).polytope
    z = 256
    rng = np.random.default_rng(33)
    X = _interior(p, z, rng)
    H = np.asfortranarray(rng.standard_normal((p.dim(), z)))
    U = rng.uniform(0, 1, z)
    with mh.Engine(p, z, f64_engine="int8") as eng:
        eng.set_state(X)
        _compare(p, X, H, U, eng, orc)


def test_i8_injected_step_config5_subset(orc):
    # the headline polytope (n = 2000, m_I = 2e5) on 64 walks
    p = workloads.config(5).polytope
    z = 64
    rng = np.random.default_rng(55)
    X = _interior(p, z, rng, shrink=0.3)
    H = np.asfortranarray(rng.standard_normal((p.dim(), z)))
    U = rng.uniform(0, 1, z)
    with mh.Engine(p, z, f64_engine="int8") as eng:
        eng.set_state(X)
        _compare(p, X, H, U, eng, orc)


@pytest.mark.parametrize("scale,eps", [(1.0, 1e-11), (1e-100, 1e-300), (1e150, 1e-11)])
def test_i8_bounds_match_dmma_to_a_few_ulps(scale, eps):
    # fp64-grade: the slice products agree with the fp64 tensor-core product
    # to 1e-12 of the chord width, on badly scaled rows and directions too
    n, m, z = 96, 2500, 256
    rng = np.random.default_rng(7)
    p = workloads.random_polytope(n, m, seed=11)
    rs = 10.0 ** rng.uniform(-6, 6, m)  # rows over 12 decades (same body)
    p = mh.Polytope(np.asfortranarray(p.a_in * rs[:, None]), p.b_in * rs)
    X = _interior(p, z, rng)
    H = np.asfortranarray(rng.standard_normal((n, z)) * 10.0 ** rng.uniform(-3, 3, (n, 1)) * scale)
    U = rng.uniform(0, 1, z)
    out = {}
    for eng_name in ["dmma", "int8"]:
        with mh.Engine(p, z, f64_engine=eng_name, eps_dir=eps) as eng:
            eng.set_state(X)
            out[eng_name] = eng.step_injected(H, U)[:2]
    (lo_d, hi_d), (lo_i, hi_i) = out["dmma"], out["int8"]
    w = hi_d - lo_d
    assert np.all(w > 0)
    assert np.abs(lo_i - lo_d).max() <= 1e-12 * w.max()
    assert np.all(np.abs(lo_i - lo_d) <= 1e-12 * w)
    assert np.all(np.abs(hi_i - hi_d) <= 1e-12 * w)


def test_i8_trajectory_tracks_dmma_and_stays_inside():
    # incremental iterates: same seed, same uniforms; the int8 engine moves
    # along the 53-bit-rounded direction, so trajectories agree to rounding
    p = workloads.random_polytope(200, 6000, seed=21)
    z = 512
    X0 = np.zeros((200, z), order="F")
    out = {}
    for eng_name in ["dmma", "int8"]:
        with mh.Engine(p, z, seed=9, f64_engine=eng_name, refresh_every=16) as eng:
            eng.set_state(X0)
            eng.step(40)
            bad, viol, _ = eng.check_state(1e-9)
            assert bad == -1 and viol.max() <= 1e-9
            out[eng_name] = eng.get_state()
    assert np.abs(out["int8"]).max() > 0.1
    assert np.abs(out["int8"] - out["dmma"]).max() <= 1e-8


def test_i8_run_box_moments():
    # uniform on [-1, 1]^12: mean 0, variance 1/3 (proj/tests/test_sampler.cpp:320-336)
    p = mh.make_hypercube(12)
    with mh.Engine(p, 512, seed=5, f64_engine="int8") as eng:
        S, st = eng.run(np.zeros(12), phi=40, windows=20, burn_in=100)
    assert S.shape == (20 * 512, 12)
    assert (S @ p.a_in.T - p.b_in).max() <= 1e-9
    assert np.abs(S.mean(0)).max() <= 0.03
    assert np.abs(S.var(0) - 1.0 / 3.0).max() <= 0.03


def test_i8_dimension_limit():
    p = workloads.random_polytope(4700, 4, seed=1)
    with pytest.raises(mh.MharError) as e:
        mh.Engine(p, 8, f64_engine="int8")
    assert e.value.code == mh.ErrorCode.invalid_argument


def test_contexts_alive_together_do_not_interfere():
    # regression: ctx_create uploaded A_I with a legacy-stream cudaMemcpy whose
    # DMA could still be landing when the packing kernel ran on the context's
    # non-blocking stream -- with two contexts alive the first iterate's bounds
    # changed from run to run.  Every combination must give one outcome.
    p = workloads.random_polytope(200, 6000, seed=21)
    z = 512
    X0 = np.zeros((200, z), order="F")
    seen = set()
    for combo in [("dmma",), ("dmma", "int8"), ("int8", "int8"), ("dmma", "dmma")]:
        for _ in range(2):
            engs = [mh.Engine(p, z, seed=9, f64_engine=e) for e in combo]
            for e in engs:
                e.set_state(X0)
                e.step(1)
                _, lo, hi, _ = e.debug_last_iterate()
                seen.add((lo.tobytes() if e.f64_engine == "dmma" else None, hi.sum()))
            for e in engs:
                e.close()
    his = {round(h, 9) for _, h in seen}
    los = {l for l, _ in seen if l is not None}
    assert len(his) == 1 and len(los) == 1


def test_i8_injected_step_with_equalities(orc):
    # config 4 shape (n = 1000, m_I = 52000 with the box rows, m_E = 100):
    # D = P H is projected, then quantised; one step vs the oracle at 1e-9
    from paper_2104_07097_b200 import workloads as wl
    w = wl.config(4)
    p = w.polytope
    z = 128
    rng = np.random.default_rng(44)
    op = mh.compute_projection(p.a_eq)
    X = np.asfortranarray(op.p @ rng.uniform(-0.02, 0.02, (p.dim(), z)))
    H = np.asfortranarray(rng.standard_normal((p.dim(), z)))
    U = rng.uniform(0, 1, z)
    with mh.Engine(p, z, projector=op, f64_engine="int8") as eng:
        eng.set_state(X)
        lo, hi, th, fl = eng.step_injected(H, U)
        Xg = eng.get_state()
    st, Xr, lor, hir, thr, flr, _ = orc.step_injected(p.a_in, p.b_in, op.p, EPS_DIR, X, H, U)
    assert st == 0
    np.testing.assert_array_equal(fl, flr)
    ok = (flr & mh.FLAG_DEGENERATE) == 0
    w_ = np.where(ok, hir - lor, 1.0)
    assert np.all(np.abs(lo - lor)[ok] <= RTOL * w_[ok])
    assert np.all(np.abs(hi - hir)[ok] <= RTOL * w_[ok])
    assert np.abs(Xg - Xr).max() <= RTOL * np.abs(Xr).max()


def test_i8_run_simplex_moments_and_drift():
    # simplex(6) with the equality sum x = 1: reprojection cadence, moments
    p = mh.make_simplex(6)
    op = mh.compute_projection(p.a_eq)
    with mh.Engine(p, 256, seed=21, projector=op, f64_engine="int8") as eng:
        S, st = eng.run(np.full(6, 1.0 / 6), phi=30, windows=20, burn_in=60, reproject_every=30)
    assert np.abs(S.sum(1) - 1.0).max() <= 1e-9
    assert (S @ p.a_in.T - p.b_in).max() <= 1e-9
    assert np.abs(S.mean(0) - 1.0 / 6).max() <= 0.02


def test_i8_redraw_keeps_the_rate_cache_consistent():
    # eps_dir 0.6 on box(8): directions with every |d_i| <= 0.6 are degenerate
    # and redrawn from the walk's own stream; the redrawn walk's rates go into
    # the tile-layout fp64 cache.  The incremental int8 engine must follow the
    # DMMA engine that recomputes the slack every iterate (with eps this large
    # walks may leave the box -- the reference skips rows with |a d| <= eps --
    # so the check is trajectory agreement, over a few iterates).
    p = mh.make_hypercube(8)
    out = {}
    for name, kw in [("int8", dict(f64_engine="int8", refresh_every=1000)),
                     ("dmma", dict(slack="recompute"))]:
        with mh.Engine(p, 256, seed=3, eps_dir=0.6, **kw) as eng:
            eng.set_state(np.zeros((8, 256)))
            eng.step(4)
            out[name] = (eng.get_state(), eng.stats()["redraw_count"])
    assert out["int8"][1] > 0 and out["int8"][1] == out["dmma"][1]
    assert np.abs(out["int8"][0] - out["dmma"][0]).max() <= 1e-9


def test_i8_uniformity_screening_against_direct_draws():
    # acceptance #3's screen (proj/tests/acceptance_main.cpp:160-203) on the
    # int8 engine: box(8) samples vs direct uniform draws, 10 seeds, at least
    # 9 runs with Friedman-Rafsky z >= -1.64
    from paper_2104_07097_b200 import stats
    n = 8
    p = mh.make_hypercube(n)
    ok = 0
    for rep in range(10):
        with mh.Engine(p, 256, seed=500 + rep, f64_engine="int8") as eng:
            S, _ = eng.run(np.zeros(n), phi=64, windows=8, burn_in=64)
        S = S[:2000]
        ref = stats.sample_uniform_hypercube(np.random.default_rng(rep), n, 2000)
        if stats.friedman_rafsky(S, ref).z_value >= stats.kUniformityZThreshold:
            ok += 1
    assert ok >= 9, f"{ok}/10"


def test_env_switch_selects_the_int8_engine(monkeypatch):
    # MHAR_F64_ENGINE=int8: every eligible fp64 context uses the int8 engine
    # (the C++ drop-in needs no code change); walk tiles of the tcgen05 pair
    # pad z to 256 instead of 64
    p = workloads.random_polytope(50, 600, seed=2)
    with mh.Engine(p, 100) as eng:
        assert eng.stats()["z_padded"] == 128
    monkeypatch.setenv("MHAR_F64_ENGINE", "int8")
    with mh.Engine(p, 100) as eng:
        assert eng.stats()["z_padded"] == 256
        assert eng.stats()["chord_kernel"] == "chord_i8_kernel"
        eng.set_state(np.zeros((50, 100)))
        eng.step(5)
        assert eng.check_state(1e-9)[0] == -1
    big = workloads.random_polytope(4700, 4, seed=1)  # beyond n <= 4608: stays on DMMA
    with mh.Engine(big, 8) as eng:
        assert eng.stats()["z_padded"] == 128  # chord3's 128-walk units (n_pad >= 384)
