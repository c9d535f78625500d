"""GPU parity: the CUDA engine (through the C ABI) against the CPU oracle on
the same seeded inputs.  Tolerances (north star): one iterate with injected
normals H and chord positions U matches the reference step within 1e-9
relative in fp64 -- relative to the chord width for the bounds/theta and to
the walk's max-norm for the moved point; flags are identical.

Reference tests restated are cited per test (proj/tests/...)."""
import math

import numpy as np
import pytest

import oracle
import paper_2104_07097_b200 as mh
from paper_2104_07097_b200 import workloads
from scalar_walk import ScalarWalk

pytestmark = pytest.mark.gpu
RTOL = 1e-9
EPS_DIR = 1e-11


def _interior_points(p: mh.Polytope, z, rng, shrink=0.5):
    """Random interior points: short random walks from x0 = the origin-ish
    center, by pulling random directions back inside."""
    n = p.dim()
    if p.num_equalities() == 0:
        X = rng.uniform(-1, 1, (n, z))
        # scale each column so max(A x) <= shrink * min(b)
        ax = p.a_in @ X
        s = np.max(ax / p.b_in[:, None], axis=0)
        X = X * (shrink / np.maximum(s, 1e-300))
        return np.asfortranarray(X)
    # simplex-like bodies: convex combination of the center and a random point
    c = np.full(n, 1.0 / n)
    w = rng.dirichlet(np.ones(n), z).T
    return np.asfortranarray(shrink * w + (1 - shrink) * c[:, None])


def _compare(p, X, H, U, projector, eng, orc):
    lo, hi, th, fl = eng.step_injected(H, U)
    Xg = eng.get_state()
    P = None if projector is None else projector.p
    st, Xr, lor, hir, thr, flr, err = orc.step_injected(p.a_in, p.b_in, P, EPS_DIR, X, H, U)
    assert st == 0
    np.testing.assert_array_equal(fl, flr)
    ok = (flr & mh.FLAG_DEGENERATE) == 0
    width = np.where(ok, hir - lor, 1.0)
    assert np.all(np.abs(lo - lor)[ok] <= RTOL * width[ok])
    assert np.all(np.abs(hi - hir)[ok] <= RTOL * width[ok])
    assert np.all(np.abs(th - thr)[ok] <= RTOL * width[ok])
    scale = np.maximum(np.abs(Xr).max(axis=0), 1e-12)
    assert np.all(np.abs(Xg - Xr).max(axis=0) <= RTOL * scale)
    return lo, hi, fl


def test_box2_hand_geometry():
    # proj/tests/test_sampler.cpp:93-107 through the engine
    p = mh.make_hypercube(2)
    with mh.Engine(p, 2) as eng:
        iv = eng.lambda_intervals(np.array([[0.0, 0.5], [0.0, 0.0]]),
                                  np.array([[1.0, 1.0], [0.0, 0.0]]))
    assert iv.lower[0] == -1.0 and iv.upper[0] == 1.0
    assert iv.lower[1] == -1.5 and iv.upper[1] == 0.5
    assert list(iv.degenerate) == [0, 0]


def test_all_parallel_flagged_and_unbounded():
    # proj/tests/test_sampler.cpp:128-154
    p = mh.make_hypercube(2)
    with mh.Engine(p, 1, eps_dir=1e9) as eng:
        iv = eng.lambda_intervals(np.zeros((2, 1)), np.array([[1.0], [0.0]]))
        assert iv.degenerate[0] == 1 and iv.lower[0] == 0.0 and iv.upper[0] == 0.0
    quadrant = mh.Polytope(-np.eye(2), np.zeros(2))
    with mh.Engine(quadrant, 3) as eng:
        X = np.ones((2, 3))
        D = np.array([[1.0, 0.3, -1.0], [-1.0, 1.0, 1.0]])
        with pytest.raises(mh.MharError) as e:
            eng.lambda_intervals(X, D)
        assert e.value.code == mh.ErrorCode.unbounded_polytope
        assert "walk 1" in str(e.value)  # the first one-sided walk, as the reference raises


@pytest.mark.parametrize("n,m,z", [(10, 20, 100), (37, 301, 77), (64, 1000, 129), (5, 10, 1)])
def test_injected_step_random_bodies(orc, n, m, z):
    rng = np.random.default_rng(n * 7 + m + z)
    if m == 2 * n:
        p = mh.make_hypercube(n)
    else:
        p = workloads.random_polytope(n, m, seed=n + m)
    X = _interior_points(p, z, rng)
    H = np.asfortranarray(rng.standard_normal((n, z)))
    U = rng.uniform(0, 1, z)
    with mh.Engine(p, z) as eng:
        eng.set_state(X)
        _compare(p, X, H, U, None, eng, orc)


def test_injected_step_simplex_projected(orc):
    # config 2 shape: simplex n = 100, z = 1000, P = I - J/n
    n, z = 100, 1000
    p = mh.make_simplex(n)
    op = mh.compute_projection(p.a_eq)
    rng = np.random.default_rng(2)
    X = _interior_points(p, z, rng)
    H = np.asfortranarray(rng.standard_normal((n, z)))
    H[:, 3] = 1.0  # entirely in the row space: collapses (test_projection.cpp:87-108)
    U = rng.uniform(0, 1, z)
    with mh.Engine(p, z, projector=op) as eng:
        eng.set_state(X)
        lo, hi, fl = _compare(p, X, H, U, op, eng, orc)
    assert fl[3] & mh.FLAG_COLLAPSED and fl[3] & mh.FLAG_DEGENERATE


def test_injected_step_endpoint_and_degenerate_semantics(orc):
    p = mh.make_hypercube(2)
    X = np.zeros((2, 3), order="F")
    H = np.asfortranarray([[1.0, 0.0, 1.0], [0.0, 0.0, 1.0]])
    U = np.array([0.5, 0.3, 0.0])
    with mh.Engine(p, 3) as eng:
        eng.set_state(X)
        _compare(p, X, H, U, None, eng, orc)


@pytest.mark.parametrize("cfg", [3, 4])
def test_injected_step_baseline_shapes(orc, cfg):
    # configs 3 and 4 at full polytope size on a walk subset the oracle
    # finishes in seconds
    w = workloads.config(cfg)
    p = w.polytope
    z = 256 if cfg == 3 else 128
    rng = np.random.default_rng(cfg)
    n = p.dim()
    if p.num_equalities():
        op = mh.compute_projection(p.a_eq)
        X = np.asfortranarray(op.p @ rng.uniform(-0.02, 0.02, (n, z)))
    else:
        op = None
        X = _interior_points(p, z, rng)
    H = np.asfortranarray(rng.standard_normal((n, z)))
    U = rng.uniform(0, 1, z)
    with mh.Engine(p, z, projector=op) as eng:
        eng.set_state(X)
        _compare(p, X, H, U, op, eng, orc)


def test_injected_step_config5_subset(orc):
    # config 5 polytope (n = 2000, m_I = 2e5) on 64 walks
    w = workloads.config(5)
    p = w.polytope
    z = 64
    rng = np.random.default_rng(5)
    X = _interior_points(p, z, rng, shrink=0.3)
    H = np.asfortranarray(rng.standard_normal((2000, z)))
    U = rng.uniform(0, 1, z)
    with mh.Engine(p, z) as eng:
        eng.set_state(X)
        _compare(p, X, H, U, None, eng, orc)


@pytest.mark.parametrize("body", ["box", "simplex"])
def test_reference_streams_z1_match_scalar_walk(orc, body):
    # proj/tests/test_sampler.cpp:413-485: the engine at z = 1 on the
    # reference's SplitMix streams retraces the loop-only scalar walk.
    seed, steps = 4242, 1000
    if body == "box":
        p = mh.make_hypercube(5)
        op, x = None, [0.0] * 5
        walk = ScalarWalk(p.a_in.tolist(), p.b_in.tolist())
    else:
        p = mh.make_simplex(4)
        op = mh.compute_projection(p.a_eq)
        x = [0.25] * 4
        walk = ScalarWalk(p.a_in.tolist(), p.b_in.tolist(), op.p.tolist())
    col, theta = orc.Stream(seed, 0), orc.Stream(seed, oracle.THETA_STREAM_ID)
    worst = 0.0
    with mh.Engine(p, 1, seed=seed, projector=op, rng="reference") as eng:
        eng.set_state(np.array(x)[:, None])
        for it in range(steps):
            eng.step(1)
            assert walk.advance(col, theta, x, EPS_DIR)
            if it % 100 == 99 or it == steps - 1:
                g = eng.get_state()[:, 0]
                worst = max(worst, max(abs(g[j] - x[j]) for j in range(len(x))))
    assert worst <= 1e-12


def test_reference_streams_multi_walk_match_oracle(orc):
    # The full engine on the reference's streams vs the oracle's step()
    # (redraw-free random body): same uniforms bit for bit, so trajectories
    # agree to rounding over 50 iterates (incremental slack included).
    n, m, z, seed = 24, 300, 200, 77
    p = workloads.random_polytope(n, m, seed=3)
    X0 = _interior_points(p, z, np.random.default_rng(1), shrink=0.2)
    Xr = X0.copy(order="F")
    rng = orc.WalkRng(seed, z)
    for mode in ["incremental", "recompute"]:
        with mh.Engine(p, z, seed=seed, rng="reference", slack=mode, refresh_every=16) as eng:
            eng.set_state(X0)
            Xr = X0.copy(order="F")
            rng = orc.WalkRng(seed, z)
            for it in range(50):
                eng.step(1)
                st, red, _ = orc.step(p.a_in, p.b_in, None, EPS_DIR, rng, Xr)
                assert st == 0 and red == 0
            Xg = eng.get_state()
        assert np.abs(Xg - Xr).max() <= 1e-9 * np.abs(Xr).max()


def test_retry_exhausted_after_16_redraws():
    # proj/tests/test_sampler.cpp:244-258
    p = mh.make_hypercube(2)
    for rng in ["reference", "philox"]:
        with mh.Engine(p, 1, seed=55, eps_dir=1e9, rng=rng) as eng:
            eng.set_state(np.zeros((2, 1)))
            with pytest.raises(mh.MharError) as e:
                eng.step(1)
            assert e.value.code == mh.ErrorCode.retry_exhausted
            assert eng.stats()["redraw_count"] == 16


def test_redraw_recovers_and_matches_reference_streams(orc):
    # A walk whose first direction is degenerate (eps_dir between its rates)
    # is redrawn from its own stream; on the reference streams the engine and
    # the oracle pick the same replacement.
    p = mh.make_hypercube(2)
    X0 = np.zeros((2, 4), order="F")
    seed = 9
    # eps just below 1: only directions with some |d_i| > eps qualify, so
    # some first draws are degenerate and get redrawn.
    eps = 0.9
    with mh.Engine(p, 4, seed=seed, eps_dir=eps, rng="reference") as eng:
        eng.set_state(X0)
        eng.step(3)
        Xg = eng.get_state()
        red = eng.stats()["redraw_count"]
    rng = orc.WalkRng(seed, 4)
    Xr = X0.copy(order="F")
    total = 0
    for _ in range(3):
        st, r, _ = orc.step(p.a_in, p.b_in, None, eps, rng, Xr)
        assert st == 0
        total += r
    assert total > 0 and red == total
    assert np.abs(Xg - Xr).max() <= 1e-12


def test_unbounded_body_step_raises():
    quadrant = mh.Polytope(-np.eye(2), np.zeros(2))
    with mh.Engine(quadrant, 8, seed=1) as eng:
        eng.set_state(np.ones((2, 8)))
        with pytest.raises(mh.MharError) as e:
            eng.step(1)
        assert e.value.code == mh.ErrorCode.unbounded_polytope


def test_incremental_matches_recompute():
    # The streamed slack b - A x_t = slack_{t-1} - theta rate_{t-1} differs
    # from a fresh product only by rounding; trajectories agree to 1e-9 over
    # 30 iterates (longer runs separate slowly, as any two summation orders
    # do: chords whose binding rate is tiny amplify ulp differences).
    p = workloads.random_polytope(64, 3000, seed=8)
    X0 = np.zeros((64, 300), order="F")
    out = {}
    for mode in ["incremental", "recompute"]:
        with mh.Engine(p, 300, seed=5, slack=mode, refresh_every=50) as eng:
            eng.set_state(X0)
            eng.step(30)
            out[mode] = eng.get_state()
            bad, viol, _ = eng.check_state(1e-9)
            assert bad == -1
    assert np.abs(out["incremental"] - out["recompute"]).max() <= 1e-9


@pytest.mark.parametrize("n,m,z", [(64, 3000, 300), (200, 5000, 1000), (401, 4000, 300),
                                   (800, 9000, 257), (400, 1000, 1), (420, 1200, 5)])
def test_chord3_equals_chord2(monkeypatch, n, m, z):
    # The two incremental DMMA chord kernels (chord3: 128-walk units with the
    # accumulator handed through TMEM to epilogue warps and an integer
    # log-domain ratio prefilter; chord2: 64-walk units, in-register
    # epilogue) accumulate every rate in the same k order and find the same
    # bounds, so the trajectories are bit-identical, refresh passes included.
    pol = workloads.random_polytope(n, m, seed=n)
    X0 = np.zeros((n, z), order="F")
    out = {}
    for flag in ["0", "1"]:
        monkeypatch.setenv("MHAR_CHORD3", flag)
        with mh.Engine(pol, z, seed=7, refresh_every=8) as eng:
            eng.set_state(X0)
            eng.step(20)
            out[flag] = eng.get_state()
            st = eng.stats()
            assert st["chord_launches"] > 0
            assert st["chord_kernel"] == ("chord3_kernel" if flag == "1" else "chord2_kernel")
            bad, _, _ = eng.check_state(1e-9)
            assert bad == -1
    assert np.array_equal(out["0"], out["1"])
    # default choice: chord3 from n_pad >= 384 on
    monkeypatch.delenv("MHAR_CHORD3")
    with mh.Engine(pol, z, seed=7) as eng:
        assert eng.stats()["chord_kernel"] == ("chord3_kernel" if n >= 384 else "chord2_kernel")


def test_run_box_moments_and_containment(orc):
    # proj/tests/test_sampler.cpp:320-336 + acceptance #4 bounds
    p = mh.make_hypercube(5)
    cfg = mh.SamplerConfig(z=100, phi=125, t_target=10000, seed=11)
    out = mh.run(p, cfg, x0=np.zeros(5))
    S = out.samples
    assert S.shape == (10000, 5) and out.windows == 100 and out.iterate_count == 100 * 125 * 100
    assert np.abs(S.mean(0)).max() <= 0.05
    assert np.abs(S.var(0, ddof=1) - 1 / 3).max() <= 0.05
    assert (S @ p.a_in.T - p.b_in).max() <= 1e-9


def test_run_simplex_moments_and_drift():
    # proj/tests/test_sampler.cpp:338-356, :380-392
    p = mh.make_simplex(3)
    out = mh.run(p, mh.SamplerConfig(z=100, phi=8, t_target=5000, seed=12), x0=np.full(3, 1 / 3))
    assert np.abs(out.samples.mean(0) - 1 / 3).max() <= 0.02
    assert np.abs(out.samples.sum(1) - 1.0).max() <= 1e-8
    p = mh.make_simplex(8)
    out = mh.run(p, mh.SamplerConfig(z=20, phi=50, t_target=500, seed=14), x0=np.full(8, 1 / 8))
    assert np.abs(out.samples.sum(1) - 1.0).max() <= 1e-9
    assert (out.samples @ p.a_in.T - p.b_in).max() <= 1e-8


def test_run_counting_and_reproducibility():
    # proj/tests/test_sampler.cpp:260-302
    p = mh.make_hypercube(3)
    out = mh.run(p, mh.SamplerConfig(z=2, phi=3, t_target=4, burn_in=0, seed=7), x0=np.zeros(3))
    assert out.samples.shape == (4, 3) and out.windows == 2 and out.iterate_count == 12
    out3 = mh.run(p, mh.SamplerConfig(z=2, phi=3, t_target=3, burn_in=0, seed=7), x0=np.zeros(3))
    assert out3.samples.shape == (4, 3)
    p4 = mh.make_hypercube(4)
    a = mh.run(p4, mh.SamplerConfig(z=3, phi=10, t_target=30, seed=99), x0=np.zeros(4)).samples
    b = mh.run(p4, mh.SamplerConfig(z=3, phi=10, t_target=30, seed=99), x0=np.zeros(4)).samples
    c = mh.run(p4, mh.SamplerConfig(z=3, phi=10, t_target=30, seed=100), x0=np.zeros(4)).samples
    assert np.array_equal(a, b) and np.abs(a - c).max() > 0


def test_run_reference_streams_matches_oracle_run(orc):
    # run() on the reference streams vs the oracle's run(): same law, same
    # uniforms; samples agree to rounding (box(4): exact arithmetic rows).
    p = mh.make_hypercube(4)
    kw = dict(z=3, phi=10, t_target=30, burn_in=10, reproject_every=10, seed=99)
    st, Sr, _ = orc.run(p.a_in, p.b_in, np.zeros(4), **kw)
    out = mh.run(p, mh.SamplerConfig(z=3, phi=10, t_target=30, burn_in=10, seed=99),
                 x0=np.zeros(4), rng="reference")
    assert st == 0 and np.abs(out.samples - Sr).max() <= 1e-12


def test_config3_full_width_stays_inside():
    # config 3 at full width: 4096 walks, 30 iterates, exact containment
    w = workloads.config(3)
    with mh.Engine(w.polytope, w.z, seed=3) as eng:
        eng.set_state(np.zeros((500, w.z)))
        eng.step(30)
        bad, viol, _ = eng.check_state(1e-9)
        X = eng.get_state()
    assert bad == -1 and viol.max() <= 1e-9
    # host recheck of a few walks against the raw rows
    ax = w.polytope.a_in @ X[:, :16]
    assert (ax - w.polytope.b_in[:, None]).max() <= 1e-9
    assert np.abs(X).max() > 0.05  # the walks moved


def test_sharding_invariance_global_walk_ids():
    # Philox is keyed on the global walk id: one engine over 192 walks and
    # three shards of 64 (chain_offset 0, 64, 128) produce the same walks --
    # the multi-GPU sample set does not depend on the GPU count.
    p = workloads.random_polytope(40, 900, seed=4)
    z, steps = 192, 12
    with mh.Engine(p, z, seed=21) as eng:
        eng.set_state(np.zeros((40, z)))
        eng.step(steps)
        whole = eng.get_state()
    parts = []
    for off in (0, 64, 128):
        with mh.Engine(p, 64, seed=21, chain_offset=off) as eng:
            eng.set_state(np.zeros((40, 64)))
            eng.step(steps)
            parts.append(eng.get_state())
    assert np.array_equal(whole, np.hstack(parts))


def test_state_rows_to_device_and_gather_layout():
    import torch
    p = mh.make_hypercube(6)
    with mh.Engine(p, 70, seed=3) as eng:
        eng.set_state(np.zeros((6, 70)))
        eng.step(5)
        X = eng.get_state()
        rows = torch.empty((70, 6), dtype=torch.float64, device="cuda:0")
        eng.state_rows_to_device(rows.data_ptr())
    assert np.array_equal(rows.cpu().numpy(), X.T)


@pytest.mark.parametrize("slack,tol", [("recompute", 0.0), ("incremental", 1e-9)])
def test_checkpoint_resume_continues_the_chain(slack, tol):
    # with Philox, X plus the iterate counter is the whole state;
    # 10 iterates == 6 iterates, checkpoint, a fresh context restored, 4 more
    # (bit-exact when the slack is recomputed; the incremental cache is
    # refreshed on restore, so that run agrees to rounding)
    p = workloads.random_polytope(40, 900, seed=12)
    z = 96
    X0 = np.zeros((40, z), order="F")
    with mh.Engine(p, z, seed=77, slack=slack) as eng:
        eng.set_state(X0)
        eng.step(10)
        ref = eng.get_state()
        assert eng.iteration == 10
    with mh.Engine(p, z, seed=77, slack=slack) as eng:
        eng.set_state(X0)
        eng.step(6)
        ck = eng.checkpoint()
    with mh.Engine(p, z, seed=77, slack=slack) as eng:
        eng.restore(ck)
        eng.step(4)
        out = eng.get_state()
    assert np.abs(out - ref).max() <= tol
    with mh.Engine(p, z, seed=77, rng="reference") as eng:
        with pytest.raises(mh.MharError):
            eng.iteration = 3
