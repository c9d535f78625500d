"""The reference's chord semantics (compute_lambda_intervals,
/root/reference/proj/src/sampler.cpp:182-200) on every large-body engine --
the DMMA chord, the int8-slice engine, the fp32 variant and the stacked-
diagonal fast path -- not only on the walk-resident small kernel:

- a walk whose rows all bound one side raises UNBOUNDED_POLYTOPE naming the
  first such walk (proj/tests/test_sampler.cpp:128-154);
- rows with |a d| <= eps_dir are skipped, and a walk with no row left is
  flagged degenerate with lo = hi = 0, like the oracle."""
import numpy as np
import pytest

import paper_2104_07097_b200 as mh

pytestmark = pytest.mark.gpu

ENGINES = [dict(), dict(f64_engine="int8"), dict(precision=32)]
IDS = ["dmma", "int8", "fp32"]


def _one_sided_body(n=300, m=1000, seed=4):
    # A = -|G|: every row has a d < 0 for an all-positive direction
    g = np.random.default_rng(seed).standard_normal((m, n))
    return mh.Polytope(np.asfortranarray(-np.abs(g)), np.ones(m))


@pytest.mark.parametrize("kw", ENGINES, ids=IDS)
def test_unbounded_walk_raises_on_large_bodies(kw):
    p = _one_sided_body()
    n, z = p.dim(), 300
    rng = np.random.default_rng(1)
    H = np.asfortranarray(rng.standard_normal((n, z)))
    H[:, 7] = 1.0   # only lower bounds: unbounded
    H[:, 40] = 1.0  # a later one: the first is reported
    with mh.Engine(p, z, **kw) as eng:
        eng.set_state(np.zeros((n, z)))
        with pytest.raises(mh.MharError) as e:
            eng.step_injected(H, rng.uniform(0, 1, z))
    assert e.value.code == mh.ErrorCode.unbounded_polytope
    assert "walk 7" in str(e.value)


def test_unbounded_walk_raises_on_the_diagonal_fast_path():
    n, z = 300, 200  # x >= 0: stacked-diagonal body beyond the walk-resident kernel
    quadrant = mh.Polytope(-np.eye(n), np.zeros(n))
    rng = np.random.default_rng(2)
    H = np.asfortranarray(rng.standard_normal((n, z)))
    H[:, 11] = np.abs(H[:, 11])
    with mh.Engine(quadrant, z) as eng:
        eng.set_state(np.ones((n, z)))
        with pytest.raises(mh.MharError) as e:
            eng.step_injected(H, rng.uniform(0, 1, z))
    assert e.value.code == mh.ErrorCode.unbounded_polytope
    assert "walk 11" in str(e.value)


@pytest.mark.parametrize("kw", ENGINES, ids=IDS)
def test_all_rows_skipped_is_degenerate(orc, kw):
    from paper_2104_07097_b200 import workloads
    p = workloads.random_polytope(200, 3000, seed=3)
    n, z = p.dim(), 256
    rng = np.random.default_rng(3)
    H = np.asfortranarray(rng.standard_normal((n, z)))
    H[:, 5] *= 1e-30  # every |a d| below eps_dir for this walk only
    U = rng.uniform(0, 1, z)
    X = np.zeros((n, z), order="F")
    with mh.Engine(p, z, eps_dir=1e-20, **kw) as eng:
        eng.set_state(X)
        lo, hi, th, fl = eng.step_injected(H, U)
        Xg = eng.get_state()
    st, Xr, lor, hir, thr, flr, _ = orc.step_injected(p.a_in, p.b_in, None, 1e-20, X, H, U)
    assert st == 0
    np.testing.assert_array_equal(fl, flr)
    assert fl[5] & mh.FLAG_DEGENERATE and lo[5] == 0.0 and hi[5] == 0.0
    assert np.all(Xg[:, 5] == 0.0)  # a degenerate walk stays put
    ok = (flr & mh.FLAG_DEGENERATE) == 0
    assert ok.sum() == z - 1
    if kw.get("precision", 64) == 32:
        return  # fp32 bounds (margin, rounded body): tests/test_gpu_fp32.py
    tol = 1e-9
    w = hir - lor
    assert np.all(np.abs(lo - lor)[ok] <= tol * w[ok])
    assert np.all(np.abs(hi - hir)[ok] <= tol * w[ok])


def _quadrant_path(slack, **kw):
    # Half the directions are one-sided on the quadrant {x >= 0}
    # (UNBOUNDED), so errors are frequent; after each, the caller hands back
    # the unchanged state, as the reference's loop would (WalkState is
    # untouched on a throw, sampler.cpp:235-272).
    n, z = 2, 1
    quadrant = mh.Polytope(-np.eye(n), np.zeros(n))
    errors = 0
    with mh.Engine(quadrant, z, seed=17, slack=slack, refresh_every=1000, small_path=False,
                   **kw) as eng:
        x = np.ones((n, z))
        eng.set_state(x)
        traj = []
        for _ in range(60):
            try:
                eng.step(1)
            except mh.MharError as e:
                assert e.code == mh.ErrorCode.unbounded_polytope
                errors += 1
                eng.set_state(x)
            x = eng.get_state()
            assert x.min() >= -1e-12  # inside the quadrant
            traj.append(x.copy())
    assert 5 < errors < 55
    return np.array(traj)


@pytest.mark.parametrize("kw", [dict(), dict(f64_engine="int8")], ids=["dmma", "int8"])
def test_caught_error_then_same_state_refreshes_the_slack_cache(kw):
    # A failed iterate has already written the chord kernel's S_t / R_t while
    # theta and X stayed at t-1: the incremental cache must not be reused
    # when the same state comes back.  The incremental run equals
    # the fresh-product (recompute) run.
    ref = _quadrant_path("recompute")
    got = _quadrant_path("incremental", **kw)
    np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-12)


def _quadrant3_path(slack):
    # the quadrant with a redundant third row (m % n != 0: not the diagonal
    # fast path, so the incremental DMMA chord kernels run); one-sided
    # directions (UNBOUNDED) are frequent and the caller hands back the
    # unchanged state after each
    quadrant = mh.Polytope(np.array([[-1.0, 0.0], [0.0, -1.0], [-1.0, -1.0]]), np.zeros(3))
    errors = 0
    with mh.Engine(quadrant, 1, seed=23, slack=slack, refresh_every=1000,
                   small_path=False) as eng:
        x = np.ones((2, 1))
        eng.set_state(x)
        traj = []
        for _ in range(60):
            try:
                eng.step(1)
            except mh.MharError as e:
                assert e.code == mh.ErrorCode.unbounded_polytope
                assert "walk 0" in str(e)
                errors += 1
                eng.set_state(x)
            x = eng.get_state()
            assert x.min() >= -1e-12
            traj.append(x.copy())
        kernel = eng.stats()["chord_kernel"]
    assert 5 < errors < 55
    return np.array(traj), kernel


@pytest.mark.parametrize("chord3", ["0", "1"])
def test_unbounded_and_cache_reset_on_both_dmma_chord_kernels(monkeypatch, chord3):
    # one-sided walks raise UNBOUNDED from the incremental kernels' side bits
    # (chord2's fp64 scan, chord3's integer-key scan), and the slack cache is
    # rebuilt after every caught error: equal to the recompute path
    monkeypatch.setenv("MHAR_CHORD3", chord3)
    got, kernel = _quadrant3_path("incremental")
    assert kernel == ("chord3_kernel" if chord3 == "1" else "chord2_kernel")
    ref, _ = _quadrant3_path("recompute")
    np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-12)
