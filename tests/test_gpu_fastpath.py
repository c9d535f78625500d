"""Structure-aware paths (csrc/fastpath.cuh) for the paper's own bodies at
sizes beyond the walk-resident kernel:

- stacked diagonal blocks (the reference's own fast path,
  proj/src/sampler.cpp:47-71, :166-172): bounds bit-identical to the
  general DMMA product, and to the oracle;
- the factored projection D = H - A_E' G A_E H for small m_E: equal to the
  dense P H to rounding (the 1e-9 parity bar)."""
import os

import numpy as np
import pytest

import paper_2104_07097_b200 as mh

pytestmark = pytest.mark.gpu
EPS_DIR = 1e-11


def _engine(*args, fastpath=True, **kw):
    old = os.environ.pop("MHAR_NO_FASTPATH", None)
    if not fastpath:
        os.environ["MHAR_NO_FASTPATH"] = "1"
    try:
        return mh.Engine(*args, **kw)
    finally:
        os.environ.pop("MHAR_NO_FASTPATH", None)
        if old is not None:
            os.environ["MHAR_NO_FASTPATH"] = old


def test_diag_blocks_injected_step_matches_oracle_bitwise(orc):
    n, z = 300, 257  # [I; -I]: 600 x 300, too big for the walk-resident kernel
    p = mh.make_hypercube(n)
    rng = np.random.default_rng(3)
    X = np.asfortranarray(rng.uniform(-0.9, 0.9, (n, z)))
    H = np.asfortranarray(rng.standard_normal((n, z)))
    U = rng.uniform(0, 1, z)
    with _engine(p, z) as eng:
        eng.set_state(X)
        lo, hi, th, fl = eng.step_injected(H, U)
        Xg = eng.get_state()
    st, Xr, lor, hir, thr, flr, _ = orc.step_injected(p.a_in, p.b_in, None, EPS_DIR, X, H, U)
    assert st == 0
    np.testing.assert_array_equal(fl, flr)
    np.testing.assert_array_equal(lo, lor)
    np.testing.assert_array_equal(hi, hir)
    assert np.abs(Xg - Xr).max() <= 1e-15


@pytest.mark.parametrize("body", ["three_blocks", "box_ragged_bounds", "box_uniform"])
def test_diag_blocks_trajectory_equals_general_product(body):
    # stacked diagonal blocks: three with mixed coefficients [2I; -I; 0.5 I]
    # (per-row loads), a box with per-coordinate bounds [I; -I] x <= [u; -l]
    # (per-row bounds), a uniform box (the constant-block instantiation)
    n, z = 260, 200
    rng = np.random.default_rng(5)
    if body == "three_blocks":
        a = np.vstack([2.0 * np.eye(n), -np.eye(n), 0.5 * np.eye(n)])
        b = np.concatenate([np.full(n, 2.0), np.full(n, 1.0), np.full(n, 0.7)])
    elif body == "box_ragged_bounds":
        a = np.vstack([np.eye(n), -np.eye(n)])
        b = np.concatenate([rng.uniform(0.5, 2.0, n), rng.uniform(0.5, 2.0, n)])
    else:
        a = np.vstack([3.0 * np.eye(n), -3.0 * np.eye(n)])
        b = np.full(2 * n, 1.5)
    p = mh.Polytope(a, b)
    out = {}
    for fast in (True, False):  # the general path recomputes the slack like the fast path
        with _engine(p, z, seed=11, fastpath=fast, slack="recompute") as eng:
            eng.set_state(np.zeros((n, z)))
            eng.step(25)
            out[fast] = eng.get_state()
            bad, viol, _ = eng.check_state(1e-9)
            assert bad == -1 and viol.max() <= 1e-9
    np.testing.assert_array_equal(out[True], out[False])
    assert np.abs(out[True]).max() > 0.1


def test_factored_projection_injected_step_matches_oracle(orc):
    n, z = 300, 130  # simplex: A_E = 1', A_I = -I (diagonal too)
    p = mh.make_simplex(n)
    op = mh.compute_projection(p.a_eq)
    rng = np.random.default_rng(8)
    w = rng.dirichlet(np.ones(n), z).T
    X = np.asfortranarray(0.5 * w + 0.5 / n)
    H = np.asfortranarray(rng.standard_normal((n, z)))
    U = rng.uniform(0, 1, z)
    with _engine(p, z, projector=op) as eng:
        eng.set_state(X)
        lo, hi, th, fl = eng.step_injected(H, U)
        Xg = eng.get_state()
    st, Xr, lor, hir, thr, flr, _ = orc.step_injected(p.a_in, p.b_in, op.p, EPS_DIR, X, H, U)
    assert st == 0
    np.testing.assert_array_equal(fl, flr)
    ok = (flr & mh.FLAG_DEGENERATE) == 0
    wd = np.where(ok, hir - lor, 1.0)
    assert np.all(np.abs(lo - lor)[ok] <= 1e-9 * wd[ok])
    assert np.all(np.abs(hi - hir)[ok] <= 1e-9 * wd[ok])
    assert np.abs(Xg - Xr).max() <= 1e-9 * np.abs(Xr).max()


@pytest.mark.parametrize("me", [2, 3, 4])
def test_factored_projection_several_equalities(orc, me):
    # m_E = 2..4 random equality rows: the factored projection's split-partial
    # sums (proj_dot_kernel / proj_apply_kernel<ME>) against the oracle's
    # dense P H on one injected step
    n, m, z = 300, 2500, 193
    rng = np.random.default_rng(40 + me)
    a_in = rng.standard_normal((m, n))
    a_in /= np.linalg.norm(a_in, axis=1, keepdims=True)
    a_eq = rng.standard_normal((me, n))
    p = mh.Polytope(np.asfortranarray(a_in), np.ones(m), np.asfortranarray(a_eq), np.zeros(me))
    op = mh.compute_projection(p.a_eq)
    X = np.asfortranarray(op.p @ rng.uniform(-0.02, 0.02, (n, z)))  # on the slice, inside
    H = np.asfortranarray(rng.standard_normal((n, z)))
    U = rng.uniform(0, 1, z)
    with _engine(p, z, projector=op) as eng:
        eng.set_state(X)
        lo, hi, th, fl = eng.step_injected(H, U)
        Xg = eng.get_state()
    st, Xr, lor, hir, thr, flr, _ = orc.step_injected(p.a_in, p.b_in, op.p, EPS_DIR, X, H, U)
    assert st == 0
    np.testing.assert_array_equal(fl, flr)
    ok = (flr & mh.FLAG_DEGENERATE) == 0
    wd = np.where(ok, hir - lor, 1.0)
    assert np.all(np.abs(lo - lor)[ok] <= 1e-9 * wd[ok])
    assert np.all(np.abs(hi - hir)[ok] <= 1e-9 * wd[ok])
    assert np.abs(Xg - Xr).max() <= 1e-9 * np.abs(Xr).max()
    assert np.abs(a_eq @ Xg).max() <= 1e-12  # still on the slice


def test_factored_projection_run_stays_on_the_slice():
    n = 400
    p = mh.make_simplex(n)
    op = mh.compute_projection(p.a_eq)
    with _engine(p, 512, seed=2, projector=op) as eng:
        S, _ = eng.run(np.full(n, 1.0 / n), phi=20, windows=4, burn_in=20, reproject_every=20)
    assert np.abs(S.sum(1) - 1.0).max() <= 1e-9
    assert (S @ p.a_in.T - p.b_in).max() <= 1e-9
    assert abs(S.mean() - 1.0 / n) <= 0.1 / n


def test_multi_kernel_structured_run_large_simplex():
    # n = 3000 does not fit the walk-resident kernel: the multi-kernel path
    # with the diagonal chord and the factored projection, run() with
    # reprojection; against the general path (dense P H, DMMA chord)
    n = 3000
    p = mh.make_simplex(n)
    op = mh.compute_projection(p.a_eq)
    out = {}
    for fast in (True, False):
        with _engine(p, 256, seed=9, projector=op, fastpath=fast, slack="recompute") as eng:
            S, _ = eng.run(np.full(n, 1.0 / n), phi=10, windows=2, burn_in=10, reproject_every=10)
        assert np.abs(S.sum(1) - 1.0).max() <= 1e-9
        assert (S @ p.a_in.T - p.b_in).max() <= 1e-9
        out[fast] = S
    assert np.abs(out[True] - out[False]).max() <= 1e-9
