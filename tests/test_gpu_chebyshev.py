"""Chebyshev-centre start point on the GPU against the
reference's own test cases (tests/test_chebyshev.cpp, acceptance #5 in
tests/acceptance_main.cpp:251-290) and an independent LP solver (scipy's
HiGHS) at the configs' sizes.  Every call goes through the C ABI."""
import itertools

import numpy as np
import pytest

import paper_2104_07097_b200 as mh
from paper_2104_07097_b200 import workloads

pytestmark = pytest.mark.gpu


def _err(p):
    with pytest.raises(mh.MharError) as e:
        mh.chebyshev_center(p)
    return e.value.code


def _highs_radius(p):
    from scipy.optimize import linprog
    n = p.dim()
    norms = np.linalg.norm(p.a_in, axis=1)
    a_ub = np.hstack([p.a_in, norms[:, None]])
    a_eq = np.hstack([p.a_eq, np.zeros((p.num_equalities(), 1))]) if p.num_equalities() else None
    c = np.zeros(n + 1)
    c[n] = -1.0
    res = linprog(c, A_ub=a_ub, b_ub=p.b_in, A_eq=a_eq,
                  b_eq=p.b_eq if p.num_equalities() else None,
                  bounds=[(None, None)] * n + [(0, None)], method="highs")
    assert res.status == 0
    return res.x[:n], res.x[n]


def _enumerate(p):
    """tests/oracles.hpp:295-371 restated: best feasible active set."""
    n = p.dim()
    rows = [np.append(a, np.linalg.norm(a)) for a in p.a_in] + [np.append(np.zeros(n), -1.0)]
    rhs = list(p.b_in) + [0.0]
    eq = [np.append(a, 0.0) for a in p.a_eq]
    best = (-np.inf, None)
    for idx in itertools.combinations(range(len(rows)), n + 1 - len(eq)):
        sys = np.array(eq + [rows[k] for k in idx])
        r = np.array(list(p.b_eq) + [rhs[k] for k in idx])
        try:
            sol = np.linalg.solve(sys, r)
        except np.linalg.LinAlgError:
            continue
        if sol[n] < -1e-9:
            continue
        if all(rows[i] @ sol <= rhs[i] + 1e-9 for i in range(len(rows))) and \
                all(abs(e[:n] @ sol[:n] - b) <= 1e-9 for e, b in zip(eq, p.b_eq)):
            if sol[n] > best[0]:
                best = (sol[n], sol[:n])
    return best


@pytest.mark.parametrize("n", [2, 10, 100])
def test_unit_box_centres_exactly(n):
    c = mh.chebyshev_center(mh.make_hypercube(n))
    assert c.radius == 1.0
    assert np.abs(c.x).max() == 0.0


@pytest.mark.parametrize("n", [3, 4, 10])
def test_simplex_barycentre(n):
    c = mh.chebyshev_center(mh.make_simplex(n))
    assert abs(c.radius - 1.0 / n) <= 1e-8
    assert np.abs(c.x - 1.0 / n).max() <= 1e-8


@pytest.mark.parametrize("n", [3, 4])
def test_simplex_matches_active_set_enumeration(n):
    p = mh.make_simplex(n)
    c = mh.chebyshev_center(p)
    r, x = _enumerate(p)
    assert abs(c.radius - r) <= 1e-8
    assert np.abs(c.x - x).max() <= 1e-8


def test_random_planar_bodies_match_highs():
    rng = np.random.default_rng(41)
    for rep in range(8):
        extra = int(rng.uniform() * 3)
        a = np.vstack([[[1, 0], [-1, 0], [0, 1], [0, -1]], rng.uniform(-1, 1, (extra, 2))])
        b = np.concatenate([np.ones(4), 0.3 + rng.uniform(size=extra)])
        p = mh.Polytope(a, b)
        c = mh.chebyshev_center(p)
        _, r = _highs_radius(p)
        assert abs(c.radius - r) <= 1e-8, rep
        assert (a @ c.x - b).max() <= 1e-9


def test_scaling_scales_centre_and_radius():
    rng = np.random.default_rng(42)
    a = np.vstack([rng.uniform(-1, 1, (6, 3)), np.kron(np.eye(3), [[1.0], [-1.0]])])
    b = np.concatenate([0.5 + rng.uniform(size=6), 2.0 * np.ones(6)])
    base = mh.chebyshev_center(mh.Polytope(a, b))
    scaled = mh.chebyshev_center(mh.Polytope(a, 3.5 * b))
    assert abs(scaled.radius - 3.5 * base.radius) <= 1e-8
    assert np.abs(scaled.x - 3.5 * base.x).max() <= 1e-8


def test_error_codes():
    assert _err(mh.Polytope(np.array([[1.0], [-1.0]]), np.array([0.0, -1.0]))) == \
        mh.ErrorCode.empty_polytope
    flat = mh.Polytope(np.array([[1.0, 0], [-1, 0], [0, 1], [0, -1]]), np.array([0.0, 0, 1, 1]))
    assert _err(flat) == mh.ErrorCode.no_interior
    assert _err(mh.Polytope(np.array([[-1.0]]), np.array([0.0]))) == \
        mh.ErrorCode.unbounded_polytope


def test_equality_centre_stays_on_slice():
    p = mh.make_simplex(6)
    c = mh.chebyshev_center(p)
    assert np.abs(p.a_eq @ c.x - p.b_eq).max() <= 1e-9
    assert mh.contains(p, c.x, 1e-9)


@pytest.mark.parametrize("config", [2, 3])
def test_config_bodies_match_highs(config):
    """The constraint-generation LP at the configs' sizes: same optimal radius
    as HiGHS on the full LP, and the centre keeps that radius to every row."""
    p = workloads.config(config).polytope
    c = mh.chebyshev_center(p)
    _, r = _highs_radius(p)
    assert abs(c.radius - r) <= 1e-9 * max(1.0, r)
    norms = np.linalg.norm(p.a_in, axis=1)
    margin = ((p.b_in - p.a_in @ c.x) / norms).min()
    assert margin >= c.radius - 1e-9
    if config == 3:
        assert c.working_rows < p.num_inequalities()


def test_run_without_start_uses_the_centre():
    """sampler.cpp:276 + test_sampler.cpp:275: start_radius of the unit box is 1."""
    cube = mh.make_hypercube(3)
    cfg = mh.SamplerConfig(z=2, phi=3, t_target=4, burn_in=0, seed=7)
    out = mh.run(cube, cfg)
    assert out.start_radius == 1.0
    assert np.abs(out.start).max() == 0.0
    warm = mh.run(cube, cfg, x0=np.zeros(3))
    assert np.array_equal(out.samples, warm.samples)
