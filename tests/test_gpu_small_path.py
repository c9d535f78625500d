"""The walk-resident small-body kernel (csrc/small_kernel.cuh) against the
per-iterate kernel chain on the same Philox streams, and its error
semantics (proj/tests/test_sampler.cpp:139-154, :244-258)."""
import numpy as np
import pytest

import paper_2104_07097_b200 as mh
from paper_2104_07097_b200 import workloads

pytestmark = pytest.mark.gpu


def _both(p, z, x0, steps, seed=17, projector=None, reproject=0, **kw):
    out = {}
    for small in (True, False):
        with mh.Engine(p, z, seed=seed, projector=projector, small_path=small, **kw) as eng:
            X = np.empty((p.dim(), z), order="F")
            X[:] = np.asarray(x0)[:, None]
            eng.set_state(X)
            eng.step(steps, reproject)
            out[small] = (eng.get_state(), eng.stats())
    return out


@pytest.mark.parametrize("n", [3, 10, 33])
def test_small_path_matches_kernel_chain_box(n):
    p = mh.make_hypercube(n)
    out = _both(p, 150, np.zeros(n), 40)
    assert out[True][1]["kernel_launches"] < out[False][1]["kernel_launches"]
    np.testing.assert_allclose(out[True][0], out[False][0], rtol=0, atol=1e-12)


def test_small_path_matches_kernel_chain_simplex_with_reprojection():
    p = mh.make_simplex(20)
    op = mh.compute_projection(p.a_eq)
    out = _both(p, 64, np.full(20, 0.05), 30, projector=op, reproject=10)
    np.testing.assert_allclose(out[True][0], out[False][0], rtol=0, atol=1e-12)
    assert np.abs(out[True][0].sum(0) - 1.0).max() <= 1e-12


def test_small_path_random_body():
    p = workloads.random_polytope(12, 200, seed=6)
    out = _both(p, 100, np.zeros(12), 25)
    np.testing.assert_allclose(out[True][0], out[False][0], rtol=0, atol=1e-11)


def test_small_path_retry_exhausted_and_redraw_count():
    p = mh.make_hypercube(2)
    with mh.Engine(p, 1, seed=55, eps_dir=1e9) as eng:
        eng.set_state(np.zeros((2, 1)))
        with pytest.raises(mh.MharError) as e:
            eng.step(1)
        assert e.value.code == mh.ErrorCode.retry_exhausted
        assert eng.stats()["redraw_count"] == 16


def test_small_path_unbounded_names_walk():
    # both paths raise for the same (earliest iterate, lowest) walk
    quadrant = mh.Polytope(-np.eye(2), np.zeros(2))
    msgs = []
    for small in (True, False):
        with mh.Engine(quadrant, 5, seed=2, small_path=small) as eng:
            eng.set_state(np.ones((2, 5)))
            with pytest.raises(mh.MharError) as e:
                eng.step(3)
            assert e.value.code == mh.ErrorCode.unbounded_polytope
            msgs.append(str(e.value))
    assert msgs[0] == msgs[1]


def test_small_path_redraws_match_kernel_chain():
    # eps_dir between the rates forces redraws (box(2): rates are +-d_i)
    p = mh.make_hypercube(2)
    out = _both(p, 64, np.zeros(2), 5, eps_dir=0.9)
    assert out[True][1]["redraw_count"] == out[False][1]["redraw_count"] > 0
    np.testing.assert_allclose(out[True][0], out[False][0], rtol=0, atol=1e-12)


def test_config1_run_moments():
    # BASELINE config 1: hypercube n = 10, z = 100, 1000 burn-in + 1000 kept
    # (phi = 1, 1000 windows -> 1e5 samples): marginals mean 0, variance 1/3.
    p = mh.make_hypercube(10)
    out = mh.run(p, mh.SamplerConfig(z=100, phi=1, t_target=100_000, burn_in=1000, seed=1),
                 x0=np.zeros(10))
    S = out.samples
    assert S.shape == (100_000, 10)
    assert (S @ p.a_in.T - p.b_in).max() <= 1e-9
    # consecutive samples of a walk are correlated (phi = 1); the bound
    # allows for the effective sample size
    assert np.abs(S.mean(0)).max() <= 0.03
    assert np.abs(S.var(0) - 1 / 3).max() <= 0.03


def test_config2_run_mean():
    # BASELINE config 2: simplex n = 100, x0 = 1/n, z = 1000, 5000 iterations
    p = mh.make_simplex(100)
    out = mh.run(p, mh.SamplerConfig(z=1000, phi=50, t_target=100_000, burn_in=0, seed=2),
                 x0=np.full(100, 0.01))
    S = out.samples
    assert np.abs(S.sum(1) - 1.0).max() <= 1e-9
    assert (S @ p.a_in.T - p.b_in).max() <= 1e-9
    assert np.abs(S.mean(0) - 0.01).max() <= 0.002
