"""The API twins of SURVEY 8(a) row A10 through the C ABI:
generate_directions (proj/tests/test_sampler.cpp:78-91) and select_points
(test_sampler.cpp:164-215)."""
import math

import numpy as np
import pytest

import oracle
import paper_2104_07097_b200 as mh
from scalar_walk import ks_statistic_uniform

pytestmark = pytest.mark.gpu


def test_generate_directions_reference_streams(orc):
    # same streams as the reference's WalkRng: the fill matches the oracle's
    # fill_standard_normal_matrix to transcendental rounding, and successive
    # batches keep consuming 2*ceil(n/2) draws per column
    p = mh.make_hypercube(7)
    with mh.Engine(p, 4, seed=51, rng="reference") as eng:
        h1 = eng.generate_directions()
        h2 = eng.generate_directions()
    rng = orc.WalkRng(51, 4)
    r1 = rng.fill_standard_normal_matrix(7)
    r2 = rng.fill_standard_normal_matrix(7)
    np.testing.assert_allclose(h1, r1, rtol=1e-14, atol=1e-15)
    np.testing.assert_allclose(h2, r2, rtol=1e-14, atol=1e-15)


def test_generate_directions_moments():
    p = mh.make_hypercube(64)
    with mh.Engine(p, 1024, seed=3) as eng:
        h = eng.generate_directions()
        h2 = eng.generate_directions()
    assert abs(h.mean()) < 0.01 and abs(h.var() - 1) < 0.02
    assert not np.array_equal(h, h2)


def test_select_points_inside_and_flag_refusal():
    # proj/tests/test_sampler.cpp:164-197
    p = mh.make_hypercube(2)
    X = np.zeros((2, 3))
    D = np.array([[1.0, 0.0, 1.0], [0.0, 1.0, 1.0]])
    with mh.Engine(p, 3, seed=52, rng="reference") as eng:
        iv = eng.lambda_intervals(X, D)
        moved = eng.select_points(X, D, iv)
        for k in range(3):
            assert mh.contains(p, moved[:, k], 0.0)
            assert np.linalg.norm(moved[:, k]) > 0
        iv.degenerate[1] = 1
        with pytest.raises(mh.MharError) as e:
            eng.select_points(X, D, iv)
        assert e.value.code == mh.ErrorCode.direction_degenerate


def test_select_points_uniform_along_chord_and_theta_stream(orc):
    # proj/tests/test_sampler.cpp:199-215 (KS at 1%), and the draws are the
    # reference theta stream's, in walk order
    reps = 4000
    p = mh.make_hypercube(2)
    X = np.zeros((2, reps))
    D = np.tile([[1.0], [0.0]], (1, reps))
    with mh.Engine(p, reps, seed=54, rng="reference") as eng:
        iv = eng.lambda_intervals(X, D)
        moved = eng.select_points(X, D, iv)
    u = (moved[0] + 1.0) / 2.0
    assert ks_statistic_uniform(list(u)) < 1.63 / math.sqrt(reps)
    s = orc.Stream(54, oracle.THETA_STREAM_ID)
    want = np.array([-1.0 + s.next_uniform() * 2.0 for _ in range(reps)])
    assert np.abs(moved[0] - want).max() <= 1e-15


def test_step_runs_the_engine_body_and_rejects_another():
    # step(p, op, cfg, engine, state): one iterate of the engine's body; a
    # different polytope (same shape, other rows) is refused, not silently
    # sampled with the engine's device copy
    p = mh.make_hypercube(3)
    cfg = mh.resolve(mh.SamplerConfig(), p)
    with mh.Engine(p, 8, seed=5) as eng:
        st = mh.WalkState(x=np.zeros((3, 8), order="F"))
        mh.step(p, None, cfg, eng, st)
        assert st.j == 1 and np.abs(st.x).max() <= 1.0 and np.abs(st.x).max() > 0.0
        other = mh.Polytope(p.a_in.copy(), np.full(6, 0.5))
        with pytest.raises(mh.MharError) as e:
            mh.step(other, None, cfg, eng, st)
        assert e.value.code == mh.ErrorCode.invalid_argument
        assert st.j == 1
