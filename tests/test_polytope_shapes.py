"""Polytope construction checks of the Python host API, as the reference's
constructor makes them (proj/src/polytope.cpp:16-33, :90-97): a right-hand
side that does not match its matrix, or equalities of another width, raise
DIMENSION_MISMATCH before anything reaches the C ABI (which reads exactly
those extents).  CPU only."""
import numpy as np
import pytest

import paper_2104_07097_b200 as mh


@pytest.mark.parametrize("args", [
    (np.eye(3), np.ones(2)),
    (np.eye(3), np.ones(3), np.ones((1, 2)), np.ones(1)),
    (np.eye(3), np.ones(3), np.ones((1, 3)), np.ones(2)),
    (np.ones(3), np.ones(3)),
])
def test_shape_mismatch_raises(args):
    with pytest.raises(mh.MharError) as e:
        mh.Polytope(*args)
    assert e.value.code == mh.ErrorCode.dimension_mismatch


def test_valid_bodies_and_empty_equalities_take_the_width():
    p = mh.Polytope(np.eye(4), np.ones(4), np.zeros((0, 0)), np.zeros(0))
    assert p.a_eq.shape == (0, 4) and p.num_equalities() == 0
    s = mh.make_simplex(5)
    assert s.a_eq.shape == (1, 5) and s.b_eq.shape == (1,)
    c = mh.make_hypercube(3)
    assert c.a_in.shape == (6, 3) and c.b_in.shape == (6,)


def test_step_guard_tells_the_engine_body_from_another():
    # step(p, ..., engine, state) refuses a body other than the engine's
    # before touching the device; a re-wrap of the same arrays is the same body
    p = mh.make_hypercube(3)

    class Bound:  # stands in for an Engine: the guard runs before any device call
        pass
    eng = Bound()
    eng.p = p
    st = mh.WalkState(x=np.zeros((3, 2), order="F"))
    with pytest.raises(mh.MharError) as e:
        mh.step(mh.Polytope(p.a_in.copy(), p.b_in), None, None, eng, st)
    assert e.value.code == mh.ErrorCode.invalid_argument
    with pytest.raises(AttributeError):  # got past the guard, to the engine call
        mh.step(mh.Polytope(p.a_in, p.b_in), None, None, eng, st)
