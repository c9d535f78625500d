"""CUDA-graph replay of steady iterates (csrc/abi.cu graph_iterate): the
multi-kernel path's trajectories are bit-identical with and without graphs
(MHAR_NO_GRAPHS=1), across slack refreshes, reprojection, state resets,
checkpoint/resume and every engine."""
import os

import numpy as np
import pytest

import paper_2104_07097_b200 as mh
from paper_2104_07097_b200 import workloads

pytestmark = pytest.mark.gpu


def _engine(*args, graphs=True, **kw):
    old = os.environ.pop("MHAR_NO_GRAPHS", None)
    if not graphs:
        os.environ["MHAR_NO_GRAPHS"] = "1"
    try:
        return mh.Engine(*args, **kw)
    finally:
        os.environ.pop("MHAR_NO_GRAPHS", None)
        if old is not None:
            os.environ["MHAR_NO_GRAPHS"] = old


def _trajectory(p, z, graphs, chunks, reproject=0, reset_at=None, **kw):
    n = p.dim()
    x0 = kw.pop("x0", np.zeros(n))
    out = []
    with _engine(p, z, graphs=graphs, seed=21, **kw) as eng:
        eng.set_state(np.repeat(np.asarray(x0, dtype=np.float64)[:, None], z, axis=1))
        for i, k in enumerate(chunks):
            if reset_at is not None and i == reset_at:
                ck = eng.checkpoint()
                X = eng.get_state()
                eng.set_state(X * 0.5)          # state swap: the graph is recaptured
                eng.step(5, reproject)
                eng.restore(ck)                 # counter rewound: the device copy follows
            eng.step(k, reproject)
            out.append(eng.get_state())
        st = eng.stats()
    return out, st


@pytest.mark.parametrize("kw", [dict(), dict(f64_engine="int8"), dict(precision=32),
                                dict(slack="recompute")],
                         ids=["dmma", "int8", "fp32", "recompute"])
def test_graph_trajectories_bit_identical(kw):
    p = workloads.random_polytope(96, 6000, seed=4)
    chunks = [37, 64, 5, 130, 9]  # crosses the 128-iterate refresh
    a, sa = _trajectory(p, 256, True, chunks, **dict(kw))
    b, sb = _trajectory(p, 256, False, chunks, **dict(kw))
    for xa, xb in zip(a, b):
        np.testing.assert_array_equal(xa, xb)
    assert sa["iterations"] == sb["iterations"] == sum(chunks)
    assert np.abs(a[-1]).max() > 0.05


def test_graph_chord3_bit_identical():
    # n_pad >= 384: the graph replays chord3_kernel (its unit ticket counter
    # is rewound by the last CTA of every launch), across refreshes and a
    # state reset
    p = workloads.random_polytope(400, 4000, seed=8)
    chunks = [30, 70, 40]
    a, sa = _trajectory(p, 300, True, chunks, reset_at=1)
    b, _ = _trajectory(p, 300, False, chunks, reset_at=1)
    assert sa["chord_kernel"] == "chord3_kernel"
    for xa, xb in zip(a, b):
        np.testing.assert_array_equal(xa, xb)
    assert np.abs(a[-1]).max() > 0.05


def test_graph_structured_path_with_reprojection_and_reset():
    n = 3000
    p = mh.make_simplex(n)
    op = mh.compute_projection(p.a_eq)
    chunks = [20, 33, 7, 40]
    kw = dict(projector=op, x0=np.full(n, 1.0 / n))
    a, _ = _trajectory(p, 256, True, chunks, reproject=10, reset_at=2, **dict(kw))
    b, _ = _trajectory(p, 256, False, chunks, reproject=10, reset_at=2, **dict(kw))
    for xa, xb in zip(a, b):
        np.testing.assert_array_equal(xa, xb)
    assert np.abs(a[-1].sum(0) - 1.0).max() <= 1e-9
