"""The fp32 variant (precision=32): the rates A_I d on tcgen05 tensor cores
with fp32 accuracy (csrc/chord_tc32.cuh; kind::f16 with per-row / per-walk
scales, or kind::tf32 under MHAR_TC_F16=0), fp64 slack/state from the
caller's A_I, chords of {A x <= b - mu}.  North-star bar: one iterate within
1e-4 relative of the reference step on the fp32 body with the injected
direction; every emitted sample exactly inside the caller's body; moments
within Monte-Carlo error.  The fast form (fp32_direction="rounded") moves
along a rounded direction and is tested against the reference step with that
direction."""
import numpy as np
import pytest

import oracle
import paper_2104_07097_b200 as mh
from paper_2104_07097_b200 import workloads

pytestmark = pytest.mark.gpu
RTOL32 = 1e-4


def _tf32(x):
    u = np.asarray(x, dtype=np.float32).view(np.uint32) & np.uint32(0xFFFFE000)
    return u.view(np.float32)


@pytest.fixture(autouse=True, params=["f16", "tf32"])
def form(request, monkeypatch):
    """Both forms of the variant: kind::f16 with per-row / per-walk scales
    (default) and kind::tf32 (MHAR_TC_F16=0)."""
    monkeypatch.setenv("MHAR_TC_F16", "1" if request.param == "f16" else "0")
    return request.param


def _f16_split(x, axis):
    """x scaled by 2^(14 - e) (max |x| < 2^e along `axis`), split into two
    halves below the fp16 normal range flushed: (hi, hi + lo), unscaled."""
    mx = np.abs(x).max(axis=axis, keepdims=True)
    e = np.where(mx > 0, np.floor(np.log2(np.where(mx > 0, mx, 1.0))) + 1, 0)
    s = 2.0 ** (14 - e)
    h = (x * s).astype(np.float16).astype(np.float64)
    h[np.abs(h) < 2.0 ** -14] = 0.0
    lo = (x * s - h).astype(np.float16).astype(np.float64)
    lo[np.abs(lo) < 2.0 ** -14] = 0.0
    return h / s, (h + lo) / s


def dir_used(H, form="tf32"):
    """The direction moved along: TF32-rounded, or the per-walk-scaled half."""
    if form == "f16":
        return _f16_split(np.asarray(H, dtype=np.float64), 0)[0]
    return _tf32(H).astype(np.float64)


def _interior(p, z, rng, shrink=0.4):
    X = rng.uniform(-1, 1, (p.dim(), z))
    s = np.max((p.a_in @ X) / p.b_in[:, None], axis=0)
    return np.asfortranarray(X * (shrink / s))


@pytest.mark.parametrize("n,m,z", [(16, 300, 128), (37, 1000, 200), (500, 20000, 256)])
def test_fp32_injected_step_parity(orc, form, n, m, z):
    # north star: one iterate within 1e-4 of the reference step on the same
    # fp32 body with the injected (un-quantised) direction.  The default
    # (split-direction) variant differs from the fp64 path only in the
    # products A_I d (sampler.cpp:174-176): the walk moves along the fp64
    # direction, the slack comes from the caller's A_I.
    p = workloads.random_polytope(n, m, seed=n)
    rng = np.random.default_rng(m)
    X = _interior(p, z, rng)
    H = np.asfortranarray(rng.standard_normal((n, z)))
    U = rng.uniform(0.05, 0.95, z)
    with mh.Engine(p, z, precision=32) as eng:
        eng.set_state(X)
        lo, hi, th, fl = eng.step_injected(H, U)
        Xg = eng.get_state()
        bad, viol, _ = eng.check_state(0.0)  # fresh fp64 product on the caller's A_I
    A32 = np.asfortranarray(np.asarray(p.a_in, dtype=np.float32).astype(np.float64))
    st, Xr, lor, hir, thr, flr, _ = orc.step_injected(A32, p.b_in, None, 1e-11, X, H, U)
    assert st == 0
    assert np.array_equal(fl & mh.FLAG_DEGENERATE, flr & mh.FLAG_DEGENERATE)
    w = hir - lor
    assert np.all(np.abs(lo - lor) <= RTOL32 * w)
    assert np.all(np.abs(hi - hir) <= RTOL32 * w)
    assert np.all(np.abs(th - thr) <= RTOL32 * w)
    assert np.abs(Xg - Xr).max() <= RTOL32 * np.abs(Xr).max()
    # every walk strictly inside the caller's body (not a perturbed copy)
    assert bad == -1 and viol.max() < 0.0
    assert (p.a_in @ Xg - p.b_in[:, None]).max() < 0.0


@pytest.mark.parametrize("n,m,z", [(16, 300, 128), (500, 20000, 256)])
def test_fp32_rounded_direction_form(orc, form, n, m, z):
    # the fast form (fp32_direction="rounded"): the direction is rounded to
    # one operand and the walk moves along that rounded direction; against
    # the reference step on the same body with that direction injected
    p = workloads.random_polytope(n, m, seed=n)
    rng = np.random.default_rng(m)
    X = _interior(p, z, rng)
    H = np.asfortranarray(rng.standard_normal((n, z)))
    U = rng.uniform(0.05, 0.95, z)
    with mh.Engine(p, z, precision=32, fp32_direction="rounded") as eng:
        eng.set_state(X)
        lo, hi, th, fl = eng.step_injected(H, U)
        Xg = eng.get_state()
        bad, viol, _ = eng.check_state(0.0)
    D_used = np.asfortranarray(dir_used(H, form))  # the direction moved along
    A32 = np.asfortranarray(np.asarray(p.a_in, dtype=np.float32).astype(np.float64))
    st, Xr, lor, hir, thr, flr, _ = orc.step_injected(A32, p.b_in, None, 1e-11, X, D_used, U)
    assert st == 0
    w = hir - lor
    assert np.all(np.abs(lo - lor) <= RTOL32 * w)
    assert np.all(np.abs(hi - hir) <= RTOL32 * w)
    # the margin only ever shrinks the chord (to fp32 accuracy of the rates)
    assert np.all(hi <= hir + 1e-6 * w) and np.all(lo >= lor - 1e-6 * w)
    assert np.abs(Xg - Xr).max() <= RTOL32 * np.abs(Xr).max()
    assert bad == -1 and viol.max() < 0.0


@pytest.mark.parametrize("direction", ["split", "rounded"])
def test_fp32_walks_stay_exactly_feasible(form, direction):
    p = workloads.random_polytope(64, 4000, seed=3)
    with mh.Engine(p, 256, seed=4, precision=32, refresh_every=64,
                   fp32_direction=direction) as eng:
        eng.set_state(np.zeros((64, 256)))
        for _ in range(5):
            eng.step(60)
            bad, viol, _ = eng.check_state(1e-9)   # fresh fp64 product on the caller's A_I
            assert bad == -1 and viol.max() <= 0.0
        X = eng.get_state()
    assert (p.a_in @ X - p.b_in[:, None]).max() <= 0.0
    assert np.abs(X).max() > 0.1


def test_fp32_run_box_moments():
    p = mh.make_hypercube(12)
    with mh.Engine(p, 512, seed=5, precision=32) as eng:
        S, st = eng.run(np.zeros(12), phi=40, windows=20, burn_in=100)
    assert S.shape == (20 * 512, 12)
    assert (S @ p.a_in.T - p.b_in).max() <= 1e-9
    assert np.abs(S.mean(0)).max() <= 0.03
    assert np.abs(S.var(0) - 1 / 3).max() <= 0.03


def test_fp32_matches_fp64_in_law():
    # same Philox streams, fp32 vs fp64 chords: trajectories stay close over
    # a few iterates (rate errors ~1e-6 relative, margin 1e-6)
    p = workloads.random_polytope(40, 1500, seed=9)
    out = {}
    for prec in (64, 32):
        with mh.Engine(p, 128, seed=12, precision=prec, small_path=False) as eng:
            eng.set_state(np.zeros((40, 128)))
            eng.step(4)
            out[prec] = eng.get_state()
    assert np.abs(out[32] - out[64]).max() <= 1e-3


def test_fp32_config5_full_width_feasible():
    w = workloads.config(5)
    with mh.Engine(w.polytope, w.z, seed=5, precision=32) as eng:
        eng.set_state(np.zeros((2000, w.z)))
        eng.step(10)
        bad, viol, _ = eng.check_state(1e-9)
    assert bad == -1 and viol.max() <= 0.0


def test_fp32_with_equalities_stays_on_the_slice_and_inside():
    # bodies with equalities: the projected direction is split (d_hi + d_lo)
    # rather than rounded to TF32, so it stays in the null space of A_E and
    # the reprojection cadence only removes rounding drift
    n, me = 120, 6
    rng = np.random.default_rng(12)
    a_eq = rng.standard_normal((me, n))
    base = workloads.random_polytope(n, 3000, seed=13)
    p = mh.Polytope(base.a_in, base.b_in, a_eq, np.zeros(me))
    op = mh.compute_projection(p.a_eq)
    with mh.Engine(p, 256, seed=4, projector=op, precision=32, refresh_every=64) as eng:
        eng.set_state(np.zeros((n, 256)))
        for _ in range(4):
            eng.step(75, 25)
            bad, viol, eqv = eng.check_state(1e-9)
            assert bad == -1 and viol.max() <= 0.0 and eqv.max() <= 1e-9
        X = eng.get_state()
    assert np.abs(a_eq @ X).max() <= 1e-9
    assert np.abs(X).max() > 0.05


def test_fp32_relay_path_without_tma(monkeypatch, form):
    # MHAR_TC_TMA=0: plain bulk copies and the odd CTA's "stage landed" relay
    # (the round-1 protocol) -- the same trajectory as the 2-CTA TMA loads
    p = workloads.random_polytope(300, 5000, seed=21)
    out = {}
    for tma in ("1", "0"):
        monkeypatch.setenv("MHAR_TC_TMA", tma)
        with mh.Engine(p, 512, seed=8, precision=32) as eng:
            eng.set_state(np.zeros((300, 512)))
            eng.step(12)
            out[tma] = eng.get_state()
            bad, viol, _ = eng.check_state(1e-9)
            assert bad == -1 and viol.max() <= 0.0
    np.testing.assert_array_equal(out["1"], out["0"])
