"""Pins the CPU oracle (oracle/mhar_oracle.c) to the reference's own
known-answer tests for the hot path.  Each test names the reference test it
restates (proj/tests/...).  CPU only."""
import math

import numpy as np
import pytest

import oracle
from scalar_walk import ScalarWalk, box_muller as py_box_muller, ks_statistic_uniform, \
    ray_march_chord, sample_moments

EPS_DIR = 1e-11


# ----------------------------------------------------------------- rng ------

def test_streams_deterministic_and_decorrelated(orc):
    # proj/tests/test_rng.cpp:13-27
    a, b = orc.Stream(123, 0), orc.Stream(123, 0)
    other_stream, other_seed = orc.Stream(123, 1), orc.Stream(124, 0)
    ds = dsd = 0
    for _ in range(64):
        v = a.next_u64()
        assert v == b.next_u64()
        ds += v != other_stream.next_u64()
        dsd += v != other_seed.next_u64()
    assert ds >= 63 and dsd >= 63


def test_stream_known_values(orc):
    # SplitMix64 finaliser constants of proj/src/rng.cpp:17-21, checked by hand
    # against the published splitmix64 mix of 0 and of the golden increment.
    assert orc.lib().orc_mix64(0) == 0
    s = orc.Stream(0, 0)
    init = orc.lib().orc_mix64(0x9E3779B97F4A7C15) ^ orc.lib().orc_mix64(0x6A09E667F3BCC909)
    assert s.state.value == init
    assert s.next_u64() == orc.lib().orc_mix64((init + 0x9E3779B97F4A7C15) % 2**64)


def test_uniform_ranges(orc):
    # proj/tests/test_rng.cpp:29-39
    s = orc.Stream(7, 3)
    for _ in range(10000):
        u = s.next_uniform()
        assert 0.0 <= u < 1.0
        v = s.next_uniform_open()
        assert 0.0 < v <= 1.0


def test_box_muller_kat_and_rejects(orc):
    # proj/tests/test_rng.cpp:41-51
    c, s = orc.box_muller(0.5, 0.25)
    assert abs(c) <= 1e-15
    assert s == pytest.approx(math.sqrt(2.0 * math.log(2.0)), rel=1e-12)
    for u1, u2 in [(0.0, 0.5), (1.5, 0.5), (0.5, 1.0), (0.5, -0.1)]:
        with pytest.raises(ValueError):
            orc.box_muller(u1, u2)


def test_normal_moments(orc):
    # proj/tests/test_rng.cpp:53-63
    draws = orc.Stream(2024, 0).fill_standard_normal(100000)
    assert abs(draws.mean()) <= 0.02
    assert abs(draws.var(ddof=1) - 1.0) <= 0.03


def test_fill_consumes_fixed_draw_count(orc):
    # proj/tests/test_rng.cpp:65-74
    a = orc.Stream(5, 9)
    a.fill_standard_normal(5)
    b = orc.Stream(5, 9)
    for _ in range(6):
        b.next_u64()
    assert a.next_u64() == b.next_u64()


@pytest.mark.parametrize("n", [2, 3, 4, 5])
def test_single_walk_fill_matches_scalar_bitwise(orc, n):
    # proj/tests/test_rng.cpp:76-101
    rng = orc.WalkRng(99, 1)
    h = rng.fill_standard_normal_matrix(n)
    ref = orc.Stream(99, 0)
    want = [0.0] * n
    for p in range((n + 1) // 2):
        c, s = orc.box_muller(ref.next_uniform_open(), ref.next_uniform())
        want[2 * p] = c
        if 2 * p + 1 < n:
            want[2 * p + 1] = s
    assert list(h[:, 0]) == want
    # and the independent python restatement agrees bit for bit
    ref2 = orc.Stream(99, 0)
    sw = ScalarWalk([[1.0] * n], [1.0])
    assert sw.normals(ref2, n) == want


def test_matrix_fill_close_at_vector_sizes(orc):
    # proj/tests/test_rng.cpp:103-120
    n = 64
    rng = orc.WalkRng(1234, 2)
    h = rng.fill_standard_normal_matrix(n)
    for k in range(2):
        ref = orc.Stream(1234, k)
        for p in range(n // 2):
            c, s = py_box_muller(ref.next_uniform_open(), ref.next_uniform())
            assert h[2 * p, k] == pytest.approx(c, rel=1e-12, abs=1e-300)
            assert h[2 * p + 1, k] == pytest.approx(s, rel=1e-12, abs=1e-300)


def test_walk_columns_advance_independently(orc):
    # proj/tests/test_rng.cpp:122-133
    a, b = orc.WalkRng(42, 4), orc.WalkRng(42, 4)
    st = oracle.C.c_uint64(int(a.cols[2]))
    oracle.lib().orc_fill_standard_normal(oracle.C.byref(st), oracle._d(np.empty(6)), 6)
    a.cols[2] = st.value
    for k in (0, 1, 3):
        assert a.cols[k] == b.cols[k]
    assert a.cols[2] != b.cols[2]
    assert a.theta[0] == b.theta[0]


# ---------------------------------------------------------------- gemm ------

@pytest.mark.parametrize("m,n,z", [(1, 1, 1), (7, 5, 3), (50, 300, 9), (25, 257, 17), (97, 33, 2)])
def test_gemm_is_sequential_fma_chain(orc, m, n, z):
    rng = np.random.default_rng(m * 1000 + n + z)
    A = np.asfortranarray(rng.standard_normal((m, n)))
    B = np.asfortranarray(rng.standard_normal((n, z)))
    got = orc.gemm(A, B)
    # naive ascending-k FMA chain (math.fma, Python >= 3.13 absent -> use numpy
    # longdouble-free emulation via fractions for a few entries)
    from fractions import Fraction
    for i, j in [(0, 0), (m - 1, z - 1), (m // 2, z // 2)]:
        acc = 0.0
        for k in range(n):
            exact = Fraction(A[i, k]) * Fraction(B[k, j]) + Fraction(acc)
            acc = float(exact)  # round-to-nearest of the exact fma
        assert got[i, j] == acc
    np.testing.assert_allclose(got, A @ B, rtol=1e-12, atol=1e-12)


# --------------------------------------------------------------- chords -----

def test_chord_bounds_box_hand_geometry(orc):
    # proj/tests/test_sampler.cpp:93-107
    A, b = orc.make_hypercube(2)
    X = np.asfortranarray([[0.0, 0.5], [0.0, 0.0]])
    D = np.asfortranarray([[1.0, 1.0], [0.0, 0.0]])
    st, lo, hi, dg, _, _ = orc.lambda_intervals(A, b, X, D, EPS_DIR)
    assert st == 0
    assert lo[0] == -1.0 and hi[0] == 1.0
    assert lo[1] == -1.5 and hi[1] == 0.5
    assert dg[0] == 0 and dg[1] == 0


def test_chord_bounds_simplex_vs_ray_march(orc):
    # proj/tests/test_sampler.cpp:109-126
    A, b, AE, bE = orc.make_simplex(3)
    x = np.array([1 / 3, 1 / 3, 1 / 3])
    d = np.array([2 / 3, -1 / 3, -1 / 3])
    d /= np.linalg.norm(d)
    st, lo, hi, _, _, _ = orc.lambda_intervals(A, b, x[:, None], d[:, None], EPS_DIR)
    rows = [[-1, 0, 0], [0, -1, 0], [0, 0, -1]]
    mlo, mhi = ray_march_chord(rows, [0, 0, 0], list(x), list(d), 1e-6)
    assert abs(hi[0] - mhi) <= 1e-6 and abs(lo[0] - mlo) <= 1e-6


def test_all_parallel_flagged(orc):
    # proj/tests/test_sampler.cpp:128-137
    A, b = orc.make_hypercube(2)
    st, lo, hi, dg, sd, _ = orc.lambda_intervals(A, b, np.zeros((2, 1)), np.array([[1.0], [0.0]]),
                                                 1e9)
    assert st == 0 and dg[0] == 1 and lo[0] == 0.0 and hi[0] == 0.0 and sd[0] == 0


def test_one_sided_chord_unbounded(orc):
    # proj/tests/test_sampler.cpp:139-154
    A = -np.eye(2)
    b = np.zeros(2)
    st, *_ , err = orc.lambda_intervals(A, b, np.array([[1.0], [1.0]]), np.array([[0.3], [1.0]]),
                                       EPS_DIR)
    assert st == 7 and err == 0


def test_chord_scan_masks_and_sides(orc):
    # vmath.hpp:83-155: rows inside +-eps are skipped; order independent
    num = np.array([1.0, 2.0, -0.5, 3.0, 7.0])
    den = np.array([0.5, -1.0, 1e-12, 2.0, -7.0])
    lo, hi, p, q = orc.chord_scan(num, den, 1e-11)
    assert (lo, hi, p, q) == (-1.0, 1.5, True, True)
    lo2, hi2, _, _ = orc.chord_scan(num[::-1], den[::-1], 1e-11)
    assert (lo2, hi2) == (lo, hi)


# ----------------------------------------------------------- projection -----

def _invariants(P, AE):
    assert np.abs(P - P.T).max() <= 1e-10
    assert np.abs(P @ P - P).max() <= 1e-9
    assert np.abs(AE @ P).max() <= 1e-9


def test_projection_ones_row_closed_form(orc):
    # proj/tests/test_projection.cpp:32-44
    AE = np.ones((1, 3))
    st, P, _ = orc.compute_projection(AE)
    assert st == 0
    np.testing.assert_allclose(P, np.eye(3) - 1 / 3, rtol=1e-14, atol=1e-15)
    _invariants(P, AE)


def test_projection_axis_row(orc):
    # proj/tests/test_projection.cpp:46-53
    st, P, _ = orc.compute_projection(np.array([[1.0, 0.0, 0.0]]))
    want = np.eye(3)
    want[0, 0] = 0.0
    assert np.abs(P - want).max() <= 1e-15


def test_projection_simplex4_bit_exact(orc):
    # proj/tests/acceptance_main.cpp:122-125 / test_sampler.cpp:448-452
    _, _, AE, _ = orc.make_simplex(4)
    st, P, _ = orc.compute_projection(AE)
    want = np.full((4, 4), -0.25)
    np.fill_diagonal(want, 0.75)
    assert st == 0 and np.array_equal(P, want)


def test_projection_random_invariants_and_errors(orc):
    # proj/tests/test_projection.cpp:55-85, 162-172
    s = orc.Stream(24, 0)
    for me, n in [(1, 2), (1, 40), (5, 12), (20, 60), (99, 100)]:
        AE = np.array([[2.0 * s.next_uniform() - 1.0 for _ in range(n)] for _ in range(me)])
        st, P, G = orc.compute_projection(AE)
        assert st == 0
        _invariants(P, AE)
        assert np.abs((AE @ AE.T) @ G - np.eye(me)).max() <= 1e-10
    assert orc.compute_projection(np.eye(3))[0] == 4  # RANK_DEFICIENT_EQ
    assert orc.compute_projection(np.array([[1, 1, 0, 0], [2, 2, 0, 0.0]]))[0] == 4


def test_projected_direction_kat(orc):
    # proj/tests/test_projection.cpp:87-108
    AE = np.ones((1, 3))
    _, P, _ = orc.compute_projection(AE)
    H = np.asfortranarray([[1.0, 1.0, 0.5], [0.0, 1.0, -0.25], [0.0, 1.0, 0.75]])
    D = orc.gemm(P, H)
    np.testing.assert_allclose(D[:, 0], [2 / 3, -1 / 3, -1 / 3], rtol=1e-14)
    assert np.linalg.norm(D[:, 1]) <= 1e-12
    assert np.abs(AE @ D).max() <= 1e-9


def test_reprojection_kat(orc):
    # proj/tests/test_projection.cpp:128-144
    _, _, AE, bE = orc.make_simplex(3)
    _, P, G = orc.compute_projection(AE)
    kept = orc.reproject(AE, G, bE, np.array([[0.2], [0.3], [0.5]]))
    assert np.abs(kept[:, 0] - [0.2, 0.3, 0.5]).max() <= 1e-12
    fixed = orc.reproject(AE, G, bE, np.array([[0.4], [0.4], [0.4]]))
    np.testing.assert_allclose(fixed[:, 0], [1 / 3] * 3, rtol=1e-14)
    assert abs(fixed.sum() - 1.0) <= 1e-10


def test_reprojection_columns_independent(orc):
    # proj/tests/test_projection.cpp:146-160
    s = orc.Stream(23, 0)
    AE = np.array([[2.0 * s.next_uniform() - 1.0 for _ in range(6)] for _ in range(2)])
    bE = np.array([0.5, -1.0])
    _, _, G = orc.compute_projection(AE)
    batch = np.asfortranarray(np.array([[2.0 * s.next_uniform() - 1.0 for _ in range(3)]
                                        for _ in range(6)]))
    allx = orc.reproject(AE, G, bE, batch)
    for k in range(3):
        single = orc.reproject(AE, G, bE, batch[:, k:k + 1])
        assert np.array_equal(allx[:, k], single[:, 0])
        assert np.abs(AE @ allx[:, k] - bE).max() <= 1e-10


def test_contains_semantics(orc):
    # proj/tests/test_polytope.cpp:65-83
    A, b = orc.make_hypercube(3)
    assert orc.contains(A, b, np.zeros(3), 1e-9)
    assert not orc.contains(A, b, np.array([1.001, 0, 0]), 1e-9)
    A, b, AE, bE = orc.make_simplex(3)
    assert orc.contains(A, b, np.full(3, 1 / 3), 1e-9, AE, bE)
    assert not orc.contains(A, b, np.full(3, 0.5), 1e-9, AE, bE)
    A, b = orc.make_hypercube(2)
    x = np.array([1.0 + 1e-7, 0.0])
    assert not orc.contains(A, b, x, 1e-9) and orc.contains(A, b, x, 1e-6)


# ----------------------------------------------------------------- step -----

def test_steps_stay_inside_box(orc):
    # proj/tests/test_sampler.cpp:217-228
    A, b = orc.make_hypercube(4)
    rng = orc.WalkRng(0, 6)
    X = np.zeros((4, 6), order="F")
    for _ in range(50):
        st, _, _ = orc.step(A, b, None, EPS_DIR, rng, X)
        assert st == 0
        for k in range(6):
            assert orc.contains(A, b, X[:, k], 1e-12)


def test_projected_steps_stay_on_slice(orc):
    # proj/tests/test_sampler.cpp:230-242
    A, b, AE, bE = orc.make_simplex(5)
    _, P, _ = orc.compute_projection(AE)
    rng = orc.WalkRng(0, 4)
    X = np.asfortranarray(np.full((5, 4), 0.2))
    for _ in range(200):
        assert orc.step(A, b, P, EPS_DIR, rng, X)[0] == 0
    for k in range(4):
        assert abs(X[:, k].sum() - 1.0) <= 1e-9
        assert orc.contains(A, b, X[:, k], 1e-9, AE, bE)


def test_retry_exhausted_after_16(orc):
    # proj/tests/test_sampler.cpp:244-258
    A, b = orc.make_hypercube(2)
    rng = orc.WalkRng(55, 1)
    X = np.zeros((2, 1), order="F")
    st, redraws, err = orc.step(A, b, None, 1e9, rng, X)
    assert st == 9 and redraws == 16 and err == 0


@pytest.mark.parametrize("body", ["box", "simplex"])
def test_z1_engine_matches_scalar_walk(orc, body):
    # proj/tests/test_sampler.cpp:413-485 (acceptance #2 at 1e3 steps)
    seed, steps = 4242, 1000
    if body == "box":
        A, b = orc.make_hypercube(5)
        P = None
        x = [0.0] * 5
        walk = ScalarWalk(A.tolist(), b.tolist())
    else:
        A, b, AE, _ = orc.make_simplex(4)
        _, P, _ = orc.compute_projection(AE)
        x = [0.25] * 4
        walk = ScalarWalk(A.tolist(), b.tolist(), P.tolist())
    rng = orc.WalkRng(seed, 1)
    X = np.asfortranarray(np.array(x)[:, None])
    col, theta = orc.Stream(seed, 0), orc.Stream(seed, oracle.THETA_STREAM_ID)
    worst = 0.0
    for _ in range(steps):
        assert orc.step(A, b, P, EPS_DIR, rng, X)[0] == 0
        assert walk.advance(col, theta, x, EPS_DIR)
        worst = max(worst, max(abs(X[j, 0] - x[j]) for j in range(len(x))))
    assert worst <= 1e-12


def test_theta_uniform_along_chord(orc):
    # proj/tests/test_sampler.cpp:199-215 via the injected step: U is the chord
    # position, so theta maps affinely; KS on the reference stream's uniforms.
    A, b = orc.make_hypercube(2)
    s = orc.Stream(54, oracle.THETA_STREAM_ID)
    reps = 4000
    U = np.array([s.next_uniform() for _ in range(reps)])
    X = np.zeros((2, reps), order="F")
    H = np.asfortranarray(np.tile([[1.0], [0.0]], (1, reps)))
    st, Xn, lo, hi, th, fl, _ = orc.step_injected(A, b, None, EPS_DIR, X, H, U)
    assert st == 0 and np.all(lo == -1.0) and np.all(hi == 1.0)
    u = (Xn[0] + 1.0) / 2.0
    assert ks_statistic_uniform(list(u)) < 1.63 / math.sqrt(reps)


def test_injected_step_semantics(orc):
    A, b = orc.make_hypercube(2)
    X = np.zeros((2, 3), order="F")
    H = np.asfortranarray([[1.0, 0.0, 1.0], [0.0, 0.0, 1.0]])
    U = np.array([0.5, 0.3, 0.0])
    st, Xn, lo, hi, th, fl, _ = orc.step_injected(A, b, None, EPS_DIR, X, H, U)
    assert st == 0
    assert fl[0] == 6 and th[0] == 0.0  # both sides, theta = midpoint of (-1, 1)
    assert fl[1] & 1 and np.all(Xn[:, 1] == 0.0)  # zero direction: degenerate, unmoved
    assert fl[2] & 16 and th[2] == 0.0  # u = 0 hits the endpoint -> midpoint


# ------------------------------------------------------------------ run ------

def test_run_counting(orc):
    # proj/tests/test_sampler.cpp:260-286 (warm start at the centre 0)
    A, b = orc.make_hypercube(3)
    st, S, stats = orc.run(A, b, np.zeros(3), z=2, phi=3, t_target=4, burn_in=0,
                           reproject_every=3, seed=7)
    assert st == 0 and S.shape == (4, 3) and stats.windows == 2 and stats.iterate_count == 12
    for row in S:
        assert orc.contains(A, b, row, 1e-9)
    st, S, stats = orc.run(A, b, np.zeros(3), z=2, phi=3, t_target=3, burn_in=0,
                           reproject_every=3, seed=7)
    assert S.shape == (4, 3) and stats.windows == 2


def test_run_reproducible_per_seed(orc):
    # proj/tests/test_sampler.cpp:288-302
    A, b = orc.make_hypercube(4)
    kw = dict(z=3, phi=10, t_target=30, burn_in=10, reproject_every=10)
    _, a1, _ = orc.run(A, b, np.zeros(4), seed=99, **kw)
    _, a2, _ = orc.run(A, b, np.zeros(4), seed=99, **kw)
    _, c, _ = orc.run(A, b, np.zeros(4), seed=100, **kw)
    assert np.array_equal(a1, a2) and np.abs(a1 - c).max() > 0


def test_box_moments(orc):
    # proj/tests/test_sampler.cpp:320-336
    A, b = orc.make_hypercube(5)
    st, S, _ = orc.run(A, b, np.zeros(5), z=100, phi=125, t_target=10000, burn_in=125,
                       reproject_every=125, seed=11)
    assert st == 0 and S.shape[0] == 10000
    assert np.abs(S.mean(0)).max() <= 0.05
    assert np.abs(S.var(0, ddof=1) - 1 / 3).max() <= 0.05


def test_simplex_moments_and_drift(orc):
    # proj/tests/test_sampler.cpp:338-356 and :380-392
    A, b, AE, bE = orc.make_simplex(3)
    st, S, _ = orc.run(A, b, np.full(3, 1 / 3), z=100, phi=8, t_target=5000, burn_in=8,
                       reproject_every=8, seed=12, AE=AE, bE=bE)
    assert st == 0
    assert np.abs(S.mean(0) - 1 / 3).max() <= 0.02
    assert np.abs(S.sum(1) - 1.0).max() <= 1e-8
    A, b, AE, bE = orc.make_simplex(8)
    st, S, _ = orc.run(A, b, np.full(8, 1 / 8), z=20, phi=50, t_target=500, burn_in=50,
                       reproject_every=50, seed=14, AE=AE, bE=bE)
    assert st == 0 and np.abs(S.sum(1) - 1.0).max() <= 1e-9


def test_philox4x32_10_known_answers(orc):
    # Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11): the authors'
    # published known-answer vectors (Random123 kat_vectors, philox4x32 10
    # rounds).  The engine's production-mode draws and oracle.step_philox
    # rest on this function.
    assert orc.philox4x32_10([0, 0, 0, 0], [0, 0]) == [0x6627E8D5, 0xE169C58D, 0xBC57AC4C,
                                                       0x9B00DBD8]
    assert orc.philox4x32_10([0xFFFFFFFF] * 4, [0xFFFFFFFF] * 2) == [0x408F276D, 0x41C83B0E,
                                                                     0xA20BC7C6, 0x6D5451FD]
    assert orc.philox4x32_10([0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344],
                             [0xA4093822, 0x299F31D0]) == [0xD16CFE09, 0x94FDCCEB, 0x5001E420,
                                                           0x24126EA1]


def test_philox_step_is_the_reference_step_on_philox_draws(orc):
    # orc_step_philox == orc_step_injected fed the same Philox normals and
    # the first theta draw (no redraws / rejections on this body): only the
    # random source differs from the reference step
    import numpy as np
    from paper_2104_07097_b200 import workloads
    p = workloads.random_polytope(9, 60, seed=3)
    z, seed, off, it = 7, 5, 11, 3
    X = np.zeros((9, z), order="F")
    H = np.stack([orc.philox_normals(seed, off + k, it, 0, 9) for k in range(z)], 1)
    import ctypes as C
    U = np.empty(z)
    for k in range(z):
        a, b = C.c_uint64(), C.c_uint64()
        orc.lib().orc_philox_u64x2(seed, 0, off + k, it, 0, 1, C.byref(a), C.byref(b))
        U[k] = (a.value >> 11) * 2.0 ** -53
    st, Xi, *_ = orc.step_injected(p.a_in, p.b_in, None, 1e-11, X, H, U)
    Xp = X.copy(order="F")
    st2, red, _ = orc.step_philox(p.a_in, p.b_in, None, 1e-11, seed, off, it, Xp)
    assert st == 0 and st2 == 0 and red == 0
    assert np.array_equal(Xi, Xp)
