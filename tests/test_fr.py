"""Two-sample tree test: the oracle restatement of
proj/src/stats.cpp pinned to the reference's own cases
(proj/tests/test_stats.cpp, acceptance #7), and the GPU implementation
against the oracle and the reference's acceptance #3 gate."""
import itertools

import numpy as np
import pytest

import oracle


# ------------------------------------------------------------ oracle (CPU) --

def test_fr_hand_instance(orc):
    # proj/tests/test_stats.cpp:137-148, acceptance_main.cpp:333-345
    st, r = orc.friedman_rafsky(np.array([0.0, 10.0]), np.array([1.0, 11.0]))
    assert st == 0 and r.cross_edges == 3 and r.expected_cross == 3.0
    assert r.variance_cross == 2.0 / 3.0 and r.z_value == 0.0 and r.shared_end_pairs == 2


def test_mst_collinear_and_two_points(orc):
    # proj/tests/test_stats.cpp:65-90
    a, b, w = orc.minimum_spanning_tree(np.array([0.0, 3.0, 1.0, 6.0]))
    assert sorted(zip(a.tolist(), b.tolist())) == [(0, 2), (1, 3), (2, 1)]
    assert sorted(w.tolist()) == [1.0, 2.0, 3.0]
    a, b, w = orc.minimum_spanning_tree(np.array([[0.0, 0.0], [3.0, 4.0]]))
    assert (a[0], b[0], w[0]) == (0, 1, 5.0)


def test_mst_matches_exhaustive_tiny_trees(orc):
    # proj/tests/test_stats.cpp:91-104: the minimum over all spanning trees
    rng = np.random.default_rng(3)
    for _ in range(20):
        P = rng.uniform(0, 1, (5, 2))
        _, _, w = orc.minimum_spanning_tree(P)
        D = np.linalg.norm(P[:, None] - P[None], axis=2)
        best = np.inf
        for edges in itertools.combinations(list(itertools.combinations(range(5), 2)), 4):
            parent = list(range(5))

            def find(x):
                while parent[x] != x:
                    x = parent[x]
                return x
            ok = True
            for i, j in edges:
                ri, rj = find(i), find(j)
                if ri == rj:
                    ok = False
                    break
                parent[ri] = rj
            if ok:
                best = min(best, sum(D[i, j] for i, j in edges))
        assert abs(w.sum() - best) <= 1e-12


def test_mst_duplicates_zero_weight(orc):
    # proj/tests/test_stats.cpp:123-135
    P = np.array([[1.0, 1.0], [1.0, 1.0], [2.0, 1.0], [1.0, 1.0]])
    _, _, w = orc.minimum_spanning_tree(P)
    assert sorted(w.tolist()) == [0.0, 0.0, 1.0]


def test_fr_separated_symmetric_degenerate(orc):
    # proj/tests/test_stats.cpp:150-192, 194-210
    rng = np.random.default_rng(4)
    a = rng.normal(0, 1, (60, 3))
    b = rng.normal(20, 1, (50, 3))
    st, r = orc.friedman_rafsky(a, b)
    assert st == 0 and r.z_value < -5
    st2, r2 = orc.friedman_rafsky(b, a)
    assert r2.cross_edges == r.cross_edges and abs(r2.z_value - r.z_value) < 1e-12
    assert orc.friedman_rafsky(a[:1], b)[0] == 11


# ------------------------------------------------------------------- GPU ----

@pytest.mark.gpu
@pytest.mark.parametrize("N,n", [(50, 1), (400, 3), (3000, 10)])
def test_gpu_mst_equals_oracle(orc, N, n):
    from paper_2104_07097_b200 import stats
    P = np.random.default_rng(N + n).uniform(-1, 1, (N, n))
    ga, gb, gw = stats.minimum_spanning_tree(P)
    oa, ob, ow = orc.minimum_spanning_tree(P)
    assert np.array_equal(ga, oa) and np.array_equal(gb, ob) and np.array_equal(gw, ow)


@pytest.mark.gpu
@pytest.mark.parametrize("form", ["cta", "grid", "grid_l2"])
@pytest.mark.parametrize("case", ["lattice_ties", "wide", "ragged"])
def test_gpu_mst_forms_equal_oracle(orc, monkeypatch, form, case):
    # both Prim forms (one CTA; cooperative grid over every SM) edge for edge
    # against the oracle: an integer lattice with many equal distances (the
    # tie rule), n beyond the staged-coordinate limit, a ragged pool size
    from paper_2104_07097_b200 import stats
    rng = np.random.default_rng(len(case))
    if case == "lattice_ties":
        P = rng.integers(0, 12, (4000, 2)).astype(np.float64)
    elif case == "wide":
        P = rng.uniform(-1, 1, (300, 4500))
    else:
        P = rng.standard_normal((5003, 7))
    monkeypatch.setenv("MHAR_PRIM", form)
    ga, gb, gw = stats.minimum_spanning_tree(P)
    oa, ob, ow = orc.minimum_spanning_tree(P)
    assert np.array_equal(ga, oa) and np.array_equal(gb, ob) and np.array_equal(gw, ow)


@pytest.mark.gpu
def test_gpu_fr_kats_and_oracle(orc):
    import paper_2104_07097_b200 as mh
    from paper_2104_07097_b200 import stats
    r = stats.friedman_rafsky(np.array([0.0, 10.0]), np.array([1.0, 11.0]))
    assert (r.cross_edges, r.expected_cross, r.variance_cross, r.z_value, r.shared_end_pairs) == \
        (3, 3.0, 2.0 / 3.0, 0.0, 2)
    rng = np.random.default_rng(9)
    a, b = rng.uniform(-1, 1, (700, 6)), rng.uniform(-1, 1, (500, 6))
    g = stats.friedman_rafsky(a, b)
    st, o = orc.friedman_rafsky(a, b)
    assert st == 0 and g.cross_edges == o.cross_edges and g.z_value == o.z_value
    with pytest.raises(mh.MharError) as e:
        stats.friedman_rafsky(a[:1], b)
    assert e.value.code == mh.ErrorCode.degenerate_test


@pytest.mark.gpu
def test_acceptance3_uniformity_screening():
    # proj/tests/acceptance_main.cpp:160-203: engine samples (z = 100, phi =
    # walk_dim^3, 5000 points) against 5000 direct uniform draws, 10 seeds per
    # body; a body passes when at least 9 of 10 runs score z >= -1.64.
    import paper_2104_07097_b200 as mh
    from paper_2104_07097_b200 import stats
    for c, (fig, n) in enumerate([("hypercube", 5), ("hypercube", 15), ("hypercube", 25),
                                  ("simplex", 5), ("simplex", 15), ("simplex", 25)]):
        cube = fig == "hypercube"
        p = mh.make_hypercube(n) if cube else mh.make_simplex(n)
        walk_dim = n if cube else n - 1
        x0 = np.zeros(n) if cube else np.full(n, 1.0 / n)
        ok = 0
        for rep in range(10):
            seed = 1000 * (c + 1) + rep
            cfg = mh.SamplerConfig(z=100, phi=walk_dim ** 3, t_target=5000, burn_in=0, seed=seed)
            S = mh.run(p, cfg, x0=x0).samples
            rng = np.random.default_rng(seed)
            ref = (stats.sample_uniform_hypercube(rng, n, 5000) if cube
                   else stats.sample_uniform_simplex(rng, n, 5000))
            if stats.friedman_rafsky(S, ref).z_value >= stats.kUniformityZThreshold:
                ok += 1
        assert ok >= 9, f"{fig}({n}): {ok}/10"
