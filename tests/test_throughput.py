"""The reference's throughput harness (proj/src/bench.cpp:9-61) on the
engine: measure_throughput / sweep_padding with the reference's scripted-clock
cases (proj/tests/test_bench.cpp) and acceptance check #8, "padding raises
throughput" (proj/tests/acceptance_main.cpp:349-375)."""
import pytest

import paper_2104_07097_b200 as mh


def scripted(instants):
    it = iter(instants)
    return lambda: next(it)


def test_non_positive_counts_are_rejected():
    cube = mh.make_hypercube(2)
    cfg = mh.BenchConfig(repetitions=0)
    with pytest.raises(mh.MharError) as e:
        mh.measure_throughput(cube, 1, cfg, "hypercube(2)")
    assert e.value.code == mh.ErrorCode.invalid_argument
    cfg.repetitions = 1
    with pytest.raises(mh.MharError):
        mh.measure_throughput(cube, 0, cfg, "hypercube(2)")
    with pytest.raises(mh.MharError) as e:
        mh.sweep_padding(cube, [], cfg, "hypercube(2)")
    assert e.value.code == mh.ErrorCode.invalid_argument


@pytest.mark.gpu
def test_scripted_thousand_seconds():
    cfg = mh.BenchConfig(phi=30000, windows=1, repetitions=1, seed=3)
    r = mh.measure_throughput(mh.make_hypercube(2), 100, cfg, "hypercube(2)",
                              clock=scripted([0.0, 1000.0]))
    assert r.total_samples == 3000000
    assert r.run_seconds == [1000.0] and r.mean_sps == 3000.0 and r.std_sps == 0.0


@pytest.mark.gpu
def test_equal_durations_zero_spread_and_exact_rates():
    cube = mh.make_hypercube(3)
    r = mh.measure_throughput(cube, 4, mh.BenchConfig(phi=5, windows=2, repetitions=3),
                              "hypercube(3)", clock=scripted([0, 2, 10, 12, 20, 22]))
    assert len(r.run_sps) == 3 and r.std_sps == 0.0 and r.mean_sps == r.run_sps[0]
    r = mh.measure_throughput(cube, 5, mh.BenchConfig(phi=7, windows=3, repetitions=2),
                              "hypercube(3)", clock=scripted([0, 4, 0, 8]))
    assert r.total_samples == 5 * 7 * 3
    assert all(r.run_sps[k] == r.total_samples / r.run_seconds[k] for k in range(2))
    assert r.mean_sps == (r.run_sps[0] + r.run_sps[1]) / 2.0


@pytest.mark.gpu
def test_one_element_sweep_equals_direct_and_one_record_per_z():
    simplex = mh.make_simplex(3)
    cfg = mh.BenchConfig(phi=4, windows=1, repetitions=2, seed=9)
    d = mh.measure_throughput(simplex, 2, cfg, "simplex(3)", clock=scripted([0, 1, 1, 3]))
    s = mh.sweep_padding(simplex, [2], cfg, "simplex(3)", clock=scripted([0, 1, 1, 3]))
    assert len(s) == 1 and s[0] == d
    recs = mh.sweep_padding(mh.make_hypercube(4), [1, 2, 4],
                            mh.BenchConfig(phi=2, windows=1, repetitions=1), "hypercube(4)",
                            clock=scripted([0, 1, 0, 1, 0, 1]))
    assert [r.z for r in recs] == [1, 2, 4]


@pytest.mark.gpu
def test_acceptance8_padding_raises_throughput():
    cfg = mh.BenchConfig(phi=1000, windows=1, repetitions=5, seed=20240818)
    cube = mh.make_hypercube(50)
    narrow = mh.measure_throughput(cube, 1, cfg, "hypercube(50)")
    wide = mh.measure_throughput(cube, 16, cfg, "hypercube(50)")
    assert wide.mean_sps >= narrow.mean_sps
    assert narrow.total_samples == 1000 and wide.total_samples == 16000
