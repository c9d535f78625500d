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


def test_bench_csv_and_json_formats(tmp_path):
    # proj/tests/test_io.cpp throughput cases
    r = mh.BenchRecord(figure="hypercube(50)", n=50, z=16, phi=1000, windows=1,
                       total_samples=16000, run_seconds=[1.0, 2.0], run_sps=[16000.0, 8000.0],
                       mean_sps=12000.0, std_sps=4000.0)
    header = "figure,n,z,phi,windows,total_samples,mean_sps,std_sps,runs\n"
    text = mh.bench_csv_string([r])
    assert text == header + "hypercube(50),50,16,1000,1,16000,12000,4000,2\n"
    assert mh.bench_csv_string([]) == header
    q = mh.BenchRecord(figure="simplex(10)", n=10, z=4, phi=729, windows=2, total_samples=5832,
                       run_seconds=[0.5, 0.25, 0.125], run_sps=[11664.0, 23328.0, 46656.0],
                       mean_sps=27216.0, std_sps=17750.0)
    import json
    doc = json.loads(mh.bench_json_string([q]))
    assert doc["format_version"] == 1 and len(doc["records"]) == 1
    rec = doc["records"][0]
    assert rec["figure"] == "simplex(10)" and len(rec["run_seconds"]) == 3
    assert rec["run_sps"][2] == 46656.0 and rec["mean_sps"] == 27216.0
    p = tmp_path / "bench.json"
    mh.write_bench_json(str(p), [q])
    assert json.loads(p.read_text()) == doc
    with pytest.raises(mh.MharError) as e:
        mh.write_bench_csv("/nonexistent/dir/b.csv", [q])
    assert e.value.code == mh.ErrorCode.io_failure
