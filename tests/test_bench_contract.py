"""The bench.py contract the driver depends on, checked on CPU: the reference
arm (`--impl reference`, the CPU restatement of the reference step timed on
the host cores) prints one JSON line with the base keys, and the roofline
helpers read the committed peaks and ncu captures."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run(
        [sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "3",
         "--steps", "1", "--warmup", "3", "--cpu-walks", "8"],
        cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "dtype", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["steps"] == 1 and d["warmup"] == 3
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["cores"] >= 1
    assert d["config"]["workload"].startswith("random n=500")


def test_roofline_peaks_and_traffic_are_committed():
    sys.path.insert(0, ROOT)
    import bench
    assert 30.0 < bench.fp64_peak() < 45.0          # DMMA TFLOP/s
    assert 3000.0 < bench.int8_dense_peak() < 5000.0  # int8 TOPS
    assert 800.0 < bench.tf32_dense_peak() < 1300.0   # TF32 TFLOP/s
    assert 1600.0 < bench.f16_dense_peak() < 2600.0   # FP16 TFLOP/s
    for cap in ("chord2_full", "tc32_full", "i8_full"):
        t = bench.ncu_traffic(cap)
        assert t is not None and t > 1.0


def test_reference_arm_under_torchrun_two_ranks():
    # the driver launches the reference arm like the engine arm: rank 0
    # prints the one line, rank 1 exits 0 without work or a device
    out = subprocess.run(
        [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
         "--master-addr", "127.0.0.1", "--master-port", "29533", os.path.join(ROOT, "bench.py"),
         "--impl", "reference", "--gpus", "2", "--config", "3", "--steps", "1", "--warmup", "3",
         "--cpu-walks", "8"],
        cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
