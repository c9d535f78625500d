"""chord2 vs chord3 across the dimension n (m = 20000 unit-norm rows, 4096
walks): average incremental chord launch time and fraction of the DMMA peak.
Behind the n_pad threshold that selects chord3 (csrc/abi.cu)."""
import json, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_07097_b200 as mh
from paper_2104_07097_b200 import workloads

PEAK = 37.061  # TFLOP/s, profiles/fp64_peaks_r01.json
m, z = int(os.environ.get("SWEEP_M", 20000)), int(os.environ.get("SWEEP_Z", 4096))
for n in [int(a) for a in sys.argv[1:]] or [64, 128, 256, 384, 512, 768]:
    p = workloads.random_polytope(n, m, seed=n)
    for flag in ("0", "1"):
        os.environ["MHAR_CHORD3"] = flag
        with mh.Engine(p, z, seed=3, small_path=False) as eng:
            eng.set_state(np.zeros((n, z), order="F"))
            eng.step(3)
            eng.set_timing(True)
            eng.reset_stats()
            eng.step(10)
            st = eng.stats()
        ms = st["chord_ms"] / max(st["chord_timed"], 1)
        tf = st["chord_flops"] / max(st["chord_ms"] * 1e-3, 1e-30) / 1e12
        print(json.dumps({"n": n, "m": m, "z": z, "kernel": st["chord_kernel"],
                          "avg_launch_ms": ms, "tflops": tf, "frac": tf / PEAK}), flush=True)
