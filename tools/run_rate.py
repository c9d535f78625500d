"""run() end to end on config 5 (the reference's own bench rate z*phi*windows/time,
proj/src/bench.cpp:20-35): burn-in, windows of phi iterates, containment check
and collection of every walk per window (samples copied to the host)."""
import json, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_07097_b200 as mh
from paper_2104_07097_b200 import workloads

w = workloads.config(5)
phi = int(sys.argv[1]) if len(sys.argv) > 1 else 64
windows = int(sys.argv[2]) if len(sys.argv) > 2 else 2
for engine in ["dmma", "int8", "fp32"]:
    kw = dict(precision=32) if engine == "fp32" else dict(f64_engine=engine)
    with mh.Engine(w.polytope, w.z, seed=7, **kw) as eng:
        eng.run(w.x0, 2, 1, 0, 0)  # warm-up
        t0 = time.perf_counter()
        S, st = eng.run(w.x0, phi, windows, 0, 0)
        wall = time.perf_counter() - t0
    print(json.dumps({"engine": engine, "phi": phi, "windows": windows, "walks": w.z,
                      "device_seconds": st.seconds, "wall_seconds": wall,
                      "chain_steps_per_s_device": w.z * phi * windows / st.seconds,
                      "chain_steps_per_s_wall": w.z * phi * windows / wall,
                      "samples_shape": list(S.shape)}), flush=True)
