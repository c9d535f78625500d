"""Large walk counts on one B200 (config 5): the slack/rate caches grow to
m_I x z x 16 B (52 GB at z = 16384, 105 GB at z = 32768); checks 64-bit
indexing, containment after the timed iterates, and the rate per engine."""
import json, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_07097_b200 as mh
from paper_2104_07097_b200 import workloads

cases = [("dmma", 64, 16384), ("int8", 64, 16384), ("dmma", 32, 16384), ("dmma", 64, 32768)]
w = workloads.config(5, z=4096)
p = w.polytope
for eng_name, prec, z in cases:
    t0 = time.perf_counter()
    with mh.Engine(p, z, seed=5, precision=prec, f64_engine=eng_name) as eng:
        eng.set_state(np.zeros((p.dim(), z), order="F"))
        eng.step_timed(4)
        ms = eng.step_timed(5)
        bad, viol, _ = eng.check_state(1e-9)
        X = eng.get_state()
    print(json.dumps({"engine": eng_name, "precision": prec, "z": z,
                      "chain_steps_per_s": z * 5 / (ms * 1e-3), "ms_per_iterate": ms / 5,
                      "first_bad": int(bad), "max_violation": float(np.max(viol)),
                      "moved": float(np.abs(X).max()), "wall_s": time.perf_counter() - t0}),
          flush=True)
