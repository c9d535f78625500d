"""fp32 variant at large walk counts (config 5): chain-steps/s against z, with
and without the walk-pair bands (MHAR_TC_WALK_BAND=0 disables them)."""
import json, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_07097_b200 as mh
from paper_2104_07097_b200 import workloads

w = workloads.config(5, z=4096)
p = w.polytope
for z in [int(a) for a in sys.argv[1:]] or [4096, 16384]:
    for direction in ("split", "rounded"):
        with mh.Engine(p, z, seed=5, precision=32, fp32_direction=direction) as eng:
            eng.set_state(np.zeros((p.dim(), z), order="F"))
            eng.step_timed(4)
            ms = eng.step_timed(5)
            bad, viol, _ = eng.check_state(1e-9)
        print(json.dumps({"z": z, "direction": direction,
                          "walk_band_env": os.environ.get("MHAR_TC_WALK_BAND"),
                          "chain_steps_per_s": z * 5 / (ms * 1e-3), "ms_per_iterate": ms / 5,
                          "first_bad": int(bad), "max_violation": float(np.max(viol))}), flush=True)
