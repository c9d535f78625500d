"""Determinism of iterate 0 bounds across engine pairs / reps."""
import sys
import numpy as np
sys.path.insert(0, '.')
import paper_2104_07097_b200 as mh
from paper_2104_07097_b200 import workloads

p = workloads.random_polytope(200, 6000, seed=21)
z = 512
X0 = np.zeros((200, z), order="F")


def bounds(eng):
    eng.set_state(X0)
    eng.step(1)
    _, lo, hi, _ = eng.debug_last_iterate()
    return lo, hi


for combo in [("dmma",), ("int8",), ("dmma", "dmma"), ("int8", "int8"), ("dmma", "int8")]:
    seen = []
    for r in range(8):
        engs = [mh.Engine(p, z, seed=9, f64_engine=e, refresh_every=16) for e in combo]
        res = [bounds(e) for e in engs]
        for e in engs:
            e.close()
        for lo, hi in res:
            key = (round(float(hi[0]), 9), round(float(lo[0]), 9), round(float(hi.sum()), 6))
            if key not in seen:
                seen.append(key)
    print(combo, "distinct iterate-0 outcomes:", len(seen), seen[:4], flush=True)
