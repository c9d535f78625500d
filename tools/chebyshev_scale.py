"""Times the GPU Chebyshev-centre LP on the BASELINE configs and checks the
centre's margin to every row (prints one JSON line per config)."""
import json
import sys
import time

import os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2104_07097_b200 as mh
from paper_2104_07097_b200 import workloads


def main(configs):
    for idx in configs:
        p = workloads.config(idx).polytope
        t0 = time.perf_counter()
        c = mh.chebyshev_center(p)
        dt = time.perf_counter() - t0
        norms = np.linalg.norm(p.a_in, axis=1)
        margin = float(((p.b_in - p.a_in @ c.x) / norms).min())
        eq = float(np.abs(p.a_eq @ c.x - p.b_eq).max()) if p.num_equalities() else 0.0
        print(json.dumps({"config": idx, "n": p.dim(), "m_in": p.num_inequalities(),
                          "m_eq": p.num_equalities(), "seconds": round(dt, 3),
                          "radius": c.radius, "min_margin": margin, "eq_residual": eq,
                          "rounds": c.rounds, "pivots": c.pivots,
                          "working_rows": c.working_rows}), flush=True)


if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]] or [1, 2, 3, 4, 5])
