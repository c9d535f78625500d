"""One body of the paper table, a few iterates, for an ncu launch list."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_07097_b200 as mh
fig, n, z = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
small = (sys.argv[4] != "0") if len(sys.argv) > 4 else True  # 0: force the multi-kernel path
p = mh.make_hypercube(n) if fig == "hypercube" else mh.make_simplex(n)
x0 = np.zeros(n) if fig == "hypercube" else np.full(n, 1.0 / n)
proj = mh.compute_projection(p.a_eq) if p.num_equalities() else None
with mh.Engine(p, z, seed=1, projector=proj, small_path=small) as eng:
    eng.run(x0, 5, 1, 0, 5 if proj else 0)
    _, st = eng.run(x0, 200, 1, 0, 200 if proj else 0)
    print("us per iterate", 1e6 * st.seconds / 200)
