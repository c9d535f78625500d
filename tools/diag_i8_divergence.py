import numpy as np, sys
sys.path.insert(0, '.')
import paper_2104_07097_b200 as mh
from paper_2104_07097_b200 import workloads
p = workloads.random_polytope(200, 6000, seed=21)
z = 512
X0 = np.zeros((200, z), order="F")
for its in [5, 10, 20, 40]:
    out = {}
    for name, kw in [("dmma", dict(f64_engine="dmma")), ("int8", dict(f64_engine="int8")), ("recomp", dict(slack="recompute"))]:
        with mh.Engine(p, z, seed=9, refresh_every=16, **kw) as eng:
            eng.set_state(X0)
            eng.step(its)
            out[name] = eng.get_state()
    d1 = np.abs(out["int8"] - out["dmma"]).max(0)
    d2 = np.abs(out["recomp"] - out["dmma"]).max(0)
    q = lambda d: [float(np.quantile(d, t)) for t in (0.5, 0.9, 0.99, 1.0)] + [int((d > 1e-9).sum())]
    print(its, "int8-vs-dmma", q(d1), "recompute-vs-dmma", q(d2), flush=True)
