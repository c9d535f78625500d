import os, sys
import numpy as np
sys.path.insert(0, '.')
import paper_2104_07097_b200 as mh
from paper_2104_07097_b200 import workloads
p = workloads.random_polytope(200, 6000, seed=21)
z = 512
X0 = np.zeros((200, z), order="F")
for e in sys.argv[1:]:
    eng = mh.Engine(p, z, seed=9, f64_engine=e, refresh_every=16)
    eng.set_state(X0)
    eng.step(1)
    _, lo, hi, _ = eng.debug_last_iterate()
    eng.step(5)
    _, lo5, hi5, _ = eng.debug_last_iterate()
    eng.close()
    print(os.environ.get("MHAR_POISON", "-"), e, round(float(hi.sum()), 6), round(float(lo.sum()), 6), round(float(hi5.sum()), 6), flush=True)
