"""Stress: repeated DMMA vs int8-slice trajectories (determinism / race hunt)."""
import sys, time
import numpy as np
sys.path.insert(0, '.')
import paper_2104_07097_b200 as mh
from paper_2104_07097_b200 import workloads

p = workloads.random_polytope(200, 6000, seed=21)
z = 512
X0 = np.zeros((200, z), order="F")
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20


def traj(name, its=40, per_step=False):
    with mh.Engine(p, z, seed=9, f64_engine=name, refresh_every=16) as eng:
        eng.set_state(X0)
        if not per_step:
            eng.step(its)
            return eng.get_state()
        out = []
        for _ in range(its):
            eng.step(1)
            out.append(eng.get_state())
        return out


ref_d = traj("dmma")
ref_i = traj("int8")
bad = 0
for r in range(reps):
    for name, ref in (("dmma", ref_d), ("int8", ref_i)):
        try:
            x = traj(name)
        except mh.MharError as e:
            bad += 1
            print(f"rep {r} {name}: {e}", flush=True)
            continue
        d = np.abs(x - ref).max(0)
        if d.max() > 0:
            bad += 1
            print(f"rep {r} {name}: nondeterministic, walks differing: {(d > 0).sum()}, max {d.max():.3e}",
                  flush=True)
            # find the first iterate where it differs
            a = traj(name, per_step=True)
            b = traj(name, per_step=True)
            for t in range(40):
                dd = np.abs(a[t] - b[t]).max(0)
                if dd.max() > 0:
                    print(f"   first differing iterate {t}: walks {np.nonzero(dd)[0][:20]} max {dd.max():.3e}",
                          flush=True)
                    break
print("cross", float(np.abs(ref_d - ref_i).max()), "nondeterministic runs:", bad, flush=True)
