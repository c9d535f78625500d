"""Find the first iterate where the int8-slice engine leaves the DMMA trajectory."""
import sys
import numpy as np
sys.path.insert(0, '.')
import paper_2104_07097_b200 as mh
from paper_2104_07097_b200 import workloads

p = workloads.random_polytope(200, 6000, seed=21)
z = 512
X0 = np.zeros((200, z), order="F")
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
for r in range(reps):
    ed = mh.Engine(p, z, seed=9, f64_engine="dmma", refresh_every=16)
    ei = mh.Engine(p, z, seed=9, f64_engine="int8", refresh_every=16)
    ed.set_state(X0); ei.set_state(X0)
    for t in range(40):
        ed.step(1)
        try:
            ei.step(1)
        except mh.MharError as e:
            print(f"rep {r} iterate {t}: {e}", flush=True)
            break
        a, b = ed.get_state(), ei.get_state()
        d = np.abs(a - b).max(0)
        if d.max() > 1e-10:
            w = np.nonzero(d > 1e-10)[0]
            print(f"rep {r} iterate {t}: {len(w)} walks off, first {w[:16]}, max {d.max():.3e}", flush=True)
            Dd, lod, hid, thd = ed.debug_last_iterate()
            Di, loi, hii, thi = ei.debug_last_iterate()
            dd = np.abs(Dd - Di).max(0) / np.abs(Dd).max(0)
            print(f"   D rel diff: max {dd.max():.3e}, walks > 1e-12: {(dd > 1e-12).sum()}", flush=True)
            print(f"   lower diff max {np.abs(lod - loi).max():.3e} upper {np.abs(hid - hii).max():.3e} theta {np.abs(thd - thi).max():.3e}", flush=True)
            k = w[0]
            print(f"   walk {k}: dmma lo {lod[k]:.6f} hi {hid[k]:.6f} th {thd[k]:.6f} | int8 lo {loi[k]:.6f} hi {hii[k]:.6f} th {thi[k]:.6f}", flush=True)
            print(f"   D walk {k} dmma {Dd[:4, k]} int8 {Di[:4, k]}", flush=True)
            break
    ed.close(); ei.close()
print("done", flush=True)
