"""Long runs of every engine on BASELINE configs 3, 4 (and 5 with SOAK_CFGS):
containment and equality residuals of all walks every 100 iterates
(refreshes every 128, reprojection every 100 on config 4)."""
import json, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_07097_b200 as mh
from paper_2104_07097_b200 import workloads

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 600
for cfg in [int(c) for c in os.environ.get("SOAK_CFGS", "3 4").split()]:
    w = workloads.config(cfg)
    p = w.polytope
    proj = mh.compute_projection(p.a_eq) if p.num_equalities() else None
    for kw in (dict(), dict(f64_engine="int8"), dict(precision=32)):
        worst, worst_eq = -np.inf, 0.0
        with mh.Engine(p, w.z, seed=3, projector=proj, **kw) as eng:
            X0 = np.zeros((p.dim(), w.z), order="F")
            X0[:] = w.x0[:, None]
            eng.set_state(X0)
            for t in range(iters // 100):
                eng.step(100, 100 if proj else 0)
                bad, viol, eqv = eng.check_state(1e-9)
                assert bad == -1, (cfg, kw, t, bad)
                worst = max(worst, float(viol.max()))
                worst_eq = max(worst_eq, float(eqv.max()))
            X = eng.get_state()
            kernel = eng.stats()["chord_kernel"]
        print(json.dumps({"config": cfg, "engine": kw or "dmma", "chord_kernel": kernel,
                          "iterates": iters,
                          "max_violation": worst, "max_eq_residual": worst_eq,
                          "spread": float(np.abs(X).max())}), flush=True)
