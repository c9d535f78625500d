"""Times the GPU Prim MST / Friedman-Rafsky test at the reference's acceptance
sizes (5000 + 5000 points) and larger pools."""
import json, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2104_07097_b200 import stats

for form in ("cta", "grid_l2", "grid"):
    os.environ["MHAR_PRIM"] = form
    sizes = [(2 * 5000, 10), (2 * 5000, 100), (2 * 20000, 10)]
    if form != "cta":
        sizes += [(2 * 50000, 10), (2 * 5000, 1000)]
    for N, n in sizes:
        rng = np.random.default_rng(N + n)
        a = rng.uniform(-1, 1, (N // 2, n))
        b = rng.uniform(-1, 1, (N // 2, n))
        stats.friedman_rafsky(a[:100], b[:100])  # warm-up
        t0 = time.perf_counter()
        r = stats.friedman_rafsky(a, b)
        dt = time.perf_counter() - t0
        print(json.dumps({"form": form, "pooled": N, "n": n, "seconds": round(dt, 4),
                          "z": r.z_value, "cross_edges": r.cross_edges}), flush=True)
