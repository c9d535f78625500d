"""Mid-size structured bodies on the multi-kernel path (hypercube / simplex,
n in the thousands): per-iterate time with the walk-resident kernel off,
for ncu captures of diag_chord_kernel / normals_kernel / axpy_kernel.
usage: python tools/mid_body_probe.py [hypercube|simplex] n z iters [small]
("small": let the context take the walk-resident kernel when it fits)"""
import json, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_07097_b200 as mh

body = sys.argv[1] if len(sys.argv) > 1 else "hypercube"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 5000
z = int(sys.argv[3]) if len(sys.argv) > 3 else 1000
iters = int(sys.argv[4]) if len(sys.argv) > 4 else 50
small = len(sys.argv) > 5 and sys.argv[5] == "small"
p = mh.make_hypercube(n) if body == "hypercube" else mh.make_simplex(n)
op = mh.compute_projection(p.a_eq) if p.num_equalities() else None
x0 = np.zeros(n) if body == "hypercube" else np.full(n, 1.0 / n)
with mh.Engine(p, z, seed=1, projector=op, small_path=small) as eng:
    eng.set_state(np.repeat(x0[:, None], z, 1))
    eng.step(5)
    eng.sync()
    t = time.perf_counter()
    eng.step(iters)
    eng.sync()
    dt = time.perf_counter() - t
    st = eng.stats()
print(json.dumps({"body": body, "n": n, "z": z, "us_per_iterate": dt / iters * 1e6,
                  "chain_steps_per_s": z * iters / dt, "chord_kernel": st["chord_kernel"],
                  "launches_per_iterate": st["kernel_launches"] / (iters + 5)}))
