"""Small end-to-end exercise of every engine kernel for compute-sanitizer:
multi-kernel path (fused, incremental, check, projection, redraw, reference
streams, reprojection), walk-resident path, injected hook, run(), and the
tcgen05 engines (fp32 variant, int8-slice fp64)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_07097_b200 as mh
from paper_2104_07097_b200 import workloads

p = workloads.random_polytope(37, 700, seed=1)
for slack in ("incremental", "recompute"):
    with mh.Engine(p, 77, seed=1, slack=slack, refresh_every=3) as e:
        e.set_state(np.zeros((37, 77))); e.step(7); e.check_state(1e-9)
        H = np.random.default_rng(0).standard_normal((37, 77)); e.step_injected(H, np.full(77, 0.3))
s = mh.make_simplex(40); op = mh.compute_projection(s.a_eq)
with mh.Engine(s, 65, seed=2, projector=op, small_path=False, eps_dir=0.02) as e:
    e.set_state(np.full((40, 65), 1 / 40)); e.step(6, 2); e.check_state(1e-9)
with mh.Engine(mh.make_hypercube(6), 33, seed=3, rng="reference", eps_dir=0.5) as e:
    e.set_state(np.zeros((6, 33))); e.step(5)
with mh.Engine(s, 65, seed=2, projector=op) as e:
    e.run(np.full(40, 1 / 40), 5, 2, 3, 2)
# tcgen05 engines: fp32 variant and int8-slice fp64 engine (ragged sizes)
q = workloads.random_polytope(45, 1300, seed=4)
for kw in (dict(precision=32), dict(f64_engine="int8")):
    with mh.Engine(q, 300, seed=5, refresh_every=4, **kw) as e:
        e.set_state(np.zeros((45, 300))); e.step(9); e.check_state(1e-9)
        H = np.random.default_rng(1).standard_normal((45, 300)); e.step_injected(H, np.full(300, 0.6))
print("sanitize smoke ok")
