"""Diagnostic for the fp16 form of the fp32 variant: per-walk bound errors of
one injected step against the oracle on the f16-quantized operands."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle
import paper_2104_07097_b200 as mh
from paper_2104_07097_b200 import workloads

def q16(x, axis):
    mx = np.abs(x).max(axis=axis, keepdims=True)
    e = np.where(mx > 0, np.floor(np.log2(np.where(mx > 0, mx, 1))) + 1, 0)
    s = 2.0 ** (14 - e)
    h = (x * s).astype(np.float16).astype(np.float64)
    h[np.abs(h) < 2.0 ** -14] = 0
    l = (x * s - h).astype(np.float16).astype(np.float64)
    l[np.abs(l) < 2.0 ** -14] = 0
    return h / s, (h + l) / s

n, m, z = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
p = workloads.random_polytope(n, m, seed=n)
rng = np.random.default_rng(m)
X = rng.uniform(-1, 1, (n, z)); X *= 0.4 / np.max((p.a_in @ X) / p.b_in[:, None], axis=0)
X = np.asfortranarray(X)
H = np.asfortranarray(rng.standard_normal((n, z)))
U = rng.uniform(0.05, 0.95, z)
with mh.Engine(p, z, precision=32) as eng:
    eng.set_state(X)
    lo, hi, th, fl = eng.step_injected(H, U)
Dq, _ = q16(H, 0)
_, Aq = q16(p.a_in, 1)
orc = oracle.lib() and oracle
st, Xr, lor, hir, thr, flr, _ = oracle.step_injected(np.asfortranarray(Aq), p.b_in, None, 1e-11, X, np.asfortranarray(Dq), U)
w = hir - lor
err = np.maximum(np.abs(lo - lor), np.abs(hi - hir)) / w
print("max rel err", err.max(), "median", np.median(err))
bad = np.where(err > 1e-4)[0]
print("bad walks", len(bad), bad[:40])
