"""Long-run containment of every engine on BASELINE config 4 (box rows,
50000 random rows, 100 equalities): 200 iterates with refreshes every 64 and
reprojection every 50, every walk checked on a fresh fp64 product
(tools/soak.py runs the 600-iterate version on configs 3 and 4)."""
import numpy as np
import pytest

import paper_2104_07097_b200 as mh
from paper_2104_07097_b200 import workloads

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("kw", [dict(), dict(f64_engine="int8"), dict(precision=32)],
                         ids=["dmma", "int8", "fp32"])
def test_config4_long_run_containment(kw):
    w = workloads.config(4)
    p = w.polytope
    op = mh.compute_projection(p.a_eq)
    z = 1024
    with mh.Engine(p, z, seed=6, projector=op, refresh_every=64, **kw) as eng:
        eng.set_state(np.zeros((p.dim(), z)))
        for _ in range(4):
            eng.step(50, 50)
            bad, viol, eqv = eng.check_state(1e-9)
            assert bad == -1 and viol.max() <= 1e-9 and eqv.max() <= 1e-9
        X = eng.get_state()
    assert np.abs(p.a_eq @ X).max() <= 1e-9
    assert np.abs(X).max() > 0.1
