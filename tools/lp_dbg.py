"""Debug aid for the centring LP: prints the centre of a small body (the
pivot trace with MHAR_LP_TRACE=1)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_07097_b200 as mh
kind, n = sys.argv[1], int(sys.argv[2])
p = mh.make_simplex(n) if kind == "simplex" else mh.make_hypercube(n)
try:
    c = mh.chebyshev_center(p)
    print("RESULT", kind, n, c.x[:4], c.radius, c.pivots)
except mh.MharError as e:
    print("ERROR", kind, n, e)
