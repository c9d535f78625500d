"""Sweeps the fp32 (tcgen05) chord kernel's L2 policy for the A stream and its
rasterisation band on config 5; prints one JSON line per setting."""
import json
import os
import sys

import numpy as np

import paper_2104_07097_b200 as mh
from paper_2104_07097_b200 import workloads


def main():
    w = workloads.config(5)
    settings = [tuple(map(int, s.split(":"))) for s in sys.argv[1:]] or \
        [(a, g) for a in (0, 1, 2) for g in (1, 2, 4)]
    for apol, group in settings:
        os.environ["MHAR_TC_APOL"] = str(apol)
        os.environ["MHAR_TC_GROUP"] = str(group)
        with mh.Engine(w.polytope, w.z, seed=1, precision=32) as eng:
            eng.set_state(np.repeat(w.x0[:, None], w.z, axis=1))
            eng.step(3)
            eng.sync()
            eng.set_timing(True)
            eng.reset_stats()
            ms = eng.step_timed(6)
            st = eng.stats()
        print(json.dumps({"a_policy": apol, "group_n": group, "ms_per_iterate": ms / 6,
                          "chord_ms_per_launch": st["chord_ms"] / max(1, st["chord_timed"]),
                          "chain_steps_per_s": w.z * 6 / (ms / 1e3)}), flush=True)


if __name__ == "__main__":
    main()
