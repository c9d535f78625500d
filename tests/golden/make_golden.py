"""Regenerates the golden fixtures in tests/golden/ from the CPU oracle.

The reference ships no stored trajectories and cannot be built here, so the
pinned ground truth is (1) the reference's own known-answer tests
(tests/test_oracle_kats.py) and (2) these frozen oracle outputs, which make
any later change of the oracle or of the engine visible.

    python tests/golden/make_golden.py      # rewrites the .npz files
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402


def random_body(n, m, seed):
    rng = np.random.default_rng(seed)
    a = rng.standard_normal((m, n))
    a /= np.linalg.norm(a, axis=1, keepdims=True)
    return np.asfortranarray(a), np.ones(m)


def main():
    # 1. injected single iterates (the GPU test hook semantics)
    cases = {}
    for name, (n, m, z, seed) in {"rand13": (13, 57, 9, 1), "rand40": (40, 300, 70, 2)}.items():
        A, b = random_body(n, m, seed)
        rng = np.random.default_rng(seed + 100)
        X = np.asfortranarray(rng.uniform(-0.1, 0.1, (n, z)))
        H = np.asfortranarray(rng.standard_normal((n, z)))
        U = rng.uniform(0, 1, z)
        st, Xn, lo, hi, th, fl, _ = oracle.step_injected(A, b, None, 1e-11, X, H, U)
        assert st == 0
        cases[name] = dict(A=A, b=b, X=X, H=H, U=U, X_next=Xn, lower=lo, upper=hi, theta=th,
                           flags=fl)
    A, b, AE, bE = oracle.make_simplex(6)
    st, P, G = oracle.compute_projection(AE)
    rng = np.random.default_rng(7)
    X = np.asfortranarray(np.full((6, 5), 1 / 6))
    H = np.asfortranarray(rng.standard_normal((6, 5)))
    U = rng.uniform(0, 1, 5)
    st, Xn, lo, hi, th, fl, _ = oracle.step_injected(A, b, P, 1e-11, X, H, U)
    cases["simplex6"] = dict(A=A, b=b, AE=AE, bE=bE, P=P, X=X, H=H, U=U, X_next=Xn, lower=lo,
                             upper=hi, theta=th, flags=fl)
    for name, d in cases.items():
        np.savez(os.path.join(HERE, f"step_injected_{name}.npz"), **d)

    # 2. reference-stream trajectory: box(5), z = 3, seed 4242, 20 iterates
    A, b = oracle.make_hypercube(5)
    rng = oracle.WalkRng(4242, 3)
    X = np.zeros((5, 3), order="F")
    traj = []
    for _ in range(20):
        assert oracle.step(A, b, None, 1e-11, rng, X)[0] == 0
        traj.append(X.copy())
    np.savez(os.path.join(HERE, "trajectory_box5_z3_seed4242.npz"), A=A, b=b,
             states=np.stack(traj))

    # 3. normals of WalkRng(99, 2), n = 7 (odd: last sine dropped)
    rng = oracle.WalkRng(99, 2)
    np.savez(os.path.join(HERE, "normals_seed99_z2_n7.npz"), H=rng.fill_standard_normal_matrix(7))


if __name__ == "__main__":
    main()
