"""Generate tests/golden/optimize_v1.npz from the UNMODIFIED reference optimizer (oracle/_ref shim).

Run in the container that has /root/reference (make -C oracle builds the shim first):
    python tests/gen_golden_optimize.py
Every output below is returned by the reference's own hygt::optimize (optimizer.hpp:311-371)
and hygt::variance_permutation (:378-390) on the stored covariance; the GPU tests compare the
device trainer (hygt_optimize_f64) with these arrays without needing /root/reference.
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "optimize_v1.npz")


def ar1(bs, rho):
    """statistics.hpp:287-305 (ar1_covariance_2d) through the reference itself."""
    n = bs * bs
    out = np.zeros((n, n))
    O.ref().ref_ar1_covariance_2d(bs, rho, out.ctypes.data)
    return out


def main():
    O.build()
    rng = np.random.Generator(np.random.PCG64(2505_21728))
    g = {}
    cases = []
    # name, phi, log2n, rounds, kwargs
    cases.append(("n16r2_acceptance", ar1(4, 0.95), 4, 2, dict(restarts=4, seed=1)))  # acceptance.cpp:197-203
    cases.append(("n16r2_seed7", ar1(4, 0.9), 4, 2, dict(restarts=3, seed=7)))  # test_optimizer.cpp:140-151
    cases.append(("n4r2_seed99", ar1(2, 0.85), 2, 2, dict(restarts=3, seed=99)))  # test_optimizer.cpp:164-173
    g8 = rng.standard_normal((8, 8))
    cases.append(("n8r2_psd", g8 @ g8.T, 3, 2, dict(restarts=2, seed=3)))
    g4 = rng.standard_normal((4, 4))
    cases.append(("n4r1_random_init", g4 @ g4.T + 0.1 * np.eye(4), 2, 1, dict(restarts=2, seed=5, init_mode="random")))
    cases.append(("n4r2_zero_init", ar1(2, 0.7), 2, 2, dict(restarts=1, init_mode="zero")))
    d = np.diag(np.arange(1.0, 9.0))
    cases.append(("n8r1_diagonal", d, 3, 1, dict(restarts=1)))  # test_optimizer.cpp:95-108
    cases.append(("n64r1_two_sweeps", ar1(8, 0.9), 6, 1, dict(restarts=2, seed=2, max_sweeps=2)))
    for k in range(6):  # test_optimizer.cpp:110-121: N = 2 reaches the KLT gain
        g2 = rng.standard_normal((2, 2))
        cases.append((f"n2r1_psd{k}", g2 @ g2.T + 1e-3 * np.eye(2), 1, 1, dict(restarts=2, seed=64 + k)))
    names = []
    for name, phi, log2n, rounds, kw in cases:
        angles, rep = O.ref_optimize(phi, log2n, rounds, **kw)
        perm, var = O.ref_variance_permutation(phi, log2n, rounds, angles)
        names.append(name)
        g[f"{name}/phi"] = phi
        g[f"{name}/shape"] = np.array([log2n, rounds, kw.get("restarts", 4), kw.get("max_sweeps", 50)])
        g[f"{name}/seed"] = np.array([kw.get("seed", 0)], np.uint64)
        g[f"{name}/init_mode"] = np.array(kw.get("init_mode", "greedy_jacobi"))
        g[f"{name}/angles"] = angles
        g[f"{name}/gains"] = rep["restart_gains_db"]
        g[f"{name}/best"] = np.array([rep["best_restart"]])
        g[f"{name}/klt"] = np.array([rep["klt_gain_db"]])
        g[f"{name}/traj_len"] = np.array([len(t) for t in rep["trajectories"]])
        g[f"{name}/traj_last"] = np.array([t[-1] for t in rep["trajectories"]])
        g[f"{name}/perm"] = perm
        g[f"{name}/variances"] = var
        print(name, rep["restart_gains_db"], rep["best_restart"], flush=True)
    g["names"] = np.array(names)
    np.savez_compressed(OUT, **g)
    print("wrote", OUT, os.path.getsize(OUT), "bytes")


if __name__ == "__main__":
    main()
