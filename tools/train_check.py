"""Device trainer (hygt_optimize_f64) against the oracle restatement of hygt::optimize, per
restart, plus the reference's acceptance pins (tests/acceptance.cpp:66-68)."""
import json, sys, time
import numpy as np
sys.path.insert(0, ".")
from paper_2505_21728_b200 import train as T
from oracle import oracle as O


def ar1(bs, rho):
    a = rho ** np.abs(np.subtract.outer(np.arange(bs), np.arange(bs)))
    return np.kron(a, a)


def case(name, phi, log2_n, rounds, oracle=True, **kw):
    cfg = T.OptimizerConfig(**kw)
    t = time.time(); model, rep = T.optimize(phi, log2_n, rounds, cfg); tg = time.time() - t
    out = {"case": name, "gpu_s": round(tg, 4), "gpu_gains": rep.restart_gains_db, "gpu_best": rep.best_restart,
           "gpu_klt": rep.klt_gain_db, "gpu_sweeps": [len(x) for x in rep.trajectories]}
    if oracle:
        t = time.time(); a, r = O.optimize(phi, log2_n, rounds, **kw); to = time.time() - t
        out.update({"oracle_s": round(to, 3), "oracle_gains": r["restart_gains_db"].tolist(), "oracle_best": r["best_restart"],
                    "oracle_klt": r["klt_gain_db"], "oracle_sweeps": [len(x) for x in r["trajectories"]],
                    "max_gain_diff": float(np.max(np.abs(np.array(rep.restart_gains_db) - r["restart_gains_db"]))),
                    "angle_diff_best": float(np.max(np.abs(model.angles - a)))})
    print(json.dumps(out), flush=True)


case("n16r2_acceptance", ar1(4, 0.95), 4, 2, restarts=4, seed=1)
case("n16r2_rho09_seed7", ar1(4, 0.9), 4, 2, restarts=3, seed=7)
rng = np.random.default_rng(5)
g = rng.standard_normal((8, 8)); case("n8r2_random_psd", g @ g.T, 3, 2, restarts=2, seed=3)
case("n64r3_acceptance", ar1(8, 0.95), 6, 3, oracle=False, restarts=4, seed=1)
case("n64r1_2sweeps", ar1(8, 0.9), 6, 1, restarts=2, seed=2, max_sweeps=2)
case("n256r1_1sweep", ar1(16, 0.9), 8, 1, oracle=False, restarts=1, seed=2, max_sweeps=2)
