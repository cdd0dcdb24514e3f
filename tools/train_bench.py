"""Trainer benchmark: hygt_optimize_f64 on the GPU against the reference's own
hygt::optimize (oracle/_ref shim) on the host's cores, same problems, same config.

Workloads (per-class 2-D AR(1) covariances, rho_c ~ U[0.5, 0.95] seeded, like config 2's classes):
  cfg2_train: 35 classes, N=16, R=3, restarts 4, up to 50 sweeps (the `hygt train` defaults)
  cfg3_train: 35 classes, N=64, R=4, restarts 4, up to 50 sweeps (GPU); the reference arm runs a
              bounded sample (restarts 1, max_sweeps 2) and is compared per candidate evaluation
  acceptance: N=64, R=3, restarts 4, seed 1 (acceptance.cpp:207-228), GPU only here; the
              reference's time for it is in profiles/r01/train_bench.jsonl when measured.
Unit of work: one candidate-angle evaluation (candidate_gain, optimizer.hpp:257-266); each
position of a sweep evaluates 64 (the current angle, 33 grid points, 30 golden-section steps).
Prints one JSON line per measurement.
"""
import json
import os
import sys
import threading
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_21728_b200 import train as T  # noqa: E402


def ar1(bs, rho):
    a = rho ** np.abs(np.subtract.outer(np.arange(bs), np.arange(bs)))
    return np.kron(a, a)


def phis(classes, bs, seed):
    rng = np.random.default_rng(seed)
    return np.stack([ar1(bs, r) for r in rng.uniform(0.5, 0.95, classes)])


def candidates(reports, log2n, rounds):
    a = rounds * log2n * (1 << (log2n - 1))
    return sum(64 * a * (len(t) - 1) for rep in reports for t in rep)


def gpu_run(name, P, log2n, rounds, cfg, seeds, reps=3):
    T.optimize_batch(P[:1], log2n, rounds, T.OptimizerConfig(restarts=1, max_sweeps=1))  # warm-up
    times = []
    for _ in range(reps):
        t = time.perf_counter()
        out = T.optimize_batch(P, log2n, rounds, cfg, seeds=seeds)
        times.append(time.perf_counter() - t)
    t = float(np.median(times))
    cand = candidates([rep.trajectories for _, rep in out], log2n, rounds)
    print(json.dumps({"workload": name, "impl": "gpu", "seconds": t, "candidates": cand,
                      "candidates_per_s": cand / t, "problems": int(P.shape[0]),
                      "best_gains": [round(rep.restart_gains_db[rep.best_restart], 6) for _, rep in out][:4],
                      "config": cfg.__dict__}), flush=True)
    return out


def ref_run(name, P, log2n, rounds, cfg, seeds, threads):
    from oracle import oracle as O
    if not O.ref_available():
        print(json.dumps({"workload": name, "impl": "reference", "unavailable": "oracle/_ref not built"}))
        return
    res = [None] * P.shape[0]
    nxt = [0]
    lock = threading.Lock()

    def worker():
        while True:
            with lock:
                i = nxt[0]
                nxt[0] += 1
            if i >= P.shape[0]:
                return
            res[i] = O.ref_optimize(P[i], log2n, rounds, restarts=cfg.restarts, max_sweeps=cfg.max_sweeps,
                                    gain_tolerance_db=cfg.gain_tolerance_db, seed=int(seeds[i]))

    t = time.perf_counter()
    ths = [threading.Thread(target=worker) for _ in range(threads)]
    for th in ths:
        th.start()
    for th in ths:
        th.join()
    t = time.perf_counter() - t
    cand = candidates([r["trajectories"] for _, r in res], log2n, rounds)
    print(json.dumps({"workload": name, "impl": "reference", "seconds": t, "candidates": cand,
                      "candidates_per_s": cand / t, "problems": int(P.shape[0]), "threads": threads,
                      "best_gains": [round(float(r["restart_gains_db"][r["best_restart"]]), 6) for _, r in res][:4],
                      "config": cfg.__dict__}), flush=True)


def main():
    threads = os.cpu_count()
    seeds = [T.derive_seed(0, c) for c in range(35)]
    P16 = phis(35, 4, 2)
    P64 = phis(35, 8, 3)
    full = T.OptimizerConfig(restarts=4)
    sample = T.OptimizerConfig(restarts=1, max_sweeps=2)
    gpu_run("cfg2_train", P16, 4, 3, full, seeds)
    gpu_run("cfg3_train", P64, 6, 4, full, seeds, reps=1)
    gpu_run("cfg3_train_sample", P64, 6, 4, sample, seeds)
    gpu_run("acceptance_n64r3", ar1(8, 0.95)[None], 6, 3, T.OptimizerConfig(restarts=4, seed=1), None, reps=1)
    if "--no-ref" not in sys.argv:
        ref_run("cfg2_train", P16, 4, 3, full, seeds, threads)
        ref_run("cfg3_train_sample", P64, 6, 4, sample, seeds, threads)


if __name__ == "__main__":
    main()
