"""The coordinate-descent trainer: hygt::optimize on the GPU.

Mirrors include/hygt/optimizer.hpp: ``OptimizerConfig`` (:35-42), ``TrainingReport`` (:44-50),
``optimize`` (:311-371), ``variance_permutation`` (:378-390) and the per-class loop of
``hygt train`` (tools/hygt_main.cpp:73-103). The search runs in libhygt_gpu.so
(``hygt_optimize_f64``, csrc/hygt_train.cu); this module only marshals host arrays. There is
no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _lib
from .errors import ArgumentError, raise_for
from .model import HyGTModel, num_parameters

INIT_MODES = {"greedy_jacobi": 0, "random": 1, "zero": 2}


class _Config(C.Structure):  # hygt_optimize_config (include/hygt_gpu.h)
    _fields_ = [("restarts", C.c_int), ("max_sweeps", C.c_int), ("gain_tolerance_db", C.c_double),
                ("seed", C.c_uint64), ("init_mode", C.c_int)]


@dataclass
class OptimizerConfig:
    """optimizer.hpp:35-42."""
    restarts: int = 4
    max_sweeps: int = 50
    gain_tolerance_db: float = 1e-4
    seed: int = 0
    init_mode: str = "greedy_jacobi"  # restart 0; the others are random


@dataclass
class TrainingReport:
    """optimizer.hpp:44-50, plus the propagated variances of the best model."""
    restart_gains_db: List[float] = field(default_factory=list)
    best_restart: int = 0
    trajectories: List[List[float]] = field(default_factory=list)
    klt_gain_db: float = 0.0
    gain_ratio: float = 0.0
    variances: Optional[np.ndarray] = None


def splitmix64(state: int) -> int:
    """rng.hpp:26-31."""
    m = (1 << 64) - 1
    z = (state + 0x9E3779B97F4A7C15) & m
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & m
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & m
    return z ^ (z >> 31)


def derive_seed(base: int, stream: int) -> int:
    """rng.hpp:36-38."""
    return splitmix64(base ^ splitmix64(stream + 1))


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def optimize_batch(phis, log2_n: int, rounds: int, config: OptimizerConfig = OptimizerConfig(),
                   seeds: Optional[Sequence[int]] = None) -> List[Tuple[HyGTModel, TrainingReport]]:
    """optimize() for every covariance of phis [P][N][N] in one device launch (one CTA per
    problem and restart). seeds: per-problem OptimizerConfig::seed (default config.seed)."""
    phis = np.ascontiguousarray(phis, dtype=np.float64)
    n = 1 << log2_n
    if phis.ndim == 2:
        phis = phis[None]
    if phis.ndim != 3 or phis.shape[1:] != (n, n):
        raise ArgumentError("optimize: dimension mismatch")
    if config.init_mode not in INIT_MODES:
        raise ArgumentError(f"optimize: unknown init_mode {config.init_mode!r}")
    problems = phis.shape[0]
    restarts = max(int(config.restarts), 0)
    sweeps = max(int(config.max_sweeps), 0)
    a_count = num_parameters(log2_n, rounds) if 1 <= log2_n <= 16 and rounds >= 1 else 0
    cfg = _Config(int(config.restarts), int(config.max_sweeps), float(config.gain_tolerance_db),
                  int(config.seed) & ((1 << 64) - 1), INIT_MODES[config.init_mode])
    seed_arr = None if seeds is None else np.ascontiguousarray(seeds, dtype=np.uint64)
    if seed_arr is not None and seed_arr.size != problems:
        raise ArgumentError("optimize: one seed per problem")
    angles = np.zeros((problems, max(a_count, 1)), np.float64)
    gains = np.zeros((problems, max(restarts, 1)), np.float64)
    best = np.zeros(problems, np.int32)
    klt = np.zeros(problems, np.float64)
    traj = np.full((problems, max(restarts, 1), sweeps + 1), np.nan)
    tlen = np.zeros((problems, max(restarts, 1)), np.int32)
    var = np.zeros((problems, n), np.float64)
    st = _lib.lib().hygt_optimize_f64(log2_n, rounds, problems, _ptr(phis), C.byref(cfg), _ptr(seed_arr),
                                      _ptr(angles), _ptr(gains), _ptr(best), _ptr(klt), _ptr(traj),
                                      _ptr(tlen), _ptr(var), None)
    if st:
        raise_for(st, _lib.last_error())
    out = []
    for p in range(problems):
        b = int(best[p])
        rep = TrainingReport(
            restart_gains_db=gains[p, :restarts].tolist(), best_restart=b,
            trajectories=[traj[p, r, :tlen[p, r]].tolist() for r in range(restarts)],
            klt_gain_db=float(klt[p]),
            gain_ratio=float(gains[p, b] / klt[p]) if klt[p] > 1e-15 else 1.0,
            variances=var[p].copy())
        out.append((HyGTModel(log2_n, rounds, angles[p, :a_count]), rep))
    return out


def optimize(phi, log2_n: int, rounds: int,
             config: OptimizerConfig = OptimizerConfig()) -> Tuple[HyGTModel, TrainingReport]:
    """hygt::optimize(phi, log2_n, rounds, config) (optimizer.hpp:311-371)."""
    return optimize_batch(np.asarray(phi, dtype=np.float64)[None], log2_n, rounds, config)[0]


def variance_permutation(model: HyGTModel, variances) -> HyGTModel:
    """optimizer.hpp:378-390: attach the permutation that orders the propagated variances
    (TrainingReport.variances) non-increasingly, ties by ascending index."""
    if model.permutation is not None:
        raise ArgumentError("variance_permutation: model already has one")
    v = np.asarray(variances, dtype=np.float64)
    perm = sorted(range(v.size), key=lambda i: (-v[i], i))
    return HyGTModel(model.log2_n, model.rounds, model.angles, perm)


def train_classes(phis, counts, log2_n: int, rounds: int, restarts: int = 4, seed: int = 0):
    """The per-class loop of `hygt train` (tools/hygt_main.cpp:83-103): classes with fewer than
    N samples keep the identity transform; the others are optimized with the seed
    derive_seed(seed, c) and get the variance-sorting permutation. Returns [(model, report or
    None)] per class."""
    phis = np.ascontiguousarray(phis, dtype=np.float64)
    n = 1 << log2_n
    counts = np.asarray(counts).reshape(-1)
    todo = [c for c in range(phis.shape[0]) if counts[c] >= n]
    results = {}
    if todo:
        cfg = OptimizerConfig(restarts=restarts)
        batch = optimize_batch(phis[todo], log2_n, rounds, cfg, seeds=[derive_seed(seed, c) for c in todo])
        for c, (model, rep) in zip(todo, batch):
            results[c] = (variance_permutation(model, rep.variances), rep)
    return [results.get(c, (HyGTModel.zeros(log2_n, rounds), None)) for c in range(phis.shape[0])]
