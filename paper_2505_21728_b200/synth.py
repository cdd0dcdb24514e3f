"""Synthetic workloads of BASELINE.json's five configs.

The paper's codec datasets are not available (and not needed): seeded synthetic inputs with the
configs' shapes and distributions stand in. Model parameters (angles U[-pi, pi), Fisher-Yates
style permutations, per-class rho ~ U[0.5, 0.95]) are drawn on the host from numpy's PCG64;
rows and class ids are generated on the device by counter-based kernels in libhygt_gpu.so so any
row range of a 16 GB batch can be produced (and re-produced) without host staging.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np
import torch

from . import _lib
from .errors import raise_for
from .model import HyGTModel, num_parameters


@dataclass
class Config:
    name: str
    log2_n: int
    classes: int
    rounds: int
    count: int
    inter_round_perms: bool
    rho: Optional[float]          # None => per-class U[0.5, 0.95]
    sigma: float = 16.0
    edge_fraction: float = 0.0
    edge_amplitude: float = 32.0  # not given by config 3; documented choice
    edge_noise: float = 4.0
    energy: bool = False
    klt: bool = False
    description: str = ""


CONFIGS = {
    1: Config("cfg1_n16_c1_r2", 4, 1, 2, 1 << 20, True, 0.9,
              description="N=16, C=1, R=2, one fixed inter-round permutation, 2^20 AR(1) rows"),
    2: Config("cfg2_n16_c35_r3", 4, 35, 3, 1 << 24, True, None,
              description="N=16, C=35, R=3, seeded inter-round permutations, per-class rho, 2^24 rows"),
    3: Config("cfg3_n64_c35_r4", 6, 35, 4, 1 << 22, True, 0.9, edge_fraction=0.1,
              description="N=64, C=35, R=4, per-class permutations, 10% directional edges, 2^22 rows"),
    4: Config("cfg4_klt_n64_c35", 6, 35, 4, 1 << 22, True, 0.9, edge_fraction=0.1, klt=True,
              description="dense per-class 64x64 KLT on config 3's rows"),
    5: Config("cfg5_n256_c35_r4", 8, 35, 4, 1 << 24, False, 0.9, energy=True,
              description="N=256, C=35, R=4, 2^24 rows, per-class energy sums"),
}


@dataclass
class Workload:
    cfg: Config
    seed: int
    angles: np.ndarray                 # [C][A] fp64
    perms: Optional[np.ndarray]        # [C][R-1][N] or None
    rho: np.ndarray                    # [C] fp32
    models: list = field(default_factory=list)

    @property
    def n(self) -> int:
        return 1 << self.cfg.log2_n

    def block_size(self) -> int:
        return int(round(math.sqrt(self.n)))

    def make_classes(self, count: int, row0: int = 0, device="cuda") -> torch.Tensor:
        cls = torch.empty(count, dtype=torch.uint16, device=device)
        st = _lib.lib().hygt_synth_classes(cls.data_ptr(), count, row0, self.cfg.classes,
                                           self.seed ^ 0xC1A55, torch.cuda.current_stream().cuda_stream)
        raise_for(st, _lib.last_error())
        return cls

    def make_rows(self, count: int, cls: torch.Tensor, row0: int = 0, device="cuda") -> torch.Tensor:
        x = torch.empty((count, self.n), dtype=torch.float32, device=device)
        rho = torch.from_numpy(self.rho.astype(np.float32)).to(device)
        st = _lib.lib().hygt_synth_rows_f32(
            x.data_ptr(), count, row0, self.block_size(), cls.data_ptr(), rho.data_ptr(),
            self.cfg.classes, self.cfg.sigma, self.cfg.edge_fraction, self.cfg.edge_amplitude,
            self.cfg.edge_noise, self.seed, torch.cuda.current_stream().cuda_stream)
        raise_for(st, _lib.last_error())
        return x

    def klt_bases(self) -> np.ndarray:
        """35 random orthogonal N x N matrices: Q of the QR of seeded Gaussians, diag(R) > 0."""
        rng = np.random.Generator(np.random.PCG64(self.seed ^ 0x4B17))
        out = np.empty((self.cfg.classes, self.n, self.n))
        for c in range(self.cfg.classes):
            q, r = np.linalg.qr(rng.standard_normal((self.n, self.n)))
            out[c] = q * np.sign(np.diag(r))[None, :]
        return out


def make_workload(config: int, seed: int = 2505_21728) -> Workload:
    cfg = CONFIGS[config]
    rng = np.random.Generator(np.random.PCG64(seed + config))
    n = 1 << cfg.log2_n
    a = num_parameters(cfg.log2_n, cfg.rounds)
    angles = rng.uniform(-math.pi, math.pi, size=(cfg.classes, a))
    perms = None
    if cfg.inter_round_perms and cfg.rounds > 1:
        if cfg.classes == 1:  # config 1: one fixed permutation between the rounds
            p = rng.permutation(n)
            perms = np.tile(p, (1, cfg.rounds - 1, 1))
        else:
            perms = np.stack([np.stack([rng.permutation(n) for _ in range(cfg.rounds - 1)])
                              for _ in range(cfg.classes)])
        perms = perms.astype(np.uint16)
    if cfg.rho is None:
        rho = rng.uniform(0.5, 0.95, size=cfg.classes)
    else:
        rho = np.full(cfg.classes, cfg.rho)
    w = Workload(cfg, seed, angles, perms, rho.astype(np.float32))
    w.models = [HyGTModel(cfg.log2_n, cfg.rounds, angles[c]) for c in range(cfg.classes)]
    return w
