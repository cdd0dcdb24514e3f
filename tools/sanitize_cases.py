"""Small invocations of every kernel family for compute-sanitizer (memcheck / racecheck /
synccheck), one case per process:
    compute-sanitizer --tool racecheck python tools/sanitize_cases.py stage
Cases: stage (N=16 TMA-staged, config-2 shape), clsjit (N=64 per-class NVRTC chain), segment
(N=256 butterfly kernel with fused energy), gemm64 / gemm256 (the tensor-core path, CTA pairs,
energy), gemm256_1cta (single CTAs), klt (N=64 grouped GEMM), fixed (per-class integer chain),
fixed_row (int32 row kernel), corr (fp64 correlation)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_21728_b200 import (FixedPlan, HyGTModel, HyGTPlan, KLTPlan, QuantizedHyGTModel,  # noqa: E402
                                   TrigTable, correlation)
import paper_2505_21728_b200._lib as L  # noqa: E402


def float_case(log2n, rounds, classes, rows, kernel="auto", perms=False, energy=False, pairs=True):
    rng = np.random.default_rng(log2n * 7 + rows)
    n = 1 << log2n
    ms = [HyGTModel(log2n, rounds, rng.uniform(-np.pi, np.pi, rounds * log2n * n // 2)) for _ in range(classes)]
    inter = np.stack([np.stack([rng.permutation(n) for _ in range(rounds - 1)]) for _ in range(classes)]) if perms else None
    plan = HyGTPlan(ms, inter, kernel=kernel, cta_pairs=pairs)
    x = torch.from_numpy((rng.standard_normal((rows, n)) * 16).astype(np.float32)).cuda()
    cls = torch.from_numpy(rng.integers(0, classes, rows).astype(np.int16)).cuda().view(torch.uint16)
    if energy:
        e = torch.zeros(classes, n, dtype=torch.float64, device="cuda")
        y = plan.forward_energy(x, cls, e)
    else:
        y = plan.forward(x, cls)
    z = plan.inverse(y, cls)
    plan.sync_status()
    torch.cuda.synchronize()
    return plan.path, float((z - x).abs().max())


def main(case):
    if case == "stage":
        r = float_case(4, 3, 35, 6000, perms=True)
    elif case == "clsjit":
        r = float_case(6, 4, 5, 3000, perms=True)
    elif case == "segment":
        r = float_case(8, 2, 3, 1500, kernel="butterfly", energy=True)
    elif case == "gemm64":
        r = float_case(6, 3, 4, 3000, kernel="tensor", perms=True, energy=True)
    elif case == "gemm256":
        r = float_case(8, 2, 3, 1500, kernel="tensor", energy=True)
    elif case == "gemm256_1cta":
        r = float_case(8, 2, 3, 1500, kernel="tensor", energy=True, pairs=False)
    elif case == "klt":
        rng = np.random.default_rng(1)
        k = np.stack([np.linalg.qr(rng.standard_normal((64, 64)))[0] for _ in range(3)])
        plan = KLTPlan(k)
        x = torch.randn(2000, 64, device="cuda")
        cls = torch.randint(0, 3, (2000,), device="cuda").to(torch.int16).view(torch.uint16)
        y = plan.forward(x, cls)
        z = plan.inverse(y, cls)
        torch.cuda.synchronize()
        r = ("klt", float((z - x).abs().max()))
    elif case in ("fixed", "fixed_row"):
        if case == "fixed_row":
            L.set_knob("HYGT_FIXED_JIT", 0)
            L.set_knob("HYGT_FIXED_STAGE", 0)
        rng = np.random.default_rng(2)
        codes = rng.integers(0, 256, (3, 3 * 6 * 32)).astype(np.uint16)
        plan = FixedPlan([QuantizedHyGTModel(6, 3, 8, codes[c]) for c in range(3)], TrigTable(8, 10))
        x = torch.from_numpy(rng.integers(-1000, 1000, (2000, 64))).cuda()
        cls = torch.from_numpy(rng.integers(0, 3, 2000).astype(np.int16)).cuda().view(torch.uint16)
        y = plan.forward(x, cls)
        plan.inverse(y, cls)
        r = ("fixed", 0.0)
    elif case == "corr":
        x = torch.randn(3000, 64, device="cuda")
        cls = torch.randint(0, 4, (3000,), device="cuda").to(torch.int16).view(torch.uint16)
        correlation(x, cls, 4)
        torch.cuda.synchronize()
        r = ("corr", 0.0)
    else:
        raise SystemExit(f"unknown case {case}")
    print(case, r)


if __name__ == "__main__":
    main(sys.argv[1])
