"""Kernel-level sweep (development tool): forward-kernel GB/s of HyGTPlan for a grid of
(log2n, rounds, classes, permutations, env layout) on synthetic data already in HBM.
    python tools/kbench.py 4:3:35:perm 4:3:1:noperm ...
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_21728_b200 import HyGTModel, HyGTPlan  # noqa: E402


def run(spec, rows=None, iters=10):
    parts = spec.split(":")
    log2n, rounds, classes, perm = parts[:4]
    pattern = parts[4] if len(parts) > 4 else "rand"
    log2n, rounds, classes = int(log2n), int(rounds), int(classes)
    n = 1 << log2n
    rows = rows or (1 << 30) // (4 * n)  # 1 GiB per array
    rng = np.random.default_rng(1)
    models = [HyGTModel(log2n, rounds, rng.uniform(-np.pi, np.pi, rounds * n * log2n // 2))
              for _ in range(classes)]
    inter = None
    if perm == "perm" and rounds > 1:
        inter = np.stack([np.stack([rng.permutation(n) for _ in range(rounds - 1)]) for _ in range(classes)])
    plan = HyGTPlan(models, inter)
    x = torch.randn(rows, n, device="cuda")
    if pattern == "rand":
        cls = torch.randint(0, classes, (rows,), device="cuda", dtype=torch.int32).to(torch.uint16)
    elif pattern == "sorted":
        cls = (torch.arange(rows, device="cuda") * classes // rows).to(torch.int32).to(torch.uint16)
    elif pattern == "runs64":  # runs of 64 equal ids
        cls = ((torch.arange(rows, device="cuda") // 64) % classes).to(torch.int32).to(torch.uint16)
    else:
        cls = torch.zeros(rows, device="cuda", dtype=torch.int32).to(torch.uint16)
    y = torch.empty_like(x)
    ws = torch.zeros(plan.workspace_bytes(rows), dtype=torch.uint8, device="cuda")
    for _ in range(3):
        plan.forward(x, cls, out=y, workspace=ws)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        plan.forward(x, cls, out=y, workspace=ws)
    e.record()
    e.synchronize()
    ms = s.elapsed_time(e) / iters
    gbs = rows * (8 * n + (2 if classes > 1 else 0)) / (ms * 1e-3) / 1e9
    env = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("HYGT_"))
    print(f"{spec:18s} {env:40s} {ms:7.3f} ms  {gbs:7.0f} GB/s  {gbs / 6552:.3f}", flush=True)


if __name__ == "__main__":
    for sp in sys.argv[1:]:
        run(sp)
