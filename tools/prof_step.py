"""One bucket + forward(+energy) + inverse step of a config on resident rows, for ncu captures
(development tool): python tools/prof_step.py --config 5 [--steps 2]"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_21728_b200 import HyGTPlan  # noqa: E402
from paper_2505_21728_b200.synth import make_workload  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=5)
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--rows", type=int, default=0)
a = ap.parse_args()
w = make_workload(a.config)
rows = a.rows or w.cfg.count
cls = w.make_classes(rows)
x = w.make_rows(rows, cls)
y = torch.empty_like(x)
xr = torch.empty_like(x)
plan = HyGTPlan(w.models, w.perms)
ws = torch.zeros(plan.workspace_bytes(rows), dtype=torch.uint8, device="cuda")
e = torch.zeros(w.cfg.classes, w.n, dtype=torch.float64, device="cuda") if w.cfg.energy else None
for _ in range(a.steps):
    plan.bucket(cls, rows, ws)
    if e is not None:
        plan.forward_energy(x, cls, e, out=y, workspace=ws, reuse_buckets=True)
    else:
        plan.forward(x, cls, out=y, workspace=ws, reuse_buckets=True)
    plan.inverse(y, cls, out=xr, workspace=ws, reuse_buckets=True)
plan.sync_status(ws)
torch.cuda.synchronize()
print("ok", plan.path, (xr - x).abs().max().item())
