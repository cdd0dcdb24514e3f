"""One bucket + forward(+energy) + inverse step of a config on resident rows, for ncu captures
(development tool): python tools/prof_step.py --config 5 [--steps 2] [--range]
--range brackets the last step's forward with cudaProfilerStart/Stop, so `ncu --replay-mode
range --profile-from-start off` measures a whole launch chain (config 3's per-class grids) as
one result."""
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
ap.add_argument("--range", action="store_true", help="bracket the last step with cudaProfilerStart/Stop")
ap.add_argument("--kernel", default="auto", choices=["auto", "butterfly", "tensor"])
a = ap.parse_args()
w = make_workload(a.config)
rows = a.rows or w.cfg.count
cls = w.make_classes(rows)
x = w.make_rows(rows, cls)
y = torch.empty_like(x)
xr = torch.empty_like(x)
if w.cfg.klt:  # config 4: the KLT comparison path
    from paper_2505_21728_b200 import KLTPlan
    kplan = KLTPlan(w.klt_bases())
    kws = torch.zeros(max(256, kplan.workspace_bytes(rows)), dtype=torch.uint8, device="cuda")
    for i in range(a.steps):
        kplan.bucket(cls, rows, kws)
        if a.range and i == a.steps - 1:
            torch.cuda.synchronize()
            torch.cuda.profiler.start()
        kplan.forward(x, cls, out=y, workspace=kws, reuse_buckets=True)
        if a.range and i == a.steps - 1:  # the measured range: one forward, as for the HyGT configs
            torch.cuda.synchronize()
            torch.cuda.profiler.stop()
        kplan.inverse(y, cls, out=xr, workspace=kws, reuse_buckets=True)
    torch.cuda.synchronize()
    print("ok klt", (xr - x).abs().max().item())
    raise SystemExit(0)
plan = HyGTPlan(w.models, w.perms, kernel=a.kernel)
ws = torch.zeros(plan.workspace_bytes(rows), dtype=torch.uint8, device="cuda")
e = torch.zeros(w.cfg.classes, w.n, dtype=torch.float64, device="cuda") if w.cfg.energy else None
for i in range(a.steps):
    plan.bucket(cls, rows, ws)
    if a.range and i == a.steps - 1:  # the measured range: one forward (the bucketing excluded)
        torch.cuda.synchronize()
        torch.cuda.profiler.start()
    if e is not None:
        plan.forward_energy(x, cls, e, out=y, workspace=ws, reuse_buckets=True)
    else:
        plan.forward(x, cls, out=y, workspace=ws, reuse_buckets=True)
    if a.range and i == a.steps - 1:
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
    plan.inverse(y, cls, out=xr, workspace=ws, reuse_buckets=True)
plan.sync_status(ws)
torch.cuda.synchronize()
print("ok", plan.path, (xr - x).abs().max().item())
