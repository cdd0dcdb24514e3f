"""Fixed-point (bit-exact integer) HyGT throughput: forward+inverse over a config's shape with
8-bit codes and a p=10 TrigTable."""
import argparse
import json
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2505_21728_b200 import TrigTable, quantize_model  # noqa: E402
from paper_2505_21728_b200.plan import FixedPlan  # noqa: E402
from paper_2505_21728_b200.synth import make_workload  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--rows", type=int, default=0)
ap.add_argument("--steps", type=int, default=10)
a = ap.parse_args()
w = make_workload(a.config)
rows = a.rows or w.cfg.count
table = TrigTable(8, 10)
qm = [quantize_model(m, 8) for m in w.models]
plan = FixedPlan(qm, table, w.perms)
cls = w.make_classes(rows)
x = torch.round(w.make_rows(rows, cls)).to(torch.int64).clamp_(-(1 << 20), 1 << 20)
y = torch.empty_like(x)
xr = torch.empty_like(x)
for _ in range(3):
    plan.forward(x, cls, out=y)
    plan.inverse(y, cls, out=xr)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
tf = ti = 0.0
for _ in range(a.steps):
    ev[0].record()
    plan.forward(x, cls, out=y)
    ev[1].record()
    plan.inverse(y, cls, out=xr)
    ev[2].record()
    torch.cuda.synchronize()
    tf += ev[0].elapsed_time(ev[1])
    ti += ev[1].elapsed_time(ev[2])
ms = (tf + ti) / a.steps
n = w.n
bpr = 2 * (8 * n * 2 + (2 if w.cfg.classes > 1 else 0))  # int64 in + out, both directions
print(json.dumps({"metric": "fixed-point HyGT fwd+inv vectors/s", "workload": w.cfg.name, "rows": rows,
                  "value": rows / (ms * 1e-3), "ms_fwd": tf / a.steps, "ms_inv": ti / a.steps,
                  "hbm_gbs": rows * bpr / (ms * 1e-3) / 1e9,
                  "roundtrip_exact": bool(torch.equal(xr, x))}))
