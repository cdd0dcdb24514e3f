"""Relative-L2 / max-abs errors of every float kernel path against the oracle on a config shape
(forward, inverse and round trip), for DESIGN.md's precision table.
    python tools/precision_report.py [--config 5] [--rows 16384]"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402
from paper_2505_21728_b200 import HyGTPlan  # noqa: E402
from paper_2505_21728_b200.synth import make_workload  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=5)
ap.add_argument("--rows", type=int, default=1 << 14)
ap.add_argument("--knob", action="append", default=[])
ap.add_argument("--kernels", default="butterfly,tensor")
a = ap.parse_args()
import paper_2505_21728_b200._lib as L  # noqa: E402
for kv in a.knob:
    L.set_knob(kv.split("=")[0], int(kv.split("=")[1]))
w = make_workload(a.config)
cls = w.make_classes(a.rows)
x = w.make_rows(a.rows, cls)
full, mask = None, 0
if w.perms is not None:
    full = np.concatenate([w.perms, np.tile(np.arange(w.n, dtype=np.uint16), (w.cfg.classes, 1, 1))], 1)
    mask = (1 << (w.cfg.rounds - 1)) - 1
xh, ch = x.cpu().numpy(), cls.cpu().numpy()
ref = O.apply_batch(w.cfg.log2_n, w.cfg.rounds, w.angles, full, mask, xh, ch, hoist=True)
refi = O.apply_batch(w.cfg.log2_n, w.cfg.rounds, w.angles, full, mask, xh, ch, inverse=True, hoist=True)


def err(y, r):
    e = y.astype(np.float64) - r
    return {"rel_l2": float(np.linalg.norm(e) / np.linalg.norm(r)), "max_abs_over_max_x": float(np.abs(e).max() / np.abs(xh).max())}


for kernel in a.kernels.split(","):
    plan = HyGTPlan(w.models, w.perms, kernel=kernel)
    y = plan.forward(x, cls)
    z = plan.inverse(x, cls)
    b = plan.inverse(y, cls)
    plan.sync_status()
    print(json.dumps({"config": w.cfg.name, "path": plan.path, "rows": a.rows,
                      "forward": err(y.cpu().numpy(), ref), "inverse": err(z.cpu().numpy(), refi),
                      "roundtrip": err(b.cpu().numpy(), xh.astype(np.float64))}))
