"""Per-tile pipeline timeline of the tensor-core kernel (CTA 0) on a config (development tool):
    python tools/gemm_trace.py --config 5"""
import argparse
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_21728_b200._lib as L  # noqa: E402
from paper_2505_21728_b200 import HyGTPlan  # noqa: E402
from paper_2505_21728_b200.synth import make_workload  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=5)
ap.add_argument("--inverse", action="store_true")
ap.add_argument("--energy", action="store_true")
ap.add_argument("--knob", action="append", default=[])
a = ap.parse_args()
for kv in a.knob:
    L.set_knob(kv.split("=")[0], int(kv.split("=")[1]))
w = make_workload(a.config)
rows = w.cfg.count
cls = w.make_classes(rows)
x = w.make_rows(rows, cls)
y = torch.empty_like(x)
plan = HyGTPlan(w.models, w.perms, kernel="tensor")
ws = torch.zeros(plan.workspace_bytes(rows), dtype=torch.uint8, device="cuda")
plan.forward(x, cls, out=y, workspace=ws)
tr = torch.zeros(64 * 16, dtype=torch.int64, device="cuda")
lib = L.lib()
lib.hygt_debug_gemm_trace.argtypes = [C.c_void_p]
lib.hygt_debug_gemm_trace(tr.data_ptr())
if a.energy:
    en = torch.zeros(w.cfg.classes, w.n, dtype=torch.float64, device="cuda")
    plan.forward_energy(x, cls, en, out=y, workspace=ws)
else:
    (plan.inverse if a.inverse else plan.forward)(x, cls, out=y, workspace=ws)
torch.cuda.synchronize()
lib.hygt_debug_gemm_trace(None)
t = tr.view(64, 16).cpu().numpy()
t0 = t[0, 0]
names = ["p1s", "p1e", "p2e", "mmaS", "mmaC", "epiS", "epiE", "-", "b00", "b01", "b02", "b03", "a0free", "a0done", "a1free", "a1done"]
print("tile " + " ".join(f"{n:>8s}" for n in names) + "   (cycles since tile 0 pass-1 start; b0x: MMA issue points, aN: split atom N slot free / written)")
for k in range(64):
    if t[k, 6] == 0:
        break
    print(f"{k:4d} " + " ".join(f"{int(v - t0) if v else 0:8d}" for v in t[k, :16]))
