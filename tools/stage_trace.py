"""Timeline of the staged kernel's roles on CTA 0 (debug hook hygt_debug_stage_trace)."""
import ctypes
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2505_21728_b200 import _lib  # noqa: E402
from paper_2505_21728_b200.synth import make_workload  # noqa: E402
from paper_2505_21728_b200.plan import HyGTPlan  # noqa: E402

w = make_workload(2)
cls = w.make_classes(w.cfg.count)
x = w.make_rows(w.cfg.count, cls)
plan = HyGTPlan(w.models, w.perms)
print("path", plan.path)
ws = torch.zeros(plan.workspace_bytes(w.cfg.count), dtype=torch.uint8, device="cuda")
y = plan.forward(x, cls, workspace=ws)
plan.bucket(cls, w.cfg.count, ws)
tr = torch.zeros(64 * 16, dtype=torch.int64, device="cuda")
lib = _lib.lib()
lib.hygt_debug_stage_trace.argtypes = [ctypes.c_void_p]
lib.hygt_debug_stage_trace(ctypes.c_void_p(tr.data_ptr()))
torch.cuda.synchronize()
y = plan.forward(x, cls, out=y, workspace=ws, reuse_buckets=True)
torch.cuda.synchronize()
lib.hygt_debug_stage_trace(None)
t = tr.view(64, 16).cpu().numpy()
t0 = t[0, 0]
names = ["load", "cons.start", "cons.end", "computed@prod", "store.read"]
cols = [0, 3, 4, 5, 6]
print("k    " + " ".join(f"{n:>13}" for n in names) + "  compute  load->start")
for k in range(40):
    r = t[k]
    print(f"{k:3d}  " + " ".join(f"{(r[c] - t0) / 1000 if r[c] else float('nan'):13.1f}" for c in cols) +
          f"  {(r[4] - r[3]) / 1000:7.1f} {(r[3] - r[0]) / 1000:8.1f}")
