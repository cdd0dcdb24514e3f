"""Per-class correlation accumulation throughput on a config's rows, with the
reference CorrelationAccumulator timed on a host sample (oracle/_ref/libhygt_ref.so)."""
import argparse
import ctypes
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = __file__.rsplit("/tools/", 1)[0]
sys.path.insert(0, ROOT)
from paper_2505_21728_b200 import correlation  # noqa: E402
from paper_2505_21728_b200.synth import make_workload  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--rows", type=int, default=0)
ap.add_argument("--steps", type=int, default=5)
ap.add_argument("--knob", action="append", default=[])
a = ap.parse_args()
import paper_2505_21728_b200._lib as _L  # noqa: E402
for kv in a.knob:
    _L.set_knob(kv.split("=")[0], int(kv.split("=")[1]))
w = make_workload(a.config)
rows = a.rows or w.cfg.count
cls = w.make_classes(rows)
x = w.make_rows(rows, cls)
C, n = w.cfg.classes, w.n
ws = torch.zeros(1 << 20, dtype=torch.uint8, device="cuda")
s, k = correlation(x, cls, C, workspace=ws)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.steps):
    s.zero_()
    k.zero_()
    correlation(x, cls, C, sums=s, counts=k, workspace=ws)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.steps
out = {"metric": "per-class correlation accumulation rows/s", "workload": w.cfg.name, "rows": rows,
       "value": rows / (ms * 1e-3), "ms": ms, "gb_s": rows * (4 * n + 2) / (ms * 1e-3) / 1e9,
       "fp64_gflops": rows * n * n * 2 / (ms * 1e-3) / 1e9}
ref = os.path.join(ROOT, "oracle", "_ref", "libhygt_ref.so")
if os.path.exists(ref):
    L = ctypes.CDLL(ref)
    p = ctypes.c_void_p
    L.ref_correlation.argtypes = [ctypes.c_int, ctypes.c_int, p, p, ctypes.c_uint64, p, p]
    m = min(rows, max(2000, int(2e8 / (n * n))))
    xs = x[:m].cpu().numpy()
    cs = cls[:m].cpu().numpy().astype(np.uint16)
    phi = np.zeros((C, n, n))
    kk = np.zeros(C, np.uint64)
    t = time.perf_counter()
    L.ref_correlation(w.cfg.log2_n, C, xs.ctypes.data, cs.ctypes.data, m, phi.ctypes.data, kk.ctypes.data)
    dt = time.perf_counter() - t
    out["cpu_reference"] = {"value": m / dt, "unit": "rows/s", "cores": 1, "sample": f"{m} rows"}
print(json.dumps(out))
