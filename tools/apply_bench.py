"""File-to-file drop-in timing: paper_2505_21728_b200/hygt_gpu_apply against the reference CLI's
`apply` (oracle/_ref/ref_apply, the unmodified headers, serial as the CLI is) on the same RBLK /
HYGT files, wall clock per process (parse, transform, write)."""
import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2505_21728_b200.formats import write_bundle, write_rblk  # noqa: E402

GPU = os.path.join(ROOT, "paper_2505_21728_b200", "hygt_gpu_apply")
REF = os.path.join(ROOT, "oracle", "_ref", "ref_apply")

ap = argparse.ArgumentParser()
ap.add_argument("--log2n", type=int, default=4)
ap.add_argument("--classes", type=int, default=35)
ap.add_argument("--rounds", type=int, default=3)
ap.add_argument("--rows", type=int, default=1 << 22)
ap.add_argument("--ref-rows", type=int, default=1 << 20, help="rows of the reference run (serial CLI)")
a = ap.parse_args()
n = 1 << a.log2n
rng = np.random.default_rng(5)
tmp = tempfile.mkdtemp(prefix="hygt_apply_")


def dataset(path, rows):
    cls = rng.integers(0, a.classes, rows).astype(np.uint16)
    x = (rng.standard_normal((rows, n)) * 16).astype(np.float32)
    write_rblk(path, a.log2n, a.classes, cls, x)


big, small = os.path.join(tmp, "big.rblk"), os.path.join(tmp, "small.rblk")
dataset(big, a.rows)
dataset(small, a.ref_rows)
A = a.rounds * a.log2n * n // 2
fmodel, qmodel = os.path.join(tmp, "f.hygt"), os.path.join(tmp, "q.hygt")
write_bundle(fmodel, a.log2n, angles=[rng.uniform(-np.pi, np.pi, A) for _ in range(a.classes)],
             perms=[rng.permutation(n) for _ in range(a.classes)])
write_bundle(qmodel, a.log2n, codes=[rng.integers(0, 256, A) for _ in range(a.classes)], angle_bits=8,
             precision_bits=10)


def run(exe, model, data, arith):
    out = os.path.join(tmp, "out.rblk")
    t = time.perf_counter()
    r = subprocess.run([exe, "--model", model, "--data", data, "--direction", "forward",
                        "--arithmetic", arith, "--out", out], capture_output=True, text=True)
    dt = time.perf_counter() - t
    assert r.returncode == 0, r.stderr
    return dt


for arith, model in (("float", fmodel), ("fixed", qmodel)):
    run(GPU, model, small, arith)  # warm the page cache and the CUDA context path
    g = min(run(GPU, model, big, arith) for _ in range(3))
    ref = run(REF, model, small, arith)
    print(json.dumps({"metric": "apply blocks/s (file to file, forward)", "arithmetic": arith, "N": n,
                      "classes": a.classes, "rounds": a.rounds, "rblk_mb": os.path.getsize(big) / 1e6,
                      "gpu_apply": {"rows": a.rows, "s": g, "blocks_per_s": a.rows / g},
                      "reference_apply": {"rows": a.ref_rows, "s": ref, "blocks_per_s": a.ref_rows / ref,
                                          "threads": 1},
                      "speedup": (a.rows / g) / (a.ref_rows / ref)}), flush=True)
