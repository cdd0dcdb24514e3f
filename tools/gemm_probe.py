"""Tensor-core path probe (development tool): per-direction kernel times of one config with and
without the fused energy, SM clocks sampled during each, optional knobs.
    python tools/gemm_probe.py --config 5 [--knob NAME=V ...] [--iters 10]"""
import argparse
import os
import statistics
import sys
import threading
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_21728_b200._lib as L  # noqa: E402
from paper_2505_21728_b200 import HyGTPlan  # noqa: E402
from paper_2505_21728_b200.synth import make_workload  # noqa: E402


def clocks_during(fn):
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
    except Exception:
        return fn(), None
    s, stop = [], False

    def poll():
        while not stop:
            s.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
            time.sleep(0.002)
    th = threading.Thread(target=poll)
    th.start()
    r = fn()
    stop = True
    th.join()
    return r, (statistics.median(s) if s else None)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--knob", action="append", default=[])
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--kernel", default="auto")
    ap.add_argument("--interleave", action="store_true")
    ap.add_argument("--sorted", action="store_true", help="class ids sorted by row (bucketed order = row order)")
    a = ap.parse_args()
    for kv in a.knob:
        k, v = kv.split("=")
        L.set_knob(k, int(v))
    w = make_workload(a.config)
    rows = w.cfg.count
    cls = w.make_classes(rows)
    if a.sorted:
        cls = torch.sort(cls.view(torch.int16).to(torch.int32)).values.to(torch.int16).view(torch.uint16)
    x = w.make_rows(rows, cls)
    y = torch.empty_like(x)
    xr = torch.empty_like(x)
    plan = HyGTPlan(w.models, w.perms, kernel=a.kernel)
    ws = torch.zeros(plan.workspace_bytes(rows), dtype=torch.uint8, device="cuda")
    energy = torch.zeros(w.cfg.classes, w.n, dtype=torch.float64, device="cuda")
    plan.bucket(cls, rows, ws)
    bpr = 8 * w.n + (2 if w.cfg.classes > 1 else 0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def timeit(name, f):
        for _ in range(3):
            f()
        torch.cuda.synchronize()

        def run():
            ts = []
            for _ in range(a.iters):
                flush.fill_(1)
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                f()
                e.record()
                ts.append((s, e))
            torch.cuda.synchronize()
            return statistics.mean(s.elapsed_time(e) for s, e in ts)
        ms, mhz = clocks_during(run)
        print(f"{name:22s} {ms:8.3f} ms  {rows * bpr / ms / 1e6 / 6546.2:6.3f} of HBM  sm {mhz} MHz  "
              f"[{plan.path}, knobs {a.knob}]", flush=True)

    ops = [("forward", lambda: plan.forward(x, cls, out=y, workspace=ws, reuse_buckets=True)),
           ("forward+energy", lambda: plan.forward_energy(x, cls, energy, out=y, workspace=ws, reuse_buckets=True)),
           ("inverse", lambda: plan.inverse(y, cls, out=xr, workspace=ws, reuse_buckets=True))]
    if a.interleave:  # round robin, so that the power-capped clock affects all three alike
        for _ in range(3):
            for _, f in ops:
                f()
        torch.cuda.synchronize()

        def run():
            ev = {k: [] for k, _ in ops}
            for _ in range(a.iters):
                for k, f in ops:
                    flush.fill_(1)
                    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    s.record()
                    f()
                    e.record()
                    ev[k].append((s, e))
            torch.cuda.synchronize()
            return {k: statistics.mean(s.elapsed_time(e) for s, e in v) for k, v in ev.items()}
        res, mhz = clocks_during(run)
        for k, ms in res.items():
            print(f"{k:22s} {ms:8.3f} ms  {rows * bpr / ms / 1e6 / 6546.2:6.3f} of HBM  sm {mhz} MHz (round robin)  "
                  f"[{plan.path}, knobs {a.knob}]", flush=True)
    else:
        for k, f in ops:
            timeit(k, f)
    plan.sync_status(ws)


if __name__ == "__main__":
    main()
