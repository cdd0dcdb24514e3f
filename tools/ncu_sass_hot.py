"""Hottest SASS instructions of an ncu report (development tool): by stall samples and by shared
wavefronts. python tools/ncu_sass_hot.py report.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
h = r[1]
rows = [dict(zip(h, x)) for x in r[2:] if len(x) == len(h)]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25


def f(d, k):
    try:
        return float(d.get(k, 0) or 0)
    except ValueError:
        return 0.0


tot = sum(f(d, "Warp Stall Sampling (All Samples)") for d in rows) or 1
print("== top stall instructions ==")
for i, d in sorted(enumerate(rows), key=lambda kv: -f(kv[1], "Warp Stall Sampling (All Samples)"))[:n]:
    top = sorted(((k, f(d, k)) for k in h if k.startswith("stall_") and "Not Issued" not in k), key=lambda kv: -kv[1])[:2]
    print(f"{i:5d} {f(d, 'Warp Stall Sampling (All Samples)') / tot:6.1%} {d['Source'].strip()[:70]:70s} {top}")
print("== shared wavefronts (excessive) ==")
for i, d in sorted(enumerate(rows), key=lambda kv: -f(kv[1], "L1 Wavefronts Shared"))[:12]:
    print(f"{i:5d} {d['Source'].strip()[:60]:60s} wf {f(d, 'L1 Wavefronts Shared'):.3e} ideal {f(d, 'L1 Wavefronts Shared Ideal'):.3e} exec {f(d, 'Instructions Executed'):.3e}")
