"""Summarise a gemm_trace.py log (development tool): mean per-tile intervals over tiles 8..63.
    python tools/trace_summary.py gpurun_out/trace.log"""
import sys

import numpy as np

rows = []
for line in open(sys.argv[1]):
    f = line.split()
    if len(f) == 17 and f[0].isdigit():
        rows.append([int(v) for v in f])
t = np.array(rows, dtype=np.int64)
t = t[t[:, 0] >= 8]
d = lambda a, b: float(np.mean(t[:, 1 + b] - t[:, 1 + a]))  # noqa: E731
per = float(np.mean(np.diff(t[:, 1])))
print(f"tiles {len(t)}: period {per:.0f} cycles")
print(f"  split: loads->max {d(0, 1):.0f}, max->atoms written {d(1, 2):.0f}")
print(f"  MMA: start->first corr atom issued {d(3, 8):.0f}, corr ka0->ka1 {d(8, 9):.0f}, "
      f"first corr->first main {d(8, 10):.0f}, main ka0->ka1 {d(10, 11):.0f}, issue span {d(3, 4):.0f}")
print(f"  split atoms: loads->atom0 slot free {d(0, 12):.0f}, atom0 convert {d(12, 13):.0f}, "
      f"atom0 done->atom1 slot free {d(13, 14):.0f}, atom1 convert {d(14, 15):.0f}")
print(f"  epilogue: MMA committed->epilogue start {d(4, 5):.0f}, epilogue span {d(5, 6):.0f}")
