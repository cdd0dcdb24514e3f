"""Summarise a gemm_trace.py log of the N = 256 TS kernel (development tool): mean per-tile
intervals over tiles 8..63 (events: 0 split start, 1 row maxima, 12 data slot free, 2 tile
written, 3 / 4 MMA issue start / committed, 5 / 6 epilogue start / end).
    python tools/trace_ts.py gpurun_out/trace.log"""
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
print(f"tiles {len(t)}: period {float(np.mean(np.diff(t[:, 1]))):.0f} cycles (split), "
      f"{float(np.mean(np.diff(t[:, 4]))):.0f} (MMA), {float(np.mean(np.diff(t[:, 6]))):.0f} (epilogue)")
print(f"  split: start->maxima {d(0, 1):.0f}, maxima->slot free {d(1, 12):.0f}, slot free->written {d(12, 2):.0f}")
print(f"  MMA: written->issue start {d(2, 3):.0f}, issue span {d(3, 4):.0f}, committed->epilogue start {d(4, 5):.0f}")
print(f"  epilogue span {d(5, 6):.0f}; split start -> epilogue end {d(0, 6):.0f}")
