"""Shared-memory wavefronts per opcode (per row) from an ncu source-page CSV."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]
num = lambda v: float(v.replace(",", "")) if v else 0.0
nrows = float(sys.argv[2]) if len(sys.argv) > 2 else 2 ** 24
agg = {}
for d in data:
    wf = num(d["L1 Wavefronts Shared"])
    if wf == 0:
        continue
    toks = d["Source"].split()
    op = toks[1] if toks[0].startswith("@") else toks[0]
    a = agg.setdefault(op, [0, 0, 0])
    a[0] += num(d["Instructions Executed"])
    a[1] += wf
    a[2] += num(d["L1 Wavefronts Shared Ideal"])
tot = sum(v[1] for v in agg.values())
print(f"total shared wavefronts/row {tot / nrows:.3f}")
for k, (ex, wf, ide) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:12} inst/row {ex / nrows:6.3f}  wf/row {wf / nrows:6.3f} ideal/row {ide / nrows:6.3f}  wf/inst {wf / max(ex, 1):5.2f}")
if len(sys.argv) > 3:
    top = sorted(data, key=lambda d: -(num(d["L1 Wavefronts Shared"]) - num(d["L1 Wavefronts Shared Ideal"])))[:int(sys.argv[3])]
    for d in top:
        print("  excess", int(num(d["L1 Wavefronts Shared"]) - num(d["L1 Wavefronts Shared Ideal"])), d["Source"][:60],
              int(num(d["Instructions Executed"])))
