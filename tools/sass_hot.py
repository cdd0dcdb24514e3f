"""Summarise an ncu source-page CSV (--page source --print-source sass): stall samples per
instruction, grouped into regions, and the top instructions."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]
num = lambda v: float(v.replace(",", "")) if v not in ("", None) else 0.0
tot = sum(num(d["Warp Stall Sampling (All Samples)"]) for d in data)
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
print(f"instructions {len(data)}  samples {tot:.0f}")
agg = {c: sum(num(d[c]) for d in data) for c in stall_cols}
print("stalls:", ", ".join(f"{c[6:]} {v / tot:.1%}" for c, v in sorted(agg.items(), key=lambda kv: -kv[1])[:8]))
top = sorted(data, key=lambda d: -num(d["Warp Stall Sampling (All Samples)"]))[: int(sys.argv[2]) if len(sys.argv) > 2 else 30]
for d in top:
    s = num(d["Warp Stall Sampling (All Samples)"])
    main = sorted(((num(d[c]), c[6:]) for c in stall_cols), reverse=True)[:2]
    print(f"{d['Address']:>6} {s / tot:6.2%} {d['Source'][:60]:60} ex={d['Instructions Executed']:>10} "
          f"wf={d['L1 Wavefronts Shared']:>9} ideal={d['L1 Wavefronts Shared Ideal']:>9} "
          + " ".join(f"{n}:{v:.0f}" for v, n in main))
