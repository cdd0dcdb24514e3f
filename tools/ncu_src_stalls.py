"""Warp-stall samples of an ncu report attributed to CUDA source lines (development tool; needs
a -lineinfo build): python tools/ncu_src_stalls.py report.ncu-rep [N] [FILE_SUBSTRING]"""
import collections
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
want = sys.argv[3] if len(sys.argv) > 3 else ""
rows = list(csv.reader(io.StringIO(out)))
tot = collections.Counter()
kinds = collections.defaultdict(collections.Counter)
src = {}
fname = ""
hdr = None
cur = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 4:
        continue
    if r[0]:  # a source line
        cur = (fname, int(r[0]))
        src[cur] = r[1]
    if r[2] and cur is not None:  # a SASS row under the current source line
        d = dict(zip(hdr[2:], r[2:]))
        try:
            s = float(d.get("Warp Stall Sampling (All Samples)", 0) or 0)
        except ValueError:
            s = 0
        tot[cur] += s
        for k, v in d.items():
            if k.startswith("stall_") and "Not Issued" not in k:
                try:
                    kinds[cur][k] += float(v or 0)
                except ValueError:
                    pass
total = sum(tot.values()) or 1
print(f"total samples {total:.0f}")
for key, s in tot.most_common():
    if want and want not in key[0]:
        continue
    top = ", ".join(f"{k[6:]} {v / s:.0%}" for k, v in kinds[key].most_common(3) if v)
    print(f"{s / total:6.1%} {key[0].split('/')[-1]}:{key[1]:<5d} {src[key].strip()[:70]:70s} [{top}]")
    n -= 1
    if n == 0:
        break
