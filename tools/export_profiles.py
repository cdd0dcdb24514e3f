"""Turn one tools/profile_round.sh output directory (gpurun_out/<dir>) into the tracked summaries
under profiles/rNN: the bench line, the ncu launch list and its per-kernel summary, raw / details
CSV pages of every --set full capture, the whole-chain range CSVs, traffic.json.
    python tools/export_profiles.py gpurun_out/r02b profiles/r02"""
import collections
import csv
import glob
import os
import shutil
import subprocess
import sys

src, dst = sys.argv[1], sys.argv[2]
os.makedirs(dst, exist_ok=True)
for f in ["bench_default.json", "launches_default.csv"] + [os.path.basename(p) for p in glob.glob(f"{src}/range_cfg*.csv")] + \
        [os.path.basename(p) for p in glob.glob(f"{src}/corr_cfg*.json")] + [os.path.basename(p) for p in glob.glob(f"{src}/gputest.log")]:
    if os.path.exists(f"{src}/{f}"):
        shutil.copy(f"{src}/{f}", f"{dst}/{f}")

# per-kernel summary of the launch list
p = f"{src}/launches_default.csv"
if os.path.exists(p):
    lines = [l for l in open(p) if l.startswith('"')]
    rows = list(csv.reader(lines))
    h = rows[0]
    ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.OrderedDict()
    for r in rows[1:]:
        v = float(r[iv].replace(",", ""))
        v *= {"ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6}.get(r[iu], 1e-3)
        name = r[ik].split("(")[0]
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(a[1] for a in agg.values())
    with open(f"{dst}/launches_default_summary.txt", "w") as o:
        o.write("ncu --metrics gpu__time_duration.sum --clock-control none launch list of `python bench.py --steps 2 "
                "--warmup 3 --no-e2e --no-cpu` (cold-cache, serialised launches; includes the synthetic-row "
                "generator and torch helper kernels outside the timed steps)\n")
        o.write(f"{'kernel':<72} {'launches':>8} {'mean us':>10} {'total us':>11}  share\n")
        for name, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            o.write(f"{name[:70]:<72} {n:>8} {t / n:>10.1f} {t:>11.1f} {t / tot:>6.1%}\n")

# raw / details pages of the full captures
for rep in sorted(glob.glob(f"{src}/ncu_*.ncu-rep")):
    name = os.path.basename(rep)[4:-8]
    for page in ("raw", "details"):
        out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv"], capture_output=True, text=True).stdout
        open(f"{dst}/ncu_full_{name}_{page}.csv", "w").write(out)
    brief = subprocess.run([sys.executable, os.path.join(os.path.dirname(__file__), "ncu_brief.py"), rep],
                           capture_output=True, text=True).stdout
    open(f"{dst}/ncu_{name}_brief.txt", "w").write(brief)
subprocess.run([sys.executable, os.path.join(os.path.dirname(__file__), "traffic_json.py"), dst], check=False)
print("exported", src, "->", dst)
