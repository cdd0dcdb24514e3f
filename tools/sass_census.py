"""SASS opcode census of the built kernels (cuobjdump -sass over paper_2505_21728_b200/csrc/build/*.o):
per kernel, the instructions that show which hardware path it uses -- tcgen05 (UTC*MMA, UTCBAR,
LDTM/STTM, UTCCP), bulk copies / TMA (UBLKCP, UBLKPF, UTMALDG/UTMASTG), mbarriers (SYNCS.*),
packed FFMA2, shared-memory vectors (LDS.128/STS.128), shuffles, wide integer multiplies.
    python tools/sass_census.py > profiles/r02/sass_census.txt"""
import collections
import glob
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["UTCHMMA", "UTCQMMA", "UTCIMMA", "UTCBAR", "LDTM", "STTM", "UTCCP", "UBLKCP", "UBLKPF", "UTMALDG", "UTMASTG",
        "SYNCS.ARRIVE", "SYNCS.PHASECHK", "FFMA2", "FFMA", "FMUL2", "HMMA", "LDS.128", "STS.128", "LDS.64", "STS.64",
        "LDG.E.128", "STG.E.128", "LDGSTS", "SHFL", "IMAD.WIDE", "F2FP", "DFMA", "DADD"]


def demangle(names):
    try:
        out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.split("\n")
        return out[: len(names)]
    except Exception:
        return names


def main():
    rows = []
    for obj in sorted(glob.glob(os.path.join(ROOT, "paper_2505_21728_b200", "csrc", "build", "*.o"))):
        sass = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
        if not sass:
            continue
        for m in re.finditer(r"Function : (\S+)\n(.*?)(?=\n\s+Function : |\Z)", sass, re.S):
            name, body = m.group(1), m.group(2)
            ops = re.findall(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", body)
            c = collections.Counter()
            for op in ops:
                for k in KEYS:
                    if op == k or op.startswith(k + "."):
                        c[k] += 1
                        break
            rows.append((os.path.basename(obj), name, len(ops), c))
    names = demangle([r[1] for r in rows])
    print("# SASS census (cuobjdump -sass, sm_100a). Columns: total instructions, then counts of the")
    print("# opcodes that identify the hardware path. Kernels grouped by object file.")
    for (obj, _, total, c), nm in zip(rows, names):
        nm = re.sub(r"\(.*", "", nm.replace("(anonymous namespace)::", ""))
        parts = [f"{k}={c[k]}" for k in KEYS if c[k]]
        print(f"{obj:26s} {nm[:90]:90s} n={total:6d}  " + " ".join(parts))


if __name__ == "__main__":
    sys.exit(main())
