"""Summarise an nvcc -Xptxas -v log: registers / spills per kernel (demangled-ish)."""
import re
import sys

cur = None
rows = {}
for line in open(sys.argv[1]):
    m = re.search(r"Compiling entry function '([^']+)'", line)
    if m:
        cur = m.group(1)
        rows.setdefault(cur, {})
        continue
    m = re.search(r"Function properties for (\S+)", line)
    if m:
        cur = m.group(1)
        rows.setdefault(cur, {})
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur:
        rows[cur]["spill"] = f"{m.group(1)}/{m.group(2)}"
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        rows[cur]["regs"] = int(m.group(1))
for k, v in rows.items():
    m = re.search(r"hygt_apply_kernelILi(\d+)ELi(\d+)ELb(\d)ELb(\d)ELb(\d)", k)
    name = (f"apply N=2^{m.group(1)} L={m.group(2)} std={m.group(3)} fwd={m.group(4)} energy={m.group(5)}"
            if m else k[:70])
    print(f"{name:60s} regs={v.get('regs')} spill={v.get('spill', '0/0')}")
