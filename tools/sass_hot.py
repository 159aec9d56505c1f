"""Summarise an `ncu --page source --print-source sass --csv` dump: opcode mix
and top stall lines (first kernel section only)."""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = []
for r in rows[2:]:
    if r and r[0] == "Kernel Name":
        break
    if len(r) == len(hdr) and r[0] != "Address":
        data.append(r)
iS, iE, iW, iA = (hdr.index(k) for k in ("Source", "Instructions Executed", "Warp Stall Sampling (All Samples)", "Address"))
f = lambda x: float(x.replace(",", "") or 0)
tot = sum(f(r[iE]) for r in data) or 1
totw = sum(f(r[iW]) for r in data) or 1
print("warp instructions", tot, "stall samples", totw, "sass lines", len(data))
c, w = Counter(), Counter()
for r in data:
    t = r[iS].split()
    if not t:
        continue
    op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
    c[op] += f(r[iE])
    w[op] += f(r[iW])
for op, v in c.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 20):
    print(f"{op:10s} inst {v / tot * 100:5.1f}%  stall {w[op] / totw * 100:5.1f}%")
print("--- top stall lines")
for r in sorted(data, key=lambda r: -f(r[iW]))[:14]:
    print(r[iA], r[iS][:90], r[iW], r[iE])
