"""Top SASS instructions by warp-stall samples from `ncu -i rep --page source --csv` output.
    ncu -i rep --page source --csv --kernel-name regex:K --launch-count 1 | python scripts/ncu_hot.py [n]"""
import csv
import sys
from collections import Counter

n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
rows = list(csv.reader(sys.stdin))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hdr]
iS, iN, iE = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
data = []
for r in rows[hdr + 1:]:
    if r and r[0] in ("Kernel Name", "Address"):
        break                      # first kernel only
    if len(r) > iN and r[iN].isdigit():
        data.append(r)
tot = sum(int(r[iN] or 0) for r in data)
ops = Counter()
for r in data:
    ops[r[iS].split()[0] if r[iS].split() else "?"] += int(r[iN] or 0)
print("total samples", tot, " instructions", sum(int(r[iE] or 0) for r in data))
print("by opcode:", ", ".join(f"{k} {v / tot:.1%}" for k, v in ops.most_common(14)))
top = sorted(range(len(data)), key=lambda i: -int(data[i][iN] or 0))[:n]
for i in sorted(top):
    print(f"{i:5d} {int(data[i][iN]) / tot:6.2%}  {data[i][iS].strip()[:90]}")
