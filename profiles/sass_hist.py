"""Opcode histogram of an `ncu --page source --csv` export (SASS view):
    python profiles/sass_hist.py src.csv"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hi]
data = [r for r in rows[hi + 1:] if len(r) == len(h) and r[0] != "Address"]
iS, iE, iW = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
num = lambda x: int(float(x.replace(",", "") or 0))  # noqa: E731
tot = sum(num(r[iE]) for r in data)
print("total warp instructions", tot)
c, w = collections.Counter(), collections.Counter()
for r in data:
    parts = r[iS].split()
    if not parts:
        continue
    op = parts[1] if parts[0].startswith("@") else parts[0]
    c[op.split(".")[0]] += num(r[iE])
    w[op.split(".")[0]] += num(r[iW])
for k, v in c.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 25):
    print(f"{k:10s} {v:12d} {100 * v / max(tot, 1):5.1f}%  stall-samples {w[k]}")
