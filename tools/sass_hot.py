"""Rank SASS instructions of an ncu source-page CSV export by executed count
and stall samples; also totals per opcode.
    ncu -i rep --page source --csv --print-source sass -k regex:K > k.csv
    python tools/sass_hot.py k.csv [top]"""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
h = rows[1]
iA, iS, iE, iW = h.index("Address"), h.index("Source"), h.index("Instructions Executed"), h.index(
    "Warp Stall Sampling (All Samples)")
data = []
for r in rows[2:]:
    try:
        data.append((int(r[iE] or 0), int(r[iW] or 0), r[iA], r[iS]))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data)
stall = sum(d[1] for d in data)
print(f"total warp-instructions {tot}, stall samples {stall}")
ops = Counter()
for e, w, a, s in data:
    ops[s.split()[0] if not s.startswith("@") else s.split()[1]] += e
for op, n in ops.most_common(25):
    print(f"  {op:22s} {n:12d} {100 * n / tot:5.1f}%")
print("-- top by stall samples")
for e, w, a, s in sorted(data, key=lambda d: -d[1])[:top]:
    print(f"{a:>6s} exec {e:10d} stall {w:7d}  {s[:90]}")
