"""Attribute executed instructions / stall samples to CUDA source lines from an
ncu `--page source --csv --print-source cuda,sass` export.
    python tools/line_hot.py export.csv [top]"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
inst = defaultdict(int)
stall = defaultdict(int)
text = {}
fname = "?"
h = None
cur = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        h = r
        iE = h.index("Instructions Executed")
        iW = h.index("Warp Stall Sampling (All Samples)")
        continue
    if h is None or r[0] == "Function Name":
        continue
    if r[0]:  # a source line row
        cur = (fname, int(r[0]))
        text[cur] = r[1].strip()[:90]
    try:
        e = int(r[iE] or 0)
        w = int(r[iW] or 0)
    except (ValueError, IndexError):
        continue
    if cur is not None and not r[0]:
        inst[cur] += e
        stall[cur] += w
tot = sum(inst.values()) or 1
st = sum(stall.values()) or 1
print(f"total inst {tot} stall samples {st}")
for k in sorted(inst, key=lambda k: -inst[k])[:top]:
    print(f"{k[0]}:{k[1]:<5} {100 * inst[k] / tot:5.1f}% inst {100 * stall[k] / st:5.1f}% stall  {text.get(k, '')}")
