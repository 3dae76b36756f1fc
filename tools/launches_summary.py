"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV)."""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0}.get(r[ui], 1e-6)
        name = r[ki].split("(")[0][:70]
        tot[name] += float(r[vi].replace(",", "")) * scale
        cnt[name] += 1
    allt = sum(tot.values())
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"{v:10.3f} ms {100 * v / allt:5.1f}%  x{cnt[k]:<4d} {k}")


if __name__ == "__main__":
    main(sys.argv[1])
