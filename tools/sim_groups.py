"""Offline model of the forward program's edge entries under grouping rules.

Builds the emitted steps (ancestor cone of the outputs, non-input) of the
config-2 synthetic population with their topological levels and incoming
edge counts, then counts the padded edge entries (sum over groups of
columns x rounds) for the current join rule and for column-split grouping.
"""
import sys
from collections import defaultdict

import numpy as np

sys.path.insert(0, ".")
from paper_2404_01817_b200.synthetic import synthetic_population  # noqa: E402

I, O = 32, 8


def steps_of(nodes, conns):
    live = ~np.isnan(nodes[:, 0])
    key2row = {int(nodes[r, 0]): r for r in np.nonzero(live)[0]}
    ins = defaultdict(list)
    for c in conns:
        if np.isnan(c[0]) or c[2] != 1.0:
            continue
        a, b = key2row.get(int(c[0])), key2row.get(int(c[1]))
        if a is None or b is None:
            continue
        ins[b].append(a)
    # cone of outputs
    need = set()
    stack = [key2row[k] for k in range(I, I + O)]
    while stack:
        r = stack.pop()
        if r in need:
            continue
        need.add(r)
        stack.extend(ins[r])
    lvl = {}

    def level(r):
        if r in lvl:
            return lvl[r]
        if int(nodes[r, 0]) < I:
            lvl[r] = 0
            return 0
        lvl[r] = 1 + max([level(a) for a in ins[r]], default=0)
        return lvl[r]
    out = []
    for r in need:
        if int(nodes[r, 0]) < I:
            continue
        out.append((level(r), len(ins[r])))
    return out


def current(steps):
    by = defaultdict(list)
    for lv, c in steps:
        by[lv].append(c)
    total = 0
    for lv, cs in by.items():
        cs.sort(reverse=True)
        groups = []
        for c in cs:
            if groups and len(groups[-1]) < 4 and 2 * c >= groups[-1][0]:
                groups[-1].append(c)
            else:
                groups.append([c])
        for g in groups:
            gw = 4 if len(g) == 3 else len(g)
            total += gw * g[0]
    return total


def split_cols(steps, ncol=4):
    """Greedy: per level, fill groups of ncol columns; a step may own k
    contiguous columns (its list split in k chunks)."""
    by = defaultdict(list)
    for lv, c in steps:
        by[lv].append(c)
    total = 0
    for lv, cs in by.items():
        cs.sort(reverse=True)
        i = 0
        while i < len(cs):
            # take up to ncol steps; give spare columns to the longest
            g = cs[i:i + ncol]
            i += len(g)
            cols = [1] * len(g)
            for _ in range(ncol - len(g)):
                j = max(range(len(g)), key=lambda j: -(-g[j] // cols[j]))
                cols[j] += 1
            rounds = max(-(-g[j] // cols[j]) for j in range(len(g)))
            total += ncol * rounds
    return total


def main():
    n, c = synthetic_population(300, 128, 512, I, O, seed=20261018)
    real = cur = sp = 0
    for p in range(300):
        st = steps_of(n[p], c[p])
        real += sum(x for _, x in st)
        cur += current(st)
        sp += split_cols(st)
    print(f"real {real/300:.1f} current {cur/300:.1f} split4 {sp/300:.1f} per genome")


if __name__ == "__main__":
    main()
