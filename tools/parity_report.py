"""fp32 forward error distribution against the reference / oracle (GPU box).

For every fp32 parity case of the test suite (reference goldens, the
randomised shapes, §8d populations in both variants) this prints and writes
profiles/r02_parity_report.json: the error e = |y - ref| / max(1, |ref|) per
output element (max, quantiles, count above 1e-5), and for elements above
1e-5 the conditioning of the computation that produced them: the largest
sum of |w * v| (plus |bias|) over the nodes the sample evaluates -- fp32
rounding scales with that magnitude, not with the output's.

    python tools/parity_report.py [--out profiles/r02_parity_report.json]
"""

from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))

from oracle import arrayneat_oracle as orc  # noqa: E402


def scale_of(nodes, tr, x):
    """(B,) max over evaluated nodes of |bias| + |resp| * sum |w v| (f64)."""
    x = np.asarray(x, dtype=np.float64)
    val = {r: x[:, i] for i, r in enumerate(tr["input_rows"])}
    into = {}
    for s, d, w, _ in tr["edges"]:
        into.setdefault(d, []).append((s, w))
    ins = set(tr["input_rows"])
    worst = np.zeros(x.shape[0])
    for r in tr["order"]:
        if r in ins:
            continue
        terms = [w * val[s] for s, w in sorted(into.get(r, []))]
        mag = np.abs(nodes[r, orc.BIAS]) + abs(nodes[r, orc.RESP]) * (
            np.sum(np.abs(terms), axis=0) if terms else 0.0)
        worst = np.maximum(worst, mag)
        agg = orc.agg_apply(int(nodes[r, orc.AGG]), terms, x.shape[0])
        val[r] = orc.act_apply(int(nodes[r, orc.ACT]), nodes[r, orc.BIAS] + nodes[r, orc.RESP] * agg)
    return worst


def summarise(name, err, scale):
    flat = err.reshape(-1)
    over = flat > 1e-5
    rec = {"case": name, "elements": int(flat.size), "max": float(flat.max()) if flat.size else 0.0,
           "p50": float(np.quantile(flat, 0.5)) if flat.size else 0.0,
           "p99": float(np.quantile(flat, 0.99)) if flat.size else 0.0,
           "p99_9": float(np.quantile(flat, 0.999)) if flat.size else 0.0,
           "over_1e-5": int(over.sum())}
    if over.any():
        s = np.broadcast_to(scale[..., None], err.shape).reshape(-1)[over]
        rec["over_scale_min"] = float(s.min())
        rec["over_err_div_scale_max"] = float((flat[over] / s).max())
    # the fp32 bound a condition-aware test can state: err <= 1e-5 * max(1, scale / 64)
    allscale = np.broadcast_to(scale[..., None], err.shape).reshape(-1)
    rec["max_err_over_cond_bound"] = float((flat / (1e-5 * np.maximum(1.0, allscale / 64.0))).max()) \
        if flat.size else 0.0
    return rec


def run_case(tn, name, nodes, conns, x, n_in, n_out, variant=0):
    st, cyc = tn.transform_arrays(nodes, conns, n_in, n_out)
    ok = np.setdiff1d(np.arange(nodes.shape[0]), cyc)
    y = tn.forward_arrays(st, None, x.astype(np.float32), variant=variant)
    errs, scales = [], []
    for p in ok:
        tr = orc.transform_genome(nodes[p], conns[p], n_in, n_out)
        ref = orc.forward_genome(nodes[p], tr, x[p].astype(np.float64))
        errs.append(np.abs(y[p] - ref) / np.maximum(1.0, np.abs(ref)))
        scales.append(scale_of(nodes[p], tr, x[p]))
    return summarise(name, np.stack(errs), np.stack(scales))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(REPO, "profiles", "r02_parity_report.json"))
    args = ap.parse_args()
    import paper_2404_01817_b200 as tn
    from conftest import load_golden
    recs = []
    for name in ("forward_small.npz", "forward_cfg2_T.npz", "forward_cfg2_M.npz", "corpus.npz"):
        g = load_golden(name)
        x = g["inputs_f32"] if "inputs_f32" in g else g["inputs"]
        recs.append(run_case(tn, name, g["nodes"], g["conns"], x.astype(np.float64), int(g["num_inputs"]),
                             int(g["num_outputs"])))
    for variant in ("T", "M"):
        nodes, conns = orc.synthetic_population(192, 128, 512, 32, 8, seed=77, variant=variant)
        x = np.random.default_rng(78).standard_normal((192, 512, 32)).astype(np.float32)
        for kv in (5, 8):
            recs.append(run_case(tn, f"synthetic_{variant}_192x512_variant{kv}", nodes, conns, x.astype(np.float64),
                                 32, 8, kv))
    for r in recs:
        print(json.dumps(r))
    with open(args.out, "w") as fh:
        json.dump({"what": "fp32 forward error e = |y-ref|/max(1,|ref|) per output element vs the f64 "
                           "oracle (pinned to the reference goldens); scale = max over evaluated nodes of "
                           "|bias| + |resp| * sum|w v|", "cases": recs}, fh, indent=1)


if __name__ == "__main__":
    main()
