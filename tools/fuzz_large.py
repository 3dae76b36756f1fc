"""Large randomised parity run (evidence, not a test): populations of 200-1500
genomes with tensor-core-eligible input widths go through the device-planned
forward (every plan class, dynamic task scheduling, programmatic dependent class
launches); genomes sampled from every class are compared with the oracle.
    python tools/fuzz_large.py [cases] > report.json"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2404_01817_b200 as tn  # noqa: E402
from oracle import arrayneat_oracle as orc  # noqa: E402

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 30
report = []
worst_all = 0.0
for seed in range(cases):
    rng = np.random.default_rng(5000 + seed)
    n_in = int(rng.choice([4, 8, 16, 24, 32]))
    n_out = int(rng.integers(1, 9))
    max_nodes = int(rng.integers(n_in + n_out + 8, 181))
    max_conns = int(rng.integers(64, 601))
    pop = int(rng.integers(200, 1501))
    batch = int(rng.choice([256, 384, 512, 1024]))
    variant = str(rng.choice(["T", "T", "M"]))
    prune = bool(rng.integers(0, 2))
    precision = "f64" if rng.random() < 0.15 else "f32"
    nodes, conns = orc.synthetic_population(pop, max_nodes, max_conns, n_in, n_out, seed=seed, variant=variant,
                                            min_conns=min(32, max_conns), max_conns_drawn=max_conns)
    st, cyc = tn.transform_arrays(nodes, conns, n_in, n_out, precision=precision, prune=prune)
    dt = torch.float64 if precision == "f64" else torch.float32
    x = torch.randn((pop, batch, n_in), device="cuda", dtype=dt, generator=torch.Generator("cuda").manual_seed(seed))
    out = tn.forward_device(st, x).cpu().numpy()
    if st.precision & tn.inference.FMT_TC:
        counts = tn.inference.tc_plan_counts(st)
        ids = st._cache["tcplan"][0].view(tn.inference.TC_NCLASS, -1).cpu().numpy()
        picks = [int(p) for c in range(tn.inference.TC_NCLASS) for p in ids[c, :counts[c]][:6]]
        counts = counts.tolist()
    else:
        counts = None
        picks = [int(p) for p in rng.choice(pop, size=min(12, pop), replace=False)]
    xs = x.cpu().numpy().astype(np.float64)
    tol = 1e-9 if precision == "f64" else 1e-5
    worst = 0.0
    for p in picks:
        ref = orc.forward_genome(nodes[p], orc.transform_genome(nodes[p], conns[p], n_in, n_out), xs[p])
        if ref.size:
            worst = max(worst, float(np.max(np.abs(out[p] - ref) / np.maximum(1.0, np.abs(ref)))))
    worst_all = max(worst_all, worst / tol)
    report.append({"seed": seed, "inputs": n_in, "outputs": n_out, "max_nodes": max_nodes, "max_conns": max_conns,
                   "pop": pop, "batch": batch, "variant": variant, "prune": prune, "precision": precision,
                   "plan_class_counts": counts, "checked_genomes": len(picks), "max_rel_err": worst,
                   "tolerance": tol, "ok": worst <= tol})
    print(json.dumps(report[-1]), file=sys.stderr, flush=True)
print(json.dumps({"cases": report, "all_ok": all(r["ok"] for r in report),
                  "worst_err_over_tolerance": worst_all}, indent=1))
