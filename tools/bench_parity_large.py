"""The benchmarked launch against the oracle on a large sample (evidence, not a
test; tests/test_bench_parity_gpu.py checks 256 genomes): bench.py's
population (pop 10k, 128/512, I=32, O=8, seed 20261018, tanh/sum) through
transform_arrays + the device-planned forward over 4096 device-generated inputs
per genome (seed 20261019), then --n random genomes x all 4096 inputs compared
with the oracle at |d| <= 1e-5 * max(1, |ref|).
    python tools/bench_parity_large.py [--n 2048] > report.json"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2404_01817_b200 as tn  # noqa: E402
from oracle import arrayneat_oracle as orc  # noqa: E402
from paper_2404_01817_b200.synthetic import synthetic_population  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=2048)
a = ap.parse_args()
POP, MAXN, MAXC, NIN, NOUT, BATCH = 10_000, 128, 512, 32, 8, 4096
dev = torch.device("cuda", 0)
nodes_h, conns_h = synthetic_population(POP, MAXN, MAXC, NIN, NOUT, seed=20261018)
nodes, conns = torch.from_numpy(nodes_h).to(dev), torch.from_numpy(conns_h).to(dev)
x = torch.randn((POP, BATCH, NIN), device=dev, dtype=torch.float32,
                generator=torch.Generator(device=dev).manual_seed(20261019))
st, _ = tn.transform_arrays(nodes, conns, NIN, NOUT, sync=False)
out = tn.forward_device(st, x, torch.empty((POP, BATCH, NOUT), device=dev))
torch.cuda.synchronize()
counts = tn.inference.tc_plan_counts(st).tolist()
picks = np.sort(np.random.default_rng(11).choice(POP, size=a.n, replace=False))
errs = []
for p in picks:
    tr = orc.transform_genome(nodes_h[p], conns_h[p], NIN, NOUT)
    ref = orc.forward_genome(nodes_h[p], tr, x[p].cpu().numpy().astype(np.float64))
    errs.append(float(np.max(np.abs(out[p].cpu().numpy() - ref) / np.maximum(1.0, np.abs(ref)))))
errs = np.array(errs)
print(json.dumps({"population": POP, "inputs_per_genome": BATCH, "plan_class_counts": counts,
                  "genomes_checked": int(a.n), "outputs_checked": int(a.n * BATCH * NOUT),
                  "max_rel_err": float(errs.max()), "p99_rel_err": float(np.percentile(errs, 99)),
                  "median_rel_err": float(np.median(errs)), "tolerance": 1e-5, "all_ok": bool(errs.max() <= 1e-5)},
                 indent=1))
