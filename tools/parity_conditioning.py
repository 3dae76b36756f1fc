"""Conditioning of one forward output (evidence for the parity report): the
f64 oracle of bench genome G at sample S / output O against the same network
evaluated with every node value rounded to fp32, with fp32 weights, and with
a random +-2^-24 relative perturbation per node (the noise floor any fp32
evaluation carries).  Defaults: the one output of the benchmarked population
over 1e-5 (profiles/r02_bench_parity_large.json).
    python tools/parity_conditioning.py [G S O]"""
import sys, os, json
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from oracle import arrayneat_oracle as orc
from paper_2404_01817_b200.synthetic import synthetic_population
POP, MAXN, MAXC, NIN, NOUT, BATCH = 10_000, 128, 512, 32, 8, 4096
nodes_h, conns_h = synthetic_population(POP, MAXN, MAXC, NIN, NOUT, seed=20261018)
x = torch.randn((POP, BATCH, NIN), device="cuda", dtype=torch.float32, generator=torch.Generator(device="cuda").manual_seed(20261019))
p, smp, o = (int(v) for v in sys.argv[1:4]) if len(sys.argv) > 3 else (6165, 2012, 5)
xs = x[p].cpu().numpy().astype(np.float64)
nodes, tr = nodes_h[p], orc.transform_genome(nodes_h[p], conns_h[p], NIN, NOUT)
def fwd(round_nodes, round_weights, seed=None):
    rng = np.random.default_rng(seed) if seed is not None else None
    value = {}
    for i, r in enumerate(tr["input_rows"]): value[r] = xs[:, i]
    into = {}
    for s, d, w, _ in tr["edges"]:
        w = float(np.float32(w)) if round_weights else w
        into.setdefault(d, []).append((s, w))
    for r in tr["order"]:
        if r in set(tr["input_rows"]): continue
        terms = [w * value[s] for s, w in sorted(into.get(r, []))]
        agg = orc.agg_apply(int(nodes[r, orc.AGG]), terms, BATCH)
        b, rs = nodes[r, orc.BIAS], nodes[r, orc.RESP]
        if round_weights: b, rs = float(np.float32(b)), float(np.float32(rs))
        v = orc.act_apply(int(nodes[r, orc.ACT]), b + rs * agg)
        if round_nodes: v = v.astype(np.float32).astype(np.float64)
        if rng is not None: v = v * (1 + rng.uniform(-2**-24, 2**-24, v.shape))
        value[r] = v
    return np.stack([value[r] for r in tr["output_rows"]], axis=-1)
ref = fwd(False, False)
def err(y): return float(np.abs(y[smp, o] - ref[smp, o]) / max(1.0, abs(ref[smp, o])))
res = {"ref": float(ref[smp, o]), "exact_then_round_each_node": err(fwd(True, False)),
       "fp32_weights_exact_math": err(fwd(False, True)), "fp32_weights_round_nodes": err(fwd(True, True)),
       "random_half_ulp_per_node_max_over_20": max(err(fwd(False, False, seed=s)) for s in range(20)),
       "steps": len([r for r in tr["order"] if r not in set(tr["input_rows"])])}
print(json.dumps(res, indent=1))
