"""Synthetic workloads of BASELINE.json -- input generation only.

``synthetic_population`` builds the config-2 population: io keys at rows
0..I+O-1, H~U{0..Hmax} hidden nodes with distinct random keys at random rows,
E~U{256..512} acyclic conns (src not an output, dst not an input, random
topological rank) at random conn rows, enabled~Bern(0.9), weight/bias~N(0,1)
clipped to +-30, response 1, act tanh / agg sum (variant "T") or uniform codes
0..3 (variant "M").  tests/test_synthetic.py checks it is identical to the
oracle's copy used by the parity tests.
"""

from __future__ import annotations

import numpy as np

KEY, BIAS, RESP, AGG, ACT = range(5)
CIN, COUT, CEN, CW = range(4)


def synthetic_population(pop: int, max_nodes: int, max_conns: int, num_inputs: int,
                         num_outputs: int, seed: int = 20261018, variant: str = "T",
                         min_conns: int = 256, max_conns_drawn: int = 512,
                         max_hidden: int | None = None) -> tuple[np.ndarray, np.ndarray]:
    """SURVEY.md §8d generator: io keys at rows 0..io-1, H~U{0..Hmax} hidden nodes
    with distinct random keys at random rows, E~U{min..max} acyclic conns
    (src not output, dst not input, random topological rank) at random rows,
    enabled~Bern(0.9), weight/bias~N(0,1), response 1; variant "T" = tanh/sum,
    "M" = act, agg ~ U{0..3}."""
    rng = np.random.default_rng(seed)
    io = num_inputs + num_outputs
    hmax = max_nodes - io if max_hidden is None else min(max_hidden, max_nodes - io)
    nodes = np.full((pop, max_nodes, 5), np.nan)
    conns = np.full((pop, max_conns, 4), np.nan)
    for p in range(pop):
        h = int(rng.integers(0, hmax + 1))
        hidden_keys = io + rng.choice(2 ** 20, size=h, replace=False)
        hidden_rows = io + rng.choice(max_nodes - io, size=h, replace=False)
        nkeys = np.concatenate([np.arange(io), hidden_keys]).astype(np.float64)
        nrows = np.concatenate([np.arange(io), hidden_rows])
        nn = nkeys.size
        nodes[p, nrows, KEY] = nkeys
        nodes[p, nrows, BIAS] = np.clip(rng.standard_normal(nn), -30, 30)
        nodes[p, nrows, RESP] = 1.0
        if variant == "M":
            nodes[p, nrows, AGG] = rng.integers(0, 4, nn)
            nodes[p, nrows, ACT] = rng.integers(0, 4, nn)
        else:
            nodes[p, nrows, AGG] = 0.0
            nodes[p, nrows, ACT] = 1.0
        # topological rank: inputs first, then a random permutation of the rest
        rank = np.empty(nn)
        rank[:num_inputs] = -1.0
        rank[num_inputs:] = rng.permutation(nn - num_inputs)
        is_out = (nkeys >= num_inputs) & (nkeys < io)
        is_in = nkeys < num_inputs
        src_ok = ~is_out
        dst_ok = ~is_in
        cand = np.argwhere(src_ok[:, None] & dst_ok[None, :] & (rank[:, None] < rank[None, :]))
        e = min(int(rng.integers(min_conns, max_conns_drawn + 1)), cand.shape[0], max_conns)
        pick = cand[rng.choice(cand.shape[0], size=e, replace=False)]
        crow = rng.choice(max_conns, size=e, replace=False)
        conns[p, crow, CIN] = nkeys[pick[:, 0]]
        conns[p, crow, COUT] = nkeys[pick[:, 1]]
        conns[p, crow, CEN] = (rng.random(e) < 0.9).astype(np.float64)
        conns[p, crow, CW] = np.clip(rng.standard_normal(e), -30, 30)
    return nodes, conns
