"""Randomised shapes through the whole forward path against the oracle:
capacities, input/output counts, batch sizes (warp and tile kernels), both
precisions, tanh/sum and mixed activation/aggregation genomes, and the
staged / subset launch plans.  Seeds are fixed, so failures reproduce."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import cuda_ok

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tn():
    if not cuda_ok():
        pytest.skip("no CUDA device")
    import paper_2404_01817_b200 as tn
    return tn


def _case(seed: int):
    rng = np.random.default_rng(1000 + seed)
    n_in = int(rng.integers(1, 40))
    n_out = int(rng.integers(1, 10))
    max_nodes = int(rng.integers(n_in + n_out + 1, 200))
    max_conns = int(rng.integers(8, 700))
    batch = int(rng.choice([1, 7, 64, 130, 257, 600]))
    pop = int(rng.integers(1, 12))
    variant = str(rng.choice(["T", "M"]))
    precision = str(rng.choice(["f32", "f64"]))
    return n_in, n_out, max_nodes, max_conns, batch, pop, variant, precision


@pytest.mark.parametrize("seed", range(48))
def test_random_shapes_match_oracle(tn, seed):
    import torch
    from oracle import arrayneat_oracle as orc
    n_in, n_out, max_nodes, max_conns, batch, pop, variant, precision = _case(seed)
    lo = min(max_conns, 4)
    nodes, conns = orc.synthetic_population(pop, max_nodes, max_conns, n_in, n_out, seed=seed, variant=variant,
                                            min_conns=lo, max_conns_drawn=max(lo, max_conns))
    st, cyc = tn.transform_arrays(nodes, conns, n_in, n_out, precision=precision)
    assert cyc.size == 0
    dt = np.float64 if precision == "f64" else np.float32
    x = np.random.default_rng(seed).standard_normal((pop, batch, n_in)).astype(dt)
    out = tn.forward_device(st, torch.from_numpy(x).cuda()).cpu().numpy()
    tol = 1e-9 if precision == "f64" else 1e-5
    for p in range(pop):
        ref = orc.forward_genome(nodes[p], orc.transform_genome(nodes[p], conns[p], n_in, n_out),
                                 x[p].astype(np.float64))
        err = np.max(np.abs(out[p] - ref) / np.maximum(1.0, np.abs(ref))) if ref.size else 0.0
        assert err <= tol, (seed, p, err)
    if pop > 2:  # a subset keeps the parent's host slot counts and gives the same rows
        sub = st.select(slice(1, pop))
        xs = torch.from_numpy(x[1:]).cuda()
        assert torch.equal(tn.forward_device(sub, xs), torch.from_numpy(out[1:]).cuda())
