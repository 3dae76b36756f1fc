"""Recurrent rollouts vs the float64 CPU restatement (oracle; parity
unpinned -- the reference rejects recurrent genomes).  f64 programs within
1e-9; f32 programs within 1e-3 * max(1, |ref|) over a short horizon."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import cuda_ok

pytestmark = pytest.mark.gpu


def cyclic_population(pop, seed):
    """Synthetic genomes plus random back edges (cycles), I=27, O=8."""
    from oracle import arrayneat_oracle as orc
    nodes, conns = orc.synthetic_population(pop, 64, 256, 27, 8, seed=seed, variant="M", min_conns=60,
                                            max_conns_drawn=200)
    rng = np.random.default_rng(seed)
    for p in range(pop):
        keys = nodes[p, ~np.isnan(nodes[p, :, 0]), 0]
        free = np.nonzero(np.isnan(conns[p, :, 0]))[0]
        hid = keys[keys >= 35]
        have = {(int(a), int(b)) for a, b in conns[p][~np.isnan(conns[p, :, 0])][:, :2]}
        for r in free[:12]:
            if hid.size < 2:
                break
            u, v = rng.choice(hid, 2, replace=False)
            if (int(u), int(v)) in have:
                continue
            have.add((int(u), int(v)))
            conns[p, r] = [u, v, 1.0, rng.standard_normal()]
    return nodes, conns


@pytest.fixture(scope="module")
def tn():
    if not cuda_ok():
        pytest.skip("no CUDA device")
    import paper_2404_01817_b200 as tn
    return tn


@pytest.mark.parametrize("precision,tol", [("f64", 1e-9), ("f32", 1e-3)])
def test_rollout_matches_oracle(tn, precision, tol):
    from oracle import arrayneat_oracle as orc
    from paper_2404_01817_b200 import recurrent as rec
    nodes, conns = cyclic_population(6, 3)
    st, _ = tn.transform_arrays(nodes, conns, 27, 8, precision=precision, network_type="recurrent")
    env = rec.ant_env()
    fit = rec.rollout_fitness(st, env, steps=12, sweeps=3)
    for p in range(6):
        ref = orc.recurrent_rollout(nodes[p], conns[p], 27, 8, *env, steps=12, sweeps=3)
        assert abs(fit[p] - ref) <= tol * max(1.0, abs(ref)), (p, fit[p], ref)


def test_rollout_long_episode_runs(tn):
    from paper_2404_01817_b200 import recurrent as rec
    nodes, conns = cyclic_population(16, 4)
    st, _ = tn.transform_arrays(nodes, conns, 27, 8, network_type="recurrent")
    fit = rec.rollout_fitness(st, steps=1000, sweeps=5)
    assert fit.shape == (16,) and np.all(np.isfinite(fit)) and np.all(np.abs(fit) <= 1000)
