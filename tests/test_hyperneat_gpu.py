"""HyperNEAT: CPPN queries (forward kernel, shared inputs) + tcgen05 substrate
fitness vs the float64 CPU restatement (oracle; parity unpinned -- the
reference has no HyperNEAT).  Tolerances: CPPN weights within the fp32
forward bound 1e-4 * max(1,|w|) (mixed act/agg CPPNs); fitness within 2e-3
relative (TF32 operands + tanh.approx epilogue)."""

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


def test_query_layout_matches_oracle(tn):
    from oracle import arrayneat_oracle as orc
    from paper_2404_01817_b200 import hyperneat as hn
    assert np.allclose(hn.query_inputs(), orc.substrate_query_inputs())


@pytest.mark.parametrize("pop", [1, 7, 64])
def test_substrate_fitness_against_oracle(tn, pop):
    import torch
    from oracle import arrayneat_oracle as orc
    from paper_2404_01817_b200 import hyperneat as hn
    nodes, conns = orc.synthetic_population(pop, 32, 96, 4, 1, seed=11 + pop, variant="M",
                                            min_conns=8, max_conns_drawn=60)
    st, cyc = tn.transform_arrays(nodes, conns, 4, 1)
    assert cyc.size == 0
    w = hn.cppn_weights(st)
    x, t = hn.teacher_task(512)
    fit = hn.substrate_fitness(w, torch.from_numpy(x).cuda(), torch.from_numpy(t).cuda()).cpu().numpy()
    q = orc.substrate_query_inputs()
    for p in range(pop):
        tr = orc.transform_genome(nodes[p], conns[p], 4, 1)
        wref = orc.forward_genome(nodes[p], tr, q)[:, 0].reshape(64, 64)
        werr = np.max(np.abs(w[p].cpu().numpy() - wref) / np.maximum(1.0, np.abs(wref)))
        assert werr <= 1e-4, (p, werr)
        ref = orc.substrate_fitness(nodes[p], conns[p], x, t)
        assert abs(fit[p] - ref) <= 2e-3 * max(1.0, abs(ref)), (p, fit[p], ref)


def test_hyperneat_problem_runs(tn):
    from oracle import arrayneat_oracle as orc
    from paper_2404_01817_b200 import hyperneat as hn
    nodes, conns = orc.synthetic_population(9, 32, 96, 4, 1, seed=5, variant="M", min_conns=8,
                                            max_conns_drawn=60)
    prob = hn.HyperNEATProblem(samples=256)
    fit = prob.evaluate_population_tensors(tn.PopulationTensors(nodes, conns, None, None, 4, 1))
    assert fit.shape == (9,) and np.all(np.isfinite(fit)) and np.all(fit <= 0)
