"""GPU parity of the population operators against reference goldens
(tests/golden/evolution.npz, corpus.npz, rng.npz -- all produced by the
unmodified reference).

Bars (north_star: "bit-exact given the same RNG stream"):
  * uniforms, crossover, distances, speciation, spawn counts: bit-exact;
  * mutation / reproduction / init: structure bit-exact (padding pattern, keys,
    endpoints, enabled flags, function codes); float attributes derived from
    Box-Muller normals within 1e-12 (CUDA log/cos vs numpy SIMD log/cos can
    differ by ~1 ulp).
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import cuda_ok, load_golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tn():
    if not cuda_ok():
        pytest.skip("no CUDA device")
    import paper_2404_01817_b200 as tn
    return tn


def _cfg(tn, **kw):
    base = dict(inputs=3, outputs=2, max_nodes=32, max_conns=64, pop_size=200,
                node_add=0.5, node_delete=0.2, conn_add=0.6, conn_delete=0.2,
                bias_mutate_rate=0.8, bias_replace_rate=0.1,
                response_init_std=0.3, response_mutate_rate=0.3, response_mutate_power=0.3,
                response_replace_rate=0.05,
                weight_mutate_rate=0.8, weight_replace_rate=0.1, enabled_mutate_rate=0.05,
                activation_options=("identity", "tanh", "sigmoid", "relu"), activation_replace_rate=0.3,
                aggregation_options=("sum", "product", "max", "mean"), aggregation_replace_rate=0.3)
    base.update(kw)
    return tn.NeatConfig(**base)


def assert_genomes_match(nodes, conns, ref_nodes, ref_conns, atol=1e-12):
    assert np.array_equal(np.isnan(nodes), np.isnan(ref_nodes))
    assert np.array_equal(np.isnan(conns), np.isnan(ref_conns))
    exact_n = np.s_[..., [0, 3, 4]]
    exact_c = np.s_[..., [0, 1, 2]]
    assert np.array_equal(nodes[exact_n], ref_nodes[exact_n], equal_nan=True)
    assert np.array_equal(conns[exact_c], ref_conns[exact_c], equal_nan=True)
    np.testing.assert_allclose(nodes[..., 1:3], ref_nodes[..., 1:3], rtol=0, atol=atol)
    np.testing.assert_allclose(conns[..., 3], ref_conns[..., 3], rtol=0, atol=atol)


def test_rng_device_cells_match_reference(tn):
    import torch
    from paper_2404_01817_b200 import _native
    from paper_2404_01817_b200.rng import RngStream
    g = load_golden("rng.npz")
    for idx, row in enumerate(g["paths"]):
        seed, plen = int(row[0]), int(row[1])
        s = RngStream(seed, tuple(int(t) for t in row[2:2 + plen]))
        keys = torch.from_numpy(s._keys.view(np.int64).copy()).cuda()
        u = torch.empty(37, dtype=torch.float64, device="cuda")
        _native.call("an_rng_draw", keys.data_ptr(), 1, 0, 37, 0, u.data_ptr(), 0)
        assert np.array_equal(u.cpu().numpy(), g[f"u_{idx}"])
        z = torch.empty(19, dtype=torch.float64, device="cuda")
        _native.call("an_rng_draw", keys.data_ptr(), 1, 37, 19, 1, z.data_ptr(), 0)
        np.testing.assert_allclose(z.cpu().numpy(), g[f"n_{idx}"], rtol=0, atol=1e-14)
        # host RngStream (used for keys/counters) reproduces the reference too
        s2 = RngStream(seed, tuple(int(t) for t in row[2:2 + plen]))
        assert np.array_equal(s2.uniforms(37), g[f"u_{idx}"])


def test_init_arrays(tn):
    from paper_2404_01817_b200.genome import init_arrays
    from paper_2404_01817_b200.rng import RngStream
    g = load_golden("evolution.npz")
    n, c = init_arrays(_cfg(tn), RngStream(5).child(0, 0).split(np.arange(40)))
    assert_genomes_match(n, c, g["init_nodes"], g["init_conns"])


@pytest.mark.parametrize("net", ["feedforward", "recurrent"])
def test_mutate_arrays(tn, net):
    from paper_2404_01817_b200.rng import RngStream
    g = load_golden("evolution.npz")
    c = load_golden("corpus.npz")
    p = c["nodes"].shape[0]
    st = RngStream(77).child(3, 2).split(np.arange(p))
    st._counter = 5
    mn, mc, added = tn.evolution.mutate_arrays(c["nodes"], c["conns"], _cfg(tn, network_type=net), st,
                                               np.arange(1000, 1000 + p, dtype=np.float64))
    assert st._counter == int(g[f"mut_{net}_counter"])
    assert np.array_equal(added, g[f"mut_{net}_added"])
    assert_genomes_match(mn, mc, g[f"mut_{net}_nodes"], g[f"mut_{net}_conns"])


def test_crossover_bit_exact(tn):
    from paper_2404_01817_b200.rng import RngStream
    g = load_golden("evolution.npz")
    c = load_golden("corpus.npz")
    p = c["nodes"].shape[0]
    st = RngStream(91).child(1, 2).split(np.arange(p))
    st._counter = 2
    xn, xc = c["nodes"].copy(), c["conns"].copy()
    tn.evolution._crossover_into(xn, xc, c["nodes"][::-1].copy(), c["conns"][::-1].copy(), st)
    assert st._counter == int(g["xo_counter"])
    assert np.array_equal(xn, g["xo_nodes"], equal_nan=True)
    assert np.array_equal(xc, g["xo_conns"], equal_nan=True)


def test_distance_bit_exact(tn):
    c = load_golden("corpus.npz")
    cfg = _cfg(tn)
    n, cc = c["nodes"], c["conns"]
    assert np.array_equal(tn.evolution.distance_arrays(n, cc, n[:1], cc[:1], cfg), c["dist_to_0"])
    assert np.array_equal(tn.evolution.distance_arrays(n, cc, n[7:8], cc[7:8], cfg), c["dist_to_7"])
    assert np.array_equal(tn.evolution.distance_arrays(n[:100], cc[:100], n[100:], cc[100:], cfg),
                          c["dist_pair"])


def test_distance_representatives_kernel_equals_pairwise(tn):
    """The representative-staged kernel (P genomes x R reps, and P x 1) is
    bitwise the pair kernel, also for rows that are not aligned with the
    representative's, -0 keys, repeated keys in a representative (first row
    wins) and infinite attributes."""
    import torch
    c = load_golden("corpus.npz")
    cfg = _cfg(tn)
    n, cc = c["nodes"].copy(), c["conns"].copy()
    rng = np.random.default_rng(5)
    for i in range(0, n.shape[0], 3):  # misaligned rows
        n[i] = n[i][rng.permutation(n.shape[1])]
        cc[i] = cc[i][rng.permutation(cc.shape[1])]
    live = np.nonzero(~np.isnan(n[4, :, 0]))[0]
    n[4, live[0], 0] = -0.0 if n[4, live[0], 0] == 0.0 else n[4, live[0], 0]
    n[5, live[-1], 0] = n[5, live[-2], 0] if len(live) > 1 else n[5, live[-1], 0]  # repeated key (rep 5)
    lc = np.nonzero(~np.isnan(cc[6, :, 0]))[0]
    cc[6, lc[0], 3] = np.inf
    ev = tn.evolution
    tile = -(-65536 // n.shape[0])  # the representatives kernel runs from 64K pairs on
    nd, cd = ev._dev64(np.tile(n, (tile, 1, 1))), ev._dev64(np.tile(cc, (tile, 1, 1)))
    reps = [0, 4, 5, 6, 9, 17, 33]
    rn, rc = nd[reps].contiguous(), cd[reps].contiguous()
    mat = ev._distance_dev(nd, cd, rn, rc, cfg, 0)
    p = nd.shape[0]
    for k, r in enumerate(reps):
        pair = ev._distance_dev(nd, cd, rn[k:k + 1].expand(p, -1, -1).contiguous(),
                                rc[k:k + 1].expand(p, -1, -1).contiguous(), cfg, 1)  # pair kernel (Q == P)
        one = ev._distance_dev(nd, cd, rn[k:k + 1], rc[k:k + 1], cfg, 1)           # reps kernel (Q == 1)
        got, ref = mat[k].cpu().numpy(), pair.cpu().numpy()
        assert np.array_equal(got, ref, equal_nan=True), r
        assert np.array_equal(one.cpu().numpy(), ref, equal_nan=True), r
    assert torch.isfinite(mat).any()


@pytest.mark.parametrize("small", [8192, 0], ids=["host-bookkeeping", "device-bookkeeping"])
def test_speciate_matches_reference(tn, monkeypatch, small):
    """Both speciation paths (host bookkeeping for small populations, device
    bookkeeping for large ones) reproduce the reference exactly."""
    monkeypatch.setattr(tn.evolution, "SMALL_SPECIATE", small)
    g = load_golden("evolution.npz")
    c = load_golden("corpus.npz")
    n, cc = c["nodes"], c["conns"]
    p = n.shape[0]
    cfg = _cfg(tn, compatibility_threshold=1.2, max_species=6)
    pop = tn.PopulationTensors(n, cc, np.full(p, -1), np.full(p, np.nan), 3, 2)
    sp_pop, sp = tn.evolution.speciate(pop, [], cfg)
    assert np.array_equal(sp_pop.species_id, g["spec0_assigned"])
    assert [s.species_key for s in sp] == list(g["spec0_keys"])
    assert np.array_equal(np.stack([s.representative.nodes for s in sp]), g["spec0_reps"], equal_nan=True)
    old = [tn.evolution.SpeciesState(species_key=k, representative=pop.genome(i), member_indices=np.arange(1))
           for k, i in ((3, 17), (8, 101))]
    sp_pop, sp = tn.evolution.speciate(pop, old, cfg)
    assert np.array_equal(sp_pop.species_id, g["spec1_assigned"])
    assert [s.species_key for s in sp] == list(g["spec1_keys"])
    assert np.array_equal(np.stack([s.representative.nodes for s in sp]), g["spec1_reps_nodes"], equal_nan=True)


def test_reproduce_matches_reference(tn):
    from paper_2404_01817_b200.rng import RngStream
    g = load_golden("evolution.npz")
    c = load_golden("corpus.npz")
    n, cc = c["nodes"], c["conns"]
    p = n.shape[0]
    cfg = _cfg(tn, compatibility_threshold=1.2, max_species=6)
    fitness = g["rep_fitness"]
    pop = tn.PopulationTensors(n, cc, np.full(p, -1), np.full(p, np.nan), 3, 2)
    sp_pop, sp = tn.evolution.speciate(pop, [], cfg)
    surv = tn.evolution.update_stagnation(sp, fitness, cfg)
    alloc = tn.evolution.allocate_spawns(surv, fitness, cfg.with_overrides(pop_size=p))
    assert [s.spawn_count for s in alloc] == list(g["spawns"])
    allocator = tn.evolution.NodeKeyAllocator(500)
    off = tn.evolution.reproduce(sp_pop, alloc, fitness, cfg.with_overrides(pop_size=p), RngStream(13).child(4),
                                 allocator)
    assert allocator.next_key == int(g["rep_next_key"])
    assert_genomes_match(off.nodes, off.conns, g["rep_nodes"], g["rep_conns"])


def test_slot_tables_device_ranking_equals_host(tn, monkeypatch):
    """Large-population slot tables rank parents with device sorts; they equal
    the host ranking (fitness descending, index ascending, NaN last, -0 == +0),
    including genomes of species dropped by stagnation."""
    from paper_2404_01817_b200.evolution import SpeciesState, slot_tables
    rng = np.random.default_rng(9)
    p = 5000
    fit = rng.choice([0.0, -0.0, 1.5, 2.0, np.nan, -np.inf, 3.25], size=p)  # many ties
    fit = np.where(rng.random(p) < 0.4, rng.normal(size=p).round(1), fit)
    sp_of = rng.integers(0, 5, p)
    g = tn.GenomeTensors(np.zeros((4, 5)), np.zeros((2, 4)), 2, 1)
    species = [SpeciesState(species_key=k, representative=g, member_indices=np.nonzero(sp_of == k)[0],
                            spawn_count=0) for k in (0, 1, 2, 4)]  # species 3 was dropped
    cfg = tn.NeatConfig(pop_size=p, survival_threshold=0.3, genome_elitism=2)
    counts = np.array([s.member_indices.size for s in species], dtype=float)
    spawn = np.floor(p * counts / counts.sum()).astype(int)
    spawn[0] += p - spawn.sum()
    for s, n in zip(species, spawn):
        s.spawn_count = int(n)
    monkeypatch.setattr(tn.evolution, "SMALL_SLOT_TABLES", 10 ** 9)
    host = slot_tables(species, fit, cfg)
    monkeypatch.setattr(tn.evolution, "SMALL_SLOT_TABLES", 0)
    dev = slot_tables(species, fit, cfg)
    for a, b in zip(host, dev):
        assert np.array_equal(a, b)
    # the tables built entirely on the device (reproduce's large-population path)
    built = tn.evolution._slot_tables_device(species, fit, cfg)
    for a, b in zip(host, built):
        assert np.array_equal(a, b.cpu().numpy())


# -- max_nodes 128 / max_conns 512 with > 64 live nodes: the reference's conn-add
# closure is float32 matmul squaring there (evolution.py:370-390), the kernel's is
# the bitset Warshall for every size (tests/golden/make_goldens.py BIG_CFG)

def _big_cfg(tn, **kw):
    return _cfg(tn, inputs=32, outputs=8, max_nodes=128, max_conns=512, pop_size=48, conn_add=0.9,
                compatibility_threshold=2.0, max_species=5, **kw)


@pytest.mark.parametrize("net", ["feedforward", "recurrent"])
def test_mutate_arrays_128_512_over_64_live_nodes(tn, net):
    from paper_2404_01817_b200.rng import RngStream
    g = load_golden("evolution_big.npz")
    p = g["nodes"].shape[0]
    assert (~np.isnan(g["nodes"][:, :, 0])).sum(axis=1).min() > 64
    st = RngStream(78).child(3, 2).split(np.arange(p))
    st._counter = 3
    mn, mc, added = tn.evolution.mutate_arrays(g["nodes"], g["conns"], _big_cfg(tn, network_type=net), st,
                                               np.arange(1 << 21, (1 << 21) + p, dtype=np.float64))
    assert st._counter == int(g[f"mut_{net}_counter"])
    assert np.array_equal(added, g[f"mut_{net}_added"])
    assert_genomes_match(mn, mc, g[f"mut_{net}_nodes"], g[f"mut_{net}_conns"])


def test_reproduce_128_512_over_64_live_nodes(tn):
    from paper_2404_01817_b200.rng import RngStream
    g = load_golden("evolution_big.npz")
    n, cc = g["nodes"], g["conns"]
    p = n.shape[0]
    cfg = _big_cfg(tn)
    fitness = g["rep_fitness"]
    pop = tn.PopulationTensors(n, cc, np.full(p, -1), np.full(p, np.nan), 32, 8)
    sp_pop, sp = tn.evolution.speciate(pop, [], cfg)
    assert np.array_equal(sp_pop.species_id, g["spec_assigned"])
    surv = tn.evolution.update_stagnation(sp, fitness, cfg)
    alloc = tn.evolution.allocate_spawns(surv, fitness, cfg)
    assert [s.spawn_count for s in alloc] == list(g["spawns"])
    allocator = tn.evolution.NodeKeyAllocator(1 << 22)
    off = tn.evolution.reproduce(sp_pop, alloc, fitness, cfg, RngStream(14).child(4), allocator)
    assert allocator.next_key == int(g["rep_next_key"])
    assert_genomes_match(off.nodes, off.conns, g["rep_nodes"], g["rep_conns"])
