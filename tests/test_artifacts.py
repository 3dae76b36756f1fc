"""Run artifacts: genome JSON text format,
integrity checks and checkpoints, checked byte-for-byte / field-for-field
against the unmodified reference (oracle/_ref, used here only as the checker).
CPU-only: no kernels are called."""

from __future__ import annotations

import os
import sys

import numpy as np
import pytest

from conftest import REPO, load_golden

REF = os.path.join(REPO, "oracle", "_ref")


@pytest.fixture(scope="module")
def ref():
    if not os.path.isdir(os.path.join(REF, "arrayneat")):
        pytest.skip("reference not installed (oracle/build_ref.sh)")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import arrayneat
    return arrayneat


@pytest.fixture(scope="module")
def corpus():
    return load_golden("corpus.npz")


def _genomes(corpus, n=12):
    from paper_2404_01817_b200.genome import GenomeTensors
    return [GenomeTensors(corpus["nodes"][i], corpus["conns"][i], 3, 2) for i in range(0, 200, 200 // n)]


def test_serialize_bytes_match_reference(ref, corpus):
    from paper_2404_01817_b200.artifacts import parse_genome, serialize_genome
    for g in _genomes(corpus):
        rg = ref.GenomeTensors(g.nodes.copy(), g.conns.copy(), 3, 2)
        data = serialize_genome(g)
        assert data == ref.serialize_genome(rg)
        back = parse_genome(data)
        assert np.array_equal(back.nodes, g.nodes, equal_nan=True)
        assert np.array_equal(back.conns, g.conns, equal_nan=True)
        assert serialize_genome(back) == data
        r2 = ref.parse_genome(data)  # the reference reads our files
        assert np.array_equal(r2.nodes, g.nodes, equal_nan=True)
    assert b"null" in data and b"NaN" not in data


def test_parse_errors(corpus):
    from paper_2404_01817_b200 import ParseError
    from paper_2404_01817_b200.artifacts import parse_genome, serialize_genome
    from paper_2404_01817_b200.genome import GenomeTensors
    g = _genomes(corpus, 1)[0]
    with pytest.raises(ParseError):
        parse_genome(b"{not json")
    with pytest.raises(ParseError):
        parse_genome(b'{"num_inputs": 1}')
    bad = g.conns.copy()
    live = np.nonzero(~np.isnan(bad[:, 0]))[0][0]
    bad[live, 1] = 9999.0  # dangling endpoint
    with pytest.raises(ParseError):
        parse_genome(serialize_genome(GenomeTensors(g.nodes.copy(), bad, 3, 2)))
    nodes = g.nodes.copy()
    empty = np.nonzero(np.isnan(nodes[:, 0]))[0][0]
    nodes[empty, 0] = 77.0  # key set, attributes NaN
    with pytest.raises(ParseError):
        parse_genome(serialize_genome(GenomeTensors(nodes, g.conns.copy(), 3, 2)))


@pytest.mark.parametrize("case", ["ok", "mixed", "negkey", "dupkey", "noio", "duppair", "dangling", "enabled"])
def test_integrity_agrees_with_reference(ref, corpus, case):
    from paper_2404_01817_b200 import IntegrityError
    from paper_2404_01817_b200.artifacts import check_integrity
    from paper_2404_01817_b200.genome import GenomeTensors
    g = _genomes(corpus, 1)[0]
    nodes, conns = g.nodes.copy(), g.conns.copy()
    live_n = np.nonzero(~np.isnan(nodes[:, 0]))[0]
    live_c = np.nonzero(~np.isnan(conns[:, 0]))[0]
    if case == "mixed":
        nodes[live_n[-1], 2] = np.nan
    elif case == "negkey":
        nodes[live_n[-1], 0] = -3.0
    elif case == "dupkey":
        nodes[live_n[-1], 0] = nodes[live_n[-2], 0]
    elif case == "noio":
        nodes[live_n[0]] = np.nan
    elif case == "duppair":
        conns[live_c[1], :2] = conns[live_c[0], :2]
    elif case == "dangling":
        conns[live_c[0], 0] = 123456.0
    elif case == "enabled":
        conns[live_c[0], 2] = 0.5
    ours = GenomeTensors(nodes, conns, 3, 2)
    theirs = ref.GenomeTensors(nodes.copy(), conns.copy(), 3, 2)
    from arrayneat.genome import check_integrity as ref_check
    ref_raised = ours_raised = False
    try:
        ref_check(theirs)
    except ref.IntegrityError:
        ref_raised = True
    try:
        check_integrity(ours)
    except IntegrityError:
        ours_raised = True
    assert ours_raised == ref_raised == (case != "ok")


def _host_state(corpus):
    from paper_2404_01817_b200 import NeatConfig
    from paper_2404_01817_b200.evolution import NodeKeyAllocator, SpeciesState
    from paper_2404_01817_b200.genome import GenomeTensors, PopulationTensors
    from paper_2404_01817_b200.runner import EvolutionState
    cfg = NeatConfig(inputs=3, outputs=2, max_nodes=32, max_conns=64, pop_size=200, seed=11)
    pop = PopulationTensors(corpus["nodes"].copy(), corpus["conns"].copy(), np.arange(200) % 3,
                            np.linspace(0, 1, 200), 3, 2)
    species = [SpeciesState(species_key=k, representative=GenomeTensors(corpus["nodes"][k], corpus["conns"][k], 3, 2),
                            member_indices=np.arange(k, 200, 3), best_fitness_history=[0.1 * k, 0.2],
                            stagnation_counter=k, spawn_count=60 + k) for k in range(3)]
    return EvolutionState(config=cfg, population=pop, species=species, allocator=NodeKeyAllocator(900),
                          generation=7, stats_rows=["0,1.0,0.5,3,5.0,6.0"])


def test_checkpoint_interchangeable_with_reference(ref, corpus, tmp_path):
    from arrayneat.runner import load_checkpoint as ref_load
    from arrayneat.runner import save_checkpoint as ref_save
    from paper_2404_01817_b200.artifacts import load_checkpoint, save_checkpoint
    state = _host_state(corpus)
    save_checkpoint(tmp_path / "ours.pkl", state)
    r = ref_load(tmp_path / "ours.pkl")
    assert r.generation == 7 and r.allocator.next_key == 900 and r.stats_rows == state.stats_rows
    assert np.array_equal(r.population.nodes, corpus["nodes"], equal_nan=True)
    assert np.array_equal(r.population.species_id, state.population.species_id)
    assert [s.species_key for s in r.species] == [0, 1, 2]
    assert [s.spawn_count for s in r.species] == [60, 61, 62]
    assert r.config == ref.parse_config_text(ref.dump_config(r.config))
    ref_save(tmp_path / "theirs.pkl", r)
    back = load_checkpoint(tmp_path / "theirs.pkl", on_device=False)
    assert back.generation == 7 and back.allocator.next_key == 900
    assert np.array_equal(back.population.conns, corpus["conns"], equal_nan=True)
    assert np.array_equal(back.species[2].member_indices, np.arange(2, 200, 3))
    assert back.species[1].best_fitness_history == [0.1, 0.2]
    assert back.config == state.config


def test_custom_registry_rejected_clearly(ref):
    """user callables cannot run in the kernels -> ConfigError;
    the reference's default registry is accepted."""
    import numpy as np
    from paper_2404_01817_b200 import ConfigError
    from paper_2404_01817_b200.functions import check_registry
    check_registry(ref.DEFAULT_REGISTRY)
    check_registry(ref.FunctionRegistry())
    custom = dict(ref.FunctionRegistry().activations)
    custom[1] = ("tanh", lambda x: np.tanh(2 * x))  # built-in name, custom function
    with pytest.raises(ConfigError):
        check_registry(ref.FunctionRegistry(activations=custom))
    extra = dict(ref.FunctionRegistry().activations)
    extra[7] = ("softsign", lambda x: x / (1 + abs(x)))
    with pytest.raises(ConfigError):
        check_registry(ref.FunctionRegistry(activations=extra))
