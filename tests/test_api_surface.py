"""Drop-in surface: every in-scope name the reference package exports
(arrayneat/__init__.py:8-30) resolves on ``paper_2404_01817_b200``, and the
host-side single-genome helpers agree with the unmodified reference
(oracle/_ref, the checker).  CPU-only: no kernels are called."""

from __future__ import annotations

import math
import os
import sys

import numpy as np
import pytest

from conftest import REPO

REF = os.path.join(REPO, "oracle", "_ref")

# arrayneat/__init__.py:9-30.  Out of scope: the graph
# oracle (graphref), single-genome edit primitives and DOT export.
REFERENCE_EXPORTS = """
NeatConfig dump_config load_config parse_config_text
ArrayNeatError BadAttrIndex CapacityFull ConfigError CycleDetected DanglingEndpoint DuplicateConn
DuplicateKey ExtinctionError IntegrityError InvalidInput KeyNotFound ParseError ProtectedNode
ShapeMismatch TerminalState
GenerationStats NodeKeyAllocator SpeciesState allocate_spawns crossover distance evolve_step mutate
reproduce speciate update_stagnation
ACTIVATION_IDS AGGREGATION_IDS DEFAULT_REGISTRY FunctionRegistry
ConnRow GenomeTensors NodeRow PopulationTensors check_integrity count_live genomes_equal init_genome
parse_genome serialize_genome
StackedNetworks TransformedNetwork forward forward_batch population_forward population_transform transform
CartPoleProblem CartPoleState Problem RegressionProblem XorProblem cartpole_step eval_cartpole
eval_regression eval_xor evaluate_population make_problem
RngStream
EvolutionState RunOutcome init_state load_checkpoint run_bench run_experiment save_checkpoint
""".split()
OUT_OF_SCOPE = {"GraphNetwork", "decode", "graph_distance", "graph_forward", "graphref", "add_conn",
                "add_node", "remove_conn", "remove_node", "set_conn_attr", "set_node_attr", "to_dot",
                "parallel", "search"}


@pytest.fixture(scope="module")
def ref():
    if not os.path.isdir(os.path.join(REF, "arrayneat")):
        pytest.skip("reference not installed (oracle/build_ref.sh)")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import arrayneat
    return arrayneat


def test_reference_exports_resolve_on_package_root():
    import paper_2404_01817_b200 as pkg
    missing = [n for n in REFERENCE_EXPORTS if not hasattr(pkg, n)]
    assert not missing, f"missing at the package root: {missing}"


def test_export_list_covers_reference(ref):
    public = {n for n in dir(ref) if not n.startswith("_") and n not in ("annotations",)}
    modules = {n for n in public if type(getattr(ref, n)).__name__ == "module"}
    assert public - modules - OUT_OF_SCOPE <= set(REFERENCE_EXPORTS)


def test_eval_helpers_match_reference(ref):
    import paper_2404_01817_b200 as pkg
    w = np.array([0.7, -1.3])
    fwd = lambda x: np.tanh(x @ w + 0.25)[:, None]  # noqa: E731
    assert pkg.eval_xor(fwd) == ref.eval_xor(fwd)
    f1 = lambda x: np.sin(1.1 * x)  # noqa: E731
    assert pkg.eval_regression(f1) == ref.eval_regression(f1)
    xs = np.linspace(-2, 2, 17)
    assert pkg.eval_regression(f1, np.cos, xs) == ref.eval_regression(f1, np.cos, xs)
    with pytest.raises(pkg.ShapeMismatch):
        pkg.eval_xor(lambda x: np.zeros((3, 1)))


def test_cartpole_host_matches_reference(ref):
    import paper_2404_01817_b200 as pkg
    s, r = pkg.CartPoleState(0.01, -0.02, 0.03, 0.04), ref.CartPoleState(0.01, -0.02, 0.03, 0.04)
    for k in range(60):
        a = 1 if (k * 7) % 3 else -1
        s, r = pkg.cartpole_step(s, a), ref.cartpole_step(r, a)
        assert (s.x, s.x_dot, s.theta, s.theta_dot, s.steps) == pytest.approx(
            (r.x, r.x_dot, r.theta, r.theta_dot, r.steps), rel=0, abs=1e-15)
        if r.is_terminal:
            break
    assert s.is_terminal == r.is_terminal
    # the hand fixture of the reference tests (test_problems.py:89-97): one step from rest
    one = pkg.cartpole_step(pkg.CartPoleState(0.0, 0.0, 0.0, 0.0), 1)
    assert one.x_dot == pytest.approx(0.02 * (10 / 1.1 - 0.05 * (-(10 / 1.1) / (0.5 * (4 / 3 - 0.1 / 1.1))) / 1.1))
    fwd = lambda obs: np.array([obs[2] + 0.3 * obs[3]])  # noqa: E731
    for seed in range(4):
        assert pkg.eval_cartpole(fwd, pkg.RngStream(seed)) == ref.eval_cartpole(fwd, ref.RngStream(seed))
    with pytest.raises(ValueError):
        pkg.cartpole_step(pkg.CartPoleState(0, 0, 0, 0), 0)
    with pytest.raises(pkg.TerminalState):
        pkg.cartpole_step(pkg.CartPoleState(3.0, 0, 0, 0), 1)
    assert math.isclose(pkg.problems._THETA_LIMIT, 12 * 2 * math.pi / 360)


def test_genome_records_and_counts(ref):
    import paper_2404_01817_b200 as pkg
    from conftest import load_golden
    c = load_golden("corpus.npz")
    for i in (0, 7, 31):
        a = pkg.GenomeTensors(c["nodes"][i], c["conns"][i], 3, 2)
        b = ref.GenomeTensors(c["nodes"][i], c["conns"][i], 3, 2)
        assert pkg.count_live(a) == ref.count_live(b)
        assert pkg.genomes_equal(a, pkg.GenomeTensors(c["nodes"][i].copy(), c["conns"][i].copy(), 3, 2))
        assert not pkg.genomes_equal(a, pkg.GenomeTensors(c["nodes"][i + 1], c["conns"][i + 1], 3, 2))
    n = pkg.NodeRow(5, 0.5, 1.0, 0, 1)
    assert np.array_equal(n.as_array(), ref.NodeRow(5, 0.5, 1.0, 0, 1).as_array())
    cr = pkg.ConnRow(0, 5, 1.0, -0.25)
    assert np.array_equal(cr.as_array(), ref.ConnRow(0, 5, 1.0, -0.25).as_array())
