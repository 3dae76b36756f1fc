"""GPU fitness plugins and a short evolution run against reference goldens
(tests/golden/problems.npz).

Fitness is float64 on the device (f64 programs); the reference's tanh /
sigmoid come from numpy's SIMD libm, CUDA's from libdevice, so XOR /
regression fitness agree to 1e-9 (the reference's own oracle bound) and
cart-pole step counts agree exactly except for rare trajectories where a
1-ulp difference flips a bang-bang decision (bounded below).
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


@pytest.mark.parametrize("name,ni", [("xor", 2), ("regression", 1), ("cartpole", 4)])
def test_problem_fitness(tn, name, ni):
    g = load_golden("problems.npz")
    cfg = tn.NeatConfig(inputs=ni, outputs=1, max_nodes=24, max_conns=48, pop_size=120, problem=name)
    pop = tn.PopulationTensors(g[f"{name}_nodes"], g[f"{name}_conns"], None, None, ni, 1)
    fit = tn.make_problem(cfg).evaluate_population_tensors(pop, rng=tn.RngStream(9).child(4, 1))
    ref = g[f"{name}_fitness"]
    if name == "cartpole":
        _check_cartpole(g, fit, ref)
    else:
        np.testing.assert_allclose(fit, ref, rtol=1e-9, atol=1e-9)


def _check_cartpole(g, fit, ref):
    """Episodes are step-exact against the reference.  The only admissible
    difference is libm rounding of cos/sin (the kernel's double-double cos/sin
    vs numpy's, which can differ by 1 ulp near a rounding midpoint, and a
    chaotic episode can amplify that): each mismatching genome must be
    reproduced exactly by host replays of the same episode -- numpy's cos/sin
    giving the reference's step count and the kernel's cos/sin giving ours
    (oracle.cartpole_episode; start states = the reference's per-genome
    streams RngStream(9).child(4, 1).split(i).uniforms(4), problems.py:157)."""
    from oracle import arrayneat_oracle as orc
    nodes, conns = g["cartpole_nodes"], g["cartpole_conns"]
    bad = np.nonzero(fit != ref)[0]
    assert bad.size <= 3, bad
    for p in list(bad) + [0, 1, 2]:
        start = orc.Stream(orc.stream_key(9, 4, 1, int(p))).uniforms(4) * 0.1 - 0.05
        assert orc.cartpole_episode(nodes[p], conns[p], start) == ref[p], p
        assert orc.cartpole_episode(nodes[p], conns[p], start, orc.cos_sin_device) == fit[p], p


def test_xor_problem_fp32_path(tn):
    g = load_golden("problems.npz")
    prob = tn.XorProblem()
    prob.precision = "f32"
    pop = tn.PopulationTensors(g["xor_nodes"], g["xor_conns"], None, None, 2, 1)
    fit = prob.evaluate_population_tensors(pop)
    # fitness = 4 - sum_b (y_b - t_b)^2 over 4 cases: |d fit| <= 2 sum |y - t| |d y| <= 8e-5 for
    # outputs within north_star's 1e-5; measured well inside 1e-5 * max(1, |fit|)
    ref = g["xor_fitness"]
    assert np.max(np.abs(fit - ref) / np.maximum(1.0, np.abs(ref))) <= 1e-5


def test_short_xor_run_tracks_reference(tn):
    """Five generations from the same seed: per-generation statistics track
    the reference (exactly while every structural decision matches)."""
    from paper_2404_01817_b200.runner import init_state, stats_row  # noqa: F401
    g = load_golden("problems.npz")
    cfg = tn.NeatConfig(seed=3, pop_size=150, generation_limit=5)
    state = init_state(cfg)
    problem = tn.make_problem(cfg)
    root = tn.RngStream(cfg.seed)
    pop, species = state.population, state.species
    rows = []
    for gen in range(5):
        pop, species, stats = tn.evolve_step(pop, species, cfg, root.child(gen), state.allocator, problem)
        rows.append([stats.best_fitness, stats.mean_fitness, stats.species_count, stats.mean_live_nodes,
                     stats.mean_live_conns])
    rows = np.array(rows)
    ref = g["run_stats"]
    np.testing.assert_allclose(rows, ref, rtol=1e-9, atol=1e-9)
    nodes = pop.nodes.cpu().numpy() if hasattr(pop.nodes, "cpu") else pop.nodes
    assert np.array_equal(np.isnan(nodes), np.isnan(g["run_final_nodes"]))
    assert np.array_equal(pop.species_id, g["run_final_species"])


def test_sharded_generation_single_rank_equals_evolve_step(tn):
    """The sharded generation (distributed.py) on one rank reproduces
    evolve_step exactly (same kernels, same RNG tape)."""
    import numpy as np
    from paper_2404_01817_b200.distributed import Collective, DeviceOps, sharded_evolve_step
    from paper_2404_01817_b200.runner import init_state
    cfg = tn.NeatConfig(seed=5, pop_size=200, compatibility_threshold=2.0)
    a = init_state(cfg)
    b = init_state(cfg)
    problem = tn.make_problem(cfg)
    root = tn.RngStream(cfg.seed)
    comm, ops = Collective(), DeviceOps(cfg)
    pop, species = a.population, a.species
    nodes, conns, lo, sp_b = b.population.nodes, b.population.conns, 0, b.species
    for gen in range(3):
        pop, species, st_a = tn.evolve_step(pop, species, cfg, root.child(gen), a.allocator, problem)
        nodes, conns, lo, sp_b, st_b = sharded_evolve_step(nodes, conns, lo, sp_b, cfg, root.child(gen),
                                                           b.allocator, problem, comm, ops)
        assert st_a.best_fitness == st_b.best_fitness and st_a.mean_fitness == st_b.mean_fitness
    assert np.array_equal(pop.nodes.cpu().numpy(), nodes.cpu().numpy(), equal_nan=True)
    assert [s.species_key for s in species] == [s.species_key for s in sp_b]


def test_run_experiment_artifacts_and_resume(tn, tmp_path):
    """run_experiment writes the reference's artifacts (stats.csv schema,
    best_genome.json, checkpoint.pkl); resuming from a mid-run checkpoint
    reproduces the uninterrupted run exactly (runner.py:145-198)."""
    from paper_2404_01817_b200.artifacts import load_checkpoint, parse_genome, save_checkpoint
    from paper_2404_01817_b200.runner import EXIT_GENERATION_LIMIT, STATS_HEADER, run_experiment
    g = load_golden("problems.npz")
    cfg = tn.NeatConfig(seed=3, pop_size=150, generation_limit=5)
    full = run_experiment(cfg, tmp_path / "full")
    assert full.exit_code == EXIT_GENERATION_LIMIT and full.generations == 5
    lines = full.stats_path.read_text().splitlines()
    assert lines[0] == STATS_HEADER and len(lines) == 6
    rows = np.array([[float(v) for v in ln.split(",")[1:]] for ln in lines[1:]])
    np.testing.assert_allclose(rows[:, [0, 1, 2, 3, 4]], g["run_stats"], rtol=1e-9, atol=1e-9)
    best = parse_genome(full.genome_path.read_bytes())
    assert best.num_inputs == 2 and best.max_nodes == cfg.max_nodes
    half = run_experiment(cfg.with_overrides(generation_limit=3), tmp_path / "half")
    st = load_checkpoint(half.checkpoint_path)
    st.config = cfg
    save_checkpoint(tmp_path / "half" / "checkpoint.pkl", st)
    resumed = run_experiment(None, tmp_path / "resumed", resume_path=tmp_path / "half" / "checkpoint.pkl")
    assert resumed.stats_path.read_text() == full.stats_path.read_text()
    assert resumed.genome_path.read_bytes() == full.genome_path.read_bytes()


def test_run_bench_csv(tn, tmp_path):
    """bench.csv keeps the reference columns (filled by timing the reference
    module, the checker) and adds the GPU path's per-generation seconds."""
    import os
    import sys
    from conftest import REPO
    from paper_2404_01817_b200.runner import BENCH_HEADER, run_bench
    ref_dir = os.path.join(REPO, "oracle", "_ref")
    reference = None
    if os.path.isdir(os.path.join(ref_dir, "arrayneat")):
        sys.path.insert(0, ref_dir)
        import arrayneat as reference
    cfg = tn.NeatConfig(seed=1, pop_size=40)
    path = run_bench(cfg, [40, 60], 2, tmp_path, reference=reference)
    lines = path.read_text().splitlines()
    assert lines[0] == BENCH_HEADER and len(lines) == 5
    for ln in lines[1:]:
        cells = ln.split(",")
        assert float(cells[4]) > 0
        if reference is not None:
            assert float(cells[2]) > 0 and float(cells[3]) > 0


def test_fused_fitness_errors(tn):
    """The fused path checks the transform status after the kernel: cyclic
    genomes raise CycleDetected with their indices, unknown codes ConfigError,
    broken structure IntegrityError -- like the reference (problems.py:209-213)."""
    g = load_golden("forward_small.npz")
    nodes, conns = g["nodes"].copy(), g["conns"].copy()
    pop = tn.PopulationTensors(nodes, conns, None, None, 2, 1)
    with pytest.raises(tn.CycleDetected) as exc:
        tn.XorProblem().evaluate_population_tensors(pop)
    assert exc.value.genome_indices == [47]
    ok = np.setdiff1d(np.arange(nodes.shape[0]), [47])
    n2, c2 = nodes[ok].copy(), conns[ok].copy()
    live = np.nonzero(~np.isnan(n2[3, :, 0]))[0]
    n2[3, live[-1], 4] = 9.0  # unknown activation code
    with pytest.raises(tn.ConfigError):
        tn.XorProblem().evaluate_population_tensors(tn.PopulationTensors(n2, c2, None, None, 2, 1))
    c3 = conns[ok].copy()
    lc = np.nonzero(~np.isnan(c3[5, :, 0]))[0]
    c3[5, lc[0], 0] = 4242.0  # dangling endpoint
    with pytest.raises(tn.IntegrityError):
        tn.XorProblem().evaluate_population_tensors(tn.PopulationTensors(nodes[ok].copy(), c3, None, None, 2, 1))
