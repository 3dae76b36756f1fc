"""Generation loop with a device-resident population (reference runner.py).

``init_state`` (runner.py:54-66) builds the initial population on the GPU
(an_init) and speciates it; ``run_experiment`` (runner.py:145-198) drives
``evolve_step`` and writes the reference's artifacts -- ``stats.csv`` /
``timings.csv`` (same schema), ``best_genome.json`` (genome text format) and
``checkpoint.pkl`` (pickle payload interchangeable with the reference's).
``run_bench`` (runner.py:225-250) writes ``bench.csv`` with the reference
columns plus the GPU path's per-generation time.  Populations stay CUDA
tensors between generations; only fitness, species bookkeeping and the
per-generation statistics cross to the host.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from .artifacts import load_checkpoint, save_checkpoint, serialize_genome
from .config import NeatConfig
from .errors import ConfigError
from .evolution import STAGE_INIT, NodeKeyAllocator, evolve_step, speciate
from .genome import PopulationTensors, init_arrays
from .problems import make_problem
from .rng import RngStream

STATS_HEADER = "generation,best_fitness,mean_fitness,species_count,mean_live_nodes,mean_live_conns"
TIMINGS_HEADER = "generation,elapsed_seconds"
BENCH_HEADER = "pop_size,generation,tensorized_seconds,sequential_seconds,gpu_seconds"
EXIT_SOLVED, EXIT_ERROR, EXIT_GENERATION_LIMIT = 0, 1, 2  # runner.py:38-40


@dataclass
class EvolutionState:
    config: NeatConfig
    population: PopulationTensors
    species: list
    allocator: NodeKeyAllocator
    generation: int = 0
    stats_rows: list = field(default_factory=list)


@dataclass
class RunOutcome:
    """runner.py:131-139, plus the final state and per-generation timings."""
    exit_code: int
    generations: int
    best_fitness: float
    solved: bool
    stats_path: Path | None
    genome_path: Path | None
    checkpoint_path: Path | None
    state: EvolutionState | None = None
    timings: list = field(default_factory=list)


def init_state(config: NeatConfig, on_device: bool = True) -> EvolutionState:
    """Fresh, speciated population (runner.py:54-66): stream (0, STAGE_INIT, i)."""
    streams = RngStream(config.seed).child(0, STAGE_INIT).split(np.arange(config.pop_size))
    nodes, conns = init_arrays(config, streams, on_device=on_device)
    pop = PopulationTensors(nodes, conns, np.full(config.pop_size, -1, dtype=np.int64),
                            np.full(config.pop_size, np.nan), config.inputs, config.outputs)
    pop, species = speciate(pop, [], config)
    return EvolutionState(config=config, population=pop, species=species,
                          allocator=NodeKeyAllocator(next_key=config.inputs + config.outputs))


def stats_row(generation: int, stats) -> str:
    return (f"{generation},{stats.best_fitness!r},{stats.mean_fitness!r},{stats.species_count},"
            f"{stats.mean_live_nodes!r},{stats.mean_live_conns!r}")


def run_experiment(config: NeatConfig | None, out_dir=None, threads: int = 1, resume_path=None,
                   log=None, state: EvolutionState | None = None) -> RunOutcome:
    """Evolve until the fitness target or ``generation_limit`` (runner.py:145-198).

    Resumes from ``resume_path`` (a checkpoint of this package or of the
    reference) or continues ``state``; writes the artifacts when ``out_dir``
    is given.  ``threads`` is accepted for signature parity (the device path
    has no host thread pool)."""
    if resume_path is not None:
        state = load_checkpoint(resume_path)
        config = state.config
    elif state is not None:
        config = config or state.config
    elif config is not None:
        state = init_state(config)
    else:
        raise ConfigError("run needs a config or a checkpoint to resume")
    problem = make_problem(config)
    root = RngStream(config.seed)
    timings: list[float] = []
    timing_rows: list[str] = []
    best_genome = None
    best_fitness = -math.inf
    solved = False
    while state.generation < config.generation_limit:
        generation = state.generation
        t = time.perf_counter()
        pop, species, stats = evolve_step(state.population, state.species, config, root.child(generation),
                                          state.allocator, problem, threads=threads)
        timings.append(time.perf_counter() - t)
        state.stats_rows.append(stats_row(generation, stats))
        timing_rows.append(f"{generation},{stats.elapsed_seconds!r}")
        best_genome, best_fitness = stats.best_genome, stats.best_fitness
        state.population, state.species = pop, species
        state.generation = generation + 1
        if log:
            log(f"generation {generation}: best={stats.best_fitness:.4f} "
                f"mean={stats.mean_fitness:.4f} species={stats.species_count}")
        if stats.solved:
            solved = True
            break
    stats_path = genome_path = checkpoint_path = None
    if out_dir is not None:
        out = Path(out_dir)
        out.mkdir(parents=True, exist_ok=True)
        stats_path = out / "stats.csv"
        stats_path.write_text("\n".join([STATS_HEADER, *state.stats_rows]) + "\n", encoding="utf-8")
        (out / "timings.csv").write_text("\n".join([TIMINGS_HEADER, *timing_rows]) + "\n", encoding="utf-8")
        genome_path = out / "best_genome.json"
        if best_genome is not None:
            genome_path.write_bytes(serialize_genome(best_genome))
        checkpoint_path = out / "checkpoint.pkl"
        save_checkpoint(checkpoint_path, state)
    return RunOutcome(exit_code=EXIT_SOLVED if solved else EXIT_GENERATION_LIMIT, generations=state.generation,
                      best_fitness=best_fitness, solved=solved, stats_path=stats_path, genome_path=genome_path,
                      checkpoint_path=checkpoint_path, state=state, timings=timings)


def _gpu_generation_times(config: NeatConfig, generations: int) -> list[float]:
    import torch
    state = init_state(config)
    problem = make_problem(config)
    root = RngStream(config.seed)
    times = []
    for generation in range(generations):
        torch.cuda.synchronize()
        t = time.perf_counter()
        pop, species, _ = evolve_step(state.population, state.species, config, root.child(generation),
                                      state.allocator, problem)
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t)
        state.population, state.species = pop, species
        state.generation = generation + 1
    return times


def run_bench(config: NeatConfig, pop_sizes: list[int], generations: int, out_dir, threads: int = 1,
              log=None, reference=None) -> Path:
    """Per-generation wall time per population size (runner.py:225-250), GPU
    column added.  The reference's tensorized / per-genome columns are filled
    when its module is passed as ``reference`` (timed on the host cores with
    the same seeds), else left empty."""
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    rows = []
    for pop_size in pop_sizes:
        cfg = config.with_overrides(pop_size=pop_size, generation_limit=generations, fitness_target=math.inf)
        if log:
            log(f"pop_size={pop_size}: gpu path")
        # one untimed generation per size: first-launch costs and the GPU's clock
        # ramp after the (long) host-side reference runs stay out of the timings
        _gpu_generation_times(cfg.with_overrides(generation_limit=1), 1)
        gpu = _gpu_generation_times(cfg, generations)
        tens = seq = [None] * generations
        if reference is not None:
            rcfg = reference.NeatConfig(**{k: getattr(cfg, k) for k in cfg.__dataclass_fields__})
            from importlib import import_module
            rrun = import_module(reference.__name__ + ".runner")
            if log:
                log(f"pop_size={pop_size}: reference tensorized / sequential paths")
            tens = rrun._timed_generations(rcfg, generations, threads, False)
            seq = rrun._timed_generations(rcfg, generations, threads, True)
        for g in range(generations):
            cells = ["" if v is None else repr(v) for v in (tens[g], seq[g])]
            rows.append(f"{pop_size},{g},{cells[0]},{cells[1]},{gpu[g]!r}")
    path = out / "bench.csv"
    path.write_text("\n".join([BENCH_HEADER, *rows]) + "\n", encoding="utf-8")
    return path
