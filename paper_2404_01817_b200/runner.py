"""Generation loop with a device-resident population (reference runner.py).

``init_state`` (runner.py:54-66) builds the initial population on the GPU
(an_init) and speciates it; ``run_experiment`` (runner.py:145-198) drives
``evolve_step`` and writes the reference's ``stats.csv`` / ``timings.csv``
schema.  Populations stay CUDA tensors between generations; only fitness,
species bookkeeping and the per-generation statistics cross to the host.
"""

from __future__ import annotations

import os
import time
from dataclasses import dataclass, field

import numpy as np

from .config import NeatConfig, dump_config
from .evolution import STAGE_INIT, NodeKeyAllocator, evolve_step, speciate
from .genome import PopulationTensors, init_arrays
from .problems import make_problem
from .rng import RngStream

STATS_HEADER = "generation,best_fitness,mean_fitness,species_count,mean_live_nodes,mean_live_conns"
TIMINGS_HEADER = "generation,elapsed_seconds"


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
    state: EvolutionState
    solved: bool
    generations: int
    best_fitness: float
    timings: list


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


def run_experiment(config: NeatConfig, out_dir=None, state: EvolutionState | None = None,
                   log=None) -> RunOutcome:
    """Evolve until solved or ``generation_limit`` (runner.py:145-198)."""
    state = state or init_state(config)
    problem = make_problem(config)
    root = RngStream(config.seed)
    timings = []
    solved = False
    best = -np.inf
    while state.generation < config.generation_limit:
        t = time.perf_counter()
        pop, species, stats = evolve_step(state.population, state.species, config, root.child(state.generation),
                                          state.allocator, problem)
        timings.append(time.perf_counter() - t)
        state.stats_rows.append(stats_row(state.generation, stats))
        best = max(best, stats.best_fitness)
        if log:
            log(state.generation, stats)
        state.population, state.species = pop, species
        state.generation += 1
        if stats.solved:
            solved = True
            break
    if out_dir is not None:
        os.makedirs(out_dir, exist_ok=True)
        with open(os.path.join(out_dir, "stats.csv"), "w") as fh:
            fh.write(STATS_HEADER + "\n" + "\n".join(state.stats_rows) + "\n")
        with open(os.path.join(out_dir, "timings.csv"), "w") as fh:
            fh.write(TIMINGS_HEADER + "\n" + "\n".join(f"{i},{t!r}" for i, t in enumerate(timings)) + "\n")
        with open(os.path.join(out_dir, "config.txt"), "w") as fh:
            fh.write(dump_config(config))
    return RunOutcome(state=state, solved=solved, generations=state.generation, best_fitness=best,
                      timings=timings)
