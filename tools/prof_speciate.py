"""cProfile of one config-3 speciate call at pop P (host-side attribution;
device time shows up in the synchronising calls)."""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2404_01817_b200 as tn  # noqa: E402
from paper_2404_01817_b200 import evolution as evo  # noqa: E402
from paper_2404_01817_b200.runner import init_state  # noqa: E402

pop_n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
cfg = tn.NeatConfig(seed=0, pop_size=pop_n, inputs=2, outputs=1, problem="xor", max_nodes=50, max_conns=100,
                    compatibility_threshold=1.0, max_species=10)
state = init_state(cfg)
problem = tn.make_problem(cfg)
root = tn.RngStream(cfg.seed)
pop, species = state.population, state.species
for gen in range(2):
    rng = root.child(gen)
    fit = problem.evaluate_population_tensors(pop, rng=rng.child(evo.STAGE_EVAL))
    alloc = evo.allocate_spawns(evo.update_stagnation(species, fit, cfg), fit, cfg)
    ev = tn.PopulationTensors(pop.nodes, pop.conns, pop.species_id, fit, 2, 1)
    off = evo.reproduce(ev, alloc, fit, cfg, rng, state.allocator)
    torch.cuda.synchronize()
    if gen == 1:
        pr = cProfile.Profile()
        pr.enable()
    pop, species = evo.speciate(off, alloc, cfg)
    torch.cuda.synchronize()
    if gen == 1:
        pr.disable()
        pstats.Stats(pr).sort_stats("tottime").print_stats(14)
