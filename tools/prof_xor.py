"""cProfile of config-1 generations (XOR, pop 1000): host-side cost per phase."""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2404_01817_b200 as tn  # noqa: E402
from paper_2404_01817_b200.runner import init_state  # noqa: E402

cfg = tn.NeatConfig(seed=0, pop_size=1000, inputs=2, outputs=1, problem="xor", max_nodes=50, max_conns=100,
                    generation_limit=100)
state = init_state(cfg)
problem = tn.make_problem(cfg)
root = tn.RngStream(cfg.seed)
pop, species = state.population, state.species
for gen in range(5):
    pop, species, _ = tn.evolve_step(pop, species, cfg, root.child(gen), state.allocator, problem)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for gen in range(5, 25):
    pop, species, _ = tn.evolve_step(pop, species, cfg, root.child(gen), state.allocator, problem)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumtime").print_stats(30)
