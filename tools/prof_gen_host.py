"""cProfile of one config-3 generation (XOR, pop P): host-side attribution of
evolve_step (device time shows up in the synchronising calls)."""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2404_01817_b200 as tn  # noqa: E402
from paper_2404_01817_b200 import evolution as evo  # noqa: E402
from paper_2404_01817_b200.runner import init_state  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
cfg = tn.NeatConfig(seed=0, pop_size=P, inputs=2, outputs=1, problem="xor", max_nodes=50, max_conns=100,
                    compatibility_threshold=1.0, max_species=10)  # config 3 (tools/bench_configs.py)
state = init_state(cfg)
problem = tn.make_problem(cfg)
root = tn.RngStream(cfg.seed)
pop, species = state.population, state.species
for gen in range(4):
    pop, species, _ = evo.evolve_step(pop, species, cfg, root.child(gen), state.allocator, problem)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
pop, species, _ = evo.evolve_step(pop, species, cfg, root.child(4), state.allocator, problem)
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr).sort_stats("tottime")
st.print_stats(25)
pstats.Stats(pr).sort_stats("cumulative").print_stats(40)
st.print_callers("to|cpu|astype|full|reduce")
