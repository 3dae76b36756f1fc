import cProfile, pstats, sys, time, os
sys.path.insert(0, '/root/repo')
import torch
import paper_2404_01817_b200 as tn
from paper_2404_01817_b200 import evolution as evo
from paper_2404_01817_b200.runner import init_state
cfg = tn.NeatConfig(seed=0, pop_size=1_000_000, inputs=2, outputs=1, problem="xor", max_nodes=50, max_conns=100)
state = init_state(cfg)
problem = tn.make_problem(cfg)
root = tn.RngStream(cfg.seed)
pop, species = state.population, state.species
for gen in range(3):
    pop, species, _ = evo.evolve_step(pop, species, cfg, root.child(gen), state.allocator, problem)
torch.cuda.synchronize()
for k in range(3):
    t = time.perf_counter(); problem.evaluate_population_tensors(pop); torch.cuda.synchronize(); print("eval", time.perf_counter() - t)
pr = cProfile.Profile(); pr.enable()
problem.evaluate_population_tensors(pop); torch.cuda.synchronize()
pr.disable(); pstats.Stats(pr).sort_stats("tottime").print_stats(12)
