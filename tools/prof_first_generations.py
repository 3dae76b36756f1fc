import cProfile, pstats, sys, os, time
sys.path.insert(0, '/root/repo')
import torch
import paper_2404_01817_b200 as tn
from paper_2404_01817_b200 import evolution as evo
from paper_2404_01817_b200.runner import init_state
import math
for P in (50, 5000):
    cfg = tn.NeatConfig(seed=0, problem="xor", pop_size=P, generation_limit=20, fitness_target=math.inf)
    state = init_state(cfg)
    problem = tn.make_problem(cfg)
    root = tn.RngStream(cfg.seed)
    pop, species = state.population, state.species
    for gen in range(3):
        torch.cuda.synchronize()
        pr = cProfile.Profile(); pr.enable()
        t = time.perf_counter()
        pop, species, _ = evo.evolve_step(pop, species, cfg, root.child(gen), state.allocator, problem)
        torch.cuda.synchronize()
        pr.disable()
        print(P, gen, time.perf_counter() - t, len(species))
        if P == 5000 and gen < 2:
            pstats.Stats(pr).sort_stats("tottime").print_stats(8)
