"""Split the config-3 reproduce phase into host slot tables and the device launch."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2404_01817_b200 as tn  # noqa: E402
if os.environ.get("TNEAT_TOOL_LIB"):  # A/B of a tools/build_variant.py library
    from paper_2404_01817_b200 import _native  # noqa: E402
    _native.LIB_PATH = os.path.abspath(os.environ["TNEAT_TOOL_LIB"])
from paper_2404_01817_b200 import evolution as evo  # noqa: E402
from paper_2404_01817_b200.runner import init_state  # noqa: E402

pop_n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
cfg = tn.NeatConfig(seed=0, pop_size=pop_n, inputs=2, outputs=1, problem="xor", max_nodes=50, max_conns=100,
                    compatibility_threshold=1.0, max_species=10)
state = init_state(cfg)
problem = tn.make_problem(cfg)
root = tn.RngStream(cfg.seed)
pop, species = state.population, state.species
for gen in range(5):
    rng = root.child(gen)
    fit = problem.evaluate_population_tensors(pop, rng=rng.child(evo.STAGE_EVAL))
    ts = time.perf_counter()
    surv = evo.update_stagnation(species, fit, cfg)
    tu = time.perf_counter()
    alloc = evo.allocate_spawns(surv, fit, cfg)
    t0 = time.perf_counter()
    tabs = evo.slot_tables(alloc, fit, cfg)
    t1 = time.perf_counter()
    ev = tn.PopulationTensors(pop.nodes, pop.conns, pop.species_id, fit, 2, 1)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    off = evo.reproduce(ev, alloc, fit, cfg, rng, state.allocator)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    pop, species = evo.speciate(off, alloc, cfg)
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    print(f"gen {gen}: stagnation {1e3*(tu-ts):.1f} ms, spawns {1e3*(t0-tu):.1f} ms, "
          f"slot_tables {1e3*(t1-t0):.1f} ms, reproduce total {1e3*(t3-t2):.1f} ms, "
          f"speciate {1e3*(t4-t3):.1f} ms, species {len(species)}", flush=True)
