"""Per-phase wall time of a generation (synchronised), e.g. config 1 (pop 1000)."""
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

pop_n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
cfg = tn.NeatConfig(seed=0, pop_size=pop_n, inputs=2, outputs=1, problem="xor", max_nodes=50, max_conns=100)
state = init_state(cfg)
problem = tn.make_problem(cfg)
root = tn.RngStream(cfg.seed)
pop, species = state.population, state.species
acc = {}
GENS = int(sys.argv[2]) if len(sys.argv) > 2 else 40
for gen in range(GENS):
    rng = root.child(gen)
    t = [time.perf_counter()]
    fit = problem.evaluate_population_tensors(pop, rng=rng.child(evo.STAGE_EVAL))
    torch.cuda.synchronize(); t.append(time.perf_counter())
    surv = evo.update_stagnation(species, fit, cfg)
    alloc = evo.allocate_spawns(surv, fit, cfg)
    t.append(time.perf_counter())
    ev = tn.PopulationTensors(pop.nodes, pop.conns, pop.species_id, fit, 2, 1)
    off = evo.reproduce(ev, alloc, fit, cfg, rng, state.allocator)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    pop, species = evo.speciate(off, alloc, cfg, rng.child(evo.STAGE_SPECIATE))
    torch.cuda.synchronize(); t.append(time.perf_counter())
    if gen >= 10:
        for k, name in enumerate(["eval", "stagnation+spawns", "reproduce", "speciate"]):
            acc[name] = acc.get(name, 0) + (t[k + 1] - t[k]) / max(1, GENS - 10)
print({k: f"{1e3 * v:.3f} ms" for k, v in acc.items()}, "total", f"{1e3 * sum(acc.values()):.3f} ms")
