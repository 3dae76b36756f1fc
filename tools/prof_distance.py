"""Distance kernel timing on evolved populations: pop P x Q representatives
(speciate's pair_mode 0 launch), CUDA-event timed, with the algorithmic
bytes (every genome and representative read once) -> GB/s.
    python tools/prof_distance.py [P] [max_nodes] [max_conns] [generations] [shuffle]
shuffle=1 permutes every genome's node and connection rows (one permutation for
the population), so homologs sit at other rows and every lookup searches the
representatives' key maps."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2404_01817_b200 as tn  # noqa: E402
from paper_2404_01817_b200 import evolution as evo  # noqa: E402
from paper_2404_01817_b200.runner import init_state  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
N = int(sys.argv[2]) if len(sys.argv) > 2 else 50
C = int(sys.argv[3]) if len(sys.argv) > 3 else 100
G = int(sys.argv[4]) if len(sys.argv) > 4 else 3
SHUFFLE = len(sys.argv) > 5 and sys.argv[5] == "1"
cfg = tn.NeatConfig(seed=0, pop_size=P, inputs=2, outputs=1, problem="xor", max_nodes=N, max_conns=C,
                    compatibility_threshold=1.0, max_species=10)
state = init_state(cfg)
problem = tn.make_problem(cfg)
root = tn.RngStream(cfg.seed)
pop, species = state.population, state.species
for gen in range(G):
    pop, species, _ = evo.evolve_step(pop, species, cfg, root.child(gen), state.allocator, problem)
Q = 10
reps_n, reps_c = pop.nodes[:Q].contiguous(), pop.conns[:Q].contiguous()
if SHUFFLE:
    g = torch.Generator(device="cpu").manual_seed(1)
    pop = tn.PopulationTensors(pop.nodes[:, torch.randperm(N, generator=g)].contiguous(),
                               pop.conns[:, torch.randperm(C, generator=g)].contiguous(), None, None, 2, 1)
times = []
torch.cuda.nvtx.range_push("dist")  # ncu --nvtx --nvtx-include "dist/" captures only these launches
for _ in range(6):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    d = evo._distance_dev(pop.nodes, pop.conns, reps_n, reps_c, cfg, 0)
    e1.record()
    torch.cuda.synchronize()
    times.append(e0.elapsed_time(e1))
torch.cuda.nvtx.range_pop()
t = sorted(times)[len(times) // 2] / 1e3
gbytes = (P + Q) * (N * 5 + C * 4) * 8 / 1e9
print(f"distance P={P} Q={Q} N={N} C={C}: {1e3 * t:.3f} ms, {P * Q / t:.3g} pairs/s, "
      f"{gbytes / t:.1f} GB/s algorithmic ({gbytes:.3f} GB once)", flush=True)
