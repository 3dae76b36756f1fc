"""Small invocations of every kernel family for compute-sanitizer
(memcheck / racecheck / synccheck):
    compute-sanitizer --tool memcheck python tools/sanitize_small.py
Tensor-core forward (device plan; ragged batch; extreme rows), tile / warp
forward, transform, fused fitness, cart-pole, distance / speciation,
reproduce / mutate / init, recurrent rollout, HyperNEAT substrate."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2404_01817_b200 as tn  # noqa: E402
from paper_2404_01817_b200.synthetic import synthetic_population  # noqa: E402

which = sys.argv[1:] or ["forward", "evolution", "hyperneat", "recurrent"]
dev = torch.device("cuda", 0)
if "forward" in which:
    nodes, conns = synthetic_population(12, 128, 512, 32, 8, seed=5)
    nm, cm = synthetic_population(4, 128, 512, 32, 8, seed=6, variant="M")
    nodes, conns = np.concatenate([nodes, nm]), np.concatenate([conns, cm])
    x = torch.randn(16, 300, 32, device=dev)
    x[1, 7, 3] = float("inf")
    x[2, 9] *= 1e-30
    st, _ = tn.transform_arrays(nodes, conns, 32, 8, sync=False)
    sq = torch.zeros(16, device=dev)
    a = tn.forward_device(st, x, sq_sum=sq)
    std, _ = tn.transform_arrays(nodes, conns, 32, 8, layout="standard")
    for v in (1, 2, 5, 8):
        tn.forward_device(std, x, variant=v)
    f64, _ = tn.transform_arrays(nodes, conns, 32, 8, precision="f64")
    tn.forward_device(f64, x.double())
    torch.cuda.synchronize()
    print("forward ok", float(sq.sum()))
if "evolution" in which:
    cfg = tn.NeatConfig(seed=0, pop_size=64, inputs=2, outputs=1, problem="xor", max_nodes=20, max_conns=40,
                        compatibility_threshold=1.0)
    from paper_2404_01817_b200.runner import init_state
    state = init_state(cfg)
    problem = tn.make_problem(cfg)
    pop, species = state.population, state.species
    for g in range(2):
        pop, species, stats = tn.evolve_step(pop, species, cfg, tn.RngStream(0).child(g), state.allocator, problem)
    torch.cuda.synchronize()
    print("evolution ok", stats.best_fitness)
if "hyperneat" in which:
    from paper_2404_01817_b200 import hyperneat as hn
    nodes, conns = synthetic_population(8, 64, 256, 4, 1, seed=7, variant="M", min_conns=16, max_conns_drawn=64)
    st, _ = tn.transform_arrays(nodes, conns, 4, 1)
    x, t = hn.teacher_task(256)
    w = hn.cppn_weights(st)
    f = hn.substrate_fitness(w, torch.from_numpy(x).cuda(), torch.from_numpy(t).cuda())
    torch.cuda.synchronize()
    print("hyperneat ok", float(f.mean()))
if "recurrent" in which:
    from paper_2404_01817_b200 import recurrent as rec
    nodes, conns = synthetic_population(8, 64, 256, 27, 8, seed=8, min_conns=40, max_conns_drawn=120)
    st, _ = tn.transform_arrays(nodes, conns, 27, 8, network_type="recurrent")
    f = rec.rollout_fitness(st, rec.ant_env(), steps=5, sweeps=2)
    print("recurrent ok", float(np.mean(f)))
