import sys, numpy as np
sys.path.insert(0, '/root/repo')
import os
import paper_2404_01817_b200 as tn
if os.environ.get("TNEAT_TOOL_LIB"):
    from paper_2404_01817_b200 import _native
    _native.LIB_PATH = os.path.abspath(os.environ["TNEAT_TOOL_LIB"])
from paper_2404_01817_b200 import recurrent as rec
from paper_2404_01817_b200.synthetic import synthetic_population
from oracle import arrayneat_oracle as orc
nodes, conns = synthetic_population(4, 128, 512, 27, 8, seed=20261018, variant="T", min_conns=216, max_conns_drawn=448)
env = rec.ant_env()
for prec in ("f64", "f32"):
    st, _ = tn.transform_arrays(nodes, conns, 27, 8, network_type="recurrent", precision=prec)
    print(prec, rec.rollout_fitness(st, env, steps=1000, sweeps=5))
if not os.environ.get("TNEAT_TOOL_LIB"): print("oracle", [orc.recurrent_rollout(nodes[p], conns[p], 27, 8, *env, steps=1000, sweeps=5) for p in range(2)])
