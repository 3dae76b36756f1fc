"""Profiling driver for one bench step's kernels (transform + device-planned
forward): --steps steps of transform + forward; capture the last step with
    ncu -k regex:"transform_kernel|plan_tc|fwd_" -s <8*(steps-1)> -c 8 ..."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2404_01817_b200 as tn  # noqa: E402
from paper_2404_01817_b200.synthetic import synthetic_population  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--pop", type=int, default=10000)
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--layout", default="auto")
ap.add_argument("--prune", type=int, default=1)
a = ap.parse_args()
n, c = synthetic_population(a.pop, 128, 512, 32, 8, seed=20261018)
nodes, conns = torch.from_numpy(n).cuda(), torch.from_numpy(c).cuda()
x = torch.randn((a.pop, 4096, 32), device="cuda")
out = torch.empty((a.pop, 4096, 8), device="cuda")
for _ in range(a.steps):
    st, _ = tn.transform_arrays(nodes, conns, 32, 8, sync=False, layout=a.layout, prune=bool(a.prune))
    tn.forward_device(st, x, out)
torch.cuda.synchronize()
print("done")
