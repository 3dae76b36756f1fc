"""Profiling driver: a couple of transform + forward steps of the bench
workload (for ncu launch lists and full captures)."""
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
ap.add_argument("--variant", type=int, default=0)
ap.add_argument("--batch", type=int, default=4096)
ap.add_argument("--layout", default="auto")
ap.add_argument("--precision", default="f32")
a = ap.parse_args()
n, c = synthetic_population(a.pop, 128, 512, 32, 8, seed=20261018)
nodes, conns = torch.from_numpy(n).cuda(), torch.from_numpy(c).cuda()
dt = torch.float64 if a.precision == "f64" else torch.float32
x = torch.randn((a.pop, a.batch, 32), device="cuda", dtype=dt)
out = torch.empty((a.pop, a.batch, 8), device="cuda", dtype=dt)
for _ in range(a.steps):
    st, _ = tn.transform_arrays(nodes, conns, 32, 8, layout=a.layout, precision=a.precision)
    tn.forward_device(st, x, out, variant=a.variant)
torch.cuda.synchronize()
print("maxdims", st.maxdims)
