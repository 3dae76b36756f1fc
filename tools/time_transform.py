"""Device time of transform_arrays alone (CUDA events, median of --reps):
python tools/time_transform.py [--lib alternative.so] [--pop 10000]
(no finalize / forward: safe with diagnostic builds that stop early)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--pop", type=int, default=10000)
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--lib", default=None)
ap.add_argument("--layout", default="auto")
a = ap.parse_args()
if a.lib:
    from paper_2404_01817_b200 import _native
    _native.LIB_PATH = os.path.abspath(a.lib)
import paper_2404_01817_b200 as tn  # noqa: E402
from paper_2404_01817_b200.synthetic import synthetic_population  # noqa: E402

n, c = synthetic_population(a.pop, 128, 512, 32, 8, seed=20261018)
nodes, conns = torch.from_numpy(n).cuda(), torch.from_numpy(c).cuda()
for _ in range(3):
    tn.transform_arrays(nodes, conns, 32, 8, sync=False, layout=a.layout)
ts = []
for _ in range(a.reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    tn.transform_arrays(nodes, conns, 32, 8, sync=False, layout=a.layout)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ts.sort()
print(f"{a.lib or 'libtneat.so'} transform median {ts[len(ts) // 2]:.3f} ms min {ts[0]:.3f} ms", flush=True)
