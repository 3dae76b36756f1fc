"""The bench step loop with per-step host timestamps, to find host-side stalls."""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2404_01817_b200 as tn  # noqa: E402
from paper_2404_01817_b200.synthetic import synthetic_population  # noqa: E402

torch.set_num_threads(8)
n, c = synthetic_population(10000, 128, 512, 32, 8, seed=20261018)
nodes, conns = torch.from_numpy(n).cuda(), torch.from_numpy(c).cuda()
x = torch.randn((10000, 4096, 32), device="cuda")
out = torch.empty((10000, 4096, 8), device="cuda")
rows = []
for step in range(40):
    t0 = time.perf_counter()
    st, _ = tn.transform_arrays(nodes, conns, 32, 8, sync=False)
    t1 = time.perf_counter()
    tn.finalize_transform(st)
    t2 = time.perf_counter()
    tn.forward_device(st, x, out)
    t3 = time.perf_counter()
    rows.append((t1 - t0, t2 - t1, t3 - t2))
torch.cuda.synchronize()
for name, k in (("transform enqueue", 0), ("finalize (sync)", 1), ("plan + forward enqueue", 2)):
    v = [1e3 * r[k] for r in rows[5:]]
    print(f"{name:24s} median {statistics.median(v):.3f} ms  max {max(v):.3f} ms  p90 {sorted(v)[int(0.9*len(v))]:.3f}")
print("per-step", [round(1e3 * sum(r), 2) for r in rows[5:]])
