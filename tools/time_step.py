"""Wall/CUDA-event breakdown of one bench step (transform, finalize, plan, forward)."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2404_01817_b200 as tn  # noqa: E402
from paper_2404_01817_b200.synthetic import synthetic_population  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--pop", type=int, default=10000)
ap.add_argument("--variant", type=int, default=0)
ap.add_argument("--reps", type=int, default=4)
ap.add_argument("--layout", default="auto")
ap.add_argument("--lib", default=None, help="alternative libtneat.so build (tuning experiments)")
ap.add_argument("--fwd-reps", type=int, default=10)
ap.add_argument("--prune", type=int, default=1)
ap.add_argument("--precision", default="f32")
a = ap.parse_args()
if a.lib:
    from paper_2404_01817_b200 import _native
    _native.LIB_PATH = os.path.abspath(a.lib)
n, c = synthetic_population(a.pop, 128, 512, 32, 8, seed=20261018)
nodes, conns = torch.from_numpy(n).cuda(), torch.from_numpy(c).cuda()
dt = torch.float64 if a.precision == "f64" else torch.float32
x = torch.randn((a.pop, 4096, 32), device="cuda", dtype=dt)
out = torch.empty((a.pop, 4096, 8), device="cuda", dtype=dt)
for rep in range(a.reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    st, _ = tn.transform_arrays(nodes, conns, 32, 8, sync=False, layout=a.layout, prune=bool(a.prune), precision=a.precision)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    tn.finalize_transform(st)
    t2 = time.perf_counter()
    if st.precision & tn.inference.FMT_TC:
        plan = [c for c in tn.inference.tc_plan_counts(st) if c]
    else:
        plan = tn.inference._bucket_plan(st, (a.variant & 0xF) or 5)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    tn.forward_device(st, x, out, variant=a.variant)
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    print(f"transform {1e3*(t1-t0):.2f} ms finalize {1e3*(t2-t1):.2f} plan {1e3*(t3-t2):.2f} "
          f"forward {1e3*(t4-t3):.2f} buckets {len(plan)} maxdims {st.maxdims}", flush=True)
evs = []
for _ in range(a.fwd_reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    tn.forward_device(st, x, out, variant=a.variant)
    e1.record()
    torch.cuda.synchronize()
    evs.append(e0.elapsed_time(e1))
evs.sort()
print(f"{a.lib or 'libtneat.so'} forward median {evs[len(evs) // 2]:.3f} ms min {evs[0]:.3f} ms", flush=True)
tvs = []
for _ in range(a.fwd_reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    tn.transform_arrays(nodes, conns, 32, 8, sync=False, layout=a.layout, prune=bool(a.prune), precision=a.precision)
    e1.record()
    torch.cuda.synchronize()
    tvs.append(e0.elapsed_time(e1))
tvs.sort()
print(f"{a.lib or 'libtneat.so'} transform median {tvs[len(tvs) // 2]:.3f} ms min {tvs[0]:.3f} ms", flush=True)
