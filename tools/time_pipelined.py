"""Serial vs pipelined bench steps: step k+1's transform on a high-priority
stream overlapping step k's forward."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2404_01817_b200 as tn  # noqa: E402
from paper_2404_01817_b200.synthetic import synthetic_population  # noqa: E402

torch.set_num_threads(8)
n, c = synthetic_population(10000, 128, 512, 32, 8, seed=20261018)
nodes, conns = torch.from_numpy(n).cuda(), torch.from_numpy(c).cuda()
x = torch.randn((10000, 4096, 32), device="cuda")
out = torch.empty((10000, 4096, 8), device="cuda")
steps = 20


def serial():
    st, _ = tn.transform_arrays(nodes, conns, 32, 8, sync=False)
    tn.finalize_transform(st)
    tn.forward_device(st, x, out)


fw = torch.cuda.current_stream()
for prio in (0, -1):
    tr = torch.cuda.Stream(priority=prio)
    keep = []

    def pipelined():
        with torch.cuda.stream(tr):
            st, _ = tn.transform_arrays(nodes, conns, 32, 8, sync=False)
            tn.finalize_transform(st)
        ev = torch.cuda.Event()
        ev.record(tr)
        fw.wait_event(ev)
        for t in (st.program, st.status_dev):
            t.record_stream(fw)
        tn.forward_device(st, x, out, stream=fw)
        keep.append(st)
        if len(keep) > 2:
            keep.pop(0)

    for name, fn in (("serial", serial), (f"pipelined prio {prio}", pipelined)):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(fw)
        tr.wait_event(s0)
        for _ in range(steps):
            fn()
        ev = torch.cuda.Event()
        ev.record(tr)
        fw.wait_event(ev)
        s1.record(fw)
        torch.cuda.synchronize()
        print(f"{name}: {s0.elapsed_time(s1) / steps:.3f} ms/step", flush=True)
