"""Where the end-to-end step goes: raw PCIe copy rates (pinned, 256 MB chunks),
transform_arrays from host numpy genomes, and the pipelined forward_arrays."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2404_01817_b200 as tn  # noqa: E402
from paper_2404_01817_b200.synthetic import synthetic_population  # noqa: E402

POP, B, I, O = 10000, 4096, 32, 8
n, c = synthetic_population(POP, 128, 512, I, O, seed=20261018)
xh = torch.empty((POP, B, I), dtype=torch.float32, pin_memory=True)
xh.normal_()
oh = torch.empty((POP, B, O), dtype=torch.float32, pin_memory=True)
dev = torch.empty((POP // 10, B, I), dtype=torch.float32, device="cuda")
devo = torch.empty((POP // 10, B, O), dtype=torch.float32, device="cuda")


def timed(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t)
    return best


def h2d():
    for k in range(10):
        dev.copy_(xh[k * 1000:(k + 1) * 1000], non_blocking=True)


def d2h():
    for k in range(10):
        oh[k * 1000:(k + 1) * 1000].copy_(devo, non_blocking=True)


s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def both():
    with torch.cuda.stream(s1):
        h2d()
    with torch.cuda.stream(s2):
        d2h()


t = timed(h2d)
print(f"H2D {xh.nbytes / t / 1e9:.1f} GB/s ({1e3 * t:.1f} ms for {xh.nbytes / 1e9:.2f} GB)")
t = timed(d2h)
print(f"D2H {oh.nbytes / t / 1e9:.1f} GB/s ({1e3 * t:.1f} ms)")
t = timed(both)
print(f"H2D+D2H concurrent {1e3 * t:.1f} ms")
t = timed(lambda: tn.finalize_transform(tn.transform_arrays(n, c, I, O)[0]))
print(f"transform_arrays(numpy) + finalize {1e3 * t:.1f} ms")
st, _ = tn.transform_arrays(n, c, I, O)
t = timed(lambda: tn.forward_arrays(st, None, xh, out=oh))
print(f"forward_arrays(pinned) {1e3 * t:.1f} ms -> {POP * B / t:.3g} evals/s")
t = timed(lambda: tn.forward_arrays(tn.transform_arrays(n, c, I, O)[0], None, xh, out=oh))
print(f"e2e step {1e3 * t:.1f} ms -> {POP * B / t:.3g} evals/s")
npin, cpin = torch.from_numpy(n).pin_memory(), torch.from_numpy(c).pin_memory()
t = timed(lambda: tn.finalize_transform(tn.transform_arrays(npin, cpin, I, O)[0]))
print(f"transform_arrays(pinned) + finalize {1e3 * t:.1f} ms")
t = timed(lambda: tn.forward_arrays(tn.transform_arrays(npin, cpin, I, O)[0], None, xh, out=oh))
print(f"e2e step (pinned genomes) {1e3 * t:.1f} ms -> {POP * B / t:.3g} evals/s")
