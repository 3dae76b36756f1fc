"""Parity of the exact benchmarked launch (bench.py's step, BASELINE configs[1]).

The bench transforms the §8d population (pop 10,000, 128/512, I=32, O=8,
seed 20261018, tanh/sum) and runs the tensor-core forward from its
device-side launch plan (fwd_tc_kernel, one persistent launch per MMA-width
class) over 4096 inputs per genome
generated on the device (seed 20261019).  This test makes the same calls,
checks every genome takes the tensor-core format and the plan forms the
buckets the bench launches, and
compares a stratified 256-genome subset -- every bucket represented -- across
all 4096 inputs with the oracle at |d| <= 1e-5 * max(1, |ref|) (north_star's
fp32 bound).  It also checks the step's second half: the next transform on
the same tensors gives identical programs and bit-identical outputs (the bench
re-transforms every step)."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import cuda_ok

pytestmark = pytest.mark.gpu

POP, MAXN, MAXC, NIN, NOUT, BATCH = 10_000, 128, 512, 32, 8, 4096
TOL = 1e-5


@pytest.fixture(scope="module")
def bench_run():
    if not cuda_ok():
        pytest.skip("no CUDA device")
    import torch

    import paper_2404_01817_b200 as tn
    from paper_2404_01817_b200.synthetic import synthetic_population
    dev = torch.device("cuda", 0)
    nodes_h, conns_h = synthetic_population(POP, MAXN, MAXC, NIN, NOUT, seed=20261018)
    nodes, conns = torch.from_numpy(nodes_h).to(dev), torch.from_numpy(conns_h).to(dev)
    gen = torch.Generator(device=dev).manual_seed(20261019)
    x = torch.randn((POP, BATCH, NIN), device=dev, dtype=torch.float32, generator=gen)
    st, _ = tn.transform_arrays(nodes, conns, NIN, NOUT, sync=False)
    tn.finalize_transform(st)
    out = tn.forward_device(st, x, torch.empty((POP, BATCH, NOUT), device=dev), variant=0)
    torch.cuda.synchronize()
    return tn, st, nodes_h, conns_h, x, out


def _plan(tn, st):
    """Device launch plan of the benchmarked population: per class, its program rows."""
    counts = tn.inference.tc_plan_counts(st)
    ids = st._cache["tcplan"][0].view(tn.inference.TC_NCLASS, -1).cpu().numpy()
    return [(ids[c, :counts[c]], c) for c in range(tn.inference.TC_NCLASS) if counts[c]], counts


def test_bench_plan_has_every_bucket(bench_run):
    tn, st, *_ = bench_run
    plan, counts = _plan(tn, st)
    assert counts[6] == 0  # every tanh/sum genome takes the tensor-core format
    assert counts.sum() == POP
    assert (counts[:3] > 0).all(), counts  # MMA-width classes 32 / 48 / 64 are all launched


def test_bench_launch_matches_oracle_on_stratified_subset(bench_run):
    from oracle import arrayneat_oracle as orc
    tn, st, nodes_h, conns_h, x, out = bench_run
    plan, _ = _plan(tn, st)
    rng = np.random.default_rng(7)
    per = -(-256 // len(plan))
    picks = []
    for ids, _ in plan:
        picks += rng.choice(ids, size=min(per, ids.size), replace=False).tolist()
    picks = np.array(sorted(picks[:256] if len(picks) > 256 else picks))
    xs = x[picks].cpu().numpy().astype(np.float64)
    ys = out[picks].cpu().numpy()
    worst = 0.0
    for k, p in enumerate(picks):
        tr = orc.transform_genome(nodes_h[p], conns_h[p], NIN, NOUT)
        ref = orc.forward_genome(nodes_h[p], tr, xs[k])
        err = float(np.max(np.abs(ys[k] - ref) / np.maximum(1.0, np.abs(ref))))
        worst = max(worst, err)
        assert err <= TOL, (int(p), err)
    assert worst > 0.0  # fp32 against f64: a zero error would mean the comparison did not run


def test_bench_retransform_is_byte_identical(bench_run):
    import torch
    tn, st, nodes_h, conns_h, x, out = bench_run
    st2, _ = tn.transform_arrays(st.nodes_dev, st.conns_dev, NIN, NOUT)
    assert torch.equal(st2.program[:, :32], st.program[:, :32])  # headers (unused tails are not written)
    out2 = tn.forward_device(st2, x, variant=0)
    assert torch.equal(out2, out)  # deterministic: same programs, same plan, same bits
