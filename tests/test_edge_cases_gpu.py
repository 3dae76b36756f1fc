"""Edge cases of the transform + forward path against the oracle (pinned to
the reference by test_oracle_golden.py): empty populations and batches,
genomes without connections, empty aggregations, unpruned programs, and large
genome capacities."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import cuda_ok

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tn():
    if not cuda_ok():
        pytest.skip("no CUDA device")
    import paper_2404_01817_b200 as tn
    return tn


def _oracle_out(nodes, conns, x, ni, no):
    from oracle import arrayneat_oracle as orc
    return np.stack([orc.forward_genome(nodes[p], orc.transform_genome(nodes[p], conns[p], ni, no), x[p])
                     for p in range(nodes.shape[0])])


def test_empty_population_and_batch(tn):
    import torch
    from oracle.arrayneat_oracle import synthetic_population
    nodes, conns = synthetic_population(3, 64, 128, 4, 2, seed=1, min_conns=10, max_conns_drawn=60)
    st, _ = tn.transform_arrays(nodes[:0], conns[:0], 4, 2)
    assert st.size == 0
    out = tn.forward_device(st, torch.zeros((0, 10, 4), device="cuda"))
    assert tuple(out.shape) == (0, 10, 2)
    st, _ = tn.transform_arrays(nodes, conns, 4, 2)
    out = tn.forward_device(st, torch.zeros((3, 0, 4), device="cuda"))
    assert tuple(out.shape) == (3, 0, 2)
    x = np.random.default_rng(0).standard_normal((3, 1, 4))
    y = tn.forward_arrays(st, None, x.astype(np.float32))
    np.testing.assert_allclose(y, _oracle_out(nodes, conns, x, 4, 2), rtol=0, atol=1e-5)


def test_no_connections_and_empty_aggregations(tn):
    """Outputs without incoming edges evaluate act(bias + response * 0) for
    every aggregation (empty aggregation = 0, inference.py:238-240)."""
    from oracle.arrayneat_oracle import synthetic_population
    nodes, conns = synthetic_population(8, 32, 64, 3, 4, seed=2, variant="M", min_conns=0, max_conns_drawn=20)
    conns[:4] = np.nan  # genomes 0-3: no connections at all
    for agg in range(4):  # output nodes of genome 4 + agg: every aggregation with some empty lists
        nodes[4 + agg, 3:7, 3] = float(agg)
    x = np.random.default_rng(3).standard_normal((8, 7, 3))
    st, cyc = tn.transform_arrays(nodes, conns, 3, 4, precision="f64")
    assert cyc.size == 0
    np.testing.assert_allclose(tn.forward_arrays(st, None, x), _oracle_out(nodes, conns, x, 3, 4),
                               rtol=1e-9, atol=1e-9)


@pytest.mark.parametrize("precision,tol", [("f64", 1e-9), ("f32", 1e-5)])
def test_unpruned_programs(tn, precision, tol):
    """prune=False keeps every live node in the program (no ancestor-cone
    pruning): same outputs."""
    from oracle.arrayneat_oracle import synthetic_population
    nodes, conns = synthetic_population(10, 48, 120, 4, 3, seed=4, variant="M", min_conns=20, max_conns_drawn=100)
    x = np.random.default_rng(5).standard_normal((10, 9, 4))
    a, _ = tn.transform_arrays(nodes, conns, 4, 3, precision=precision, prune=False)
    b, _ = tn.transform_arrays(nodes, conns, 4, 3, precision=precision)
    ref = _oracle_out(nodes, conns, x, 4, 3)
    inp = x if precision == "f64" else x.astype(np.float32)
    for st in (a, b):
        out = tn.forward_arrays(st, None, inp)
        assert np.max(np.abs(out - ref) / np.maximum(1.0, np.abs(ref))) <= tol
    assert a.maxdims[1] >= b.maxdims[1]  # unpruned programs have at least as many steps


def test_large_genome_capacity(tn):
    """max_nodes 512 / max_conns 2048 (far beyond the configs): transform and
    forward stay exact against the oracle in float64."""
    from oracle.arrayneat_oracle import synthetic_population
    nodes, conns = synthetic_population(4, 512, 2048, 16, 4, seed=6, min_conns=1200, max_conns_drawn=2000)
    x = np.random.default_rng(7).standard_normal((4, 300, 16))
    st, cyc = tn.transform_arrays(nodes, conns, 16, 4, precision="f64")
    assert cyc.size == 0
    np.testing.assert_allclose(tn.forward_arrays(st, None, x), _oracle_out(nodes, conns, x, 16, 4),
                               rtol=1e-9, atol=1e-9)
    st32, _ = tn.transform_arrays(nodes, conns, 16, 4)
    out = tn.forward_arrays(st32, None, x.astype(np.float32))
    ref = _oracle_out(nodes, conns, x, 16, 4)
    assert np.max(np.abs(out - ref) / np.maximum(1.0, np.abs(ref))) <= 1e-5


def test_checked_build_traps_on_a_corrupt_program(tmp_path):
    """The checked build (-DTNEAT_CHECKS, run with TNEAT_LIB=...libtneat_checks.so)
    validates staged program indices on the device: a program whose hidden
    edge points past the genome's value slots makes the launch fail instead
    of reading out of bounds.  (Run in a subprocess: a trap poisons the context.)"""
    import os
    import subprocess
    import sys
    lib = os.environ.get("TNEAT_LIB", "")
    if "checks" not in lib:
        pytest.skip("checked build not selected (TNEAT_LIB)")
    code = r"""
import sys, torch
sys.path.insert(0, %r)
import paper_2404_01817_b200 as tn
from paper_2404_01817_b200.synthetic import synthetic_population
n, c = synthetic_population(4, 128, 512, 32, 8, seed=5)
st, _ = tn.transform_arrays(n, c, 32, 8)
L = tn.inference
hdr = st.program[:, :32].contiguous().view(torch.int32)
steps, edges, groups = (int(v) for v in hdr[0, [0, 1, 7]])
off = 128  # off_tc for O = 8
nb = (steps + 15) // 16 * 16
grp = off + 192 * nb + 4 * nb
recs = st.program[0, grp:grp + 16 * groups].contiguous().view(torch.int32).view(-1, 4).cpu()
e = int(next(r[2] for r in recs if r[1] > 0))  # first entry a group actually sweeps
src = grp + 16 * groups + 16 * steps + 4 * e
st.program[0, src:src + 4] = torch.tensor([0, 0, 0x7F, 0], dtype=torch.uint8)  # slot far past n_steps
x = torch.randn(4, 256, 32, device="cuda")
try:
    tn.forward_device(st, x)
    torch.cuda.synchronize()
    print("NO-TRAP")
except Exception as e:
    print("TRAPPED", type(e).__name__)
""" % (os.path.dirname(os.path.dirname(os.path.abspath(__file__))),)
    res = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300,
                         env=dict(os.environ))
    out = res.stdout + res.stderr
    assert "NO-TRAP" not in out, out[-2000:]
    assert "TNEAT_CHECK failed" in out, out[-2000:]


@pytest.mark.parametrize("precision", ["f32", "f64"])
@pytest.mark.parametrize("batch", [1, 256])
def test_max_min_propagate_nan_like_numpy(tn, precision, batch):
    """max / min aggregations propagate a NaN term wherever it sits, as the
    reference's np.max does (functions.py:37): 0 * inf is NaN, and a later,
    larger finite term must not replace it; relu of a NaN pre-activation stays
    NaN (np.maximum, functions.py:30).  Warp kernel at B=1, tile kernel at B=256."""
    import torch
    from oracle import arrayneat_oracle as orc
    nan = np.nan
    nodes = np.full((3, 4, 5), nan)
    conns = np.full((3, 4, 4), nan)
    for g, (agg, act) in enumerate(((2, 0), (4, 0), (0, 3))):  # max, min; sum -> relu (np.maximum(x, 0))
        nodes[g, 0] = [0, 0.0, 1.0, 0, 0]
        nodes[g, 1] = [1, 0.0, 1.0, 0, 0]
        nodes[g, 2] = [2, 0.0, 1.0, agg, act]  # the output
        conns[g, 0] = [0, 2, 1.0, 0.0]       # 0 * inf -> NaN, the first term
        conns[g, 1] = [1, 2, 1.0, 1.0]
    st, _ = tn.transform_arrays(nodes, conns, 2, 1, precision=precision)
    dt = torch.float64 if precision == "f64" else torch.float32
    x = torch.zeros((3, batch, 2), dtype=dt)
    x[:, :, 0] = float("inf")
    x[:, :, 1] = torch.linspace(-3, 3, batch, dtype=dt)
    out = tn.forward_device(st, x.cuda()).cpu().numpy()
    for g in range(3):
        ref = orc.forward_genome(nodes[g], orc.transform_genome(nodes[g], conns[g], 2, 1),
                                 x[g].numpy().astype(np.float64))
        assert np.all(np.isnan(ref)) and np.all(np.isnan(out[g])), (g, out[g][:4])
