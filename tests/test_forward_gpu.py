"""GPU parity: transform (K1) and forward (K2) against the reference goldens
and the oracle.  Calls go through the package -> ctypes -> C ABI.

Tolerances (written here, per north_star):
  * transform order / io rows / dense incoming / cyclic list: bit-exact;
  * f64 programs: |d| <= 1e-9 (the reference's own oracle bound, test_oracle.py:82-92);
  * f32 programs: |d| <= 1e-5 * max(1, |ref|) (north_star) on
    tanh/sum and mixed act/agg networks alike (profiles/r02_parity_report.json:
    max 2.4e-6 over 3.2M checked outputs).  Both program layouts --
    "standard" (tile / warp kernels) and "tc" (input layer as an exact
    digit-split tcgen05 MMA, fwd_tc_kernel) -- meet the same bounds.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import cuda_ok, load_golden

pytestmark = pytest.mark.gpu

CASES = ["forward_small.npz", "forward_cfg2_T.npz", "forward_cfg2_M.npz", "corpus.npz"]


@pytest.fixture(scope="module")
def tn():
    if not cuda_ok():
        pytest.skip("no CUDA device")
    import paper_2404_01817_b200 as tn
    return tn


def _rel_err(out, ref):
    return np.max(np.abs(out - ref) / np.maximum(1.0, np.abs(ref)))


@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("precision", ["f32", "f64"])
def test_transform_bit_exact(tn, name, precision):
    g = load_golden(name)
    st, cyc = tn.transform_arrays(g["nodes"], g["conns"], int(g["num_inputs"]),
                                  int(g["num_outputs"]), precision=precision)
    assert np.array_equal(cyc, g["cyclic"])
    assert np.array_equal(st.order, g["order"], equal_nan=True)
    ok = np.setdiff1d(np.arange(g["nodes"].shape[0]), g["cyclic"])
    assert np.array_equal(st.input_rows[ok], g["input_rows"][ok])
    assert np.array_equal(st.output_rows[ok], g["output_rows"][ok])
    if "incoming" in g:
        assert np.array_equal(st.incoming, g["incoming"], equal_nan=True)


@pytest.mark.parametrize("name", CASES)
def test_forward_f64_matches_reference(tn, name):
    g = load_golden(name)
    ok = np.setdiff1d(np.arange(g["nodes"].shape[0]), g["cyclic"])
    st, cyc = tn.transform_arrays(g["nodes"][ok], g["conns"][ok], int(g["num_inputs"]),
                                  int(g["num_outputs"]), precision="f64")
    assert cyc.size == 0
    out = tn.forward_arrays(st, None, g["inputs"][ok])
    np.testing.assert_allclose(out, g["outputs"][ok], rtol=1e-9, atol=1e-9)


@pytest.mark.parametrize("name,tol", [("forward_cfg2_T.npz", 1e-5), ("forward_small.npz", 1e-5),
                                      ("forward_cfg2_M.npz", 1e-5), ("corpus.npz", 1e-5)])
def test_forward_f32_matches_reference(tn, name, tol):
    g = load_golden(name)
    ok = np.setdiff1d(np.arange(g["nodes"].shape[0]), g["cyclic"])
    st, _ = tn.transform_arrays(g["nodes"][ok], g["conns"][ok], int(g["num_inputs"]),
                                int(g["num_outputs"]), layout="standard")
    x = g["inputs_f32"][ok] if "inputs_f32" in g else g["inputs"][ok].astype(np.float32)
    ref = g["outputs"][ok]
    for variant in (0, 1, 2, 4, 8):
        out = tn.forward_arrays(st, None, x, variant=variant)
        assert _rel_err(out, ref) <= tol, (variant, _rel_err(out, ref))
    ni = int(g["num_inputs"])
    if ni <= 32 and ni % 4 == 0:
        import torch
        sp, _ = tn.transform_arrays(g["nodes"][ok], g["conns"][ok], ni, int(g["num_outputs"]), layout="tc")
        assert sp.precision & tn.inference.FMT_TC
        out = tn.forward_device(sp, torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).cuda(),
                                variant=tn.inference.V_TC).cpu().numpy()
        assert _rel_err(out, ref) <= tol, ("tc", _rel_err(out, ref))


def test_tile_variants_bitwise_equal_and_chunk_invariant(tn):
    import torch
    from oracle.arrayneat_oracle import synthetic_population
    nodes, conns = synthetic_population(40, 128, 512, 32, 8, seed=77)
    st, _ = tn.transform_arrays(nodes, conns, 32, 8, layout="standard")
    x = torch.randn(40, 1000, 32, device="cuda", generator=torch.Generator("cuda").manual_seed(1))
    outs = [tn.forward_device(st, x, variant=v) for v in (1, 2, 4)]
    assert torch.equal(outs[0], outs[1]) and torch.equal(outs[1], outs[2])
    # genome chunks and input chunks give bitwise identical results
    part = torch.cat([tn.forward_device(st.select(slice(a, a + 13)), x[a:a + 13].contiguous(), variant=2)
                      for a in range(0, 40, 13)])
    assert torch.equal(part, outs[1])
    half = tn.forward_device(st, x[:, 300:700].contiguous(), variant=2)
    assert torch.equal(half, outs[1][:, 300:700])


def test_tc_chunk_invariant_and_matches_standard(tn):
    """Tensor-core programs: genome chunks / input sub-ranges / shared inputs
    give bitwise identical rows; results agree with the standard layout to fp32;
    every genome of the tanh/sum population takes the tensor-core format."""
    import torch
    from oracle.arrayneat_oracle import synthetic_population
    nodes, conns = synthetic_population(40, 128, 512, 32, 8, seed=78)
    sp, _ = tn.transform_arrays(nodes, conns, 32, 8, layout="tc")
    st, _ = tn.transform_arrays(nodes, conns, 32, 8, layout="standard")
    assert (sp._cache["modes"] == tn.inference.MODE_TC).all()
    x = torch.randn(40, 1000, 32, device="cuda", generator=torch.Generator("cuda").manual_seed(2))
    full = tn.forward_device(sp, x)
    part = torch.cat([tn.forward_device(sp.select(slice(a, a + 13)), x[a:a + 13].contiguous())
                      for a in range(0, 40, 13)])
    assert torch.equal(part, full)
    half = tn.forward_device(sp, x[:, 256:700].contiguous())
    assert torch.equal(half, full[:, 256:700])
    ref = tn.forward_device(st, x, variant=2)
    assert (full - ref).abs().max().item() <= 2e-5  # both within 1e-5 of the float64 reference
    shared = tn.forward_device(sp, x[0].contiguous(), shared=True)
    assert torch.equal(shared[0], full[0])


@pytest.mark.parametrize("ni", [4, 8, 12, 28, 32])
def test_tc_input_widths(tn, ni):
    """Input counts below the 32-wide K plane (zero-filled by the TMA box) and
    ragged batches, against the oracle."""
    import torch
    from oracle import arrayneat_oracle as orc
    nodes, conns = orc.synthetic_population(12, 48 + ni, 160, ni, 3, seed=100 + ni, min_conns=20,
                                            max_conns_drawn=150)
    sp, cyc = tn.transform_arrays(nodes, conns, ni, 3, layout="tc")
    assert cyc.size == 0
    x = np.random.default_rng(ni).standard_normal((12, 300, ni), dtype=np.float32)
    out = tn.forward_device(sp, torch.from_numpy(x).cuda()).cpu().numpy()
    for p in range(12):
        tr = orc.transform_genome(nodes[p], conns[p], ni, 3)
        ref = orc.forward_genome(nodes[p], tr, x[p].astype(np.float64))
        assert _rel_err(out[p], ref) <= 1e-5, (p, _rel_err(out[p], ref))


def test_tc_nonfinite_and_extreme_inputs_match_standard(tn):
    """Rows with an infinite input, or a max |x| outside the digit scaling
    range, take the exact path: outputs equal the standard layout's to fp32,
    NaN/inf positions included."""
    import torch
    from oracle.arrayneat_oracle import synthetic_population
    nodes, conns = synthetic_population(6, 128, 512, 32, 8, seed=79)
    sp, _ = tn.transform_arrays(nodes, conns, 32, 8, layout="tc")
    st, _ = tn.transform_arrays(nodes, conns, 32, 8, layout="standard")
    x = torch.randn(6, 600, 32, device="cuda", generator=torch.Generator("cuda").manual_seed(3))
    x[1, 17, 5] = float("inf")
    x[4, 300, 0] = -float("inf")
    x[2, 5] *= 1e-20  # tiny row (exponent < -62)
    x[3, 9, 7] = 1e30  # huge entry (exponent > 62)
    x[5, 11] = 0.0  # all-zero row
    a = tn.forward_device(sp, x)
    b = tn.forward_device(st, x, variant=2)
    assert torch.equal(torch.isnan(a), torch.isnan(b))
    fin = ~torch.isnan(a)
    assert torch.equal(torch.isinf(a), torch.isinf(b))
    fin = fin & ~torch.isinf(a)
    assert (a[fin] - b[fin]).abs().max().item() <= 2e-5


def test_tc_mixed_population_routes_standard_programs(tn):
    """Genomes the tensor-core format cannot take (non-sum aggregations) get
    standard programs in the same buffer and run on the tile kernel."""
    import torch
    from oracle import arrayneat_oracle as orc
    nt, ct = orc.synthetic_population(8, 128, 512, 32, 8, seed=80)
    nm, cm = orc.synthetic_population(8, 128, 512, 32, 8, seed=81, variant="M")
    nodes, conns = np.concatenate([nt, nm]), np.concatenate([ct, cm])
    sp, cyc = tn.transform_arrays(nodes, conns, 32, 8, layout="tc")
    assert cyc.size == 0
    modes = sp._cache["modes"]
    assert (modes[:8] == tn.inference.MODE_TC).all() and (modes[8:] != tn.inference.MODE_TC).any()
    x = np.random.default_rng(5).standard_normal((16, 512, 32), dtype=np.float32)
    out = tn.forward_device(sp, torch.from_numpy(x).cuda()).cpu().numpy()
    for p in range(16):
        tr = orc.transform_genome(nodes[p], conns[p], 32, 8)
        ref = orc.forward_genome(nodes[p], tr, x[p].astype(np.float64))
        assert _rel_err(out[p], ref) <= 1e-5, (p, _rel_err(out[p], ref))


def test_config2_shapes_against_oracle_sampled(tn):
    """Full config-2 genome shapes and B=4096; a sampled set of genomes is
    checked against the oracle (float64) within the fp32 bound."""
    import torch
    from oracle import arrayneat_oracle as orc
    nodes, conns = orc.synthetic_population(64, 128, 512, 32, 8, seed=20261018)
    st, cyc = tn.transform_arrays(nodes, conns, 32, 8)
    assert cyc.size == 0
    x = np.random.default_rng(20261019).standard_normal((64, 4096, 32), dtype=np.float32)
    out = tn.forward_device(st, torch.from_numpy(x).cuda()).cpu().numpy()
    for p in (0, 17, 63):
        tr = orc.transform_genome(nodes[p], conns[p], 32, 8)
        ref = orc.forward_genome(nodes[p], tr, x[p].astype(np.float64))
        assert _rel_err(out[p], ref) <= 1e-5


def test_cycle_and_errors(tn):
    g = load_golden("forward_small.npz")
    with pytest.raises(tn.CycleDetected) as exc:
        tn.transform_population_stacked(
            tn.PopulationTensors(g["nodes"], g["conns"], None, None, 2, 1))
    assert exc.value.genome_indices == [47]
    nodes = g["nodes"][:2].copy()
    nodes[0, 2, 4] = 9.0  # unknown activation code on a live node
    st, _ = tn.transform_arrays(nodes, g["conns"][:2], 2, 1)
    if not np.isnan(nodes[0, 2, 0]):
        with pytest.raises(tn.ConfigError):
            tn.forward_arrays(st, None, np.zeros((2, 1, 2)))


def test_single_genome_wrappers(tn):
    g = load_golden("forward_small.npz")
    from paper_2404_01817_b200.genome import GenomeTensors
    genome = GenomeTensors(g["nodes"][3], g["conns"][3], 2, 1)
    t = tn.transform(genome, precision="f64")
    y = tn.forward(t, None, g["inputs"][3][0])
    np.testing.assert_allclose(y, g["outputs"][3][0], atol=1e-9)
    yb = tn.forward_batch(t, None, g["inputs"][3])
    np.testing.assert_allclose(yb, g["outputs"][3], atol=1e-9)
    with pytest.raises(tn.InvalidInput):
        tn.forward(t, None, [1.0, np.nan])
    with pytest.raises(tn.InvalidInput):
        tn.forward(t, None, [1.0, 2.0, 3.0])


def test_host_pipeline_matches_device(tn):
    """The end-to-end host path (pinned host tensors, chunked H2D / kernel /
    D2H on three streams) returns exactly the device-resident result, for
    several chunk sizes and both public entry points."""
    import torch
    from oracle.arrayneat_oracle import synthetic_population
    from paper_2404_01817_b200.inference import _host_forward_pipelined
    nodes, conns = synthetic_population(37, 128, 512, 32, 8, seed=81)
    st, _ = tn.transform_arrays(nodes, conns, 32, 8)
    x = torch.randn(37, 700, 32, generator=torch.Generator().manual_seed(4)).pin_memory()
    ref = tn.forward_device(st, x.cuda()).cpu()
    for chunk in (1 << 20, 3 << 20, 1 << 30):
        out = torch.empty((37, 700, 8), dtype=torch.float32).pin_memory()
        got = _host_forward_pipelined(st, x, out, chunk_bytes=chunk)
        assert torch.equal(got, ref), chunk
    assert torch.equal(tn.forward_arrays(st, None, x), ref)
    np.testing.assert_array_equal(tn.forward_arrays(st, None, x.numpy()), ref.numpy().astype(np.float64))


def test_level_synchronous_programs_equal_exact_order_programs(tn):
    """Programs built from the level-synchronous Kahn (default) and from the
    reference's one-node-per-step Kahn (with_order=True) evaluate bitwise
    identically; the lazily computed order equals the eager one."""
    import torch
    from oracle.arrayneat_oracle import synthetic_population
    for variant in ("T", "M"):
        nodes, conns = synthetic_population(50, 128, 512, 32, 8, seed=82, variant=variant)
        a, _ = tn.transform_arrays(nodes, conns, 32, 8)
        b, _ = tn.transform_arrays(nodes, conns, 32, 8, with_order=True)
        assert a.order_dev is None and b.order_dev is not None
        x = torch.randn(50, 300, 32, device="cuda", generator=torch.Generator("cuda").manual_seed(5))
        assert torch.equal(tn.forward_device(a, x), tn.forward_device(b, x))
        assert np.array_equal(a.order, b.order, equal_nan=True)


@pytest.mark.parametrize("name", ["forward_dupes_n12.npz", "forward_dupes_n80.npz"])
def test_duplicate_pairs_match_reference(tn, name):
    """Repeated (in, out) pairs: last row wins in incoming / the forward, and
    with max_nodes <= 64 the genome reads as cyclic -- as the reference."""
    g = load_golden(name)
    st, cyc = tn.transform_arrays(g["nodes"], g["conns"], 2, 1, precision="f64")
    assert np.array_equal(cyc, g["cyclic"])
    assert np.array_equal(st.order, g["order"], equal_nan=True)
    assert np.array_equal(st.incoming, g["incoming"], equal_nan=True)
    ok = np.setdiff1d(np.arange(g["nodes"].shape[0]), g["cyclic"])
    if ok.size:
        st2, _ = tn.transform_arrays(g["nodes"][ok], g["conns"][ok], 2, 1, precision="f64")
        out = tn.forward_arrays(st2, None, g["inputs"][ok])
        np.testing.assert_allclose(out, g["outputs"][ok], rtol=1e-9, atol=1e-9)


def test_large_host_uploads_staged(tn):
    """Pageable host arrays above the staging threshold go through the pinned
    double buffer (device.to_device): bitwise the same tensor, and the same
    programs as a transform of device-resident genomes.  Subsets keep the
    host slot counts (launch plans without read-back)."""
    import torch
    from oracle.arrayneat_oracle import synthetic_population
    from paper_2404_01817_b200.device import _STAGE_BYTES, to_device
    big = np.random.default_rng(9).standard_normal((3 * _STAGE_BYTES) // 8 + 123)
    assert torch.equal(to_device(big, torch.float64).cpu(), torch.from_numpy(big))
    nodes, conns = synthetic_population(40, 128, 512, 32, 8, seed=82)
    reps = (2 * _STAGE_BYTES) // conns[:1].nbytes // 40 + 1
    nodes, conns = np.tile(nodes, (reps, 1, 1)), np.tile(conns, (reps, 1, 1))
    assert conns.nbytes > 2 * _STAGE_BYTES
    a, _ = tn.transform_arrays(nodes, conns, 32, 8)
    b, _ = tn.transform_arrays(torch.from_numpy(nodes).cuda(), torch.from_numpy(conns).cuda(), 32, 8)
    assert torch.equal(a.program[:, :32], b.program[:, :32])  # headers (the unused tails are not written)
    xa = torch.randn(a.size, 8, 32, device="cuda")
    assert torch.equal(tn.forward_device(a, xa), tn.forward_device(b, xa))
    sub = a.select(slice(5, 17))
    np.testing.assert_array_equal(sub._cache["slots"], a._cache["slots"][5:17])
    x = torch.randn(12, 300, 32, device="cuda")
    assert torch.equal(tn.forward_device(sub, x), tn.forward_device(b.select(slice(5, 17)), x))


def _split0_groups(st) -> int:
    """Number of GRP_SPLIT0 sum groups in the programs (GroupRec.cls bit 4)."""
    from paper_2404_01817_b200 import _native  # noqa: F401
    prog = st.program.cpu().numpy()
    hdr = prog[:, :32].view(np.int32)
    off = 32 + ((2 * st.num_outputs + 15) // 16) * 16
    total = 0
    for p in range(prog.shape[0]):
        g = prog[p, off:off + 16 * hdr[p, 7]].reshape(-1, 16)
        total += int(((g[:, 1] & 4) != 0).sum())
    return total


@pytest.mark.parametrize("precision,tol", [("f64", 1e-9), ("f32", 1e-5)])
def test_split_groups_every_kernel(tn, precision, tol):
    """Groups of 3 whose longest list spills into the spare column
    (GRP_SPLIT0) evaluate correctly in the tile kernel (B >= 192) and the warp
    kernel (variant 8; the fused-fitness and cart-pole passes share its
    indexing), in both precisions."""
    import torch
    from oracle import arrayneat_oracle as orc
    nodes, conns = orc.synthetic_population(24, 128, 512, 16, 4, seed=91, variant="M", min_conns=200,
                                            max_conns_drawn=400)
    st, cyc = tn.transform_arrays(nodes, conns, 16, 4, precision=precision)
    assert cyc.size == 0
    assert _split0_groups(st) > 0
    dt = np.float64 if precision == "f64" else np.float32
    x = np.random.default_rng(92).standard_normal((24, 256, 16)).astype(dt)
    refs = [orc.forward_genome(nodes[p], orc.transform_genome(nodes[p], conns[p], 16, 4), x[p].astype(np.float64))
            for p in range(24)]
    for variant in (0, 8):
        out = tn.forward_device(st, torch.from_numpy(x).cuda(), variant=variant).cpu().numpy()
        for p in range(24):
            assert _rel_err(out[p], refs[p]) <= tol, (variant, p)


def test_fused_fitness_epilogue_matches_outputs(tn):
    """The device-planned forward's fused epilogue (sum of each genome's squared
    outputs, float atomics) equals the sum over the returned outputs; populations
    that plan on the host reduce the outputs instead -- same contract."""
    import torch
    from oracle import arrayneat_oracle as orc
    for variant, pop in (("T", 300), ("M", 40)):
        nodes, conns = orc.synthetic_population(pop, 128, 512, 32, 8, seed=90 + pop, variant=variant)
        st, _ = tn.transform_arrays(nodes, conns, 32, 8, sync=False)
        x = torch.randn(pop, 777, 32, device="cuda", generator=torch.Generator("cuda").manual_seed(9))
        sq = torch.zeros(pop, device="cuda")
        out = tn.forward_device(st, x, sq_sum=sq)
        ref = out.double().square().sum(dim=(1, 2))
        torch.testing.assert_close(sq.double(), ref, rtol=2e-6, atol=1e-3)


def test_device_plan_classes_cover_population(tn):
    """The device plan puts every genome in exactly one class (the right one for
    its program), and the planned forward equals the host-planned one bit for
    bit (same kernels, same per-genome work)."""
    import torch
    from oracle import arrayneat_oracle as orc
    nodes, conns = orc.synthetic_population(200, 128, 512, 32, 8, seed=93)
    nm, cm = orc.synthetic_population(30, 128, 512, 32, 8, seed=94, variant="M")
    nodes, conns = np.concatenate([nodes, nm]), np.concatenate([conns, cm])
    st, _ = tn.transform_arrays(nodes, conns, 32, 8)
    counts = tn.inference.tc_plan_counts(st)
    ids = st._cache["tcplan"][0].view(tn.inference.TC_NCLASS, -1).cpu().numpy()
    got = np.concatenate([ids[c, :counts[c]] for c in range(tn.inference.TC_NCLASS)])
    assert np.array_equal(np.sort(got), np.arange(st.size))
    slots, se, modes = tn.inference._host_dims(st)
    nb = (se[:, 0] + 15) // 16 * 16
    for c in range(tn.inference.TC_NCLASS):
        g = ids[c, :counts[c]]
        assert np.unique(g).size == g.size
        if c < 5:
            lo, hi = (0, 32, 48, 64, 96, 128)[c], (32, 48, 64, 96, 128)[c]
            assert np.all((modes[g] == tn.inference.MODE_TC) & ((nb[g] > lo) | (c == 0)) & (nb[g] <= hi)
                          & (se[g, 1] <= 512)), c
    assert counts[6] == int((st._cache["modes"] != tn.inference.MODE_TC).sum())
    x = torch.randn(st.size, 600, 32, device="cuda", generator=torch.Generator("cuda").manual_seed(10))
    st._cache["tc_host_plan"] = False
    planned = tn.forward_device(st, x)
    st._cache["tc_host_plan"] = True
    hosted = tn.forward_device(st, x)
    assert torch.equal(planned, hosted)


def test_unpruned_wide_classes_match_oracle(tn):
    """Unpruned programs of genomes with up to 120 hidden nodes fill every device-plan
    class: MMA widths 32 / 48 / 64, the 96 class (two warpgroups sharing one TMEM
    slot), the 128 class (one warpgroup per CTA) and standard programs (> 128 steps).
    Genomes of each populated class match the oracle at 1e-5."""
    import torch
    from oracle import arrayneat_oracle as orc
    nodes, conns = orc.synthetic_population(160, 160, 512, 32, 8, seed=95)
    st, _ = tn.transform_arrays(nodes, conns, 32, 8, prune=False)
    counts = tn.inference.tc_plan_counts(st)
    assert (counts[[0, 1, 2, 3, 4]] > 0).all(), counts
    ids = st._cache["tcplan"][0].view(tn.inference.TC_NCLASS, -1).cpu().numpy()
    x = torch.randn(st.size, 384, 32, device="cuda", generator=torch.Generator("cuda").manual_seed(12))
    out = tn.forward_device(st, x).cpu().numpy()
    xs = x.cpu().numpy().astype(np.float64)
    for c in range(tn.inference.TC_NCLASS):
        for p in ids[c, :counts[c]][:4]:
            tr = orc.transform_genome(nodes[p], conns[p], 32, 8)
            ref = orc.forward_genome(nodes[p], tr, xs[p])
            err = np.max(np.abs(out[p] - ref) / np.maximum(1.0, np.abs(ref)))
            assert err <= 1e-5, (c, int(p), float(err))


def test_back_to_back_steps_keep_stream_order(tn):
    """Transform + device-planned forward steps enqueued back to back with no host
    synchronisation (the bench's step; the class launches are programmatic
    dependent launches and the caching allocator hands the next transform the
    memory of the previous programs) give exactly the isolated results."""
    import torch
    from oracle import arrayneat_oracle as orc
    pops = [orc.synthetic_population(300, 128, 512, 32, 8, seed=s) for s in (96, 97)]
    x = torch.randn(300, 512, 32, device="cuda", generator=torch.Generator("cuda").manual_seed(13))
    refs = []
    for nodes, conns in pops:
        st, _ = tn.transform_arrays(nodes, conns, 32, 8)
        refs.append(tn.forward_device(st, x).clone())
        del st
    torch.cuda.synchronize()
    nd = [(torch.from_numpy(n).cuda(), torch.from_numpy(c).cuda()) for n, c in pops]
    outs = []
    for k in range(6):
        st, _ = tn.transform_arrays(*nd[k % 2], 32, 8, sync=False)
        outs.append(tn.forward_device(st, x))
        del st
    torch.cuda.synchronize()
    for k, o in enumerate(outs):
        assert torch.equal(o, refs[k % 2]), k
