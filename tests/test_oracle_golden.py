"""Pin the CPU oracle against golden vectors produced by the reference itself.

The oracle (oracle/arrayneat_oracle.py) is only trusted because these pass:
every number compared here came out of the unmodified reference
(tests/golden/make_goldens.py).
"""

from __future__ import annotations

import math

import numpy as np
import pytest

from conftest import load_golden
from oracle import arrayneat_oracle as orc


def test_rng_uniforms_and_normals_match_reference_bits():
    g = load_golden("rng.npz")
    for idx, row in enumerate(g["paths"]):
        seed, plen = int(row[0]), int(row[1])
        path = tuple(int(t) for t in row[2:2 + plen])
        s = orc.Stream(orc.stream_key(seed, *path))
        assert np.array_equal(s.uniforms(37), g[f"u_{idx}"])          # exact
        np.testing.assert_allclose(s.normals(19), g[f"n_{idx}"], rtol=0, atol=1e-15)
        assert np.array_equal(s.uniforms(5), g[f"u2_{idx}"])


def test_rng_split_and_sparse_cells_match_reference():
    g = load_golden("rng.npz")
    keys = [orc.stream_key(99, 4, 2, i) for i in range(6)]
    streams = [orc.Stream(k) for k in keys]
    assert np.array_equal(np.stack([s.uniforms(3) for s in streams]), g["split_u"])
    base = 3
    u = [streams[r].uniform_cell(base, c) for r, c in zip(g["at_rows"], g["at_cols"])]
    assert np.array_equal(np.array(u), g["split_uat"])
    base = 13
    z = [streams[r].normal_cell(base, 10, c) for r, c in zip(g["at_rows"], g["at_cols"])]
    np.testing.assert_allclose(z, g["split_nat"], rtol=0, atol=1e-15)
    for s in streams:
        s.counter = 33
    assert np.array_equal(np.stack([s.uniforms(2) for s in streams]), g["split_after"])


@pytest.mark.parametrize("name", ["forward_small.npz", "forward_cfg2_T.npz", "forward_cfg2_M.npz",
                                  "corpus.npz", "forward_dupes_n12.npz", "forward_dupes_n80.npz"])
def test_transform_order_matches_reference(name):
    g = load_golden(name)
    n_in, n_out = int(g["num_inputs"]), int(g["num_outputs"])
    cyc = set(int(c) for c in g["cyclic"])
    for p in range(g["nodes"].shape[0]):
        tr = orc.transform_genome(g["nodes"][p], g["conns"][p], n_in, n_out)
        assert tr["cyclic"] == (p in cyc)
        ref = g["order"][p]
        assert np.array_equal(orc.order_array(tr, ref.shape[0]), ref, equal_nan=True)
        assert tr["input_rows"] == list(g["input_rows"][p])
        assert tr["output_rows"] == list(g["output_rows"][p])
        if "incoming" in g:
            assert np.array_equal(orc.incoming_dense(tr, ref.shape[0]), g["incoming"][p],
                                  equal_nan=True)


@pytest.mark.parametrize("name", ["forward_small.npz", "forward_cfg2_T.npz", "forward_cfg2_M.npz",
                                  "corpus.npz", "forward_dupes_n12.npz", "forward_dupes_n80.npz"])
def test_forward_matches_reference(name):
    g = load_golden(name)
    n_in, n_out = int(g["num_inputs"]), int(g["num_outputs"])
    cyc = set(int(c) for c in g["cyclic"])
    for p in range(g["nodes"].shape[0]):
        if p in cyc:
            continue
        tr = orc.transform_genome(g["nodes"][p], g["conns"][p], n_in, n_out)
        out = orc.forward_genome(g["nodes"][p], tr, g["inputs"][p])
        ref = g["outputs"][p]
        # sum order differs (reference: pairwise nansum; oracle: sequential)
        np.testing.assert_allclose(out, ref, rtol=1e-9, atol=1e-9)


def test_distance_matches_reference():
    g = load_golden("corpus.npz")
    nodes, conns = g["nodes"], g["conns"]
    cd, ch = float(g["c_disjoint"]), float(g["c_homologous"])
    for other, key in ((0, "dist_to_0"), (7, "dist_to_7")):
        d = [orc.distance_genome(nodes[p], conns[p], nodes[other], conns[other], cd, ch)
             for p in range(nodes.shape[0])]
        assert np.array_equal(np.array(d), g[key])      # bit-exact: same sum order
    d = [orc.distance_genome(nodes[p], conns[p], nodes[100 + p], conns[100 + p], cd, ch)
         for p in range(100)]
    assert np.array_equal(np.array(d), g["dist_pair"])


def test_synthetic_generator_is_valid_and_acyclic():
    nodes, conns = orc.synthetic_population(8, 128, 512, 32, 8, seed=3)
    for p in range(8):
        tr = orc.transform_genome(nodes[p], conns[p], 32, 8)
        assert not tr["cyclic"]
        live = ~np.isnan(conns[p, :, 0])
        assert 256 <= live.sum() <= 512
        assert not math.isnan(nodes[p, 39, 0])
