"""Generate golden vectors by running the reference ``arrayneat`` itself.

Run in the build container (the reference only exists there):

    python tests/golden/make_goldens.py

It imports the unmodified reference from ``oracle/_ref`` (built by
``oracle/build_ref.sh``) or ``/root/reference/pkg/src`` and writes small
``.npz`` fixtures next to this script.  The fixtures are committed; the GPU box
never needs the reference.  Every array here is a reference OUTPUT on seeded
inputs, so the oracle and the CUDA path are both checked against the
reference's own numbers.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
for cand in (os.path.join(REPO, "oracle", "_ref"), "/root/reference/pkg/src"):
    if os.path.isdir(os.path.join(cand, "arrayneat")):
        sys.path.insert(0, cand)
        break
sys.path.insert(0, REPO)

import arrayneat as an  # noqa: E402  (the reference)
from arrayneat import evolution as an_evo  # noqa: E402
from arrayneat.genome import init_arrays  # noqa: E402
from arrayneat.inference import forward_arrays, transform_arrays  # noqa: E402

from oracle.arrayneat_oracle import synthetic_population  # noqa: E402


def _save(name: str, **arrays) -> None:
    path = os.path.join(HERE, name)
    np.savez_compressed(path, **arrays)
    size = os.path.getsize(path)
    print(f"wrote {name} ({size / 1024:.1f} KiB)")


# -- random valid genomes through the reference's public edit API -------------------


def _random_genome(seed: int, config, n_ops: int) -> "an.GenomeTensors":
    """Same recipe as the reference's tests/conftest.py:91-141 (public ops only)."""
    rng = np.random.default_rng(seed)
    g = an.init_genome(config, an.RngStream(seed).child(0, 0, 0))
    nxt = config.inputs + config.outputs
    io = config.inputs + config.outputs

    def keys(gg):
        k = gg.nodes[:, 0]
        return [int(x) for x in k[~np.isnan(k)]]

    def pairs(gg):
        c = gg.conns
        live = ~np.isnan(c[:, 0])
        return [(int(i), int(o)) for i, o in c[live][:, [0, 1]]]

    def reaches(gg, s, d):
        adj: dict[int, list[int]] = {}
        for i, o in pairs(gg):
            adj.setdefault(i, []).append(o)
        seen, todo = set(), [s]
        while todo:
            x = todo.pop()
            if x == d:
                return True
            if x in seen:
                continue
            seen.add(x)
            todo.extend(adj.get(x, []))
        return False

    for _ in range(n_ops):
        ks, ps = keys(g), pairs(g)
        hidden = [k for k in ks if k >= io]
        choice = rng.integers(0, 6)
        if choice == 0 and np.isnan(g.nodes).all(axis=1).any():
            g = an.add_node(g, an.NodeRow(nxt, float(rng.normal()), 1.0, 0, int(rng.integers(0, 4))))
            nxt += 1
        elif choice == 1 and hidden:
            g = an.remove_node(g, int(rng.choice(hidden)))
        elif choice == 2:
            srcs = [k for k in ks if not (config.inputs <= k < io)]
            dsts = [k for k in ks if k >= config.inputs]
            cands = [(u, v) for u in srcs for v in dsts if (u, v) not in ps and not reaches(g, v, u)]
            if cands and np.isnan(g.conns).all(axis=1).any():
                u, v = cands[rng.integers(0, len(cands))]
                g = an.add_conn(g, an.ConnRow(u, v, 1.0, float(rng.normal())))
        elif choice == 3 and ps:
            i, o = ps[rng.integers(0, len(ps))]
            g = an.remove_conn(g, i, o)
        elif choice == 4 and ks:
            k = int(rng.choice(ks))
            attr = int(rng.integers(0, 4))
            val = float(rng.normal()) if attr < 2 else float(rng.integers(0, 4))
            g = an.set_node_attr(g, k, attr, val)
        elif choice == 5 and ps:
            i, o = ps[rng.integers(0, len(ps))]
            attr = int(rng.integers(0, 2))
            val = float(rng.integers(0, 2)) if attr == 0 else float(rng.normal())
            g = an.set_conn_attr(g, i, o, attr, val)
    return g


def _transform_forward_case(nodes, conns, inputs, n_in, n_out):
    stacked, cyclic = transform_arrays(nodes, conns, n_in, n_out)
    out = np.full(inputs.shape[:2] + (n_out,), np.nan)
    ok = np.setdiff1d(np.arange(nodes.shape[0]), cyclic)
    if ok.size:
        st2, cyc2 = transform_arrays(nodes[ok], conns[ok], n_in, n_out)
        assert cyc2.size == 0
        out[ok] = forward_arrays(st2, an.DEFAULT_REGISTRY, inputs[ok])
    return dict(nodes=nodes, conns=conns, inputs=inputs, order=stacked.order,
                incoming=stacked.incoming, input_rows=stacked.input_rows,
                output_rows=stacked.output_rows, cyclic=cyclic, outputs=out,
                num_inputs=np.int64(n_in), num_outputs=np.int64(n_out))


def make_forward_goldens() -> None:
    # (1) small random genomes built through the public ops (mixed act/agg codes)
    cfg = an.NeatConfig(seed=0, pop_size=20, inputs=2, outputs=1, max_nodes=12,
                        max_conns=24, generation_limit=10, max_species=4)
    gs = [_random_genome(s, cfg, 40) for s in range(48)]
    nodes = np.stack([g.nodes for g in gs])
    conns = np.stack([g.conns for g in gs])
    # genome 47 gets an enabled 2-cycle so the cyclic path is pinned too
    g = an.init_genome(cfg, an.RngStream(7).child(0, 0, 0))
    g = an.add_node(g, an.NodeRow(3, 0.1, 1.0, 0, 1))
    g = an.add_node(g, an.NodeRow(4, -0.2, 1.0, 0, 1))
    g = an.add_conn(g, an.ConnRow(3, 4, 1.0, 0.5))
    g = an.add_conn(g, an.ConnRow(4, 3, 1.0, 0.25))
    nodes[47], conns[47] = g.nodes, g.conns
    inputs = np.random.default_rng(5).standard_normal((48, 6, 2))
    _save("forward_small.npz", **_transform_forward_case(nodes, conns, inputs, 2, 1))

    # (2) config-2 shapes (I=32, O=8, 128/512), tanh/sum and mixed variants
    for variant in ("T", "M"):
        nodes, conns = synthetic_population(16, 128, 512, 32, 8, seed=20261018, variant=variant)
        x = np.random.default_rng(20261019).standard_normal((16, 24, 32), dtype=np.float32)
        case = _transform_forward_case(nodes, conns, x.astype(np.float64), 32, 8)
        case["inputs_f32"] = x
        case.pop("incoming")  # (16,128,128) is large and derivable from conns
        _save(f"forward_cfg2_{variant}.npz", **case)

    # (3) a mutated corpus (reference mutate_arrays, test_acceptance.py:36-65 recipe)
    ccfg = an.NeatConfig(
        inputs=3, outputs=2, max_nodes=32, max_conns=64, pop_size=200,
        node_add=0.5, node_delete=0.1, conn_add=0.6, conn_delete=0.1,
        bias_mutate_rate=0.8, bias_replace_rate=0.1,
        response_init_std=0.3, response_mutate_rate=0.3, response_mutate_power=0.3,
        weight_mutate_rate=0.8, weight_replace_rate=0.1,
        activation_options=("identity", "tanh", "sigmoid", "relu"),
        activation_replace_rate=0.3,
        aggregation_options=("sum", "product", "max", "mean"),
        aggregation_replace_rate=0.3)
    streams = an.RngStream(2024).child(0, 0).split(np.arange(ccfg.pop_size))
    nodes, conns = init_arrays(ccfg, streams)
    alloc = an.NodeKeyAllocator(ccfg.inputs + ccfg.outputs)
    for rnd in range(8):
        st = an.RngStream(2024).child(rnd + 1, 2).split(np.arange(ccfg.pop_size))
        base = alloc.reserve(ccfg.pop_size)
        keys = np.arange(base, base + ccfg.pop_size, dtype=np.float64)
        nodes, conns, _ = an_evo.mutate_arrays(nodes, conns, ccfg, st, keys)
    inputs = np.random.default_rng(11).standard_normal((200, 5, 3))
    case = _transform_forward_case(nodes, conns, inputs, 3, 2)
    case.pop("incoming")
    # distances of every genome to genome 0 and to genome 7 (evolution.py:425-488)
    d0 = an_evo.distance_arrays(nodes, conns, nodes[:1], conns[:1], ccfg)
    d7 = an_evo.distance_arrays(nodes, conns, nodes[7:8], conns[7:8], ccfg)
    dpair = an_evo.distance_arrays(nodes[:100], conns[:100], nodes[100:], conns[100:], ccfg)
    case.update(dist_to_0=d0, dist_to_7=d7, dist_pair=dpair,
                c_disjoint=np.float64(ccfg.compatibility_disjoint),
                c_homologous=np.float64(ccfg.compatibility_homologous))
    _save("corpus.npz", **case)


def make_rng_goldens() -> None:
    cases = []
    out = {}
    paths = [(0, ()), (123, (0, 0, 0)), (2024, (3, 2)), (7, (-1, 5)), (2 ** 40 + 3, (11,))]
    for idx, (seed, path) in enumerate(paths):
        s = an.RngStream(seed, path)
        out[f"u_{idx}"] = s.uniforms(37)
        out[f"n_{idx}"] = s.normals(19)
        out[f"u2_{idx}"] = s.uniforms(5)
        cases.append((seed, len(path)) + tuple(path) + (0,) * (3 - len(path)))
    # batched split streams + sparse cells (rng.py:77-82, 114-134)
    b = an.RngStream(99).child(4, 2).split(np.arange(6))
    out["split_u"] = b.uniforms(3)
    rows = np.array([0, 2, 5, 5, 1])
    cols = np.array([0, 7, 3, 9, 4])
    out["split_uat"] = b.uniforms_at(10, rows, cols)
    out["split_nat"] = b.normals_at(10, rows, cols)
    out["split_after"] = b.uniforms(2)
    out["at_rows"], out["at_cols"] = rows, cols
    out["paths"] = np.array(cases, dtype=np.int64)
    _save("rng.npz", **out)


if __name__ == "__main__":
    make_rng_goldens()
    make_forward_goldens()
