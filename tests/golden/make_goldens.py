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


def make_duplicate_goldens() -> None:
    """Repeated (in, out) connection pairs (a "collision" the reference does
    not reject): its dense incoming keeps the last row; with max_nodes <= 64
    the bitmask Kahn leaves the destination unready (cyclic), above 64 it does
    not (inference.py:108-141)."""
    base = np.load(os.path.join(HERE, "forward_small.npz"))
    nodes, conns = base["nodes"][:12].copy(), base["conns"][:12].copy()
    rng = np.random.default_rng(31)
    for p in range(12):
        live = np.nonzero(~np.isnan(conns[p, :, 0]))[0]
        free = np.nonzero(np.isnan(conns[p, :, 0]))[0]
        if live.size == 0 or free.size < 2:
            continue
        src = live[int(rng.integers(live.size))]
        kind = p % 4
        conns[p, free[0]] = conns[p, src]
        conns[p, free[0], 3] = float(rng.normal())
        if kind == 1:
            conns[p, free[0], 2] = 0.0      # disabled duplicate
        elif kind == 2:
            conns[p, free[1]] = conns[p, src]  # triple
            conns[p, free[1], 3] = float(rng.normal())
        elif kind == 3:
            conns[p, [src, free[0]]] = conns[p, [free[0], src]]  # duplicate in the earlier row
    inputs = np.random.default_rng(6).standard_normal((12, 5, 2))
    _save("forward_dupes_n12.npz", **_transform_forward_case(nodes, conns, inputs, 2, 1))
    wide = np.full((12, 80, 5), np.nan)
    wide[:, :nodes.shape[1]] = nodes
    _save("forward_dupes_n80.npz", **_transform_forward_case(wide, conns, inputs, 2, 1))


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


if __name__ == "__main__" and "evo" not in sys.argv and "dupes" not in sys.argv:
    make_rng_goldens()
    make_forward_goldens()
if __name__ == "__main__" and ("dupes" in sys.argv or "evo" not in sys.argv):
    make_duplicate_goldens()


# -- evolution operators --------------------------------------------------------

EVO_CFG = dict(inputs=3, outputs=2, max_nodes=32, max_conns=64, pop_size=200,
               node_add=0.5, node_delete=0.2, conn_add=0.6, conn_delete=0.2,
               bias_mutate_rate=0.8, bias_replace_rate=0.1,
               response_init_std=0.3, response_mutate_rate=0.3, response_mutate_power=0.3,
               response_replace_rate=0.05,
               weight_mutate_rate=0.8, weight_replace_rate=0.1, enabled_mutate_rate=0.05,
               activation_options=("identity", "tanh", "sigmoid", "relu"), activation_replace_rate=0.3,
               aggregation_options=("sum", "product", "max", "mean"), aggregation_replace_rate=0.3)


def make_evolution_goldens() -> None:
    from arrayneat.evolution import _crossover_into, reproduce, speciate, update_stagnation, allocate_spawns
    cfg = an.NeatConfig(**EVO_CFG)
    c = load_corpus()
    nodes, conns = c["nodes"], c["conns"]
    P = nodes.shape[0]
    out = {}
    # init_arrays
    init_rng = an.RngStream(5).child(0, 0).split(np.arange(40))
    out["init_nodes"], out["init_conns"] = init_arrays(cfg, init_rng)
    # mutate_arrays, feed-forward and recurrent
    for net in ("feedforward", "recurrent"):
        mcfg = cfg.with_overrides(network_type=net)
        st = an.RngStream(77).child(3, 2).split(np.arange(P))
        st._counter = 5  # arbitrary tape offset
        keys = np.arange(1000, 1000 + P, dtype=np.float64)
        mn, mc, added = an_evo.mutate_arrays(nodes, conns, mcfg, st, keys)
        out[f"mut_{net}_nodes"], out[f"mut_{net}_conns"], out[f"mut_{net}_added"] = mn, mc, added
        out[f"mut_{net}_counter"] = np.int64(st._counter)
    # crossover of genome i (fitter) with genome P-1-i
    st = an.RngStream(91).child(1, 2).split(np.arange(P))
    st._counter = 2
    xn, xc = nodes.copy(), conns.copy()
    _crossover_into(xn, xc, nodes[::-1].copy(), conns[::-1].copy(), st)
    out["xo_nodes"], out["xo_conns"], out["xo_counter"] = xn, xc, np.int64(st._counter)
    # speciation of the corpus from scratch and against two old species
    scfg = cfg.with_overrides(compatibility_threshold=1.2, max_species=6)
    pop = an.PopulationTensors(nodes, conns, np.full(P, -1, np.int64), np.full(P, np.nan), 3, 2)
    sp_pop, sp = speciate(pop, [], scfg)
    out["spec0_assigned"] = sp_pop.species_id
    out["spec0_keys"] = np.array([s.species_key for s in sp])
    out["spec0_reps"] = np.stack([s.representative.nodes for s in sp])
    old = [an_evo.SpeciesState(species_key=k, representative=pop.genome(g), member_indices=np.arange(1))
           for k, g in ((3, 17), (8, 101))]
    sp_pop, sp = speciate(pop, old, scfg)
    out["spec1_assigned"] = sp_pop.species_id
    out["spec1_keys"] = np.array([s.species_key for s in sp])
    out["spec1_reps_nodes"] = np.stack([s.representative.nodes for s in sp])
    # stagnation / spawns / reproduce from the from-scratch speciation with synthetic fitness
    fitness = np.round(np.random.default_rng(3).random(P) * 4.0, 2)  # ties on purpose
    sp_pop, sp = speciate(pop, [], scfg)
    surv = update_stagnation(sp, fitness, scfg)
    alloc = allocate_spawns(surv, fitness, scfg.with_overrides(pop_size=P))
    out["spawns"] = np.array([s.spawn_count for s in alloc])
    rcfg = scfg.with_overrides(pop_size=P)
    allocator = an.NodeKeyAllocator(500)
    off = reproduce(sp_pop, alloc, fitness, rcfg, an.RngStream(13).child(4), allocator)
    out["rep_nodes"], out["rep_conns"] = off.nodes, off.conns
    out["rep_fitness"] = fitness
    out["rep_next_key"] = np.int64(allocator.next_key)
    _save("evolution.npz", **out)


BIG_CFG = dict(EVO_CFG, inputs=32, outputs=8, max_nodes=128, max_conns=512, pop_size=48, conn_add=0.9,
               compatibility_threshold=2.0, max_species=5)


def make_big_evolution_goldens() -> None:
    """mutate / reproduce at max_nodes 128 / max_conns 512 on genomes with > 64
    live nodes: the reference's conn-add closure switches from the bitset
    Warshall to float32 matmul squaring above 64 live rows (evolution.py:370-390)."""
    from arrayneat.evolution import reproduce, speciate, update_stagnation, allocate_spawns
    cfg = an.NeatConfig(**BIG_CFG)
    nodes, conns = synthetic_population(160, 128, 512, 32, 8, seed=11, variant="M")
    big = np.nonzero((~np.isnan(nodes[:, :, 0])).sum(axis=1) > 64)[0][:48]
    nodes, conns = nodes[big], conns[big]
    assert nodes.shape[0] == 48
    P = nodes.shape[0]
    out = {"nodes": nodes, "conns": conns}
    for net in ("feedforward", "recurrent"):
        mcfg = cfg.with_overrides(network_type=net)
        st = an.RngStream(78).child(3, 2).split(np.arange(P))
        st._counter = 3
        keys = np.arange(1 << 21, (1 << 21) + P, dtype=np.float64)
        mn, mc, added = an_evo.mutate_arrays(nodes, conns, mcfg, st, keys)
        out[f"mut_{net}_nodes"], out[f"mut_{net}_conns"], out[f"mut_{net}_added"] = mn, mc, added
        out[f"mut_{net}_counter"] = np.int64(st._counter)
    fitness = np.round(np.random.default_rng(4).random(P) * 4.0, 1)
    pop = an.PopulationTensors(nodes, conns, np.full(P, -1, np.int64), np.full(P, np.nan), 32, 8)
    sp_pop, sp = speciate(pop, [], cfg)
    out["spec_assigned"] = sp_pop.species_id
    surv = update_stagnation(sp, fitness, cfg)
    alloc = allocate_spawns(surv, fitness, cfg)
    out["spawns"] = np.array([s.spawn_count for s in alloc])
    allocator = an.NodeKeyAllocator(1 << 22)
    off = reproduce(sp_pop, alloc, fitness, cfg, an.RngStream(14).child(4), allocator)
    out["rep_nodes"], out["rep_conns"] = off.nodes, off.conns
    out["rep_fitness"] = fitness
    out["rep_next_key"] = np.int64(allocator.next_key)
    _save("evolution_big.npz", **out)


if __name__ == "__main__" and "big" in sys.argv:
    make_big_evolution_goldens()


def load_corpus() -> dict:
    with np.load(os.path.join(HERE, "corpus.npz")) as z:
        return {k: z[k] for k in z.files}


if __name__ == "__main__":
    make_evolution_goldens()


def make_problem_goldens() -> None:
    """Fitness of mutated populations under the reference problems, plus a
    short reference XOR run (stats rows) from a fixed seed."""
    from arrayneat import problems as an_prob
    from arrayneat.runner import init_state
    out = {}
    for name, (ni, no) in {"xor": (2, 1), "regression": (1, 1), "cartpole": (4, 1)}.items():
        cfg = an.NeatConfig(inputs=ni, outputs=no, max_nodes=24, max_conns=48, pop_size=120, problem=name,
                            node_add=0.6, conn_add=0.7, bias_mutate_rate=0.8, weight_mutate_rate=0.9,
                            activation_options=("identity", "tanh", "sigmoid", "relu"),
                            activation_replace_rate=0.3)
        nodes, conns = init_arrays(cfg, an.RngStream(31).child(0, 0).split(np.arange(cfg.pop_size)))
        alloc = an.NodeKeyAllocator(ni + no)
        for rnd in range(6):
            st = an.RngStream(31).child(rnd + 1, 2).split(np.arange(cfg.pop_size))
            base = alloc.reserve(cfg.pop_size)
            nodes, conns, _ = an_evo.mutate_arrays(nodes, conns, cfg, st,
                                                   np.arange(base, base + cfg.pop_size, dtype=np.float64))
        pop = an.PopulationTensors(nodes, conns, np.full(cfg.pop_size, -1), np.full(cfg.pop_size, np.nan), ni, no)
        fit = an_prob.make_problem(cfg).evaluate_population_tensors(pop, rng=an.RngStream(9).child(4, 1))
        out[f"{name}_nodes"], out[f"{name}_conns"], out[f"{name}_fitness"] = nodes, conns, fit
    # short XOR run from init_state (runner.py:54-66, 165-169)
    cfg = an.NeatConfig(seed=3, pop_size=150, generation_limit=5)
    state = init_state(cfg)
    problem = an_prob.make_problem(cfg)
    rows = []
    pop, species, alloc = state.population, state.species, state.allocator
    root = an.RngStream(cfg.seed)
    for gen in range(5):
        pop, species, stats = an_evo.evolve_step(pop, species, cfg, root.child(gen), alloc, problem)
        rows.append([stats.best_fitness, stats.mean_fitness, stats.species_count, stats.mean_live_nodes,
                     stats.mean_live_conns])
    out["run_stats"] = np.array(rows)
    out["run_final_nodes"], out["run_final_conns"] = pop.nodes, pop.conns
    out["run_final_species"] = pop.species_id
    _save("problems.npz", **out)


if __name__ == "__main__":
    make_problem_goldens()
