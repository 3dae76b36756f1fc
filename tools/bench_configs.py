"""Secondary measurements for BASELINE.json configs 1, 3, 4 and 5 (config 2
is bench.py).  One JSON line per measurement; GPU times from CUDA events or
synchronized wall clock as stated; CPU reference on the same host.

    python tools/bench_configs.py xor|generation|hyperneat|recurrent [--pop P] ...
    python tools/bench_configs.py generation --gpus N --pop 1000000   (sharded, NCCL)
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
if os.environ.get("TNEAT_TOOL_LIB"):  # A/B of a tools/build_variant.py library
    from paper_2404_01817_b200 import _native  # noqa: E402
    _native.LIB_PATH = os.path.abspath(os.environ["TNEAT_TOOL_LIB"])


def _sync():
    import torch
    torch.cuda.synchronize()


def _ref_arrayneat():
    ref = os.path.join(REPO, "oracle", "_ref")
    if os.path.isdir(os.path.join(ref, "arrayneat")) and ref not in sys.path:
        sys.path.insert(0, ref)
    import arrayneat
    return arrayneat


def bench_xor(a):
    """Config 1: NEAT XOR, pop 1000, 50/100, 100 generations (gen/s)."""
    import paper_2404_01817_b200 as tn
    from paper_2404_01817_b200.runner import init_state
    cfg = tn.NeatConfig(seed=a.seed, pop_size=1000, inputs=2, outputs=1, problem="xor", max_nodes=50,
                        max_conns=100, generation_limit=a.gens)
    state = init_state(cfg)
    problem = tn.make_problem(cfg)
    root = tn.RngStream(cfg.seed)
    pop, species = state.population, state.species
    # warm-up generation on a throwaway copy of the state
    _ = tn.evolve_step(pop, species, cfg, root.child(0), tn.NodeKeyAllocator(state.allocator.next_key), problem)
    _sync()
    t = time.perf_counter()
    for gen in range(a.gens):
        pop, species, stats = tn.evolve_step(pop, species, cfg, root.child(gen), state.allocator, problem)
    _sync()
    dt = time.perf_counter() - t
    out = {"config": "1: XOR pop 1000 50/100", "generations": a.gens, "gen_per_s": a.gens / dt,
           "s_per_gen": dt / a.gens, "final_best": stats.best_fitness, "species": len(species)}
    if not a.no_cpu:
        an = _ref_arrayneat()
        from arrayneat.runner import init_state as ref_init
        rcfg = an.NeatConfig(seed=a.seed, pop_size=1000, inputs=2, outputs=1, problem="xor", max_nodes=50,
                             max_conns=100, generation_limit=a.gens)
        st = ref_init(rcfg)
        prob = an.make_problem(rcfg)
        rp, rs, ral = st.population, st.species, st.allocator
        rg = min(a.gens, 30)
        t = time.perf_counter()
        for gen in range(rg):
            rp, rs, rst = an.evolve_step(rp, rs, rcfg, an.RngStream(rcfg.seed).child(gen), ral, prob)
        rdt = time.perf_counter() - t
        out["cpu_reference_gen_per_s"] = rg / rdt
        out["cpu_reference_generations_timed"] = rg
        out["speedup_vs_cpu"] = out["gen_per_s"] / out["cpu_reference_gen_per_s"]
    return out


def bench_generation(a):
    """Config 3: pop P (default 1M), XOR, 50/100, threshold 1.0: per-phase times."""
    import torch

    import paper_2404_01817_b200 as tn
    from paper_2404_01817_b200 import evolution as evo
    from paper_2404_01817_b200.runner import init_state
    cfg = tn.NeatConfig(seed=0, pop_size=a.pop, inputs=2, outputs=1, problem="xor", max_nodes=50,
                        max_conns=100, compatibility_threshold=1.0, max_species=10)
    t0 = time.perf_counter()
    state = init_state(cfg)
    _sync()
    t_init = time.perf_counter() - t0
    problem = tn.make_problem(cfg)
    root = tn.RngStream(cfg.seed)
    pop, species = state.population, state.species
    phases = []
    for gen in range(a.gens):
        rng = root.child(gen)
        t = [time.perf_counter()]
        fit = problem.evaluate_population_tensors(pop, rng=rng.child(evo.STAGE_EVAL))
        _sync(); t.append(time.perf_counter())
        surv = evo.update_stagnation(species, fit, cfg)
        alloc = evo.allocate_spawns(surv, fit, cfg)
        ev = tn.PopulationTensors(pop.nodes, pop.conns, pop.species_id, fit, 2, 1)
        off = evo.reproduce(ev, alloc, fit, cfg, rng, state.allocator)
        _sync(); t.append(time.perf_counter())
        pop, species = evo.speciate(off, alloc, cfg)
        _sync(); t.append(time.perf_counter())
        phases.append({"eval_s": t[1] - t[0], "reproduce_s": t[2] - t[1], "speciate_s": t[3] - t[2],
                       "gen_s": t[3] - t[0], "species": len(species)})
    genome_bytes = (cfg.max_nodes * 5 + cfg.max_conns * 4) * 8
    last = phases[-1]
    ref = None
    if getattr(a, "ref_pop", 0):
        # the unmodified reference's evolve_step (runner.py:165-169 loop pattern)
        # on the same host, one generation at ref_pop genomes, 1 thread
        an = _ref_arrayneat()
        from arrayneat.runner import init_state as ref_init
        rcfg = an.NeatConfig(seed=0, pop_size=a.ref_pop, inputs=2, outputs=1, problem="xor", max_nodes=50,
                             max_conns=100, compatibility_threshold=1.0, max_species=10)
        st = ref_init(rcfg)
        prob = an.make_problem(rcfg)
        tt = time.perf_counter()
        an.evolve_step(st.population, st.species, rcfg, an.RngStream(0).child(0), st.allocator, prob)
        rdt = time.perf_counter() - tt
        ref = {"pop": a.ref_pop, "s_per_gen": rdt, "gen_per_s": 1.0 / rdt,
               "scaled_s_per_gen_at_pop": rdt * a.pop / a.ref_pop, "threads": 1,
               "note": "generation 0 from init_state; scaled linearly to the GPU run's population"}
    out = {"config": f"3: generation pop {a.pop} 50/100 (XOR, threshold 1.0)", "init_s": t_init,
           "phases": phases,
           # steady state: the median of the last (up to) three generations (the
           # first ones carry allocator growth; speciation time varies by run)
           "gen_per_s": 1.0 / float(np.median([p["gen_s"] for p in phases[-3:]])),
           "reproduce_GBps_min_traffic": 3 * a.pop * genome_bytes / last["reproduce_s"] / 1e9,
           "genome_bytes": genome_bytes, "gpu_mem_GB": torch.cuda.max_memory_allocated() / 1e9,
           "cpu_reference": ref}
    return out


def bench_generation_sharded(a):
    """Config 3 over N GPUs: sharded_evolve_step (one rank per GPU, NCCL):
    contiguous population shards, fitness / species-assignment all-gathers,
    founding rounds, survivor-pool gather (distributed.py); gen/s is the
    slowest rank's time per generation."""
    import torch
    import torch.distributed as dist

    import paper_2404_01817_b200 as tn
    from paper_2404_01817_b200 import distributed as dd
    from paper_2404_01817_b200.runner import init_state
    rank, world = dist.get_rank(), dist.get_world_size()
    cfg = tn.NeatConfig(seed=0, pop_size=a.pop, inputs=2, outputs=1, problem="xor", max_nodes=50,
                        max_conns=100, compatibility_threshold=1.0, max_species=10)
    state = init_state(cfg)
    lo, hi = dd.shard_range(a.pop, world, rank)
    nodes, conns = state.population.nodes[lo:hi].contiguous(), state.population.conns[lo:hi].contiguous()
    species = state.species
    comm = dd.Collective()
    ops = dd.DeviceOps(cfg)
    problem = tn.make_problem(cfg)
    root = tn.RngStream(cfg.seed)
    times = []
    for gen in range(a.gens):
        torch.cuda.synchronize()
        dist.barrier()
        t = time.perf_counter()
        nodes, conns, lo, species, stats = dd.sharded_evolve_step(nodes, conns, lo, species, cfg, root.child(gen),
                                                                  state.allocator, problem, comm, ops)
        torch.cuda.synchronize()
        dt = torch.tensor([time.perf_counter() - t], device="cuda", dtype=torch.float64)
        dist.all_reduce(dt, op=dist.ReduceOp.MAX)
        times.append(float(dt.item()))
    return {"config": f"3: sharded generation pop {a.pop} over {world} GPUs (XOR, threshold 1.0)",
            "gpus": world, "s_per_gen": times, "gen_per_s": 1.0 / times[-1], "species": len(species),
            "best_fitness": stats.best_fitness}


def bench_hyperneat(a):
    """Config 4: CPPN pop P x 4096 queries + tcgen05 substrate (S = 4096)."""
    import torch

    import paper_2404_01817_b200 as tn
    from paper_2404_01817_b200 import hyperneat as hn
    from paper_2404_01817_b200.synthetic import synthetic_population
    nodes, conns = synthetic_population(a.pop, 128, 512, 4, 1, seed=20261018, variant="M", min_conns=64,
                                        max_conns_drawn=256)
    st, _ = tn.transform_arrays(nodes, conns, 4, 1)
    x, t = hn.teacher_task(4096)
    xd, td = torch.from_numpy(x).cuda(), torch.from_numpy(t).cuda()
    for _ in range(3):
        w = hn.cppn_weights(st)
        f = hn.substrate_fitness(w, xd, td)
    _sync()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    n_rep = 5
    e[0].record()
    for _ in range(n_rep):
        w = hn.cppn_weights(st)
    e[1].record()
    for _ in range(n_rep):
        f = hn.substrate_fitness(w, xd, td)
    e[2].record()
    _sync()
    q_ms = e[0].elapsed_time(e[1]) / n_rep
    s_ms = e[1].elapsed_time(e[2]) / n_rep
    flops = 2.0 * 4096 * 64 * 64 * a.pop
    peak = json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json")))["bf16_tflops"] \
        if os.path.exists(os.path.join(REPO, "MEASURED_PEAKS.json")) else 1590.0
    out = {"config": f"4: HyperNEAT pop {a.pop}, 64x64 substrate, S=4096", "cppn_query_ms": q_ms,
           "cppn_queries_per_s": a.pop * 4096 / (q_ms / 1e3), "substrate_ms": s_ms,
           "substrate_TFLOPs": flops / (s_ms / 1e3) / 1e12,
           "substrate_frac_of_tf32_peak": flops / (s_ms / 1e3) / 1e12 / (peak / 2),
           "tf32_peak_TFLOPs_assumed": peak / 2, "pass_ms": q_ms + s_ms,
           "fitness_mean": float(f.mean())}
    if not a.no_cpu:
        from oracle import arrayneat_oracle as orc
        k = 4
        tt = time.perf_counter()
        for p in range(k):
            orc.substrate_fitness(nodes[p], conns[p], x, t)
        dt = (time.perf_counter() - tt) / k
        out["cpu_oracle_s_per_genome"] = dt
        out["cpu_oracle_kind"] = "port (no reference HyperNEAT), 1 thread"
    return out


def bench_recurrent(a):
    """Config 5: pop P recurrent genomes, I=27, O=8, 128/512, T=1000 steps, K sweeps."""
    import torch

    import paper_2404_01817_b200 as tn
    from paper_2404_01817_b200 import recurrent as rec
    from paper_2404_01817_b200.synthetic import synthetic_population
    nodes, conns = synthetic_population(a.pop, 128, 512, 27, 8, seed=20261018, variant="T", min_conns=216,
                                        max_conns_drawn=448)
    rng = np.random.default_rng(1)
    for p in range(a.pop):  # add back edges -> cycles
        free = np.nonzero(np.isnan(conns[p, :, 0]))[0][:32]
        keys = nodes[p, ~np.isnan(nodes[p, :, 0]), 0]
        hid = keys[keys >= 35]
        have = {(int(u), int(v)) for u, v in conns[p][~np.isnan(conns[p, :, 0])][:, :2]}
        for r in free:
            if hid.size < 2:
                break
            u, v = rng.choice(hid, 2, replace=False)
            if (int(u), int(v)) not in have:
                have.add((int(u), int(v)))
                conns[p, r] = [u, v, 1.0, rng.standard_normal()]
    st, _ = tn.transform_arrays(nodes, conns, 27, 8, network_type="recurrent")
    env = rec.ant_env()
    res = []
    for k in a.sweeps:
        rec.rollout_fitness(st, env, steps=10, sweeps=k)
        _sync()
        t = time.perf_counter()
        f = rec.rollout_fitness(st, env, steps=a.steps, sweeps=k)
        dt = time.perf_counter() - t
        res.append({"sweeps": k, "s": dt, "genome_steps_per_s": a.pop * a.steps / dt,
                    "fitness_mean": float(np.mean(f))})
    out = {"config": f"5: recurrent pop {a.pop}, I=27 O=8, 128/512, T={a.steps}", "runs": res}
    if not a.no_cpu:
        from oracle import arrayneat_oracle as orc
        tt = time.perf_counter()
        orc.recurrent_rollout(nodes[0], conns[0], 27, 8, *env, steps=10, sweeps=5)
        dt = time.perf_counter() - tt
        out["cpu_oracle_genome_steps_per_s_K5"] = 10 / dt
        out["cpu_oracle_kind"] = "port (no reference recurrent path), 1 thread, 10 steps of genome 0"
    return out


def main():
    if "--gpus" in sys.argv and "WORLD_SIZE" not in os.environ:
        n = int(sys.argv[sys.argv.index("--gpus") + 1])
        if n > 1:  # one rank per GPU under torch.distributed.run
            import socket
            with socket.socket() as sk:
                sk.bind(("127.0.0.1", 0))
                port = sk.getsockname()[1]
            cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
                   "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
            import subprocess
            raise SystemExit(subprocess.call(cmd))
    ap = argparse.ArgumentParser()
    ap.add_argument("which", choices=["xor", "generation", "hyperneat", "recurrent"])
    ap.add_argument("--pop", type=int, default=None)
    ap.add_argument("--gens", type=int, default=None)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--sweeps", type=int, nargs="+", default=[1, 5, 10])
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--ref-pop", type=int, default=0)
    a = ap.parse_args()
    defaults = {"xor": (1000, 100), "generation": (1_000_000, 3), "hyperneat": (10_000, 1),
                "recurrent": (10_000, 1)}
    a.pop = a.pop or defaults[a.which][0]
    a.gens = a.gens or defaults[a.which][1]
    if a.which == "generation" and "WORLD_SIZE" in os.environ:
        import torch
        import torch.distributed as dist
        local = int(os.environ.get("LOCAL_RANK", 0))
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        try:
            out = bench_generation_sharded(a)
            if dist.get_rank() == 0:
                print(json.dumps(out), flush=True)
        finally:
            dist.destroy_process_group()
        return
    out = {"xor": bench_xor, "generation": bench_generation, "hyperneat": bench_hyperneat,
           "recurrent": bench_recurrent}[a.which](a)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
