"""Sharded generation with the real kernels at world_size 2: two gloo ranks
share cuda:0 (the collectives run on the host, so neither rank's kernels wait
on the other's).  Three generations must equal the single-process
evolve_step run bit for bit (global-slot RNG keys, founding rounds,
representative argmin, parent gather)."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import REPO, cuda_ok

pytestmark = pytest.mark.gpu

GENS = 3


def _cfg():
    from paper_2404_01817_b200 import NeatConfig
    return NeatConfig(seed=5, pop_size=300, compatibility_threshold=2.0)


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_dir):
    import sys
    sys.path.insert(0, REPO)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        import paper_2404_01817_b200 as tn
        from paper_2404_01817_b200.distributed import Collective, DeviceOps, shard_range, sharded_evolve_step
        from paper_2404_01817_b200.runner import init_state
        cfg = _cfg()
        st = init_state(cfg)
        lo, hi = shard_range(cfg.pop_size, world, rank)
        nodes, conns = st.population.nodes[lo:hi].contiguous(), st.population.conns[lo:hi].contiguous()
        problem = tn.make_problem(cfg)
        root = tn.RngStream(cfg.seed)
        comm, ops = Collective(), DeviceOps(cfg)
        species = st.species
        bests = []
        for gen in range(GENS):
            nodes, conns, lo, species, stats = sharded_evolve_step(nodes, conns, lo, species, cfg, root.child(gen),
                                                                   st.allocator, problem, comm, ops)
            bests.append(stats.best_fitness)
        full = np.concatenate(comm.all_gather(nodes.cpu().numpy()))
        if rank == 0:
            np.savez(os.path.join(out_dir, f"w{world}.npz"), nodes=full, bests=np.array(bests),
                     keys=np.array([s.species_key for s in species]))
    finally:
        dist.destroy_process_group()


@pytest.fixture(scope="module")
def tn():
    if not cuda_ok():
        pytest.skip("no CUDA device")
    import paper_2404_01817_b200 as tn
    return tn


def test_two_rank_sharded_generation_equals_single_process(tn, tmp_path):
    from paper_2404_01817_b200.runner import init_state
    mp.start_processes(_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True, start_method="spawn")
    with np.load(os.path.join(tmp_path, "w2.npz")) as z:
        got = {k: z[k] for k in z.files}
    cfg = _cfg()
    st = init_state(cfg)
    problem = tn.make_problem(cfg)
    root = tn.RngStream(cfg.seed)
    pop, species, bests = st.population, st.species, []
    for gen in range(GENS):
        pop, species, stats = tn.evolve_step(pop, species, cfg, root.child(gen), st.allocator, problem)
        bests.append(stats.best_fitness)
    assert np.array_equal(np.array(bests), got["bests"])
    assert np.array_equal(pop.nodes.cpu().numpy(), got["nodes"], equal_nan=True)
    assert [s.species_key for s in species] == list(got["keys"])
