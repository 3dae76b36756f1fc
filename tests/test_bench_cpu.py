"""bench.py's multi-rank logic on CPU: strong-scaling shards of the 10k
population and the per-step fitness all-gather (gloo, world_size 2 == 1), and
the self-relaunch of ``--gpus N`` under torch.distributed.run."""

from __future__ import annotations

import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import REPO

P, NIN, NOUT, B = 12, 4, 2, 16


def _fitness_of(nodes, conns, x):
    """-mean squared output per genome (the bench step's fitness), oracle forward."""
    from oracle.arrayneat_oracle import forward_genome, transform_genome
    return np.array([-np.mean(forward_genome(nodes[p], transform_genome(nodes[p], conns[p], NIN, NOUT),
                                             x[p]) ** 2) for p in range(nodes.shape[0])], dtype=np.float32)


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_dir):
    sys.path.insert(0, REPO)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        from paper_2404_01817_b200.synthetic import synthetic_population
        nodes, conns = synthetic_population(P, 24, 60, NIN, NOUT, seed=3, min_conns=10, max_conns_drawn=40)
        x = np.random.default_rng(4).standard_normal((P, B, NIN))
        lo, shard = bench.shard_of(P, world, rank)
        fit = torch.from_numpy(_fitness_of(nodes[lo:lo + shard], conns[lo:lo + shard], x[lo:lo + shard]))
        full = torch.empty(P, dtype=torch.float32)
        bench.gather_fitness(fit, full, world)
        np.save(os.path.join(out_dir, f"w{world}_r{rank}.npy"), full.numpy())
    finally:
        dist.destroy_process_group()


def test_fitness_all_gather_world2_equals_world1(tmp_path):
    for world in (1, 2):
        mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True,
                           start_method="spawn")
    one = np.load(tmp_path / "w1_r0.npy")
    for r in range(2):
        assert np.array_equal(np.load(tmp_path / f"w2_r{r}.npy"), one)  # every rank holds the whole vector


def test_shards_are_contiguous_and_cover_the_population():
    sys.path.insert(0, REPO)
    import bench
    for world in (1, 2, 4, 8):
        spans = [bench.shard_of(10_000, world, r) for r in range(world)]
        assert [lo for lo, _ in spans] == [r * 10_000 // world for r in range(world)]
        assert sum(n for _, n in spans) == 10_000
    with pytest.raises(SystemExit):
        bench.shard_of(10_000, 3, 0)


def test_gpus_flag_relaunches_under_torchrun(monkeypatch):
    sys.path.insert(0, REPO)
    import bench
    calls = []
    monkeypatch.setattr(bench.subprocess, "call", lambda cmd: calls.append(cmd) or 0)
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "5"])
    with pytest.raises(SystemExit) as e:
        bench.main()
    assert e.value.code == 0
    cmd = calls[0]
    assert cmd[1:4] == ["-m", "torch.distributed.run", "--nnodes=1"]
    assert "--nproc-per-node=4" in cmd and "127.0.0.1" in cmd
    assert cmd[-4:] == ["--gpus", "4", "--steps", "5"]
