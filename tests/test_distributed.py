"""Multi-rank protocol of the sharded generation, on CPU with
the gloo backend and world_size 2.

The per-shard compute is swapped for CPU stand-ins (oracle distances, a
numpy model of the reproduce kernel); what is under test is the collective
protocol -- sharding, founding rounds, representative refresh, parent
gathering -- which must give the same answer for any world size, and for
speciation the reference's own answer (tests/golden/evolution.npz).
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import REPO, load_golden


class CpuOps:
    """CPU stand-in for DeviceOps (test infrastructure)."""

    def __init__(self, cd: float, ch: float):
        self.cd, self.ch = cd, ch

    def distance_rows(self, nodes, conns, rep_nodes, rep_conns):
        from oracle.arrayneat_oracle import distance_genome
        return np.array([[distance_genome(nodes[p], conns[p], rep_nodes[r], rep_conns[r], self.cd, self.ch)
                          for p in range(nodes.shape[0])] for r in range(rep_nodes.shape[0])])

    def genome(self, nodes, conns, i):
        return np.array(nodes[i]), np.array(conns[i])

    def gather(self, nodes, conns, local_idx):
        ix = np.asarray(local_idx, dtype=np.int64)
        return torch.from_numpy(np.asarray(nodes)[ix].copy()), torch.from_numpy(np.asarray(conns)[ix].copy())

    def live_counts(self, nodes, conns):
        return ((~np.isnan(nodes[:, :, 0])).sum(1).astype(np.int64),
                (~np.isnan(conns[:, :, 0])).sum(1).astype(np.int64))

    def reproduce_slots(self, pn, pc, pool, off, size, elite, slot_base, count, stage_key, new_key_base):
        """Model of an_reproduce's parent picks + elite copy (mutation omitted)."""
        from oracle.arrayneat_oracle import Stream, mix64
        pn, pc = np.asarray(pn), np.asarray(pc)
        on = np.empty((count,) + pn.shape[1:])
        oc = np.empty((count,) + pc.shape[1:])
        for i in range(count):
            key = mix64(stage_key ^ mix64((slot_base + i) + 0x9E3779B97F4A7C15))
            u = Stream(key).uniforms(2)
            a = off[i] + min(int(u[0] * size[i]), size[i] - 1)
            b = off[i] + min(int(u[1] * size[i]), size[i] - 1)
            src = pool[min(a, b)] if elite[i] < 0 else elite[i]
            on[i], oc[i] = pn[src], pc[src]
            if elite[i] < 0:
                on[i, 0, 1] = float(new_key_base + slot_base + i)  # mark slot identity
        return on, oc


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
        from paper_2404_01817_b200 import NeatConfig
        from paper_2404_01817_b200.distributed import (Collective, shard_range, sharded_reproduce,
                                                       sharded_speciate)
        from paper_2404_01817_b200.evolution import NodeKeyAllocator, SpeciesState, allocate_spawns
        from paper_2404_01817_b200.genome import GenomeTensors
        from paper_2404_01817_b200.rng import RngStream
        c = load_golden("corpus.npz")
        g = load_golden("evolution.npz")
        nodes, conns = c["nodes"], c["conns"]
        total = nodes.shape[0]
        cfg = NeatConfig(inputs=3, outputs=2, max_nodes=32, max_conns=64, pop_size=total,
                         compatibility_threshold=1.2, max_species=6)
        comm = Collective()
        ops = CpuOps(cfg.compatibility_disjoint, cfg.compatibility_homologous)
        lo, hi = shard_range(total, world, rank)
        assigned, species = sharded_speciate(nodes[lo:hi], conns[lo:hi], lo, total, [], cfg, comm, ops, 3, 2)
        old = [SpeciesState(species_key=k, representative=GenomeTensors(nodes[i], conns[i], 3, 2),
                            member_indices=np.arange(1)) for k, i in ((3, 17), (8, 101))]
        assigned1, species1 = sharded_speciate(nodes[lo:hi], conns[lo:hi], lo, total, old, cfg, comm, ops, 3, 2)
        fitness = g["rep_fitness"]
        alloc = allocate_spawns(species, fitness, cfg)
        on, oc, (slo, shi) = sharded_reproduce(nodes[lo:hi], conns[lo:hi], lo, alloc, fitness, cfg,
                                               RngStream(13).child(4), NodeKeyAllocator(500), comm, ops)
        full_n = np.concatenate(comm.all_gather(np.asarray(on)))
        if rank == 0:
            np.savez(os.path.join(out_dir, f"w{world}.npz"), assigned=assigned, assigned1=assigned1,
                     keys=np.array([s.species_key for s in species]),
                     reps=np.stack([s.representative.nodes for s in species]),
                     keys1=np.array([s.species_key for s in species1]),
                     reps1=np.stack([s.representative.nodes for s in species1]),
                     offspring=full_n)
    finally:
        dist.destroy_process_group()


def _run(world, out_dir):
    mp.start_processes(_worker, args=(world, _free_port(), out_dir), nprocs=world, join=True,
                       start_method="spawn")
    with np.load(os.path.join(out_dir, f"w{world}.npz")) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="module")
def results(tmp_path_factory):
    d = str(tmp_path_factory.mktemp("dist"))
    return _run(1, d), _run(2, d)


def test_sharded_speciation_matches_reference(results):
    g = load_golden("evolution.npz")
    for r in results:
        assert np.array_equal(r["assigned"], g["spec0_assigned"])
        assert list(r["keys"]) == list(g["spec0_keys"])
        assert np.array_equal(r["reps"], g["spec0_reps"], equal_nan=True)
        assert np.array_equal(r["assigned1"], g["spec1_assigned"])
        assert list(r["keys1"]) == list(g["spec1_keys"])
        assert np.array_equal(r["reps1"], g["spec1_reps_nodes"], equal_nan=True)


def test_sharded_reproduction_independent_of_world_size(results):
    one, two = results
    assert np.array_equal(one["offspring"], two["offspring"], equal_nan=True)
