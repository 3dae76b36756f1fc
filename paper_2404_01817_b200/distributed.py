"""Population sharding across GPUs.

One process per GPU (torch.distributed, NCCL over NVLink); rank r owns the
contiguous genome slice ``shard_range(P, world, r)``.

* transform + forward + fitness: independent per shard, no collective on the
  data path; one all-gather of the (P,) float64 fitness.
* speciation: representatives are replicated host genomes.  Each rank scores
  its shard against them; founding runs in rounds: all-reduce MIN of the
  first unassigned global index, its owner broadcasts the founder genome,
  every rank scores its shard against it.  Representative refresh: per
  species each rank proposes (min distance, global index), an all-gather
  picks the global argmin (first index on ties), the owner broadcasts it.
* reproduction: the replicated spawn / slot tables select parents from any
  rank; the genomes in the survivor pools (plus elites) are all-gathered once,
  and each rank produces its slice of next-generation slots.  Per-slot RNG
  streams are keyed by the GLOBAL slot, so offspring are identical for any
  number of GPUs.
* With ``DeviceOps`` (the product path) all of it runs on device tensors:
  distance rows, assignments, slot tables and the gathered parents never
  leave the GPU; the host sees the fitness vector, one packed copy of the
  assignment grouping and the few representative genomes.

The per-shard compute (distances, reproduction, fitness) is behind a small
``ops`` object: ``DeviceOps`` runs the CUDA kernels; the multi-process CPU
tests (gloo) substitute CPU implementations to check the collective protocol.
"""

from __future__ import annotations

import math
from dataclasses import replace

import numpy as np
import torch
import torch.distributed as dist

from .config import NeatConfig
from .evolution import (STAGE_EVAL, STAGE_REPRODUCE, STAGE_SPECIATE, GenerationStats, NodeKeyAllocator,
                        SpeciesState, allocate_spawns, slot_tables, update_stagnation)
from .genome import GenomeTensors

INF_INDEX = np.iinfo(np.int64).max


def shard_range(total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced slice of ``total`` items for ``rank``."""
    base, extra = divmod(total, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


class Collective:
    """Host-array collectives over the default process group (any backend)."""

    def __init__(self, device: torch.device | None = None):
        self.rank = dist.get_rank() if dist.is_initialized() else 0
        self.world = dist.get_world_size() if dist.is_initialized() else 1
        backend = dist.get_backend() if dist.is_initialized() else "gloo"
        self.device = device if device is not None else (
            torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu"))

    def _t(self, arr: np.ndarray) -> torch.Tensor:
        return torch.from_numpy(np.ascontiguousarray(arr)).to(self.device)

    def all_gather(self, arr: np.ndarray) -> list[np.ndarray]:
        """Gather variable-length arrays (leading axis) from every rank."""
        arr = np.ascontiguousarray(arr)
        if self.world == 1:
            return [arr]
        n = self._t(np.array([arr.shape[0]], dtype=np.int64))
        sizes = [torch.zeros_like(n) for _ in range(self.world)]
        dist.all_gather(sizes, n)
        sizes = [int(s.item()) for s in sizes]
        mx = max(sizes)
        pad = np.zeros((mx,) + arr.shape[1:], dtype=arr.dtype)
        pad[:arr.shape[0]] = arr
        t = self._t(pad)
        outs = [torch.empty_like(t) for _ in range(self.world)]
        dist.all_gather(outs, t)
        return [o.cpu().numpy()[:s] for o, s in zip(outs, sizes)]

    def all_gather_tensor(self, t: torch.Tensor) -> torch.Tensor:
        """Concatenate variable-length tensors (leading axis) from every rank,
        staying on the collective's device (NCCL: GPU memory over NVLink)."""
        if self.world == 1:
            return t
        t = t.to(self.device).contiguous()
        n = torch.tensor([t.shape[0]], dtype=torch.int64, device=self.device)
        sizes = [torch.zeros_like(n) for _ in range(self.world)]
        dist.all_gather(sizes, n)
        sizes = [int(x.item()) for x in sizes]
        pad = torch.zeros((max(sizes),) + tuple(t.shape[1:]), dtype=t.dtype, device=self.device)
        pad[:t.shape[0]] = t
        outs = [torch.empty_like(pad) for _ in range(self.world)]
        dist.all_gather(outs, pad)
        return torch.cat([o[:k] for o, k in zip(outs, sizes)])

    # -- device tensors: NCCL works on them in place; a host backend (gloo, the
    #    multi-process tests) stages them through host memory
    def _to_comm(self, t: torch.Tensor) -> torch.Tensor:
        return t if t.device == self.device else t.to(self.device)

    def all_reduce_dev(self, t: torch.Tensor, op=None) -> torch.Tensor:
        if self.world == 1:
            return t
        c = self._to_comm(t.contiguous())
        dist.all_reduce(c, op=op if op is not None else dist.ReduceOp.SUM)
        return c.to(t.device)

    def broadcast_dev(self, t: torch.Tensor, src: int) -> torch.Tensor:
        if self.world == 1:
            return t
        c = self._to_comm(t.contiguous())
        dist.broadcast(c, src)
        return c.to(t.device)

    def all_gather_dev(self, t: torch.Tensor) -> torch.Tensor:
        """Variable-length device tensors concatenated over ranks, on t's device."""
        if self.world == 1:
            return t
        return self.all_gather_tensor(t).to(t.device)

    def all_reduce_min(self, value: int) -> int:
        if self.world == 1:
            return int(value)
        t = self._t(np.array([value], dtype=np.int64))
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        return int(t.item())

    def broadcast(self, arr: np.ndarray | None, shape, dtype, src: int) -> np.ndarray:
        if self.world == 1:
            return arr
        t = self._t(arr) if self.rank == src else torch.empty(shape, dtype=torch.from_numpy(
            np.zeros(1, dtype=dtype)).dtype, device=self.device)
        dist.broadcast(t, src)
        return t.cpu().numpy()


class DeviceOps:
    """Per-shard compute on this rank's GPU (the product path)."""

    def __init__(self, config: NeatConfig):
        self.config = config

    def distance_rows(self, nodes, conns, rep_nodes: np.ndarray, rep_conns: np.ndarray) -> np.ndarray:
        from .evolution import _dev64, _distance_dev
        return _distance_dev(_dev64(nodes), _dev64(conns), _dev64(rep_nodes), _dev64(rep_conns),
                             self.config, 0).cpu().numpy()

    def genome(self, nodes, conns, i: int) -> tuple[np.ndarray, np.ndarray]:
        n, c = nodes[i], conns[i]
        if isinstance(n, torch.Tensor):
            n, c = n.cpu().numpy(), c.cpu().numpy()
        return np.array(n), np.array(c)

    def gather(self, nodes, conns, local_idx: np.ndarray):
        from .evolution import _dev64
        nd, cd = _dev64(nodes), _dev64(conns)
        ix = torch.from_numpy(np.asarray(local_idx, dtype=np.int64)).to(nd.device)
        return nd[ix], cd[ix]

    def live_counts(self, nodes, conns):
        from .evolution import _dev64
        nd, cd = _dev64(nodes), _dev64(conns)
        return ((~torch.isnan(nd[:, :, 0])).sum(1).cpu().numpy().astype(np.int64),
                (~torch.isnan(cd[:, :, 0])).sum(1).cpu().numpy().astype(np.int64))

    def reproduce_slots(self, parents_nodes, parents_conns, pool, off, size, elite, slot_base: int, count: int,
                        stage_key: int, new_key_base: int):
        import ctypes

        from . import _native
        from .device import device, ptr, stream_handle
        from .evolution import _dev64, mutate_params
        dev = device()
        pn, pc = _dev64(parents_nodes), _dev64(parents_conns)
        n, c = int(pn.shape[1]), int(pc.shape[1])
        on = torch.empty((count, n, 5), dtype=torch.float64, device=dev)
        oc = torch.empty((count, c, 4), dtype=torch.float64, device=dev)
        tabs = [torch.from_numpy(np.ascontiguousarray(a, dtype=np.int32)).to(dev) for a in (pool, off, size, elite)]
        params = mutate_params(self.config, n, c)
        _native.call("an_reproduce", ptr(pn), ptr(pc), ptr(on), ptr(oc), count, slot_base, ptr(tabs[0]),
                     ptr(tabs[1]), ptr(tabs[2]), ptr(tabs[3]), stage_key, float(new_key_base),
                     ctypes.addressof(params), None, stream_handle())
        return on, oc

    def fitness(self, problem, nodes, conns, n_in, n_out, rng) -> np.ndarray:
        from .genome import PopulationTensors
        pop = PopulationTensors(nodes, conns, None, None, n_in, n_out)
        return np.asarray(problem.evaluate_population_tensors(pop, rng=rng), dtype=np.float64)


def _owner(index: int, total: int, world: int) -> int:
    for r in range(world):
        lo, hi = shard_range(total, world, r)
        if lo <= index < hi:
            return r
    raise IndexError(index)


def sharded_speciate(nodes, conns, lo: int, total: int, species: list, config: NeatConfig, comm: Collective,
                     ops, n_in: int, n_out: int):
    """speciate (evolution.py:513-576) over a sharded population.  Returns the
    global species id array (total,) and the new species list (replicated)."""
    n_local = int(nodes.shape[0])
    thr = float(config.compatibility_threshold)
    ordered = sorted(species, key=lambda s: s.species_key)
    rows = []  # (key, previous, representative, local distance row)
    assigned = np.full(n_local, -1, dtype=np.int64)
    if ordered:
        mat = ops.distance_rows(nodes, conns, np.stack([s.representative.nodes for s in ordered]),
                                np.stack([s.representative.conns for s in ordered]))
        for k, sp in enumerate(ordered):
            rows.append((sp.species_key, sp, sp.representative, mat[k]))
        ok = mat <= thr
        hit = ok.any(axis=0)
        keys = np.array([s.species_key for s in ordered])
        assigned[hit] = keys[ok.argmax(axis=0)[hit]]
    next_key = max((r[0] for r in rows), default=-1) + 1
    while True:
        un = np.nonzero(assigned < 0)[0]
        first = comm.all_reduce_min(int(lo + un[0]) if un.size else INF_INDEX)
        if first == INF_INDEX:
            break
        if len(rows) < config.max_species:
            owner = _owner(first, total, comm.world)
            mine = ops.genome(nodes, conns, first - lo) if comm.rank == owner else (None, None)
            fn = comm.broadcast(mine[0], (nodes.shape[1], 5), np.float64, owner)
            fc = comm.broadcast(mine[1], (conns.shape[1], 4), np.float64, owner)
            d = ops.distance_rows(nodes, conns, fn[None], fc[None])[0]
            take = (assigned < 0) & (d <= thr)
            if lo <= first < lo + n_local:
                take[first - lo] = True
            assigned[take] = next_key
            rows.append((next_key, None, GenomeTensors(fn, fc, n_in, n_out), d))
            next_key += 1
        else:
            mat = np.stack([r[3] for r in rows])
            keys = np.array([r[0] for r in rows])
            rest = assigned < 0
            assigned[rest] = keys[mat[:, rest].argmin(axis=0)]
            break
    global_assigned = np.concatenate(comm.all_gather(assigned))
    result = []
    for key, previous, rep, drow in rows:
        members = np.nonzero(global_assigned == key)[0]
        if members.size == 0:
            continue
        local = np.nonzero(assigned == key)[0]
        if local.size:
            j = int(np.argmin(drow[local]))
            cand = np.array([[drow[local[j]], float(lo + local[j])]])
        else:
            cand = np.array([[np.inf, np.inf]])
        allc = np.concatenate(comm.all_gather(cand))
        best = min(range(allc.shape[0]), key=lambda i: (allc[i, 0], allc[i, 1]))
        closest = int(allc[best, 1])
        owner = _owner(closest, total, comm.world)
        mine = ops.genome(nodes, conns, closest - lo) if comm.rank == owner else (None, None)
        rn = comm.broadcast(mine[0], (nodes.shape[1], 5), np.float64, owner)
        rc = comm.broadcast(mine[1], (conns.shape[1], 4), np.float64, owner)
        new_rep = GenomeTensors(rn, rc, n_in, n_out)
        if previous is not None:
            result.append(replace(previous, representative=new_rep, member_indices=members, spawn_count=0))
        else:
            result.append(SpeciesState(species_key=key, representative=new_rep, member_indices=members))
    return global_assigned, result


def sharded_reproduce(nodes, conns, lo: int, species: list, fitness: np.ndarray, config: NeatConfig, rng,
                      allocator: NodeKeyAllocator, comm: Collective, ops):
    """reproduce (evolution.py:646-715) with parents gathered from all ranks;
    returns this rank's slice of the next generation (and its global range)."""
    total = config.pop_size
    base_key = allocator.reserve(total)
    pool, off, size, elite = slot_tables(species, fitness, config)
    needed = np.unique(np.concatenate([pool, elite[elite >= 0]]))
    n_local = int(nodes.shape[0])
    mine = needed[(needed >= lo) & (needed < lo + n_local)]
    pn, pc = ops.gather(nodes, conns, mine - lo)
    idx = comm.all_gather_tensor(torch.from_numpy(mine.astype(np.int64))).cpu().numpy()
    all_n = comm.all_gather_tensor(pn)
    all_c = comm.all_gather_tensor(pc)
    order = np.argsort(idx)
    ot = torch.from_numpy(order).to(all_n.device)
    idx, all_n, all_c = idx[order], all_n[ot], all_c[ot]
    remap = lambda a: np.searchsorted(idx, a).astype(np.int32)  # noqa: E731
    pool_r = remap(pool)
    elite_r = np.where(elite >= 0, remap(np.maximum(elite, 0)), -1).astype(np.int32)
    slo, shi = shard_range(total, comm.world, comm.rank)
    stage_key = int(np.asarray(rng.child(STAGE_REPRODUCE)._keys).reshape(-1)[0])
    on, oc = ops.reproduce_slots(all_n, all_c, pool_r, off[slo:shi], size[slo:shi], elite_r[slo:shi], slo,
                                 shi - slo, stage_key, base_key)
    return on, oc, (slo, shi)


def sharded_speciate_device(nd: torch.Tensor, cd: torch.Tensor, lo: int, total: int, species: list,
                            config: NeatConfig, comm: Collective, n_in: int, n_out: int):
    """speciate (evolution.py:513-576) over a sharded device population with
    the protocol on device tensors: distance rows and assignments stay on the
    GPU; a founding round is one all-reduce MIN of the first unassigned global
    index plus the owner's broadcast of the founder genome; the representative
    refresh all-gathers one (distance, global index) pair per species and
    broadcasts the winners.  Returns the global species ids (host, (total,))
    and the replicated species list -- the same answer as the host protocol and
    the single-GPU path for any world size."""
    from .evolution import _distance_dev
    dev = nd.device
    n_local = int(nd.shape[0])
    thr = float(config.compatibility_threshold)
    ordered = sorted(species, key=lambda s: s.species_key)
    rows = []  # (key, previous state or None, local distance row on the device)
    assigned = torch.full((n_local,), -1, dtype=torch.int64, device=dev)
    if ordered:
        rn = torch.from_numpy(np.stack([sp.representative.nodes for sp in ordered])).to(dev)
        rc = torch.from_numpy(np.stack([sp.representative.conns for sp in ordered])).to(dev)
        mat = _distance_dev(nd, cd, rn, rc, config, 0) if n_local else torch.empty((len(ordered), 0),
                                                                                     dtype=torch.float64, device=dev)
        for k, sp in enumerate(ordered):
            rows.append((sp.species_key, sp, mat[k]))
        ok = mat <= thr
        keys = torch.tensor([sp.species_key for sp in ordered], dtype=torch.int64, device=dev)
        assigned = torch.where(ok.any(dim=0), keys[ok.to(torch.int8).argmax(dim=0)], assigned)
    next_key = max((r[0] for r in rows), default=-1) + 1
    inf_t = torch.tensor([INF_INDEX], dtype=torch.int64, device=dev)
    while True:
        free = assigned < 0
        if n_local:
            has, first_l = free.to(torch.int8).max(dim=0)
            cand = torch.where(has.bool(), first_l + lo, inf_t[0]).reshape(1)
        else:
            cand = inf_t.clone()
        first = int(comm.all_reduce_dev(cand, dist.ReduceOp.MIN if comm.world > 1 else None).item())
        if first == INF_INDEX:
            break
        if len(rows) < config.max_species:
            owner = _owner(first, total, comm.world)
            if comm.rank == owner:
                fn, fc = nd[first - lo].clone(), cd[first - lo].clone()
            else:
                fn = torch.empty(tuple(nd.shape[1:]), dtype=nd.dtype, device=dev)
                fc = torch.empty(tuple(cd.shape[1:]), dtype=cd.dtype, device=dev)
            fn, fc = comm.broadcast_dev(fn, owner), comm.broadcast_dev(fc, owner)
            d = _distance_dev(nd, cd, fn[None], fc[None], config, 1) if n_local else \
                torch.empty((0,), dtype=torch.float64, device=dev)
            take = free & (d <= thr)
            if lo <= first < lo + n_local:
                take[first - lo] = True
            assigned = torch.where(take, torch.full_like(assigned, next_key), assigned)
            rows.append((next_key, None, d))
            next_key += 1
        else:
            keys = torch.tensor([r[0] for r in rows], dtype=torch.int64, device=dev)
            near = keys[torch.stack([r[2] for r in rows]).argmin(dim=0)]
            assigned = torch.where(assigned < 0, near, assigned)
            break
    # representative refresh: per species the member closest to the old
    # representative (first global index on ties) -- local candidates, one
    # all-gather of (distance, index) pairs, then the owners' broadcasts
    R = len(rows)
    keys_d = torch.tensor([r[0] for r in rows], dtype=torch.int64, device=dev)
    dist_m = torch.stack([r[2] for r in rows]) if R else torch.empty((0, n_local), dtype=torch.float64,
                                                                     device=dev)
    rowid = torch.searchsorted(keys_d, assigned)
    mine = torch.arange(R, device=dev)[:, None] == rowid[None, :]
    masked = torch.where(mine, dist_m, torch.full_like(dist_m, math.inf))
    if n_local:
        best = masked.min(dim=1).values
        loc = (mine & (masked == best[:, None])).to(torch.int8).argmax(dim=1)
    else:
        best = torch.full((R,), math.inf, dtype=torch.float64, device=dev)
        loc = torch.zeros((R,), dtype=torch.int64, device=dev)
    gidx = torch.where(torch.isinf(best), torch.full_like(best, math.inf), (loc + lo).to(torch.float64))
    cands = comm.all_gather_dev(torch.stack([best, gidx], dim=1)).view(comm.world, R, 2).cpu().numpy()
    g_assigned = comm.all_gather_dev(assigned)
    g_rowid = torch.searchsorted(keys_d, g_assigned)
    order = torch.argsort(g_rowid, stable=True)
    counts = torch.bincount(g_rowid, minlength=R)
    packed = torch.cat([g_assigned, order, counts]).cpu().numpy()  # one device->host copy
    g_assigned_h, order_h, counts_h = packed[:total], packed[total:2 * total], packed[2 * total:]
    starts = np.concatenate([[0], np.cumsum(counts_h)])
    result = []
    for k, (key, previous, _) in enumerate(rows):
        members = order_h[starts[k]:starts[k + 1]]
        if members.size == 0:
            continue
        c = cands[:, k, :]
        w = min(range(comm.world), key=lambda r: (c[r, 0], c[r, 1]))
        closest = int(c[w, 1])
        owner = _owner(closest, total, comm.world)
        if comm.rank == owner:
            rn_, rc_ = nd[closest - lo].clone(), cd[closest - lo].clone()
        else:
            rn_ = torch.empty(tuple(nd.shape[1:]), dtype=nd.dtype, device=dev)
            rc_ = torch.empty(tuple(cd.shape[1:]), dtype=cd.dtype, device=dev)
        rn_, rc_ = comm.broadcast_dev(rn_, owner), comm.broadcast_dev(rc_, owner)
        new_rep = GenomeTensors(rn_.cpu().numpy(), rc_.cpu().numpy(), n_in, n_out)
        if previous is not None:
            result.append(replace(previous, representative=new_rep, member_indices=members, spawn_count=0))
        else:
            result.append(SpeciesState(species_key=key, representative=new_rep, member_indices=members))
    return g_assigned_h, result


def sharded_reproduce_device(nd: torch.Tensor, cd: torch.Tensor, lo: int, species: list, fitness: np.ndarray,
                             config: NeatConfig, rng, allocator: NodeKeyAllocator, comm: Collective):
    """reproduce (evolution.py:646-715) for a sharded device population: the
    slot tables are built on every rank's GPU from the replicated species and
    fitness (the single-GPU path's device tables), the survivor-pool and elite
    genomes are all-gathered as device tensors, and this rank runs the fused
    kernel on its slot range.  Offspring are identical for any world size
    (global-slot RNG keys)."""
    import ctypes

    from . import _native
    from .device import ptr, stream_handle
    from .evolution import _slot_tables_device, mutate_params
    dev = nd.device
    total = config.pop_size
    base_key = allocator.reserve(total)
    pool_d, off_d, size_d, elite_d = _slot_tables_device(species, fitness, config)
    needed = torch.unique(torch.cat([pool_d.long(), elite_d[elite_d >= 0].long()]))  # sorted
    n_local = int(nd.shape[0])
    mine = needed[(needed >= lo) & (needed < lo + n_local)]
    idx_all = comm.all_gather_dev(mine)  # contiguous shards: ascending global order
    all_n = comm.all_gather_dev(nd.index_select(0, mine - lo))
    all_c = comm.all_gather_dev(cd.index_select(0, mine - lo))
    pool_r = torch.searchsorted(idx_all, pool_d.long()).to(torch.int32)
    elite_r = torch.where(elite_d >= 0, torch.searchsorted(idx_all, elite_d.clamp(min=0).long()).to(torch.int32),
                          torch.full_like(elite_d, -1))
    slo, shi = shard_range(total, comm.world, comm.rank)
    count = shi - slo
    n, c = int(nd.shape[1]), int(cd.shape[1])
    on = torch.empty((count, n, 5), dtype=torch.float64, device=dev)
    oc = torch.empty((count, c, 4), dtype=torch.float64, device=dev)
    off_s, size_s = off_d[slo:shi].contiguous(), size_d[slo:shi].contiguous()
    elite_s = elite_r[slo:shi].contiguous()
    stage_key = int(np.asarray(rng.child(STAGE_REPRODUCE)._keys).reshape(-1)[0])
    params = mutate_params(config, n, c)
    if count:
        _native.call("an_reproduce", ptr(all_n), ptr(all_c), ptr(on), ptr(oc), count, slo, ptr(pool_r),
                     ptr(off_s), ptr(size_s), ptr(elite_s), stage_key, float(base_key), ctypes.addressof(params),
                     None, stream_handle())
    return on, oc, (slo, shi)


def _sharded_evolve_step_device(nodes, conns, lo: int, species: list, config: NeatConfig, rng,
                                allocator: NodeKeyAllocator, problem, comm: Collective, ops):
    """sharded_evolve_step with the device-resident protocol (DeviceOps)."""
    from .evolution import _dev64
    total = config.pop_size
    nd, cd = _dev64(nodes), _dev64(conns)
    dev = nd.device
    fit_local = torch.from_numpy(np.ascontiguousarray(
        ops.fitness(problem, nd, cd, config.inputs, config.outputs, rng.child(STAGE_EVAL)))).to(dev)
    fitness = comm.all_gather_dev(fit_local).cpu().numpy()  # host bookkeeping is O(#species)
    best = int(fitness.argmax())
    owner = _owner(best, total, comm.world)
    if comm.rank == owner:
        bn, bc = nd[best - lo].clone(), cd[best - lo].clone()
    else:
        bn = torch.empty(tuple(nd.shape[1:]), dtype=nd.dtype, device=dev)
        bc = torch.empty(tuple(cd.shape[1:]), dtype=cd.dtype, device=dev)
    bn, bc = comm.broadcast_dev(bn, owner), comm.broadcast_dev(bc, owner)
    live = torch.stack([(~torch.isnan(nd[:, :, 0])).sum().to(torch.float64),
                        (~torch.isnan(cd[:, :, 0])).sum().to(torch.float64)])
    live = comm.all_reduce_dev(live).cpu().numpy()
    stats = GenerationStats(best_fitness=float(fitness[best]), mean_fitness=float(fitness.mean()),
                            species_count=len(species), mean_live_nodes=float(live[0] / total),
                            mean_live_conns=float(live[1] / total), elapsed_seconds=0.0, best_index=best,
                            solved=False, best_genome=GenomeTensors(bn.cpu().numpy(), bc.cpu().numpy(),
                                                                    config.inputs, config.outputs))
    if stats.best_fitness >= config.fitness_target:
        stats.solved = True
        return nodes, conns, lo, species, stats
    survivors = update_stagnation(species, fitness, config)
    if not survivors:
        from .errors import ExtinctionError
        raise ExtinctionError("all species stagnated; increase species_elitism")
    allocated = allocate_spawns(survivors, fitness, config)
    on, oc, (slo, _) = sharded_reproduce_device(nd, cd, lo, allocated, fitness, config, rng, allocator, comm)
    _, new_species = sharded_speciate_device(on, oc, slo, total, allocated, config, comm, config.inputs,
                                             config.outputs)
    return on, oc, slo, new_species, stats


def sharded_evolve_step(nodes, conns, lo: int, species: list, config: NeatConfig, rng,
                        allocator: NodeKeyAllocator, problem, comm: Collective, ops):
    """One generation over sharded populations (evolution.py:722-773).
    Returns (new local nodes, new local conns, new lo, species, stats).
    With ``DeviceOps`` the protocol runs on device tensors (the product path);
    other ``ops`` (the CPU stand-ins of the multi-process tests) use the
    host-array protocol below -- both give the single-GPU answer."""
    if isinstance(ops, DeviceOps):
        return _sharded_evolve_step_device(nodes, conns, lo, species, config, rng, allocator, problem, comm, ops)
    total = config.pop_size
    fit_local = ops.fitness(problem, nodes, conns, config.inputs, config.outputs, rng.child(STAGE_EVAL))
    fitness = np.concatenate(comm.all_gather(fit_local))
    best = int(fitness.argmax())
    owner = _owner(best, total, comm.world)
    mine = ops.genome(nodes, conns, best - lo) if comm.rank == owner else (None, None)
    bn = comm.broadcast(mine[0], (nodes.shape[1], 5), np.float64, owner)
    bc = comm.broadcast(mine[1], (conns.shape[1], 4), np.float64, owner)
    ln, lc = ops.live_counts(nodes, conns)
    live_n = np.concatenate(comm.all_gather(ln))
    live_c = np.concatenate(comm.all_gather(lc))
    stats = GenerationStats(best_fitness=float(fitness[best]), mean_fitness=float(fitness.mean()),
                            species_count=len(species), mean_live_nodes=float(live_n.mean()),
                            mean_live_conns=float(live_c.mean()), elapsed_seconds=0.0, best_index=best,
                            solved=False, best_genome=GenomeTensors(bn, bc, config.inputs, config.outputs))
    if stats.best_fitness >= config.fitness_target:
        stats.solved = True
        return nodes, conns, lo, species, stats
    survivors = update_stagnation(species, fitness, config)
    if not survivors:
        from .errors import ExtinctionError
        raise ExtinctionError("all species stagnated; increase species_elitism")
    allocated = allocate_spawns(survivors, fitness, config)
    on, oc, (slo, _) = sharded_reproduce(nodes, conns, lo, allocated, fitness, config, rng, allocator, comm, ops)
    _, new_species = sharded_speciate(on, oc, slo, total, allocated, config, comm, ops, config.inputs,
                                      config.outputs)
    return on, oc, slo, new_species, stats


__all__ = ["Collective", "DeviceOps", "shard_range", "sharded_speciate", "sharded_reproduce",
           "sharded_speciate_device", "sharded_reproduce_device", "sharded_evolve_step"]
