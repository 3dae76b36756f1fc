"""Population operators on the GPU: crossover, mutation, distance, speciation,
stagnation, spawn allocation, reproduction and the generation step.

Drop-in for reference evolution.py (same names, arguments and exceptions):
  * ``crossover_arrays`` / ``_crossover_into`` (evolution.py:101-151)  -> an_crossover
  * ``mutate_arrays`` (evolution.py:172-325, 328-407)                   -> an_mutate
  * ``distance_arrays`` (evolution.py:425-488)                          -> an_distance
  * ``speciate`` (evolution.py:513-576): existing-species assignment as one
    (R x P) distance launch; the sequential founding loop as at most
    ``max_species`` rounds of (first unassigned genome -> one distance pass);
  * ``update_stagnation`` / ``allocate_spawns`` (evolution.py:583-639): O(#species)
    host bookkeeping, as the survey prescribes;
  * ``reproduce`` (evolution.py:646-715): slot tables on the host, then one
    fused crossover + mutation + elite-overwrite launch (an_reproduce);
  * ``evolve_step`` (evolution.py:722-773).

Populations may be numpy arrays (reference behaviour: results come back as
numpy) or CUDA tensors (device-resident runs: results stay on the device).
Randomness uses the reference's counter-based tape (rng.py), so uniforms --
and therefore every structural decision -- match the reference bit for bit;
float64 attribute arithmetic rounds like numpy (no FMA); Box-Muller normals
may differ by ~1 ulp (CUDA vs numpy log/cos).
"""

from __future__ import annotations

import ctypes
import math
import time
from dataclasses import dataclass, field, replace

import numpy as np
import torch

from . import _native
from .config import NeatConfig
from .device import device, ptr, stream_handle
from .errors import ExtinctionError, ShapeMismatch
from .functions import DEFAULT_REGISTRY
from .genome import GenomeTensors, PopulationTensors

STAGE_INIT, STAGE_EVAL, STAGE_REPRODUCE, STAGE_SPECIATE = 0, 1, 2, 3
_SPAWN_EPSILON = 1e-9


@dataclass
class NodeKeyAllocator:
    """Monotone source of fresh node keys (evolution.py:41-52)."""
    next_key: int

    def reserve(self, count: int) -> int:
        first = self.next_key
        self.next_key += count
        return first

    def allocate(self) -> int:
        return self.reserve(1)


@dataclass
class SpeciesState:
    """Per-species bookkeeping (evolution.py:55-63)."""
    species_key: int
    representative: GenomeTensors
    member_indices: np.ndarray
    best_fitness_history: list = field(default_factory=list)
    stagnation_counter: int = 0
    spawn_count: int = 0


@dataclass
class GenerationStats:
    """Per-generation summary (evolution.py:66-77)."""
    best_fitness: float
    mean_fitness: float
    species_count: int
    mean_live_nodes: float
    mean_live_conns: float
    elapsed_seconds: float
    best_index: int
    solved: bool
    best_genome: GenomeTensors | None = None


# ---------------------------------------------------------------------------
# plumbing
# ---------------------------------------------------------------------------

def _dev64(x) -> torch.Tensor:
    dev = device()
    t = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.array(x, dtype=np.float64, copy=True))
    return t.to(dev, torch.float64).contiguous()


def _back(t: torch.Tensor, like):
    return t if isinstance(like, torch.Tensor) else t.cpu().numpy()


def mutate_params(config: NeatConfig, max_nodes: int | None = None, max_conns: int | None = None):
    p = _native.MutateParams()
    p.N = int(max_nodes if max_nodes is not None else config.max_nodes)
    p.C = int(max_conns if max_conns is not None else config.max_conns)
    p.I, p.O = config.inputs, config.outputs
    p.feedforward = 1 if config.network_type == "feedforward" else 0
    p.act_default, p.agg_default = config.activation_default_id, config.aggregation_default_id
    acts, aggs = config.activation_option_ids, config.aggregation_option_ids
    if len(acts) > 8 or len(aggs) > 8:
        raise ValueError("at most 8 activation / aggregation options")
    p.n_act_options, p.n_agg_options = len(acts), len(aggs)
    for i, a in enumerate(acts):
        p.act_options[i] = a
    for i, a in enumerate(aggs):
        p.agg_options[i] = a
    for name in ("node_add", "node_delete", "conn_add", "conn_delete",
                 "bias_init_mean", "bias_init_std", "bias_mutate_power", "bias_mutate_rate",
                 "bias_replace_rate", "response_init_mean", "response_init_std", "response_mutate_power",
                 "response_mutate_rate", "response_replace_rate", "weight_init_mean", "weight_init_std",
                 "weight_mutate_power", "weight_mutate_rate", "weight_replace_rate", "enabled_mutate_rate",
                 "activation_replace_rate", "aggregation_replace_rate", "attr_min", "attr_max"):
        setattr(p, name, float(getattr(config, name)))
    return p


def _keys_dev(rng, count: int) -> torch.Tensor:
    keys = np.asarray(rng._keys, dtype=np.uint64).reshape(-1)
    if keys.size == 1 and count > 1:
        keys = np.repeat(keys, count)
    if keys.size != count:
        raise ValueError(f"stream batch {keys.size} does not match {count} genomes")
    return torch.from_numpy(keys.view(np.int64).copy()).to(device())


def mutation_tape_width(config: NeatConfig, n: int, c: int) -> int:
    """Cells mutate_arrays consumes per genome."""
    w = 12
    for rep, mut, width in ((config.bias_replace_rate, config.bias_mutate_rate, n),
                            (config.response_replace_rate, config.response_mutate_rate, n),
                            (config.weight_replace_rate, config.weight_mutate_rate, c)):
        if rep == 0.0 and mut == 0.0:
            continue
        w += 2 * width + (2 * width if mut > 0.0 else 0) + (2 * width if rep > 0.0 else 0)
    if config.enabled_mutate_rate > 0.0:
        w += c
    w += 2 * n if config.activation_replace_rate > 0.0 else 0
    w += 2 * n if config.aggregation_replace_rate > 0.0 else 0
    return w


# ---------------------------------------------------------------------------
# crossover / mutation
# ---------------------------------------------------------------------------

def _crossover_into(out_nodes, out_conns, less_nodes, less_conns, rng) -> None:
    """Blend the less-fit parents into the (fitter-parent) outputs in place
    (evolution.py:101-136)."""
    on, oc = _dev64(out_nodes), _dev64(out_conns)
    ln, lc = _dev64(less_nodes), _dev64(less_conns)
    pop, n, _ = on.shape
    c = oc.shape[1]
    keys = _keys_dev(rng, pop)
    _native.call("an_crossover", ptr(on), ptr(oc), ptr(ln), ptr(lc), pop, n, c, ptr(keys), rng._counter,
                 stream_handle())
    rng._counter += 4 * n + 2 * c
    for dst, src in ((out_nodes, on), (out_conns, oc)):
        if isinstance(dst, torch.Tensor):
            if dst.data_ptr() != src.data_ptr():
                dst.copy_(src)
        else:
            dst[...] = src.cpu().numpy()


def crossover_arrays(fit_nodes, fit_conns, less_nodes, less_conns, rng):
    """Masked blend of aligned gene tensors (evolution.py:139-151)."""
    on = _dev64(fit_nodes).clone()
    oc = _dev64(fit_conns).clone()
    _crossover_into(on, oc, less_nodes, less_conns, rng)
    return _back(on, fit_nodes), _back(oc, fit_conns)


def crossover(parent_fit: GenomeTensors, parent_less: GenomeTensors, rng) -> GenomeTensors:
    """Single-pair crossover (evolution.py:154-165)."""
    if (parent_fit.num_inputs, parent_fit.num_outputs) != (parent_less.num_inputs, parent_less.num_outputs):
        raise ShapeMismatch("parents disagree on input/output counts")
    if parent_fit.nodes.shape != parent_less.nodes.shape or parent_fit.conns.shape != parent_less.conns.shape:
        raise ShapeMismatch("parents disagree on tensor capacity")
    n, c = crossover_arrays(parent_fit.nodes[None], parent_fit.conns[None], parent_less.nodes[None],
                            parent_less.conns[None], rng)
    return GenomeTensors(n[0], c[0], parent_fit.num_inputs, parent_fit.num_outputs)


def mutate_arrays(nodes, conns, config: NeatConfig, rng, new_node_keys, copy: bool = True):
    """The five mutation sub-steps for every genome (evolution.py:172-325).

    Returns (nodes, conns, can_add).  With ``copy=False`` and CUDA tensors
    the inputs are mutated in place (numpy inputs are written back)."""
    nd, cd = _dev64(nodes), _dev64(conns)
    if copy and isinstance(nodes, torch.Tensor) and nd.data_ptr() == nodes.data_ptr():
        nd, cd = nd.clone(), cd.clone()
    pop, n, _ = nd.shape
    c = cd.shape[1]
    keys = _keys_dev(rng, pop)
    nk = _dev64(np.broadcast_to(np.asarray(new_node_keys, dtype=np.float64), (pop,)) if not isinstance(
        new_node_keys, torch.Tensor) else new_node_keys)
    can_add = torch.zeros(pop, dtype=torch.uint8, device=nd.device)
    params = mutate_params(config, n, c)
    _native.call("an_mutate", ptr(nd), ptr(cd), pop, ptr(keys), rng._counter, ptr(nk),
                 ctypes.addressof(params), ptr(can_add), stream_handle())
    rng._counter += mutation_tape_width(config, n, c)
    if not copy:
        for dst, src in ((nodes, nd), (conns, cd)):
            if isinstance(dst, torch.Tensor):
                if dst.data_ptr() != src.data_ptr():
                    dst.copy_(src)
            else:
                dst[...] = src.cpu().numpy()
        nd, cd = nodes, conns
    ca = can_add.bool()
    return _back(nd, nodes), _back(cd, conns), (ca if isinstance(nodes, torch.Tensor) else ca.cpu().numpy())


def mutate(genome: GenomeTensors, config: NeatConfig, rng, allocator: NodeKeyAllocator) -> GenomeTensors:
    """One genome; consumes an allocator key only if node addition fires (evolution.py:410-418)."""
    n, c, added = mutate_arrays(genome.nodes[None], genome.conns[None], config, rng,
                                np.array([float(allocator.next_key)]))
    if added[0]:
        allocator.allocate()
    return GenomeTensors(n[0], c[0], genome.num_inputs, genome.num_outputs)


# ---------------------------------------------------------------------------
# distance and speciation
# ---------------------------------------------------------------------------

def _distance_dev(n1, c1, n2, c2, config, pair_mode: int) -> torch.Tensor:
    pop, q = int(n1.shape[0]), int(n2.shape[0])
    n, c = int(n1.shape[1]), int(c1.shape[1])
    out = torch.empty((pop if pair_mode else q * pop,), dtype=torch.float64, device=n1.device)
    _native.call("an_distance", ptr(n1), ptr(c1), pop, ptr(n2), ptr(c2), q, pair_mode, n, c,
                 float(config.compatibility_disjoint), float(config.compatibility_homologous), ptr(out),
                 stream_handle())
    return out if pair_mode else out.view(q, pop)


def distance_arrays(nodes1, conns1, nodes2, conns2, config: NeatConfig):
    """Pairwise distance with broadcasting of a batch-1 second operand
    (evolution.py:425-488); bit-exact float64."""
    n1, c1, n2, c2 = _dev64(nodes1), _dev64(conns1), _dev64(nodes2), _dev64(conns2)
    if n1.shape[1:] != n2.shape[1:] or c1.shape[1:] != c2.shape[1:]:
        raise ShapeMismatch("operands disagree on tensor capacity")
    return _back(_distance_dev(n1, c1, n2, c2, config, 1), nodes1)


def distance(g1: GenomeTensors, g2: GenomeTensors, config: NeatConfig) -> float:
    if (g1.num_inputs, g1.num_outputs) != (g2.num_inputs, g2.num_outputs):
        raise ShapeMismatch("genomes disagree on input/output counts")
    return float(distance_arrays(g1.nodes[None], g1.conns[None], g2.nodes[None], g2.conns[None], config)[0])


def _genome_host(nodes, conns, i: int, n_in: int, n_out: int) -> GenomeTensors:
    n, c = nodes[i], conns[i]
    if isinstance(n, torch.Tensor):
        n, c = n.cpu().numpy(), c.cpu().numpy()
    return GenomeTensors(np.array(n, copy=True), np.array(c, copy=True), n_in, n_out)


# populations up to this size run the speciation bookkeeping on the host (one
# read-back of the distance rows; launch latency dominates small populations);
# larger ones keep it on the device
SMALL_SPECIATE = 8192


def _speciate_host(pop, nd, cd, ordered: list, config: NeatConfig):
    """speciate() for small populations: device distance rows, host bookkeeping
    (same decisions as the device path and the reference loop)."""
    count = int(nd.shape[0])
    thr = float(config.compatibility_threshold)
    rows = []  # (key, previous state or None, distance row (P,) host)
    assigned = np.full(count, -1, dtype=np.int64)
    if ordered:
        rn = _dev64(np.stack([sp.representative.nodes for sp in ordered]))
        rc = _dev64(np.stack([sp.representative.conns for sp in ordered]))
        mat = _distance_dev(nd, cd, rn, rc, config, 0).cpu().numpy().reshape(len(ordered), count)
        rows = [(sp.species_key, sp, mat[k]) for k, sp in enumerate(ordered)]
        ok = mat <= thr
        keys = np.array([sp.species_key for sp in ordered], dtype=np.int64)
        assigned = np.where(ok.any(axis=0), keys[ok.argmax(axis=0)], assigned)
    next_key = max((r[0] for r in rows), default=-1) + 1
    while True:
        free = np.flatnonzero(assigned < 0)
        if free.size == 0:
            break
        if len(rows) < config.max_species:
            i = int(free[0])
            d = _distance_dev(nd, cd, nd[i:i + 1], cd[i:i + 1], config, 1).cpu().numpy().reshape(count)
            rows.append((next_key, None, d))
            take = (assigned < 0) & (d <= thr)
            take[i] = True
            assigned[take] = next_key
            next_key += 1
        else:
            keys = np.array([r[0] for r in rows], dtype=np.int64)
            near = keys[np.stack([r[2] for r in rows]).argmin(axis=0)]
            assigned = np.where(assigned < 0, near, assigned)
            break
    members, closest = [], []
    for key, _, d in rows:
        m = np.flatnonzero(assigned == key)
        members.append(m)
        closest.append(int(m[int(np.argmin(d[m]))]) if m.size else 0)
    return rows, assigned, members, closest


def speciate(pop: PopulationTensors, species: list, config: NeatConfig, rng=None, sequential: bool = False):
    """Assign species and refresh representatives (evolution.py:513-576)."""
    nd, cd = _dev64(pop.nodes), _dev64(pop.conns)
    count = int(nd.shape[0])
    if count <= SMALL_SPECIATE:
        ordered = sorted(species, key=lambda sp: sp.species_key)
        rows, assigned_h, members_l, closest = _speciate_host(pop, nd, cd, ordered, config)
        idx = torch.tensor(closest, dtype=torch.int64, device=nd.device)
        reps_n = nd.index_select(0, idx).cpu().numpy()
        reps_c = cd.index_select(0, idx).cpu().numpy()
        result = []
        for k, (key, previous, _) in enumerate(rows):
            if members_l[k].size == 0:
                continue
            new_rep = GenomeTensors(reps_n[k].copy(), reps_c[k].copy(), pop.num_inputs, pop.num_outputs)
            if previous is not None:
                result.append(replace(previous, representative=new_rep, member_indices=members_l[k],
                                      spawn_count=0))
            else:
                result.append(SpeciesState(species_key=key, representative=new_rep, member_indices=members_l[k]))
        return PopulationTensors(pop.nodes, pop.conns, assigned_h.astype(np.int64), pop.fitness,
                                 pop.num_inputs, pop.num_outputs), result
    thr = float(config.compatibility_threshold)
    ordered = sorted(species, key=lambda s: s.species_key)
    rows: list = []  # (key, previous state or None, representative, distance row (P,) on device)
    assigned = torch.full((count,), -1, dtype=torch.int64, device=nd.device)
    if ordered:
        rn = _dev64(np.stack([s.representative.nodes for s in ordered]))
        rc = _dev64(np.stack([s.representative.conns for s in ordered]))
        mat = _distance_dev(nd, cd, rn, rc, config, 0)  # (R, P)
        for k, sp in enumerate(ordered):
            rows.append((sp.species_key, sp, sp.representative, mat[k]))
        ok = mat <= thr
        any_ok = ok.any(dim=0)
        first = ok.to(torch.int8).argmax(dim=0)
        keys = torch.tensor([s.species_key for s in ordered], dtype=torch.int64, device=nd.device)
        assigned = torch.where(any_ok, keys[first], assigned)
    next_key = max((r[0] for r in rows), default=-1) + 1
    # founding rounds: the first still-unassigned genome founds a species and
    # takes every unassigned genome within the threshold (exactly the
    # reference's index-order loop, evolution.py:542-559)
    while True:
        has_free, first_free = (assigned < 0).to(torch.int8).max(dim=0)  # max -> first index of it
        if not bool(has_free):
            break
        if len(rows) < config.max_species:
            i = int(first_free)
            d = _distance_dev(nd, cd, nd[i:i + 1], cd[i:i + 1], config, 1)
            rows.append((next_key, None, None, d))  # representative: refreshed below
            take = (assigned < 0) & (d <= thr)
            take[i] = True
            assigned = torch.where(take, torch.full_like(assigned, next_key), assigned)
            next_key += 1
        else:
            mat = torch.stack([r[3] for r in rows])
            keys = torch.tensor([r[0] for r in rows], dtype=torch.int64, device=nd.device)
            near = keys[mat.argmin(dim=0)]
            assigned = torch.where(assigned < 0, near, assigned)
            break
    # representative refresh on the device: members of row r are the genomes
    # assigned its key; the new representative is the member closest to the
    # row's old representative, first index on ties (evolution.py:561-573)
    R = len(rows)
    keys_d = torch.tensor([r[0] for r in rows], dtype=torch.int64, device=nd.device)
    rowid = torch.searchsorted(keys_d, assigned)  # row keys are ascending
    dist = torch.stack([r[3] for r in rows])  # (R, P)
    mine = torch.arange(R, device=nd.device)[:, None] == rowid[None, :]
    masked = torch.where(mine, dist, torch.full_like(dist, math.inf))
    best = masked.min(dim=1, keepdim=True).values
    hit = mine & (masked == best)
    closest_d = hit.to(torch.int8).argmax(dim=1)  # first index reaching the minimum
    order = torch.argsort(rowid, stable=True)  # members grouped by row, ascending index
    counts = torch.bincount(rowid, minlength=R)
    # one device->host copy for the assignment, grouping and new representatives
    packed = torch.cat([assigned, order, counts, closest_d]).cpu().numpy()
    assigned_h, order_h = packed[:count], packed[count:2 * count]
    counts_h, closest_h = packed[2 * count:2 * count + R], packed[2 * count + R:]
    reps_n = nd.index_select(0, closest_d).cpu().numpy()
    reps_c = cd.index_select(0, closest_d).cpu().numpy()
    starts = np.concatenate([[0], np.cumsum(counts_h)])
    result = []
    for k, (key, previous, rep, drow) in enumerate(rows):
        members = order_h[starts[k]:starts[k + 1]]
        if members.size == 0:
            continue
        new_rep = GenomeTensors(reps_n[k].copy(), reps_c[k].copy(), pop.num_inputs, pop.num_outputs)
        if previous is not None:
            result.append(replace(previous, representative=new_rep, member_indices=members, spawn_count=0))
        else:
            result.append(SpeciesState(species_key=key, representative=new_rep, member_indices=members))
    new_pop = PopulationTensors(pop.nodes, pop.conns, assigned_h.astype(np.int64), pop.fitness,
                                pop.num_inputs, pop.num_outputs)
    return new_pop, result


# ---------------------------------------------------------------------------
# stagnation, spawn allocation (host; O(#species))
# ---------------------------------------------------------------------------

def update_stagnation(species: list, fitness, config: NeatConfig) -> list:
    """Species fitness = member max; counter resets on strict improvement; the
    top ``species_elitism`` species are always kept (evolution.py:583-604)."""
    fit = np.asarray(fitness.cpu().numpy() if isinstance(fitness, torch.Tensor) else fitness)
    scored = []
    for sp in sorted(species, key=lambda s: s.species_key):
        now = float(fit[sp.member_indices].max())
        best = max(sp.best_fitness_history) if sp.best_fitness_history else -math.inf
        scored.append((now, replace(sp, best_fitness_history=sp.best_fitness_history + [now],
                                    stagnation_counter=0 if now > best else sp.stagnation_counter + 1)))
    ranked = sorted(scored, key=lambda x: (-x[0], x[1].species_key))
    keep = {x[1].species_key for x in ranked[:config.species_elitism]}
    return [sp for _, sp in scored if sp.species_key in keep or sp.stagnation_counter < config.max_stagnation]


def allocate_spawns(species: list, fitness, config: NeatConfig) -> list:
    """Next-generation slots per species (evolution.py:607-639)."""
    if not species:
        raise ExtinctionError("no species left to allocate spawns to")
    fit = np.asarray(fitness.cpu().numpy() if isinstance(fitness, torch.Tensor) else fitness)
    ordered = sorted(species, key=lambda s: s.species_key)
    means = np.array([float(fit[s.member_indices].mean()) for s in ordered])
    old = np.array([s.member_indices.size for s in ordered], dtype=np.float64)
    shifted = means - means.min() + _SPAWN_EPSILON
    targets = shifted / shifted.sum() * config.pop_size
    r = config.spawn_number_change_rate
    step = np.clip(targets - old, -(r * old + 1.0), r * old + 1.0)
    spawn = np.maximum(np.round(old + step), 1.0).astype(np.int64)
    spawn[int(spawn.argmax())] += config.pop_size - int(spawn.sum())
    while spawn.min() < 1:
        needy, donor = int(spawn.argmin()), int(spawn.argmax())
        if donor == needy or spawn[donor] <= 1:
            raise ExtinctionError("cannot satisfy spawn floor of one per species")
        give = min(1 - int(spawn[needy]), int(spawn[donor]) - 1)
        spawn[needy] += give
        spawn[donor] -= give
    return [replace(s, spawn_count=int(n)) for s, n in zip(ordered, spawn)]


# ---------------------------------------------------------------------------
# reproduction and the generation step
# ---------------------------------------------------------------------------

def _ranked_head(m: np.ndarray, fit: np.ndarray, k: int) -> np.ndarray:
    """First k of ``m[lexsort((m, -fit[m]))]`` (fitness descending, index
    ascending on ties; NaN last) without sorting the whole species: an O(n)
    partition picks the candidates at or above the k-th value, then only
    those are sorted."""
    if k >= m.size or m.size < 4096:
        return m[np.lexsort((m, -fit[m]))][:k]
    neg = -fit[m]
    kth = np.partition(neg, k - 1)[k - 1]
    if np.isnan(kth):
        return m[np.lexsort((m, neg))][:k]
    cand = m[neg <= kth]
    return cand[np.lexsort((cand, -fit[cand]))][:k]


def _ranked_heads_device(ordered: list, fit: np.ndarray, heads: list) -> list:
    """For each species (in key order) the first heads[k] members ranked by
    (fitness descending, index ascending; NaN last): three stable device sorts
    over the population and one read-back of the heads."""
    dev = device()
    count = fit.size
    rowid = np.full(count, len(ordered), dtype=np.int64)  # genomes of dropped species sort last
    for k, sp in enumerate(ordered):
        rowid[np.asarray(sp.member_indices)] = k
    f = torch.from_numpy(np.ascontiguousarray(fit)).to(dev)
    nan = torch.isnan(f)
    key = torch.where(nan, torch.zeros_like(f), -f) + 0.0  # + 0.0: -0.0 -> +0.0, ties as in numpy
    idx = torch.argsort(key, stable=True)
    idx = idx[torch.argsort(nan[idx].to(torch.int8), stable=True)]
    rid = torch.from_numpy(rowid).to(dev)
    order = idx[torch.argsort(rid[idx], stable=True)]
    starts = np.concatenate([[0], np.cumsum([np.asarray(sp.member_indices).size for sp in ordered])])
    parts = [order[int(starts[k]):int(starts[k]) + heads[k]] for k in range(len(ordered))]
    flat = torch.cat(parts).cpu().numpy() if parts else np.zeros(0, dtype=np.int64)
    out, at = [], 0
    for h in heads:
        out.append(flat[at:at + h])
        at += h
    return out


# populations above this size rank the parent pools on the device
SMALL_SLOT_TABLES = 65536


def slot_tables(species: list, fitness, config: NeatConfig):
    """Deterministic slot layout (evolution.py:659-679): species in key order,
    elites first; parent pool = top ceil(survival * n) by (-fitness, index)."""
    fit = np.asarray(fitness.cpu().numpy() if isinstance(fitness, torch.Tensor) else fitness)
    total = config.pop_size
    ordered = sorted(species, key=lambda s: s.species_key)
    heads = [max(max(1, math.ceil(config.survival_threshold * np.asarray(sp.member_indices).size)),
                 min(config.genome_elitism, sp.spawn_count, np.asarray(sp.member_indices).size))
             for sp in ordered]
    ranked = _ranked_heads_device(ordered, fit, heads) if fit.size > SMALL_SLOT_TABLES else None
    elite = np.full(total, -1, dtype=np.int32)
    off = np.zeros(total, dtype=np.int32)
    size = np.ones(total, dtype=np.int32)
    pools = []
    slot, pooled = 0, 0
    for k, sp in enumerate(ordered):
        m = np.asarray(sp.member_indices)
        spawn = sp.spawn_count
        n_surv = max(1, math.ceil(config.survival_threshold * m.size))
        n_el = min(config.genome_elitism, spawn, m.size)
        ranking = ranked[k] if ranked is not None else _ranked_head(m, fit, max(n_surv, n_el))
        elite[slot:slot + n_el] = ranking[:n_el]
        surv = ranking[:n_surv]
        off[slot + n_el:slot + spawn] = pooled
        size[slot + n_el:slot + spawn] = surv.size
        pools.append(surv)
        pooled += surv.size
        slot += spawn
    if slot != total:
        raise ExtinctionError(f"spawn counts sum to {slot}, expected {total}")
    pool = np.concatenate(pools).astype(np.int32) if pools else np.zeros(1, dtype=np.int32)
    return pool, off, size, elite


def _slot_tables_device(species: list, fitness, config: NeatConfig) -> tuple:
    """``slot_tables`` built on the device for large populations: the same
    parent ranking (three stable device sorts), then the pool, per-slot pool
    offset/size and elite source by gathers -- no read-back of the ranked heads
    and no table upload.  Returns int32 device tensors (pool, off, size, elite)."""
    fit = np.asarray(fitness.cpu().numpy() if isinstance(fitness, torch.Tensor) else fitness)
    total = config.pop_size
    ordered = sorted(species, key=lambda s: s.species_key)
    members = [np.asarray(sp.member_indices) for sp in ordered]
    sizes = np.array([m.size for m in members], dtype=np.int64)
    spawn = np.array([sp.spawn_count for sp in ordered], dtype=np.int64)
    n_surv = np.array([max(1, math.ceil(config.survival_threshold * n)) for n in sizes], dtype=np.int64)
    n_el = np.minimum(np.minimum(config.genome_elitism, spawn), sizes)
    if int(spawn.sum()) != total:
        raise ExtinctionError(f"spawn counts sum to {int(spawn.sum())}, expected {total}")
    dev = device()
    rowid = np.full(fit.size, len(ordered), dtype=np.int64)  # genomes of dropped species sort last
    for k, m in enumerate(members):
        rowid[m] = k
    f = torch.from_numpy(np.ascontiguousarray(fit)).to(dev)
    nan = torch.isnan(f)
    key = torch.where(nan, torch.zeros_like(f), -f) + 0.0  # -0.0 -> +0.0, ties as in numpy
    idx = torch.argsort(key, stable=True)
    idx = idx[torch.argsort(nan[idx].to(torch.int8), stable=True)]
    rid = torch.from_numpy(rowid).to(dev)
    order = idx[torch.argsort(rid[idx], stable=True)]  # species rank, fitness desc, index asc
    starts = np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(np.int64)
    pooled = np.concatenate([[0], np.cumsum(n_surv)[:-1]]).astype(np.int64)
    small = torch.from_numpy(np.stack([starts, pooled, n_surv, n_el, spawn])).to(dev)
    st_d, pooled_d, surv_d, el_d, spawn_d = small
    ks = torch.arange(len(ordered), device=dev)
    # pool: the first n_surv members of every species, in species order
    pseg = torch.repeat_interleave(ks, surv_d)
    pool = order[st_d[pseg] + torch.arange(pseg.numel(), device=dev) - pooled_d[pseg]]
    # per slot: species segment, position inside it, elite or pool draw
    seg = torch.repeat_interleave(ks, spawn_d)
    slot0 = torch.cumsum(spawn_d, 0) - spawn_d
    pos = torch.arange(total, device=dev) - slot0[seg]
    is_el = pos < el_d[seg]
    elite = torch.where(is_el, order[st_d[seg] + torch.where(is_el, pos, 0)], -1)
    off = torch.where(is_el, 0, pooled_d[seg])
    size = torch.where(is_el, 1, surv_d[seg])
    if pool.numel() == 0:
        pool = torch.zeros(1, dtype=torch.int64, device=dev)
    return tuple(t.to(torch.int32) for t in (pool, off, size, elite))


def reproduce(pop: PopulationTensors, species: list, fitness, config: NeatConfig, rng,
              allocator: NodeKeyAllocator, threads: int = 1, sequential: bool = False) -> PopulationTensors:
    """Next generation (evolution.py:646-715): slot tables here, then one
    fused crossover + mutation + elite launch; slot s draws from stream
    (generation, STAGE_REPRODUCE, s) and owns node key base + s."""
    total = config.pop_size
    base_key = allocator.reserve(total)
    nd, cd = _dev64(pop.nodes), _dev64(pop.conns)
    dev = nd.device
    n, c = int(nd.shape[1]), int(cd.shape[1])
    on = torch.empty((total, n, 5), dtype=torch.float64, device=dev)
    oc = torch.empty((total, c, 4), dtype=torch.float64, device=dev)
    count = fitness.numel() if isinstance(fitness, torch.Tensor) else np.asarray(fitness).size
    if count > SMALL_SLOT_TABLES:
        pool_d, off_d, size_d, elite_d = _slot_tables_device(species, fitness, config)
    else:
        pool, off, size, elite = slot_tables(species, fitness, config)
        # one host->device copy for the four slot tables; the device views stay
        # referenced until the launch is enqueued
        tabs = torch.from_numpy(np.concatenate([pool, off, size, elite]).astype(np.int32)).to(dev)
        npool = pool.size
        pool_d, off_d = tabs[:npool], tabs[npool:npool + total]
        size_d, elite_d = tabs[npool + total:npool + 2 * total], tabs[npool + 2 * total:]
    stage_key = int(np.asarray(rng.child(STAGE_REPRODUCE)._keys).reshape(-1)[0])
    params = mutate_params(config, n, c)
    _native.call("an_reproduce", ptr(nd), ptr(cd), ptr(on), ptr(oc), total, 0, ptr(pool_d), ptr(off_d),
                 ptr(size_d), ptr(elite_d), stage_key, float(base_key), ctypes.addressof(params), None,
                 stream_handle())
    keep_dev = isinstance(pop.nodes, torch.Tensor)
    return PopulationTensors(on if keep_dev else on.cpu().numpy(), oc if keep_dev else oc.cpu().numpy(),
                             np.full(total, -1, dtype=np.int64), np.full(total, np.nan),
                             pop.num_inputs, pop.num_outputs)


def evolve_step(pop: PopulationTensors, species: list, config: NeatConfig, rng, allocator: NodeKeyAllocator,
                problem, registry=None, threads: int = 1, sequential: bool = False):
    """Evaluate, then stagnate, allocate, reproduce and re-speciate
    (evolution.py:722-773).  ``rng`` is scoped to the generation."""
    from .device import nvtx
    registry = registry or DEFAULT_REGISTRY
    start = time.perf_counter()
    with nvtx("evolve_step.evaluate"):
        fitness = np.asarray(problem.evaluate_population_tensors(pop, registry, rng.child(STAGE_EVAL),
                                                                 threads=threads, sequential=sequential),
                             dtype=np.float64)
    evaluated = PopulationTensors(pop.nodes, pop.conns, pop.species_id, fitness, pop.num_inputs,
                                  pop.num_outputs)
    nd, cd = _dev64(pop.nodes), _dev64(pop.conns)
    best = int(fitness.argmax())
    # one read-back: live node / connection counts and the best genome
    n_, c_ = int(nd.shape[1]), int(cd.shape[1])
    packed = torch.cat([(~torch.isnan(nd[:, :, 0])).sum(dim=1).to(torch.float64),
                        (~torch.isnan(cd[:, :, 0])).sum(dim=1).to(torch.float64),
                        nd[best].reshape(-1), cd[best].reshape(-1)]).cpu().numpy()
    count = nd.shape[0]
    live_nodes, live_conns = packed[:count], packed[count:2 * count]
    best_n = packed[2 * count:2 * count + 5 * n_].reshape(n_, 5).copy()
    best_c = packed[2 * count + 5 * n_:].reshape(c_, 4).copy()
    stats = GenerationStats(best_fitness=float(fitness[best]), mean_fitness=float(fitness.mean()),
                            species_count=len(species), mean_live_nodes=float(live_nodes.mean()),
                            mean_live_conns=float(live_conns.mean()), elapsed_seconds=0.0, best_index=best,
                            solved=False,
                            best_genome=GenomeTensors(best_n, best_c, pop.num_inputs, pop.num_outputs))
    if stats.best_fitness >= config.fitness_target:
        stats.solved = True
        stats.elapsed_seconds = time.perf_counter() - start
        return evaluated, species, stats
    with nvtx("evolve_step.stagnation_spawns"):
        survivors = update_stagnation(species, fitness, config)
        if not survivors:
            raise ExtinctionError("all species stagnated; increase species_elitism")
        allocated = allocate_spawns(survivors, fitness, config)
    with nvtx("evolve_step.reproduce"):
        offspring = reproduce(evaluated, allocated, fitness, config, rng, allocator, threads=threads,
                              sequential=sequential)
    with nvtx("evolve_step.speciate"):
        new_pop, new_species = speciate(offspring, allocated, config, rng.child(STAGE_SPECIATE),
                                        sequential=sequential)
    stats.elapsed_seconds = time.perf_counter() - start
    return new_pop, new_species, stats
