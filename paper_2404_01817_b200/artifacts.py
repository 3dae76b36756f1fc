"""Host-side artifacts of a run: genome text format, integrity checks and
checkpoints.

Byte-compatible with the reference so files move between the two:
  * ``serialize_genome`` / ``parse_genome`` -- the JSON genome document of
    genome.py:339-396 (one gene row per line, NaN cells as ``null``,
    round-trips bitwise including padding rows);
  * ``check_integrity`` -- the structural invariants of genome.py:289-328;
  * ``save_checkpoint`` / ``load_checkpoint`` -- the pickle payload of
    runner.py:78-127 (numpy arrays; device populations are copied to the host
    on save and come back as host arrays that the kernels accept directly).
  * ``export_genome`` -- one genome of a device population as a host
    ``GenomeTensors`` (the "export best genome from the GPU path" of §8f.3).
"""

from __future__ import annotations

import json
import math
import pickle

import numpy as np

from .config import dump_config, parse_config_text
from .errors import IntegrityError, ParseError
from .genome import GenomeTensors, PopulationTensors

NODE_KEY, CONN_IN, CONN_OUT, CONN_ENABLED = 0, 0, 1, 2
_HEADER_FIELDS = ("num_inputs", "num_outputs", "max_nodes", "max_conns")


def _host(a) -> np.ndarray:
    if hasattr(a, "detach"):
        return a.detach().cpu().numpy()
    return np.asarray(a)


def export_genome(pop: PopulationTensors, index: int) -> GenomeTensors:
    """Genome ``index`` of a (device or host) population as host float64 arrays."""
    nodes = _host(pop.nodes[index]).astype(np.float64, copy=True)
    conns = _host(pop.conns[index]).astype(np.float64, copy=True)
    return GenomeTensors(nodes, conns, pop.num_inputs, pop.num_outputs)


# ---------------------------------------------------------------------------
# integrity (genome.py:289-328)
# ---------------------------------------------------------------------------

def check_integrity(genome: GenomeTensors, exc: type[Exception] = IntegrityError) -> None:
    """Raise ``exc`` when the genome breaks a structural invariant: row shapes,
    all-or-nothing NaN rows, non-negative integer distinct keys, every io key
    present, distinct live (in, out) pairs whose endpoints are live, enabled
    flags in {0, 1}."""
    nodes, conns = np.asarray(genome.nodes), np.asarray(genome.conns)
    if nodes.ndim != 2 or nodes.shape[1] != 5:
        raise exc(f"node tensor must have shape (max_nodes, 5), got {nodes.shape}")
    if conns.ndim != 2 or conns.shape[1] != 4:
        raise exc(f"connection tensor must have shape (max_conns, 4), got {conns.shape}")
    for label, t in (("node", nodes), ("connection", conns)):
        holes = np.isnan(t)
        partial = holes.any(axis=1) != holes.all(axis=1)
        if partial.any():
            raise exc(f"{label} row {int(np.argmax(partial))} mixes NaN and live entries")
    keys = nodes[~np.isnan(nodes[:, NODE_KEY]), NODE_KEY]
    if (keys < 0).any() or (np.floor(keys) != keys).any():
        raise exc("node keys must be non-negative integers")
    if len(set(keys.tolist())) != keys.size:
        raise exc("live node keys must be pairwise distinct")
    present = set(keys.tolist())
    for k in range(genome.num_inputs + genome.num_outputs):
        if float(k) not in present:
            raise exc(f"{'input' if k < genome.num_inputs else 'output'} node key {k} is missing")
    live = conns[~np.isnan(conns[:, CONN_IN])]
    if live.shape[0]:
        pairs = {(a, b) for a, b in live[:, :2].tolist()}
        if len(pairs) != live.shape[0]:
            raise exc("live connection key pairs must be pairwise distinct")
        for col, label in ((CONN_IN, "in_key"), (CONN_OUT, "out_key")):
            for v in live[:, col].tolist():
                if v not in present:
                    raise exc(f"connection {label} {v} does not refer to a live node")
        en = live[:, CONN_ENABLED]
        if not ((en == 0.0) | (en == 1.0)).all():
            raise exc("enabled flags must be 0.0 or 1.0")


# ---------------------------------------------------------------------------
# JSON genome document (genome.py:339-396)
# ---------------------------------------------------------------------------

def _row_text(row) -> str:
    return json.dumps([None if (isinstance(v, float) and math.isnan(v)) else v for v in row])


def serialize_genome(genome: GenomeTensors) -> bytes:
    """UTF-8 JSON: header integers, then ``nodes`` and ``conns`` one row per line."""
    nodes, conns = _host(genome.nodes), _host(genome.conns)
    lines = ["{"]
    for name, value in zip(_HEADER_FIELDS, (genome.num_inputs, genome.num_outputs, nodes.shape[0],
                                            conns.shape[0])):
        lines.append(f' "{name}": {int(value)},')
    for name, t, last in (("nodes", nodes, False), ("conns", conns, True)):
        body = ",\n".join("  " + _row_text(r) for r in t.tolist())
        lines.append(f' "{name}": [\n{body}\n ]' + ("" if last else ","))
    lines.append("}")
    return ("\n".join(lines) + "\n").encode("utf-8")


def _cells_to_array(doc: dict, name: str, rows: int, cols: int) -> np.ndarray:
    cells = doc[name]
    if not isinstance(cells, list) or len(cells) != rows:
        raise ParseError(f"field {name!r}: expected {rows} rows")
    out = np.full((rows, cols), np.nan)
    for i, row in enumerate(cells):
        if not isinstance(row, list) or len(row) != cols:
            raise ParseError(f"field {name!r}, row {i}: expected {cols} cells")
        for j, v in enumerate(row):
            if v is None:
                continue
            if isinstance(v, bool) or not isinstance(v, (int, float)):
                raise ParseError(f"field {name!r}, row {i}, cell {j}: expected a number or null, got {v!r}")
            out[i, j] = float(v)
    return out


def parse_genome(data) -> GenomeTensors:
    """Inverse of ``serialize_genome`` (bitwise, padding included); ParseError on
    malformed documents or broken invariants."""
    text = data.decode("utf-8") if isinstance(data, (bytes, bytearray)) else data
    try:
        doc = json.loads(text)
    except json.JSONDecodeError as err:
        raise ParseError(f"line {err.lineno}, column {err.colno}: {err.msg}") from None
    if not isinstance(doc, dict):
        raise ParseError("genome document must be a JSON object")
    for name in (*_HEADER_FIELDS, "nodes", "conns"):
        if name not in doc:
            raise ParseError(f"missing field {name!r}")
    for name in _HEADER_FIELDS:
        v = doc[name]
        if isinstance(v, bool) or not isinstance(v, int) or v < 0:
            raise ParseError(f"field {name!r}: expected a non-negative integer")
    genome = GenomeTensors(_cells_to_array(doc, "nodes", doc["max_nodes"], 5),
                           _cells_to_array(doc, "conns", doc["max_conns"], 4),
                           doc["num_inputs"], doc["num_outputs"])
    check_integrity(genome, exc=ParseError)
    return genome


# ---------------------------------------------------------------------------
# checkpoints (runner.py:78-127)
# ---------------------------------------------------------------------------

def checkpoint_payload(state) -> dict:
    """The reference's pickle payload for an ``EvolutionState`` (host arrays)."""
    pop = state.population
    species = []
    for sp in state.species:
        rep = sp.representative
        species.append({
            "species_key": int(sp.species_key),
            "rep_nodes": _host(rep.nodes).astype(np.float64),
            "rep_conns": _host(rep.conns).astype(np.float64),
            "member_indices": _host(sp.member_indices),
            "best_fitness_history": list(sp.best_fitness_history),
            "stagnation_counter": int(sp.stagnation_counter),
            "spawn_count": int(sp.spawn_count),
        })
    fitness = pop.fitness if pop.fitness is not None else np.full(pop.size, np.nan)
    species_id = pop.species_id if pop.species_id is not None else np.full(pop.size, -1, dtype=np.int64)
    return {
        "config": dump_config(state.config),
        "generation": int(state.generation),
        "next_key": int(state.allocator.next_key),
        "nodes": _host(pop.nodes).astype(np.float64),
        "conns": _host(pop.conns).astype(np.float64),
        "species_id": _host(species_id),
        "fitness": _host(fitness).astype(np.float64),
        "stats_rows": list(state.stats_rows),
        "species": species,
    }


def save_checkpoint(path, state) -> None:
    with open(path, "wb") as fh:
        pickle.dump(checkpoint_payload(state), fh)


def load_checkpoint(path, on_device: bool = True):
    """EvolutionState from a checkpoint written by this package or the reference;
    the population is moved to the GPU when ``on_device``."""
    from .evolution import NodeKeyAllocator, SpeciesState
    from .runner import EvolutionState
    with open(path, "rb") as fh:
        payload = pickle.load(fh)
    config = parse_config_text(payload["config"])
    nodes, conns = payload["nodes"], payload["conns"]
    if on_device:
        from .device import to_device
        import torch
        nodes, conns = to_device(nodes, torch.float64), to_device(conns, torch.float64)
    pop = PopulationTensors(nodes, conns, np.asarray(payload["species_id"]), np.asarray(payload["fitness"]),
                            config.inputs, config.outputs)
    species = [SpeciesState(species_key=e["species_key"],
                            representative=GenomeTensors(e["rep_nodes"], e["rep_conns"], config.inputs,
                                                         config.outputs),
                            member_indices=e["member_indices"],
                            best_fitness_history=list(e["best_fitness_history"]),
                            stagnation_counter=e["stagnation_counter"], spawn_count=e["spawn_count"])
               for e in payload["species"]]
    return EvolutionState(config=config, population=pop, species=species,
                          allocator=NodeKeyAllocator(payload["next_key"]), generation=payload["generation"],
                          stats_rows=list(payload["stats_rows"]))
