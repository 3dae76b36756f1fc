"""Genome tensor layout (reference genome.py:1-115).

A genome is the reference's pair of NaN-padded float64 tensors: nodes
(max_nodes, 5) = (key, bias, response, aggregation_id, activation_id) and
conns (max_conns, 4) = (in_key, out_key, enabled, weight).  The device keeps
exactly this layout (float64, array-of-structs rows) so populations cross the
host/device boundary without conversion and every attribute stays the
reference's float64 value; the kernels read rows with 8/16-byte loads.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

NODE_KEY, NODE_BIAS, NODE_RESPONSE, NODE_AGG, NODE_ACT = range(5)
CONN_IN, CONN_OUT, CONN_ENABLED, CONN_WEIGHT = range(4)
NODE_ATTRS, CONN_ATTRS = 4, 2


@dataclass(frozen=True)
class NodeRow:
    """A live node gene as a record (genome.py:38-50)."""
    key: int
    bias: float
    response: float
    aggregation_id: int
    activation_id: int

    def as_array(self) -> np.ndarray:
        return np.asarray((self.key, self.bias, self.response, self.aggregation_id, self.activation_id),
                          dtype=np.float64)


@dataclass(frozen=True)
class ConnRow:
    """A live connection gene as a record; enabled is 0.0 / 1.0 (genome.py:52-63)."""
    in_key: int
    out_key: int
    enabled: float
    weight: float

    def as_array(self) -> np.ndarray:
        return np.asarray((self.in_key, self.out_key, self.enabled, self.weight), dtype=np.float64)


@dataclass(frozen=True, eq=False)
class GenomeTensors:
    """One genome (genome.py:65-79)."""
    nodes: np.ndarray
    conns: np.ndarray
    num_inputs: int
    num_outputs: int

    @property
    def max_nodes(self) -> int:
        return self.nodes.shape[0]

    @property
    def max_conns(self) -> int:
        return self.conns.shape[0]


@dataclass(eq=False)
class PopulationTensors:
    """Stacked genomes plus bookkeeping (genome.py:82-115).  ``nodes`` and
    ``conns`` may be numpy arrays or CUDA tensors (device-resident runs)."""
    nodes: object
    conns: object
    species_id: np.ndarray
    fitness: np.ndarray
    num_inputs: int
    num_outputs: int

    @property
    def size(self) -> int:
        return int(self.nodes.shape[0])

    def genome(self, index: int) -> GenomeTensors:
        n, c = self.nodes[index], self.conns[index]
        if not isinstance(n, np.ndarray):
            n, c = n.cpu().numpy(), c.cpu().numpy()
        return GenomeTensors(np.array(n, copy=True), np.array(c, copy=True),
                             self.num_inputs, self.num_outputs)

    @classmethod
    def from_genomes(cls, genomes: list) -> "PopulationTensors":
        if not genomes:
            raise ValueError("population must be non-empty")
        g0 = genomes[0]
        for g in genomes[1:]:
            if (g.nodes.shape, g.conns.shape, g.num_inputs, g.num_outputs) != \
                    (g0.nodes.shape, g0.conns.shape, g0.num_inputs, g0.num_outputs):
                raise ValueError("genomes disagree on tensor shapes or I/O counts")
        k = len(genomes)
        return cls(np.stack([g.nodes for g in genomes]), np.stack([g.conns for g in genomes]),
                   np.full(k, -1, dtype=np.int64), np.full(k, np.nan), g0.num_inputs, g0.num_outputs)


def init_arrays(config, rng, *, on_device: bool = False):
    """Fresh genomes, inputs fully connected to outputs (genome.py:129-160).

    ``rng`` is a batched stream (e.g. ``RngStream(seed).child(0, 0).split(arange(P))``);
    draws: normals(N) bias, normals(N) response, normals(C) weight per stream.
    Returns numpy arrays, or CUDA tensors with ``on_device=True``."""
    import torch

    from . import _native
    from .device import device, ptr, stream_handle
    from .evolution import mutate_params

    keys = np.asarray(rng._keys, dtype=np.uint64).reshape(-1)
    batch = tuple(rng.batch_shape)
    pop = keys.size
    dev = device()
    nodes = torch.empty((pop, config.max_nodes, 5), dtype=torch.float64, device=dev)
    conns = torch.empty((pop, config.max_conns, 4), dtype=torch.float64, device=dev)
    kd = torch.from_numpy(keys.view(np.int64).copy()).to(dev)
    params = mutate_params(config)
    _native.call("an_init", ptr(nodes), ptr(conns), pop, ptr(kd), int(rng._counter), ctypes.addressof(params),
                 stream_handle())
    rng._counter += 4 * config.max_nodes + 2 * config.max_conns
    if on_device:
        return nodes.reshape(batch + tuple(nodes.shape[1:])), conns.reshape(batch + tuple(conns.shape[1:]))
    return (nodes.cpu().numpy().reshape(batch + (config.max_nodes, 5)),
            conns.cpu().numpy().reshape(batch + (config.max_conns, 4)))


def init_genome(config, rng) -> GenomeTensors:
    """Single fresh genome (genome.py:163-166)."""
    nodes, conns = init_arrays(config, rng)
    return GenomeTensors(nodes, conns, config.inputs, config.outputs)


def genomes_equal(a: GenomeTensors, b: GenomeTensors) -> bool:
    """Bit-for-bit equality, NaN padding rows included (genome.py:118-123)."""
    if (a.num_inputs, a.num_outputs) != (b.num_inputs, b.num_outputs):
        return False
    return all(np.array_equal(np.asarray(x), np.asarray(y), equal_nan=True)
               for x, y in ((a.nodes, b.nodes), (a.conns, b.conns)))


def count_live(genome: GenomeTensors) -> tuple[int, int]:
    """Live (non-padding) node and connection rows (genome.py:279-283)."""
    live = lambda t: int(np.count_nonzero(~np.all(np.isnan(np.asarray(t)), axis=1)))  # noqa: E731
    return live(genome.nodes), live(genome.conns)
