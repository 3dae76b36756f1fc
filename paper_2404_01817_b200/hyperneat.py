"""HyperNEAT on the GPU: batched CPPN queries + tcgen05 substrate evaluation.

The reference has no HyperNEAT (the paper names it),
so the semantics here are builder-defined:

  * substrate: 64 input and 64 output nodes, each on an 8 x 8 grid over
    [-1, 1]^2 (x = linspace(-1, 1, 8) along columns, y along rows);
  * CPPN: a genome with 4 inputs (x_in, y_in, x_out, y_out) and 1 output;
    query q = k * 64 + j asks for the weight from input node j to output
    node k, so the (P, 4096, 1) forward output IS W (P, 64, 64) row-major
    [k][j] -- a plain population forward with inputs shared by all genomes
    (K2 tile kernel, ``input_genome_stride = 0``);
  * substrate batch X (S x 64, shared), teacher targets t (S,):
    Y_p = tanh(X W_p^T) and fitness_p = -mean((Y_p - t[:, None])^2), computed
    by ``an_substrate_fitness`` on the tensor cores (tf32 MMA, TMEM
    accumulators, fused epilogue) without ever writing Y.

Tolerance vs the float64 CPU restatement: ~1e-3 relative (TF32 operands,
tanh.approx in the epilogue), stated in the tests.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _native
from .device import device, ptr, stream_handle
from .inference import StackedNetworks, forward_device, transform_arrays

GRID = 8
SUBSTRATE = GRID * GRID  # 64 nodes per layer


def substrate_coords(grid: int = GRID) -> np.ndarray:
    """(grid*grid, 2) node positions (x, y) on [-1, 1]^2, row-major."""
    lin = np.linspace(-1.0, 1.0, grid)
    ys, xs = np.meshgrid(lin, lin, indexing="ij")
    return np.stack([xs.ravel(), ys.ravel()], axis=1)


def query_inputs(grid: int = GRID) -> np.ndarray:
    """(4096, 4) CPPN inputs, query q = k*64 + j -> (x_j, y_j, x_k, y_k)."""
    c = substrate_coords(grid)
    n = c.shape[0]
    k, j = np.divmod(np.arange(n * n), n)
    return np.concatenate([c[j], c[k]], axis=1)


def cppn_weights(stacked: StackedNetworks, variant: int = 0) -> torch.Tensor:
    """(P, 64, 64) fp32 substrate weights from a transformed CPPN population."""
    if (stacked.num_inputs, stacked.num_outputs) != (4, 1):
        raise ValueError("CPPNs take 4 inputs (x_in, y_in, x_out, y_out) and give 1 output")
    q = torch.from_numpy(query_inputs().astype(np.float32)).to(device())
    w = forward_device(stacked, q, shared=True, variant=variant)
    return w.view(stacked.size, SUBSTRATE, SUBSTRATE)


def substrate_fitness(weights: torch.Tensor, x: torch.Tensor, target: torch.Tensor) -> torch.Tensor:
    """fitness_p = -mean((tanh(X W_p^T) - t)^2) on the tensor cores."""
    if weights.dtype != torch.float32 or weights.shape[1:] != (SUBSTRATE, SUBSTRATE):
        raise ValueError("weights must be (P, 64, 64) float32")
    if x.shape[1] != SUBSTRATE or x.shape[0] % 128:
        raise ValueError("X must be (S, 64) with S a multiple of 128")
    w = weights.contiguous()
    xx = x.to(torch.float32).contiguous()
    tt = target.to(torch.float32).contiguous()
    out = torch.empty(w.shape[0], dtype=torch.float64, device=w.device)
    _native.call("an_substrate_fitness", ptr(w), int(w.shape[0]), ptr(xx), ptr(tt), int(xx.shape[0]),
                 ptr(out), stream_handle())
    return out


def teacher_task(samples: int = 4096, seed: int = 20261020) -> tuple[np.ndarray, np.ndarray]:
    """Synthetic substrate task: X ~ N(0,1) (S, 64),
    targets t = tanh(X u / 8) for a fixed random u."""
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((samples, SUBSTRATE)).astype(np.float32)
    u = rng.standard_normal(SUBSTRATE)
    return x, np.tanh(x.astype(np.float64) @ u / 8.0).astype(np.float32)


class HyperNEATProblem:
    """Fitness plugin: CPPN population -> substrate fitness (builder-defined)."""

    name, input_size, output_size = "hyperneat", 4, 1
    episodic = False

    def __init__(self, samples: int = 4096, seed: int = 20261020):
        x, t = teacher_task(samples, seed)
        self.x = torch.from_numpy(x).to(device())
        self.t = torch.from_numpy(t).to(device())

    def evaluate_population_tensors(self, pop, registry=None, rng=None, threads: int = 1,
                                    sequential: bool = False) -> np.ndarray:
        stacked, cyclic = transform_arrays(pop.nodes, pop.conns, 4, 1)
        if cyclic.size:
            from .errors import CycleDetected
            raise CycleDetected(f"cyclic genomes at indices {cyclic.tolist()}", genome_indices=cyclic.tolist())
        return substrate_fitness(cppn_weights(stacked), self.x, self.t).cpu().numpy()
