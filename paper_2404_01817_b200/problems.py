"""Fitness plugins on the GPU (reference problems.py:184-301).

``Problem.evaluate_population_tensors`` transforms the whole population once
(K1) and evaluates it with a fused forward + fitness kernel:
  * XOR        -> an_forward_fitness kind 1 (problems.py:54-56, 221-231)
  * regression -> an_forward_fitness kind 2 (problems.py:59-61, 234-254)
  * cart-pole  -> an_cartpole lockstep episodes (problems.py:153-177, 257-271)
The evolution loop evaluates with float64 programs by default (closest to the
reference's float64 numpy); ``precision="f32"`` selects the fast path.
Cyclic genomes raise ``CycleDetected`` with their population indices, as the
reference does (problems.py:209-213).
"""

from __future__ import annotations

import ctypes
import math

import numpy as np
import torch

from . import _native
from .config import NeatConfig
from .device import device, ptr, stream_handle
from .errors import ConfigError, CycleDetected, ShapeMismatch
from .functions import DEFAULT_REGISTRY, check_registry
from .inference import (StackedNetworks, _check_codes, _maxdims_arg, _raise_cycles,
                        finalize_transform, transform_arrays)
from .rng import RngStream

XOR_INPUTS = np.array([[0.0, 0.0], [0.0, 1.0], [1.0, 0.0], [1.0, 1.0]])
XOR_TARGETS = np.array([[0.0], [1.0], [1.0], [0.0]])
REGRESSION_TARGETS = {"sin": np.sin, "cos": np.cos, "abs": np.abs, "square": np.square}
MAX_STEPS = 500


def regression_grid(samples: int) -> np.ndarray:
    return np.linspace(-math.pi, math.pi, samples)


def _xor_fitness(outputs: np.ndarray) -> np.ndarray:
    return 4.0 - ((outputs - XOR_TARGETS) ** 2).sum(axis=(-2, -1))


def _regression_fitness(outputs: np.ndarray, targets: np.ndarray) -> np.ndarray:
    return -((outputs[:, :, 0] - targets) ** 2).mean(axis=1)


class Problem:
    """Fitness interface; higher is better (problems.py:184-218)."""

    name: str
    input_size: int
    output_size: int
    episodic: bool = False
    precision: str = "f64"

    def evaluate_stacked(self, stacked: StackedNetworks, registry, rng, indices=None) -> np.ndarray:
        raise NotImplementedError

    def evaluate_population_tensors(self, pop, registry=None, rng=None, threads: int = 1,
                                    sequential: bool = False) -> np.ndarray:
        """Transform and evaluate the whole population on the device."""
        check_registry(registry)
        rng = rng or RngStream(0)
        stacked, cyclic = transform_arrays(pop.nodes, pop.conns, pop.num_inputs, pop.num_outputs,
                                           precision=self.precision, layout="standard")
        if cyclic.size:
            _raise_cycles(cyclic, 0, f"cyclic genomes at indices {cyclic.tolist()}")
        return self.evaluate_stacked(stacked, registry, rng, indices=np.arange(stacked.size))


def _fused(stacked: StackedNetworks, inputs: np.ndarray, kind: int, targets: np.ndarray | None) -> np.ndarray:
    _check_codes(stacked)
    dt = torch.float64 if stacked.precision & 1 else torch.float32
    dev = device()
    x = torch.from_numpy(np.ascontiguousarray(inputs)).to(dev, dt)
    tg = torch.from_numpy(np.ascontiguousarray(targets, dtype=np.float64)).to(dev) if targets is not None else None
    fit = torch.empty(stacked.size, dtype=torch.float64, device=dev)
    _native.call("an_forward_fitness", ptr(stacked.program), stacked.stride, stacked.max_nodes,
                 stacked.max_conns, stacked.precision, _maxdims_arg(stacked), ptr(x), 0, stacked.size,
                 int(x.shape[0]), int(x.shape[1]), stacked.num_outputs, kind, ptr(tg), ptr(fit),
                 stream_handle())
    return fit.cpu().numpy()


class XorProblem(Problem):
    name, input_size, output_size = "xor", 2, 1

    def evaluate_stacked(self, stacked, registry, rng, indices=None):
        return _fused(stacked, XOR_INPUTS, 1, None)


class RegressionProblem(Problem):
    name, input_size, output_size = "regression", 1, 1

    def __init__(self, target: str = "sin", samples: int = 64):
        if target not in REGRESSION_TARGETS:
            raise ConfigError(f"unknown regression target {target!r}; options: {sorted(REGRESSION_TARGETS)}")
        if samples < 2:
            raise ConfigError("regression_samples must be >= 2")
        self.target_fn = REGRESSION_TARGETS[target]
        self.xs = regression_grid(samples)
        self.ys = self.target_fn(self.xs)

    def evaluate_stacked(self, stacked, registry, rng, indices=None):
        return _fused(stacked, self.xs[:, None], 2, self.ys)


class CartPoleProblem(Problem):
    name, input_size, output_size = "cartpole", 4, 1
    episodic = True

    def evaluate_stacked(self, stacked, registry, rng, indices=None):
        _check_codes(stacked)
        if indices is None:
            indices = np.arange(stacked.size)
        u = rng.split(np.asarray(indices)).uniforms(4).reshape(-1, 4)
        start = torch.from_numpy(u * 0.1 - 0.05).to(device())
        fit = torch.empty(stacked.size, dtype=torch.float64, device=start.device)
        _native.call("an_cartpole", ptr(stacked.program), stacked.stride, stacked.max_nodes, stacked.max_conns,
                     stacked.precision, _maxdims_arg(stacked), stacked.size, ptr(start), MAX_STEPS, ptr(fit),
                     stream_handle())
        return fit.cpu().numpy()


def evaluate_population(problem: Problem, transformed, registry=None, rng=None) -> np.ndarray:
    """Fitness of an already-transformed population (problems.py:274-282)."""
    stacked = transformed if isinstance(transformed, StackedNetworks) \
        else StackedNetworks.from_networks(list(transformed))
    return problem.evaluate_stacked(stacked, registry or DEFAULT_REGISTRY, rng or RngStream(0),
                                    indices=np.arange(stacked.size))


_PROBLEMS = {"xor": XorProblem, "regression": RegressionProblem, "cartpole": CartPoleProblem}


def make_problem(config: NeatConfig) -> Problem:
    """Problem named by the config, checked against its I/O counts (problems.py:288-301)."""
    if config.problem not in _PROBLEMS:
        raise ConfigError(f"unknown problem {config.problem!r}; options: {sorted(_PROBLEMS)}")
    problem = RegressionProblem(config.regression_target, config.regression_samples) \
        if config.problem == "regression" else _PROBLEMS[config.problem]()
    if (config.inputs, config.outputs) != (problem.input_size, problem.output_size):
        raise ConfigError(f"problem {problem.name!r} needs inputs={problem.input_size} "
                          f"outputs={problem.output_size}, config has inputs={config.inputs} "
                          f"outputs={config.outputs}")
    return problem
