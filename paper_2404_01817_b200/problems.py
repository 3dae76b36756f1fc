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
from dataclasses import dataclass

from .errors import ConfigError, CycleDetected, ShapeMismatch, TerminalState
from .functions import DEFAULT_REGISTRY, check_registry
from .inference import (StackedNetworks, _check_codes, _check_status_codes, _maxdims_arg, _raise_cycles,
                        status_cyclic, transform_arrays)
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


# ---------------------------------------------------------------------------
# single-genome host entry points (problems.py:72-150): a user-supplied
# forward callable, evaluated on the host one network at a time.  The
# population path below runs the same fitness on the GPU.
# ---------------------------------------------------------------------------

def _as_column(outputs, n: int) -> np.ndarray:
    y = np.asarray(outputs, dtype=np.float64)
    if y.shape not in ((n, 1), (n,)):
        raise ShapeMismatch(f"expected outputs of shape ({n}, 1), got {y.shape}")
    return y.reshape(1, n, 1)


def eval_xor(forward_fn) -> float:
    """4 - sum of squared errors over the four XOR cases (problems.py:72-77)."""
    return float(_xor_fitness(_as_column(forward_fn(XOR_INPUTS.copy()), 4))[0])


def eval_regression(forward_fn, target_fn=np.sin, samples=None) -> float:
    """-MSE against ``target_fn`` on the sample grid (problems.py:80-88)."""
    xs = regression_grid(64) if samples is None else np.asarray(samples, dtype=np.float64)
    y = _as_column(forward_fn(xs[:, None]), xs.size)
    return float(_regression_fitness(y, target_fn(xs))[0])


# cart-pole constants (problems.py:37-47); the device kernel (csrc/forward.cu
# an_cartpole) integrates the same Euler step
_G, _MC, _MP, _HL, _FORCE, _DT = 9.8, 1.0, 0.1, 0.5, 10.0, 0.02
_X_LIMIT, _THETA_LIMIT = 2.4, 12 * 2 * math.pi / 360


@dataclass(frozen=True)
class CartPoleState:
    """One cart-pole state (problems.py:93-104)."""
    x: float
    x_dot: float
    theta: float
    theta_dot: float
    steps: int = 0

    @property
    def is_terminal(self) -> bool:
        return abs(self.x) > _X_LIMIT or abs(self.theta) > _THETA_LIMIT or self.steps >= MAX_STEPS


def cartpole_step(state: CartPoleState, force_direction: int) -> CartPoleState:
    """One Euler step with force +-10 N: positions move with the old velocities,
    then velocities with the accelerations (problems.py:107-135)."""
    if force_direction not in (-1, 1):
        raise ValueError(f"force_direction must be -1 or +1, got {force_direction}")
    if state.is_terminal:
        raise TerminalState("cart-pole state is already terminal")
    f = float(force_direction) * _FORCE
    c, s = math.cos(state.theta), math.sin(state.theta)
    m = _MC + _MP
    tmp = (f + _MP * _HL * state.theta_dot ** 2 * s) / m
    th_acc = (_G * s - c * tmp) / (_HL * (4.0 / 3.0 - _MP * c ** 2 / m))
    x_acc = tmp - _MP * _HL * th_acc * c / m
    return CartPoleState(state.x + _DT * state.x_dot, state.x_dot + _DT * x_acc,
                         state.theta + _DT * state.theta_dot, state.theta_dot + _DT * th_acc,
                         state.steps + 1)


def eval_cartpole(forward_fn, rng: RngStream) -> float:
    """Steps survived (1..500) under the bang-bang policy sign(output) (problems.py:138-150)."""
    u = np.asarray(rng.uniforms(4), dtype=np.float64).reshape(4) * 0.1 - 0.05
    state = CartPoleState(*(float(v) for v in u))
    while not state.is_terminal:
        obs = np.array([state.x, state.x_dot, state.theta, state.theta_dot])
        out = float(np.asarray(forward_fn(obs)).reshape(-1)[0])
        state = cartpole_step(state, 1 if out > 0 else -1)
    return float(state.steps)


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
        stacked, _ = transform_arrays(pop.nodes, pop.conns, pop.num_inputs, pop.num_outputs,
                                      precision=self.precision, layout="standard", sync=False)
        fused = self.fused_launch(stacked)
        if fused is not None:
            # one read-back for fitness and per-genome status; the kernel ran
            # with capacity-sized launch bounds, so no transform read-back first
            fit, status = fused
            # every status bit is an error: read back the fitness and a count of
            # flagged genomes; the status array itself only when one is flagged
            host = torch.cat([fit, torch.count_nonzero(status).to(torch.float64).reshape(1)]).cpu().numpy()
            if host[stacked.size] != 0:
                self._check(status.cpu().numpy().astype(np.int64))
            return host[:stacked.size]
        from .inference import finalize_transform
        cyclic = finalize_transform(stacked)
        if cyclic.size:
            _raise_cycles(cyclic, 0, f"cyclic genomes at indices {cyclic.tolist()}")
        return self.evaluate_stacked(stacked, registry, rng, indices=np.arange(stacked.size))

    def fused_launch(self, stacked: StackedNetworks):
        """Problems with a fused device fitness return (fitness, status) device
        tensors without synchronising; others return None."""
        return None

    @staticmethod
    def _check(status: np.ndarray) -> None:
        cyclic = status_cyclic(status)
        if cyclic.size:
            _raise_cycles(cyclic, 0, f"cyclic genomes at indices {cyclic.tolist()}")
        _check_status_codes(status)


def _device_const(owner, name: str, a: np.ndarray, dt) -> torch.Tensor:
    """Problem inputs / targets, copied to the device once per owner object."""
    cache = owner.__dict__.setdefault("_device_constants", {})
    key = (name, dt, torch.cuda.current_device())
    t = cache.get(key)
    if t is None:
        t = torch.from_numpy(np.ascontiguousarray(a)).to(device(), dt)
        cache[key] = t
    return t


def _fused_launch(owner, stacked: StackedNetworks, inputs: np.ndarray, kind: int, targets: np.ndarray | None,
                  maxdims=None) -> torch.Tensor:
    dt = torch.float64 if stacked.precision & 1 else torch.float32
    x = _device_const(owner, "inputs", inputs, dt)
    tg = _device_const(owner, "targets", targets, torch.float64) if targets is not None else None
    fit = torch.empty(stacked.size, dtype=torch.float64, device=x.device)
    _native.call("an_forward_fitness", ptr(stacked.program), stacked.stride, stacked.max_nodes,
                 stacked.max_conns, stacked.precision, _maxdims_arg(stacked, maxdims), ptr(x), 0, stacked.size,
                 int(x.shape[0]), int(x.shape[1]), stacked.num_outputs, kind, ptr(tg), ptr(fit),
                 stream_handle())
    return fit


def _capacity_dims(stacked: StackedNetworks) -> tuple:
    """Launch bounds valid for every program of this shape (value slots <= N + 3)."""
    n = stacked.max_nodes
    return (n + 3, n, 3 * stacked.max_conns + 12 * n + 16)


def _fused(owner, stacked: StackedNetworks, inputs: np.ndarray, kind: int, targets: np.ndarray | None) -> np.ndarray:
    _check_codes(stacked)
    return _fused_launch(owner, stacked, inputs, kind, targets).cpu().numpy()


class XorProblem(Problem):
    name, input_size, output_size = "xor", 2, 1

    def evaluate_stacked(self, stacked, registry, rng, indices=None):
        return _fused(self, stacked, XOR_INPUTS, 1, None)

    def fused_launch(self, stacked):
        return _fused_launch(self, stacked, XOR_INPUTS, 1, None, _capacity_dims(stacked)), stacked.status_dev


class RegressionProblem(Problem):
    name, input_size, output_size = "regression", 1, 1

    def __init__(self, target: str = "sin", samples: int = 64):
        if target not in REGRESSION_TARGETS:
            raise ConfigError(f"unknown regression target {target!r}; options: {sorted(REGRESSION_TARGETS)}")
        if samples < 2:
            raise ConfigError("regression_samples must be >= 2")
        self.target_fn = REGRESSION_TARGETS[target]
        self.xs = regression_grid(samples)
        self.xs_col = np.ascontiguousarray(self.xs[:, None])
        self.ys = self.target_fn(self.xs)

    def evaluate_stacked(self, stacked, registry, rng, indices=None):
        return _fused(self, stacked, self.xs_col, 2, self.ys)

    def fused_launch(self, stacked):
        return _fused_launch(self, stacked, self.xs_col, 2, self.ys, _capacity_dims(stacked)), stacked.status_dev


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
