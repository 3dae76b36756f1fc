"""Recurrent NEAT rollouts on the GPU (builder-defined; SURVEY.md G2, §8a a-REC).

The reference rejects recurrent genomes at transform time (SPEC.md:360,
inference.py:143).  Here a genome compiled in recurrent mode
(``transform_arrays(..., network_type="recurrent")``) is run with K
synchronous activation sweeps per environment step inside the synthetic
Ant-shaped environment of BASELINE config 5:

    s_{t+1} = tanh(A s_t + M a_t),  A ~ N(0, 1/D) (D x D),  M ~ N(0, 1/D) (D x O)
    observation = s_t (D = 27), action a_t = network outputs (O = 8),
    reward = s_t[0], fitness = sum over T steps (T = 1000).

Node values start at 0 and persist across environment steps.  The kernel
(an_rollout) keeps the whole episode on chip, one warp per genome.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _native
from .device import device, ptr, stream_handle
from .inference import StackedNetworks, _check_codes, _maxdims_arg, transform_arrays

OBS, ACT = 27, 8


def ant_env(seed: int = 20261021, obs: int = OBS, act: int = ACT):
    """(A, M, s0) of the synthetic Ant-shaped environment (float64)."""
    rng = np.random.default_rng(seed)
    a = rng.standard_normal((obs, obs)) / np.sqrt(obs)
    m = rng.standard_normal((obs, act)) / np.sqrt(obs)
    s0 = np.tanh(rng.standard_normal(obs))
    return a, m, s0


def rollout_fitness(stacked: StackedNetworks, env=None, steps: int = 1000, sweeps: int = 5) -> np.ndarray:
    """Fitness (P,) of every genome of a recurrent-mode transform."""
    if stacked.mode != 1:
        raise ValueError("rollouts need programs compiled with network_type='recurrent'")
    _check_codes(stacked)
    a, m, s0 = env if env is not None else ant_env(obs=stacked.num_inputs, act=stacked.num_outputs)
    dt = torch.float64 if stacked.precision & 1 else torch.float32
    dev = device()
    at, mt, st0 = (torch.from_numpy(np.ascontiguousarray(x)).to(dev, dt) for x in (a, m, s0))
    d = int(at.shape[0])
    fit = torch.empty(stacked.size, dtype=torch.float64, device=dev)
    _native.call("an_rollout", ptr(stacked.program), stacked.stride, stacked.max_nodes, stacked.max_conns,
                 stacked.precision, _maxdims_arg(stacked), stacked.size, stacked.num_inputs,
                 stacked.num_outputs, ptr(at), ptr(mt), ptr(st0), d, int(steps), int(sweeps), ptr(fit),
                 stream_handle())
    return fit.cpu().numpy()


class RecurrentAntProblem:
    """Fitness plugin for recurrent genomes in the synthetic Ant environment."""

    name, input_size, output_size = "ant_recurrent", OBS, ACT
    episodic = True

    def __init__(self, steps: int = 1000, sweeps: int = 5, precision: str = "f32", seed: int = 20261021):
        self.steps, self.sweeps, self.precision = steps, sweeps, precision
        self.env = ant_env(seed)

    def evaluate_population_tensors(self, pop, registry=None, rng=None, threads: int = 1,
                                    sequential: bool = False) -> np.ndarray:
        stacked, _ = transform_arrays(pop.nodes, pop.conns, pop.num_inputs, pop.num_outputs,
                                      precision=self.precision, network_type="recurrent")
        return rollout_fitness(stacked, self.env, self.steps, self.sweeps)
