"""Device plumbing shared by the host modules: tensor conversion and streams.

PyTorch supplies device memory, streams and events; all compute goes through
libtneat.so.  Inputs may be numpy arrays (the reference API) or torch tensors
(device-resident use); outputs follow the input kind.
"""

from __future__ import annotations

import numpy as np
import torch

from ._native import NativeError


def device() -> torch.device:
    if not torch.cuda.is_available():
        raise NativeError("no CUDA device: the tneat GPU path has no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def stream_handle(stream: torch.cuda.Stream | None = None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def to_device(x, dtype: torch.dtype) -> torch.Tensor:
    """numpy / torch (any device) -> contiguous device tensor of ``dtype``."""
    dev = device()
    if isinstance(x, torch.Tensor):
        t = x
    else:
        t = torch.from_numpy(np.ascontiguousarray(x))
    if t.device != dev:
        t = t.to(dev, non_blocking=t.is_pinned())
    if t.dtype != dtype:
        t = t.to(dtype)
    return t.contiguous()


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else int(t.data_ptr())
