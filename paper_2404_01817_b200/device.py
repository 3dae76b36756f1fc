"""Device plumbing shared by the host modules: tensor conversion and streams.

PyTorch supplies device memory, streams and events; all compute goes through
libtneat.so.  Inputs may be numpy arrays (the reference API) or torch tensors
(device-resident use); outputs follow the input kind.
"""

from __future__ import annotations

import threading

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


_STAGE_BYTES = 32 << 20
_stage = {"bufs": None, "events": [None, None]}
_stage_lock = threading.Lock()  # the staging buffers are shared by every caller thread


def _upload_staged(t: torch.Tensor, dev: torch.device) -> torch.Tensor:
    """Large pageable host tensor -> device through two pinned 32 MB staging
    buffers: the DMA of chunk k overlaps the host copy of chunk k+1."""
    with _stage_lock:
        return _upload_staged_locked(t, dev)


def _upload_staged_locked(t: torch.Tensor, dev: torch.device) -> torch.Tensor:
    if _stage["bufs"] is None:
        _stage["bufs"] = [torch.empty(_STAGE_BYTES, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
    src = t.reshape(-1).view(torch.uint8)
    out = torch.empty(t.shape, dtype=t.dtype, device=dev)
    dst = out.reshape(-1).view(torch.uint8)
    n = src.numel()
    for k, lo in enumerate(range(0, n, _STAGE_BYTES)):
        hi = min(n, lo + _STAGE_BYTES)
        slot = k & 1
        if _stage["events"][slot] is not None:
            _stage["events"][slot].synchronize()
        buf = _stage["bufs"][slot][: hi - lo]
        buf.copy_(src[lo:hi])
        dst[lo:hi].copy_(buf, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        _stage["events"][slot] = ev
    return out


def to_device(x, dtype: torch.dtype) -> torch.Tensor:
    """numpy / torch (any device) -> contiguous device tensor of ``dtype``."""
    dev = device()
    if isinstance(x, torch.Tensor):
        t = x
    else:
        t = torch.from_numpy(np.ascontiguousarray(x))
    if t.device != dev:
        if t.device.type == "cpu" and not t.is_pinned() and t.numel() * t.element_size() > 2 * _STAGE_BYTES:
            t = _upload_staged(t.contiguous(), dev)
        else:
            t = t.to(dev, non_blocking=t.is_pinned())
    if t.dtype != dtype:
        t = t.to(dtype)
    return t.contiguous()


class _PinnedRing:
    """A few reusable pinned staging buffers for small host->device uploads:
    the copy is asynchronous on the current stream and a buffer is reused
    only after its previous copy has completed (event), so planning inside a
    copy/compute pipeline never synchronizes a stream."""

    def __init__(self, n: int = 4):
        self.bufs = [None] * n
        self.events = [None] * n
        self.k = 0
        self.lock = threading.Lock()

    def upload(self, arr: np.ndarray, dev: torch.device):
        with self.lock:
            return self._upload(arr, dev)

    def _upload(self, arr: np.ndarray, dev: torch.device):
        src = torch.from_numpy(np.ascontiguousarray(arr))
        nbytes = src.numel() * src.element_size()
        slot = self.k
        self.k = (self.k + 1) % len(self.bufs)
        if self.events[slot] is not None:
            self.events[slot].synchronize()
        buf = self.bufs[slot]
        if buf is None or buf.numel() < nbytes:
            # pinned allocations are slow (milliseconds): size every slot at once,
            # with headroom, so steady-state uploads never allocate
            size = max(2 * nbytes, 1 << 20)
            for k in range(len(self.bufs)):
                if self.bufs[k] is None or self.bufs[k].numel() < nbytes:
                    if self.events[k] is not None:
                        self.events[k].synchronize()
                    self.bufs[k] = torch.empty(size, dtype=torch.uint8, pin_memory=True)
            buf = self.bufs[slot]
        staged = buf[:nbytes].view(src.dtype).view(src.shape)
        staged.copy_(src)
        out = torch.empty(src.shape, dtype=src.dtype, device=dev)
        out.copy_(staged, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        self.events[slot] = ev
        return out, ev


_RING = _PinnedRing()


def upload_async(arr: np.ndarray, dev: torch.device) -> tuple[torch.Tensor, torch.cuda.Event]:
    """Small numpy array -> device tensor without a stream synchronization;
    consumers on other streams wait on the returned event."""
    return _RING.upload(arr, dev)


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else int(t.data_ptr())


class nvtx:
    """NVTX range around a host phase (visible in nsys / ncu timelines; a
    no-op cost of ~100 ns without a profiler attached)."""

    __slots__ = ("name",)

    def __init__(self, name: str):
        self.name = name

    def __enter__(self):
        torch.cuda.nvtx.range_push(self.name)
        return self

    def __exit__(self, *exc):
        torch.cuda.nvtx.range_pop()
        return False
