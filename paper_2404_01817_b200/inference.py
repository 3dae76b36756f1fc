"""Two-phase inference on the GPU: transform (K1) and population forward (K2).

Drop-in for reference inference.py:
  * ``transform_arrays`` (inference.py:82-147)  -> csrc/transform.cu ``an_transform``
  * ``forward_arrays``   (inference.py:185-262) -> csrc/forward.cu  ``an_forward``
  * wrappers ``transform``, ``population_transform``,
    ``transform_population_stacked``, ``forward``, ``forward_batch``,
    ``population_forward`` (inference.py:150-319) with the same argument
    checks and exceptions.

``StackedNetworks`` duck-types the reference's (``size``, ``order``,
``nodes``, ``incoming``, ``input_rows``, ``output_rows``, ``genome_view``) but
its payload is the device-resident compiled program of every genome; the dense
``incoming`` tensor is only materialised (lazily, on the host) if asked for.

Precision: ``precision="f32"`` (default) evaluates in float32 -- the north-star
path, parity ``|d| <= 1e-5 * max(1, |ref|)`` against the float64 reference;
``precision="f64"`` evaluates in float64 for reference-exact checking
(<= 1e-9 like the reference's own oracle tests, test_oracle.py:82-92).

Layout: ``layout="tc"`` compiles fp32 feed-forward programs for the
tensor-core forward (csrc/forward.cu ``fwd_tc_kernel``): the input-sourced
edges of every step become one exact digit-split tcgen05 MMA per 128-sample
tile (csrc/digits.cuh), the hidden-sourced edges run on CUDA cores.  Genomes
it cannot take (non-sum aggregations, out-of-range weights) get standard
programs in the same buffer and run on the tile kernel.  ``layout="auto"``
(default) is "tc" for fp32 feed-forward populations with I <= 32, I % 4 == 0,
else "standard".  Standard programs run on every kernel (tile / warp forward,
fused fitness, cart-pole, recurrent rollouts); a TC-layout population asked
for a standard-only kernel (small batches, explicit tile variants) is
re-transformed once into standard programs (cached).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native
from .device import nvtx, upload_async, device, ptr, stream_handle, to_device
from .errors import ConfigError, CycleDetected, IntegrityError, InvalidInput
from .functions import DEFAULT_REGISTRY, check_registry

ST_CYCLIC, ST_BAD_ACT, ST_BAD_AGG, ST_BAD_KEY, ST_DANGLING, ST_MISSING_IO = 1, 2, 4, 8, 16, 32
_PREC = {"f32": 0, "f64": 1}
FMT_F64, FMT_TC = 1, 2  # program format bits (csrc/common.cuh)
MODE_TC = 2  # ProgHeader.mode of a tensor-core program
_TORCH_DT = {0: torch.float32, 1: torch.float64, 2: torch.float32}
V_TC = 11  # forward variant of the tensor-core kernel
TC_MIN_BATCH = 64  # smaller batches run standard programs on the warp / tile kernels


def _precision_code(precision) -> int:
    if precision in _PREC:
        return _PREC[precision]
    raise ValueError(f"precision must be 'f32' or 'f64', got {precision!r}")


@dataclass(eq=False)
class StackedNetworks:
    """Transformed population: compiled per-genome programs on the device."""

    nodes_dev: torch.Tensor          # (P, N, 5) float64
    conns_dev: torch.Tensor          # (P, C, 4) float64
    num_inputs: int
    num_outputs: int
    program: torch.Tensor            # (P, stride) uint8
    order_dev: torch.Tensor | None   # (P, N) int16, -1 padded; computed on first use
    conn_rows_dev: torch.Tensor | None  # (P, C, 2) int16; computed on first use
    io_rows: torch.Tensor            # (P, I+O) int32
    status_dev: torch.Tensor         # (P,) int32
    maxdims: tuple[int, int, int]    # max (slots, steps, edges) over the population
    precision: int = 0               # program format: FMT_F64 | FMT_TC bits
    mode: int = 0
    _cache: dict = field(default_factory=dict, repr=False)

    # -- reference duck-typing (inference.py:46-75) ----------------------------
    @property
    def size(self) -> int:
        return int(self.program.shape[0])

    @property
    def max_nodes(self) -> int:
        return int(self.nodes_dev.shape[1])

    @property
    def max_conns(self) -> int:
        return int(self.conns_dev.shape[1])

    @property
    def stride(self) -> int:
        return int(self.program.shape[1])

    @property
    def status(self) -> np.ndarray:
        if "status" not in self._cache:
            self._cache["status"] = self.status_dev.cpu().numpy()
        return self._cache["status"]

    @property
    def nodes(self) -> np.ndarray:
        if "nodes" not in self._cache:
            self._cache["nodes"] = self.nodes_dev.cpu().numpy()
        return self._cache["nodes"]

    @property
    def conn_rows(self) -> torch.Tensor:
        """(P, C, 2) int16 (src row, dst row) of the enabled connections that
        enter the reference's dense incoming (-1 elsewhere).  Programs do not
        need it, so it is computed on first use by a transform pass that also
        emits it."""
        if self.conn_rows_dev is None:
            p, n, c = self.size, self.max_nodes, self.max_conns
            rows = torch.empty((p, c, 2), dtype=torch.int16, device=self.program.device)
            scratch = torch.empty_like(self.program)
            status = torch.zeros((p,), dtype=torch.int32, device=self.program.device)
            md = torch.zeros((3,), dtype=torch.int32, device=self.program.device)
            _native.call("an_transform", ptr(self.nodes_dev), ptr(self.conns_dev), p, n, c, self.num_inputs,
                         self.num_outputs, self.mode, self.precision, 1, ptr(scratch), self.stride, None,
                         ptr(rows), None, ptr(status), ptr(md), stream_handle())
            self.conn_rows_dev = rows
        return self.conn_rows_dev

    def order_device(self) -> torch.Tensor:
        """The reference's Kahn order (P, N) int16 on the device.  Programs do not
        need it (levels suffice), so it is computed on first use by a transform
        pass that also emits the order."""
        if self.order_dev is None:
            p, n, c = self.size, self.max_nodes, self.max_conns
            order = torch.empty((p, n), dtype=torch.int16, device=self.program.device)
            scratch = torch.empty_like(self.program)
            status = torch.zeros((p,), dtype=torch.int32, device=self.program.device)
            md = torch.zeros((3,), dtype=torch.int32, device=self.program.device)
            _native.call("an_transform", ptr(self.nodes_dev), ptr(self.conns_dev), p, n, c, self.num_inputs,
                         self.num_outputs, self.mode, self.precision, 1, ptr(scratch), self.stride, ptr(order),
                         None, None, ptr(status), ptr(md), stream_handle())
            self.order_dev = order
        return self.order_dev

    @property
    def order(self) -> np.ndarray:
        """(P, N) float64 row order, NaN padded (inference.py:125,133)."""
        if "order" not in self._cache:
            o = self.order_device().to(torch.float64)
            o[o < 0] = float("nan")
            self._cache["order"] = o.cpu().numpy()
        return self._cache["order"]

    @property
    def input_rows(self) -> np.ndarray:
        return self.io_rows[:, : self.num_inputs].cpu().numpy().astype(np.int64)

    @property
    def output_rows(self) -> np.ndarray:
        return self.io_rows[:, self.num_inputs:].cpu().numpy().astype(np.int64)

    @property
    def incoming(self) -> np.ndarray:
        """(P, N, N) float64, incoming[p, dst, src] = weight, NaN where no
        enabled edge (inference.py:108-112).  Materialised on demand."""
        if "incoming" not in self._cache:
            p, n = self.size, self.max_nodes
            inc = torch.full((p, n, n), float("nan"), dtype=torch.float64, device=self.program.device)
            rows = self.conn_rows.to(torch.int64)
            pm, cm = torch.nonzero(rows[:, :, 0] >= 0, as_tuple=True)
            inc[pm, rows[pm, cm, 1], rows[pm, cm, 0]] = self.conns_dev[pm, cm, 3]
            self._cache["incoming"] = inc.cpu().numpy()
        return self._cache["incoming"]

    def genome_view(self, i: int) -> "TransformedNetwork":
        sub = self.select(slice(i, i + 1))
        return TransformedNetwork(sub)

    def select(self, idx) -> "StackedNetworks":
        """Row subset (a view on the same device buffers where possible).  The
        host copies of status and slot counts carry over, so planning a subset's
        launches needs no device read-back."""
        ensure_finalized(self)
        sub = StackedNetworks(self.nodes_dev[idx], self.conns_dev[idx], self.num_inputs,
                              self.num_outputs, self.program[idx],
                              None if self.order_dev is None else self.order_dev[idx],
                              None if self.conn_rows_dev is None else self.conn_rows_dev[idx],
                              self.io_rows[idx], self.status_dev[idx],
                              self.maxdims, self.precision, self.mode)
        if isinstance(idx, slice):
            for k in ("status", "slots", "steps_edges", "modes"):
                if k in self._cache:
                    sub._cache[k] = self._cache[k][idx]
        return sub

    @classmethod
    def from_networks(cls, networks: list) -> "StackedNetworks":
        parts = [t.stacked if isinstance(t, TransformedNetwork) else t for t in networks]
        for p in parts:  # launch sizes must be known before they are combined
            ensure_finalized(p)
        first = parts[0]
        md = tuple(max(p.maxdims[k] for p in parts) for k in range(3))
        cat = lambda name: torch.cat([getattr(p, name) for p in parts])  # noqa: E731
        order = None if any(p.order_dev is None for p in parts) else cat("order_dev")
        return cls(cat("nodes_dev"), cat("conns_dev"), first.num_inputs, first.num_outputs,
                   cat("program"), order,
                   None if any(p.conn_rows_dev is None for p in parts) else cat("conn_rows_dev"), cat("io_rows"),
                   cat("status_dev"), md, first.precision, first.mode)


class TransformedNetwork:
    """Inference-ready single genome (inference.py:30-43) backed by a
    one-genome StackedNetworks."""

    def __init__(self, stacked: StackedNetworks):
        self.stacked = stacked

    @property
    def nodes(self) -> np.ndarray:
        return self.stacked.nodes[0]

    @property
    def order(self) -> np.ndarray:
        return self.stacked.order[0]

    @property
    def conns_expanded(self) -> np.ndarray:
        """(N, N, 1): [i, j, 0] = weight of the enabled edge row i -> row j."""
        return self.stacked.incoming[0].T[:, :, None]

    @property
    def input_rows(self) -> np.ndarray:
        return self.stacked.input_rows[0]

    @property
    def output_rows(self) -> np.ndarray:
        return self.stacked.output_rows[0]


# ---------------------------------------------------------------------------
# transform
# ---------------------------------------------------------------------------

def transform_arrays(nodes, conns, num_inputs: int, num_outputs: int, *,
                     precision: str = "f32", network_type: str = "feedforward",
                     prune: bool = True, stream: torch.cuda.Stream | None = None,
                     sync: bool = True, layout: str = "auto",
                     with_order: bool = False) -> tuple[StackedNetworks, np.ndarray]:
    """Kahn transform of every genome at once (inference.py:82-147).

    Returns the stacked programs and the indices of cyclic genomes (their
    programs are empty).  ``nodes``/``conns`` may be numpy or torch (any
    device).  With ``sync=False`` the cyclic list and launch sizes are not
    read back (the caller must call ``finalize_transform`` before forward).
    """
    prec = _precision_code(precision)
    mode = {"feedforward": 0, "recurrent": 1}[network_type]
    nd = to_device(nodes, torch.float64)
    cd = to_device(conns, torch.float64)
    if nd.dim() != 3 or nd.shape[2] != 5 or cd.dim() != 3 or cd.shape[2] != 4 or nd.shape[0] != cd.shape[0]:
        raise ValueError(f"expected (P,N,5) and (P,C,4) tensors, got {tuple(nd.shape)}, {tuple(cd.shape)}")
    pop, n, c = int(nd.shape[0]), int(nd.shape[1]), int(cd.shape[1])
    if layout not in ("auto", "tc", "standard"):
        raise ValueError(f"layout must be 'auto', 'tc' or 'standard', got {layout!r}")
    tc_ok = prec == 0 and mode == 0 and num_inputs <= 32 and num_inputs % 4 == 0
    if layout == "tc" and not tc_ok:
        raise ConfigError("layout='tc' needs fp32 feed-forward programs with <= 32 inputs (a multiple of 4)")
    if layout in ("tc", "auto") and tc_ok:
        prec |= FMT_TC
    with nvtx("transform_arrays"):
        return _transform_arrays(nd, cd, num_inputs, num_outputs, prec, mode, prune, stream, sync, with_order)


def _transform_arrays(nd, cd, num_inputs, num_outputs, prec, mode, prune, stream, sync, with_order):
    pop, n, c = int(nd.shape[0]), int(nd.shape[1]), int(cd.shape[1])
    stride = int(_native.lib().an_program_stride(n, c, num_outputs, prec))
    dev = nd.device
    program = torch.empty((pop, stride), dtype=torch.uint8, device=dev)
    order = torch.empty((pop, n), dtype=torch.int16, device=dev) if with_order else None
    io_rows = torch.empty((pop, num_inputs + num_outputs), dtype=torch.int32, device=dev)
    status = torch.zeros((pop,), dtype=torch.int32, device=dev)
    maxdims = torch.zeros((3,), dtype=torch.int32, device=dev)
    _native.call("an_transform", ptr(nd), ptr(cd), pop, n, c, num_inputs, num_outputs, mode, prec,
                 int(bool(prune)), ptr(program), stride, ptr(order) if order is not None else None,
                 None, ptr(io_rows),
                 ptr(status), ptr(maxdims), stream_handle(stream))
    stacked = StackedNetworks(nd, cd, num_inputs, num_outputs, program, order, None, io_rows,
                              status, (0, 0, 0), prec, mode)
    stacked._cache["maxdims_dev"] = maxdims
    if not sync:
        return stacked, np.zeros(0, dtype=np.int64)
    return stacked, finalize_transform(stacked)


def finalize_transform(stacked: StackedNetworks) -> np.ndarray:
    """Read back launch sizes and per-genome status; raise on invalid genomes;
    return the cyclic genome indices (feed-forward mode)."""
    md = stacked._cache.pop("maxdims_dev", None)
    if md is not None:
        # one read-back: launch sizes, per-genome status, value-slot counts and
        # program formats: header words 0-2 (steps, edge entries, value slots)
        # and 6 (mode) of common.cuh ProgHeader
        dims = stacked.program[:, 0:28].contiguous().view(torch.int32)[:, [0, 1, 2, 6]].reshape(-1)
        host = torch.cat([md, stacked.status_dev, dims]).cpu().numpy()
        p = stacked.size
        stacked.maxdims = tuple(int(v) for v in host[:3])
        stacked._cache["status"] = host[3:3 + p]
        d4 = host[3 + p:].reshape(p, 4)
        stacked._cache["slots"] = d4[:, 2]
        stacked._cache["steps_edges"] = d4[:, :2]
        stacked._cache["modes"] = d4[:, 3]
    return status_cyclic(stacked.status, stacked.mode)


def ensure_finalized(stacked: StackedNetworks) -> None:
    """Launch sizes come from ``finalize_transform``'s read-back; a transform
    run with ``sync=False`` is finalized here before anything is launched on it
    (a launch sized from the (0,0,0) placeholder would under-allocate shared
    memory)."""
    if "maxdims_dev" in stacked._cache:
        finalize_transform(stacked)


def status_cyclic(st: np.ndarray, mode: int = 0) -> np.ndarray:
    """Raise IntegrityError on structurally invalid genomes (per-genome status
    bits of the transform); return the cyclic genome indices (feed-forward)."""
    hard = st & (ST_BAD_KEY | ST_DANGLING | ST_MISSING_IO)
    if hard.any():
        bad = np.nonzero(hard)[0]
        raise IntegrityError(f"genome tensors violate structural invariants at indices {bad[:20].tolist()} "
                             f"(status bits {sorted(set(int(x) for x in st[bad[:20]]))})")
    if mode == 1:
        return np.zeros(0, dtype=np.int64)
    return np.nonzero(st & ST_CYCLIC)[0].astype(np.int64)


def _raise_cycles(cyclic: np.ndarray, offset: int = 0, msg: str | None = None) -> None:
    if cyclic.size:
        bad = (cyclic + offset).tolist()
        raise CycleDetected(msg or f"enabled connections contain a directed cycle in genomes {bad}",
                            genome_indices=bad)


def _genome_parts(genome):
    return genome.nodes[None], genome.conns[None], genome.num_inputs, genome.num_outputs


def transform(genome, **kw) -> TransformedNetwork:
    """One genome; raises CycleDetected on an enabled cycle (inference.py:150-158)."""
    n, c, i, o = _genome_parts(genome)
    stacked, cyclic = transform_arrays(n, c, i, o, **kw)
    if cyclic.size:
        raise CycleDetected("enabled connections contain a directed cycle")
    return TransformedNetwork(stacked)


def population_transform(pop, **kw) -> list[TransformedNetwork]:
    """Every genome; aggregated CycleDetected (inference.py:161-168)."""
    stacked = transform_population_stacked(pop, **kw)
    return [stacked.genome_view(i) for i in range(stacked.size)]


def transform_population_stacked(pop, **kw) -> StackedNetworks:
    """Stacked variant used by the evolution loop (inference.py:171-178)."""
    stacked, cyclic = transform_arrays(pop.nodes, pop.conns, pop.num_inputs, pop.num_outputs, **kw)
    _raise_cycles(cyclic)
    return stacked


# ---------------------------------------------------------------------------
# forward
# ---------------------------------------------------------------------------

def _check_codes(stacked: StackedNetworks) -> None:
    _check_status_codes(stacked.status)


def _check_status_codes(st: np.ndarray) -> None:
    if (st & ~ST_CYCLIC & (ST_BAD_ACT | ST_BAD_AGG)).any():
        which = np.nonzero(st & (ST_BAD_ACT | ST_BAD_AGG))[0][:10].tolist()
        kind = "activation" if (st & ST_BAD_ACT).any() else "aggregation"
        raise ConfigError(f"unknown {kind} code in genomes {which}")


_TILE_TT = {1: 128, 2: 256, 3: 64, 4: 256, 5: 128, 6: 128}
_SMEM_PER_SM = 228 * 1024


def _host_dims(stacked: StackedNetworks) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    """Per-genome (slots, (steps, edges), mode) from the transform's read-back
    (read here if the stacked object has none)."""
    if "steps_edges" not in stacked._cache or "modes" not in stacked._cache:
        d = stacked.program[:, 0:28].contiguous().view(torch.int32)[:, [0, 1, 2, 6]].cpu().numpy()
        stacked._cache["slots"] = d[:, 2]
        stacked._cache["steps_edges"] = d[:, :2]
        stacked._cache["modes"] = d[:, 3]
    return stacked._cache["slots"], stacked._cache["steps_edges"], stacked._cache["modes"]


def _upload_plan(stacked: StackedNetworks, key, ids_host: np.ndarray):
    # no stream sync (plans are made inside copy/compute pipelines); launches wait on the upload's event
    ids, ev = upload_async(ids_host.astype(np.int32), stacked.program.device)
    stacked._cache[("plan_ready", key)] = ev
    stacked._cache[("plan_ids", key)] = ids
    return ids


def _bucket_plan(stacked: StackedNetworks, variant: int, subset: np.ndarray | None = None,
                 key=None) -> list:
    """Occupancy buckets of the tile kernel: genomes (all, or ``subset``)
    sorted by value-slot count and split where the number of resident CTAs per
    SM changes; each bucket is one launch with its own (tighter) shared-memory
    size.  Cached on the stacked object."""
    key = key if key is not None else ("plan", variant)
    if key in stacked._cache:
        return stacked._cache[key]
    tt = _TILE_TT.get(variant, 256)
    esz = 8 if stacked.precision & FMT_F64 else 4
    slots, se, _ = _host_dims(stacked)
    members = np.arange(slots.size, dtype=np.int64) if subset is None else subset
    msl = slots[members]
    # slot counts are small integers: a 16-bit key makes numpy's stable sort a radix sort
    order = members[np.argsort(np.minimum(msl, 65535).astype(np.uint16), kind="stable")]
    sorted_slots = slots[order]
    ids = _upload_plan(stacked, key, order)
    _, ms, me = stacked.maxdims
    prog = 32 * ms + (16 * me if stacked.precision & FMT_F64 else 8 * me + 16) + 16
    pad = {1: 1, 2: 2, 3: 1, 4: 4, 5: 2, 6: 4}[variant]
    occ = _SMEM_PER_SM // (prog + np.maximum(sorted_slots, stacked.num_inputs) * (tt + pad) * esz + 1024)
    # per-bucket program extents (steps, edge entries): a launch sizes its shared
    # program area for its own genomes, not the population's largest (fp32 tile
    # kernel only; the classes above stay conservative)
    fp32 = not stacked.precision & FMT_F64
    plan = []
    lo = 0
    n = sorted_slots.size
    while lo < n:
        hi = lo + int(np.searchsorted(occ[lo:] != occ[lo], True))  # first index with another class
        hi = n if hi == lo else hi
        if fp32:
            ext = se[order[lo:hi]].max(axis=0)
            plan.append((ids[lo:hi], (int(sorted_slots[hi - 1]), int(ext[0]), int(ext[1]))))
        else:
            plan.append((ids[lo:hi], (int(sorted_slots[hi - 1]), ms, me)))
        lo = hi
    stacked._cache[key] = plan
    return plan


TC_NCLASS = 7  # device launch-plan classes (csrc/forward.cu plan_tc_kernel)


def _tc_plan_buffers(stacked: StackedNetworks, device) -> tuple[torch.Tensor, torch.Tensor]:
    """Scratch of the device-side launch plan (ids int32[7P]; counts int32[14]:
    7 class counts, then the class launches' dynamic task counters),
    allocated once per StackedNetworks; the plan itself is rebuilt on the
    device by every forward (no host read-back)."""
    bufs = stacked._cache.get("tcplan")
    if bufs is None:
        bufs = (torch.empty((TC_NCLASS * max(1, stacked.size),), dtype=torch.int32, device=device),
                torch.empty((2 * TC_NCLASS,), dtype=torch.int32, device=device))
        stacked._cache["tcplan"] = bufs
    return bufs


def tc_plan_counts(stacked: StackedNetworks) -> np.ndarray:
    """Genomes per device-plan class of an FMT_TC population (classes 0-4:
    tensor-core programs by MMA width 32/48/64/96/128, 5: tensor-core programs
    with more hidden-edge entries than the class buffer, 6: standard programs).
    Diagnostics and tests; the forward does not need it."""
    ids, counts = _tc_plan_buffers(stacked, stacked.program.device)
    _native.call("an_plan_tc", ptr(stacked.program), stacked.stride, stacked.size, ptr(ids), ptr(counts),
                 stream_handle())
    return counts[:TC_NCLASS].cpu().numpy()


def _tc_plan(stacked: StackedNetworks) -> tuple[list, list]:
    """Host launch plan of an FMT_TC population (the fallback when the device
    plan's capacity-sized classes do not fit shared memory -- very large
    genome capacities): tensor-core programs bucketed by
    their MMA width (steps rounded up to 16: it sets the TMEM columns and the
    shared-memory footprint, i.e. the resident CTAs per SM), each bucket sized
    by its own (steps, edge entries) extents; standard programs (genomes the
    tensor-core format cannot take) go to the tile kernel's buckets."""
    key = ("plan", V_TC)
    if key in stacked._cache:
        return stacked._cache[key]
    slots, se, modes = _host_dims(stacked)
    tc = np.nonzero(modes == MODE_TC)[0]
    std = np.nonzero(modes != MODE_TC)[0]
    plan_tc = []
    if tc.size:
        nb = (se[tc, 0] + 15) // 16
        order = tc[np.argsort(nb, kind="stable")]
        ids = _upload_plan(stacked, key, order)
        snb = (se[order, 0] + 15) // 16
        bounds = np.flatnonzero(np.diff(snb)) + 1
        for lo, hi in zip(np.concatenate([[0], bounds]), np.concatenate([bounds, [order.size]])):
            ext = se[order[lo:hi]].max(axis=0)
            plan_tc.append((ids[lo:hi], (int(slots[order[lo:hi]].max()), int(ext[0]), int(ext[1]))))
    plan_std = _bucket_plan(stacked, 5, std, key=("plan_tcstd", 5)) if std.size else []
    stacked._cache[key] = (plan_tc, plan_std)
    return stacked._cache[key]


def standard_programs(stacked: StackedNetworks) -> StackedNetworks:
    """Standard-layout programs of an FMT_TC population (for the kernels that
    only take standard programs), transformed once and cached."""
    if not stacked.precision & FMT_TC:
        return stacked
    std = stacked._cache.get("standard")
    if std is None:
        std, _ = transform_arrays(stacked.nodes_dev, stacked.conns_dev, stacked.num_inputs, stacked.num_outputs,
                                  network_type="feedforward", layout="standard")
        stacked._cache["standard"] = std
    return std


def forward_device(stacked: StackedNetworks, inputs: torch.Tensor, out: torch.Tensor | None = None,
                   *, shared: bool = False, variant: int = 0, bucketed: bool = True,
                   stream: torch.cuda.Stream | None = None,
                   sq_sum: torch.Tensor | None = None) -> torch.Tensor:
    """Device-resident forward: inputs (P,B,I) (or (B,I) with shared=True) on
    the GPU in the program's dtype -> outputs (P,B,O).  Tensor-core (FMT_TC)
    programs plan their launches on the device (no host sync at all, a
    transform with sync=False need not be finalized); standard programs use
    the host bucket plan (cached after the first call).

    ``sq_sum``: optional (P,) float32 CUDA tensor, accumulated with each
    genome's sum of squared outputs by the device-planned forward's fused
    epilogue (the caller zeroes it); other launch paths reduce ``out``."""
    if not stacked.precision & FMT_TC:
        ensure_finalized(stacked)
    dt = _TORCH_DT[stacked.precision]
    if inputs.dtype != dt or not inputs.is_cuda or not inputs.is_contiguous():
        raise ValueError(f"inputs must be a contiguous CUDA {dt} tensor")
    pop = stacked.size
    if shared:
        b, i = int(inputs.shape[-2]), int(inputs.shape[-1])
        gstride = 0
    else:
        if inputs.dim() != 3 or inputs.shape[0] != pop:
            raise ValueError(f"expected inputs of shape (P={pop}, B, I), got {tuple(inputs.shape)}")
        b, i = int(inputs.shape[1]), int(inputs.shape[2])
        gstride = b * i
    if i != stacked.num_inputs:
        raise InvalidInput(f"expected input length {stacked.num_inputs}, got {i}")
    if out is None:
        out = torch.empty((pop, b, stacked.num_outputs), dtype=dt, device=inputs.device)
    elif (not isinstance(out, torch.Tensor) or not out.is_cuda or out.dtype != dt or not out.is_contiguous()
          or tuple(out.shape) != (pop, b, stacked.num_outputs) or out.device != inputs.device):
        raise ValueError(f"out must be a contiguous CUDA {dt} tensor of shape (P={pop}, B={b}, "
                         f"O={stacked.num_outputs}) on {inputs.device}")
    if stacked.precision & FMT_TC:
        v = variant & 0xF
        if v not in (0, V_TC) or (v == 0 and b < TC_MIN_BATCH) or not bucketed:
            # standard-only kernels (or an unbucketed launch): standard programs
            return forward_device(standard_programs(stacked), inputs, out, shared=shared, variant=variant,
                                  bucketed=bucketed, stream=stream, sq_sum=sq_sum)
        launch = stream or torch.cuda.current_stream()
        args = (ptr(stacked.program), stacked.stride, stacked.max_nodes, stacked.max_conns, stacked.precision)
        if "tc_host_plan" not in stacked._cache and "modes" in stacked._cache:
            # finalized populations that are mostly standard programs (mixed
            # aggregations) keep the tile kernel's tight per-bucket launches
            stacked._cache["tc_host_plan"] = bool((stacked._cache["modes"] != MODE_TC).mean() > 0.5)
        if not stacked._cache.get("tc_host_plan"):
            # device-side launch plan: classes and counts never leave the GPU, so a
            # transform + forward step needs no host synchronisation
            ids, counts = _tc_plan_buffers(stacked, inputs.device)
            if launch != torch.cuda.current_stream():
                ids.record_stream(launch)
                counts.record_stream(launch)
            ret = _native.lib().an_forward_planned(*args, ptr(ids), ptr(counts), ptr(inputs), gstride, pop, b, i,
                                                   stacked.num_outputs, ptr(out),
                                                   ptr(sq_sum) if sq_sum is not None else None,
                                                   stream_handle(stream))
            if ret != -6:
                _native.check("an_forward_planned", ret)
                return out
            stacked._cache["tc_host_plan"] = True  # capacity-sized classes do not fit shared memory
        ensure_finalized(stacked)
        plan_tc, plan_std = _tc_plan(stacked)
        tpc = variant & 0xFF00
        for key, plan, vv in ((("plan", V_TC), plan_tc, V_TC), (("plan_tcstd", 5), plan_std, 5)):
            if not plan:
                continue
            launch.wait_event(stacked._cache[("plan_ready", key)])
            if launch != torch.cuda.current_stream():
                stacked._cache[("plan_ids", key)].record_stream(launch)
            for ids, md in plan:
                _native.call("an_forward", *args, _maxdims_arg(stacked, md), ptr(ids), ptr(inputs), gstride,
                             int(ids.numel()), b, i, stacked.num_outputs, ptr(out), vv | tpc,
                             stream_handle(stream))
        _sq_sum_from_out(out, sq_sum, stream)
        return out
    # fp64 value rows are twice as wide: one sample per thread keeps 2x the CTAs
    # resident (27 vs 47 ms at config 2)
    wide = 1 if stacked.precision & FMT_F64 else 5
    v = (variant & 0xF) or (wide if b >= 192 else (3 if b >= 96 else 8))
    args = (ptr(stacked.program), stacked.stride, stacked.max_nodes, stacked.max_conns, stacked.precision)
    tail = (b, i, stacked.num_outputs, ptr(out), int(variant) if variant > 15 else int(v),
            stream_handle(stream))
    v &= 0xF
    if v in _TILE_TT and bucketed and pop > 1:
        plan = _bucket_plan(stacked, v)
        launch = stream or torch.cuda.current_stream()
        launch.wait_event(stacked._cache[("plan_ready", ("plan", v))])
        if launch != torch.cuda.current_stream():
            stacked._cache[("plan_ids", ("plan", v))].record_stream(launch)  # allocated on the current stream
        for ids, md in plan:
            _native.call("an_forward", *args, _maxdims_arg(stacked, md), ptr(ids), ptr(inputs), gstride,
                         int(ids.numel()), *tail)
    else:
        _native.call("an_forward", *args, _maxdims_arg(stacked), None, ptr(inputs), gstride, pop, *tail)
    _sq_sum_from_out(out, sq_sum, stream)
    return out


def _sq_sum_from_out(out: torch.Tensor, sq_sum: torch.Tensor | None, stream) -> None:
    """sq_sum += per-genome sum of squared outputs (paths without the fused epilogue)."""
    if sq_sum is None:
        return
    with torch.cuda.stream(stream or torch.cuda.current_stream()):
        sq_sum.add_(torch.linalg.vector_norm(out.view(out.shape[0], -1).float(), dim=1).square_())


def _maxdims_arg(stacked: StackedNetworks, dims=None) -> int:
    """Host int32[3] launch sizes, kept alive on the stacked object."""
    ensure_finalized(stacked)
    dims = tuple(int(v) for v in (dims or stacked.maxdims))
    key = ("maxdims_host", dims)
    arr = stacked._cache.get(key)
    if arr is None:
        arr = (ctypes.c_int32 * 3)(*dims)
        stacked._cache[key] = arr
    return ctypes.addressof(arr)


def _chunk_bounds(pop: int, per: int, first: int) -> list:
    """Genome ranges of the copy/compute pipeline: the first chunks ramp up
    from ``first`` genomes (short pipeline fill), then ``per`` each."""
    bounds, lo, size = [], 0, max(1, min(first, per))
    while lo < pop:
        hi = min(pop, lo + size)
        bounds.append((lo, hi))
        lo, size = hi, min(per, 2 * size)
    return bounds


def _host_forward_pipelined(stacked: StackedNetworks, x: torch.Tensor, out_host: torch.Tensor,
                            chunk_bytes: int = 256 << 20, variant: int = 0) -> torch.Tensor:
    """Host (P,B,I) -> host (P,B,O) in genome chunks: H2D copy of chunk k+1
    and D2H of chunk k-1 overlap the kernel on chunk k (two copy streams,
    double-buffered device staging; chunks ramp up from 1/8 of the chunk size
    so the pipeline fills quickly).  Pinned host tensors make the copies
    asynchronous DMA; the per-chunk launch plans come from the host copy of
    the slot counts (no device read-back inside the loop)."""
    pop, b, i = x.shape
    o = stacked.num_outputs
    dt = _TORCH_DT[stacked.precision]
    dev = device()
    per = max(1, int(chunk_bytes // max(1, b * i * x.element_size())))
    _host_dims(stacked)
    bufs_in = [torch.empty((min(per, pop), b, i), dtype=dt, device=dev) for _ in range(2)]
    bufs_out = [torch.empty((min(per, pop), b, o), dtype=dt, device=dev) for _ in range(2)]
    h2d, comp, d2h = torch.cuda.Stream(), torch.cuda.current_stream(), torch.cuda.Stream()
    in_free = [None, None]
    out_free = [None, None]
    for k, (lo, hi) in enumerate(_chunk_bounds(pop, per, max(1, per // 8))):
        slot = k & 1
        with torch.cuda.stream(h2d):
            if in_free[slot] is not None:
                h2d.wait_event(in_free[slot])
            dst = bufs_in[slot][: hi - lo]
            dst.copy_(x[lo:hi], non_blocking=True)
            ready = torch.cuda.Event()
            ready.record(h2d)
        comp.wait_event(ready)
        if out_free[slot] is not None:
            comp.wait_event(out_free[slot])
        forward_device(stacked.select(slice(lo, hi)), dst, bufs_out[slot][: hi - lo],
                       variant=variant, stream=comp)
        done = torch.cuda.Event()
        done.record(comp)
        in_free[slot] = done
        with torch.cuda.stream(d2h):
            d2h.wait_event(done)
            out_host[lo:hi].copy_(bufs_out[slot][: hi - lo], non_blocking=True)
            fin = torch.cuda.Event()
            fin.record(d2h)
        out_free[slot] = fin
    d2h.synchronize()
    return out_host


def forward_arrays(stacked: StackedNetworks, registry=None, inputs=None, *, variant: int = 0,
                   out=None):
    """Batched forward, inputs (P, B, I) -> outputs (P, B, O) (inference.py:185-262).

    numpy inputs -> numpy float64 outputs (reference behaviour); torch CUDA
    inputs -> torch outputs on the device; torch CPU inputs (ideally pinned)
    -> torch CPU outputs through the chunked copy/compute pipeline.
    """
    check_registry(registry)
    _check_codes(stacked)
    dt = _TORCH_DT[stacked.precision]
    if isinstance(inputs, torch.Tensor) and inputs.is_cuda:
        x = inputs if inputs.dtype == dt else inputs.to(dt)
        return forward_device(stacked, x.contiguous(), out, variant=variant)
    if isinstance(inputs, torch.Tensor):
        x = inputs if inputs.dtype == dt else inputs.to(dt)
        if out is None:
            out = torch.empty((x.shape[0], x.shape[1], stacked.num_outputs), dtype=dt,
                              pin_memory=x.is_pinned())
        return _host_forward_pipelined(stacked, x.contiguous(), out, variant=variant)
    arr = np.asarray(inputs)
    if arr.ndim == 3 and arr.strides[0] == 0:
        # broadcast_to inputs shared by every genome (problems.py:230,253)
        shared = to_device(arr[0], dt)
        return forward_device(stacked, shared, shared=True, variant=variant).cpu().numpy().astype(np.float64)
    x = torch.from_numpy(np.ascontiguousarray(arr, dtype=np.float32 if dt == torch.float32 else np.float64))
    res = torch.empty((x.shape[0], x.shape[1], stacked.num_outputs), dtype=dt)
    if x.numel() * x.element_size() <= (64 << 20):
        res = forward_device(stacked, to_device(x, dt), variant=variant).cpu()
    else:
        res = _host_forward_pipelined(stacked, x, res, variant=variant)
    return res.numpy().astype(np.float64)


def _check_inputs(arr: np.ndarray, num_inputs: int) -> None:
    """inference.py:265-269."""
    if arr.shape[-1] != num_inputs:
        raise InvalidInput(f"expected input length {num_inputs}, got {arr.shape[-1]}")
    if np.isnan(arr).any():
        raise InvalidInput("input contains NaN")


def forward(tn: TransformedNetwork, registry=None, inputs=None) -> np.ndarray:
    """(I,) -> (O,) (inference.py:279-287)."""
    arr = np.asarray(inputs, dtype=np.float64)
    if arr.ndim != 1:
        raise InvalidInput(f"expected a 1-D input vector, got shape {arr.shape}")
    _check_inputs(arr, tn.stacked.num_inputs)
    return forward_arrays(tn.stacked, registry or DEFAULT_REGISTRY, arr[None, None, :])[0, 0]


def forward_batch(tn: TransformedNetwork, registry=None, inputs=None) -> np.ndarray:
    """(B, I) -> (B, O) (inference.py:290-300)."""
    arr = np.asarray(inputs, dtype=np.float64)
    if arr.ndim != 2:
        raise InvalidInput(f"expected a (B, I) input matrix, got shape {arr.shape}")
    if arr.shape[0] < 1:
        raise InvalidInput("batch must contain at least one row")
    _check_inputs(arr, tn.stacked.num_inputs)
    return forward_arrays(tn.stacked, registry or DEFAULT_REGISTRY, arr[None])[0]


def population_forward(transformed, registry=None, inputs=None) -> np.ndarray:
    """(P, I) or (P, B, I) -> per-genome outputs (inference.py:303-319)."""
    stacked = transformed if isinstance(transformed, StackedNetworks) \
        else StackedNetworks.from_networks(list(transformed))
    arr = np.asarray(inputs, dtype=np.float64)
    if arr.ndim == 2:
        _check_inputs(arr, stacked.num_inputs)
        return forward_arrays(stacked, registry or DEFAULT_REGISTRY, arr[:, None, :])[:, 0, :]
    if arr.ndim == 3:
        _check_inputs(arr, stacked.num_inputs)
        return forward_arrays(stacked, registry or DEFAULT_REGISTRY, arr)
    raise InvalidInput(f"expected (P, I) or (P, B, I) inputs, got shape {arr.shape}")
