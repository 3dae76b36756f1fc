"""ctypes binding of the in-tree C-ABI library ``libtneat.so`` (include/tneat.h).

The library must have been built (``python -m paper_2404_01817_b200.build`` or
``__graft_entry__.build()``).  There is deliberately NO fallback: if the
library or a CUDA device is missing, every GPU entry point raises.
"""

from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
# TNEAT_LIB: an alternative build of the library (tools/build_variant.py, e.g.
# the checked build with device bounds checks) for a whole test run
LIB_PATH = os.environ.get("TNEAT_LIB") or os.path.join(_HERE, "libtneat.so")

P, I32, I64, U64, D = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double

# name -> (restype, argtypes); keep in sync with include/tneat.h
SIGNATURES: dict[str, tuple] = {
    "an_program_stride": (I64, [I32, I32, I32, I32]),
    "an_transform": (I32, [P, P, I64, I32, I32, I32, I32, I32, I32, I32, P, I64, P, P, P, P, P, P]),
    "an_forward": (I32, [P, I64, I32, I32, I32, P, P, P, I64, I64, I32, I32, I32, P, I32, P]),
    "an_forward_planned": (I32, [P, I64, I32, I32, I32, P, P, P, I64, I64, I32, I32, I32, P, P, P]),
    "an_plan_tc": (I32, [P, I64, I64, P, P, P]),
    "an_forward_fitness": (I32, [P, I64, I32, I32, I32, P, P, I64, I64, I32, I32, I32, I32, P, P, P]),
    "an_cartpole": (I32, [P, I64, I32, I32, I32, P, I64, P, I32, P, P]),
    "an_rng_draw": (I32, [P, I64, U64, I64, I32, P, P]),
    "an_init": (I32, [P, P, I64, P, U64, P, P]),
    "an_distance": (I32, [P, P, I64, P, P, I64, I32, I32, I32, D, D, P, P]),
    "an_mutate": (I32, [P, P, I64, P, U64, P, P, P, P]),
    "an_crossover": (I32, [P, P, P, P, I64, I32, I32, P, U64, P]),
    "an_reproduce": (I32, [P, P, P, P, I64, I64, P, P, P, P, U64, D, P, P, P]),
    "an_substrate_fitness": (I32, [P, I64, P, P, I32, P, P]),
    "an_rollout": (I32, [P, I64, I32, I32, I32, P, I64, I32, I32, P, P, P, I32, I32, I32, P, P]),
}


class MutateParams(ctypes.Structure):
    """Mirror of include/tneat.h an_mutate_params."""
    _fields_ = [(n, ctypes.c_int32) for n in ("N", "C", "I", "O", "feedforward", "act_default",
                                               "agg_default", "n_act_options", "n_agg_options")] + [
        ("act_options", ctypes.c_int32 * 8), ("agg_options", ctypes.c_int32 * 8), ("pad", ctypes.c_int32)] + [
        (n, ctypes.c_double) for n in (
            "node_add", "node_delete", "conn_add", "conn_delete",
            "bias_init_mean", "bias_init_std", "bias_mutate_power", "bias_mutate_rate", "bias_replace_rate",
            "response_init_mean", "response_init_std", "response_mutate_power", "response_mutate_rate",
            "response_replace_rate",
            "weight_init_mean", "weight_init_std", "weight_mutate_power", "weight_mutate_rate",
            "weight_replace_rate",
            "enabled_mutate_rate", "activation_replace_rate", "aggregation_replace_rate",
            "attr_min", "attr_max")]

_lib = None
_lock = threading.Lock()


class NativeError(RuntimeError):
    """A libtneat entry point returned a non-zero status."""


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise NativeError(
                        f"{LIB_PATH} is not built; run `python -m paper_2404_01817_b200.build` "
                        "(the GPU path has no CPU fallback)")
                handle = ctypes.CDLL(LIB_PATH)
                for name, (res, args) in SIGNATURES.items():
                    fn = getattr(handle, name)
                    fn.restype = res
                    fn.argtypes = args
                _lib = handle
    return _lib


def call(name: str, *args) -> int:
    """Invoke ``name`` and raise NativeError on a negative status.  Only
    entry points with a declared ctypes signature may be called (an
    undeclared one would be called with C-int arguments)."""
    if name not in SIGNATURES:
        raise NativeError(f"{name} has no ctypes signature in _native.SIGNATURES")
    return check(name, getattr(lib(), name)(*args))


def check(name: str, ret: int) -> int:
    """Raise NativeError for a negative status of entry point ``name``."""
    if ret < 0:
        if ret <= -100:
            raise NativeError(f"{name}: CUDA error {-(ret + 100)}")
        raise NativeError(f"{name}: argument error {ret}")
    return ret


def exported_symbols() -> list[str]:
    return list(SIGNATURES)
