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
LIB_PATH = os.path.join(_HERE, "libtneat.so")

P, I32, I64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64

# name -> (restype, argtypes); keep in sync with include/tneat.h
SIGNATURES: dict[str, tuple] = {
    "an_program_stride": (I64, [I32, I32, I32, I32]),
    "an_transform": (I32, [P, P, I64, I32, I32, I32, I32, I32, I32, I32, P, I64, P, P, P, P, P, P]),
    "an_forward": (I32, [P, I64, I32, I32, I32, P, P, P, I64, I64, I32, I32, I32, P, I32, P]),
    "an_forward_fitness": (I32, [P, I64, I32, I32, I32, P, P, I64, I64, I32, I32, I32, I32, P, P, P]),
}

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
    """Invoke ``name`` and raise NativeError on a negative status."""
    ret = getattr(lib(), name)(*args)
    if ret < 0:
        if ret <= -100:
            raise NativeError(f"{name}: CUDA error {-(ret + 100)}")
        raise NativeError(f"{name}: argument error {ret}")
    return ret


def exported_symbols() -> list[str]:
    return list(SIGNATURES)
