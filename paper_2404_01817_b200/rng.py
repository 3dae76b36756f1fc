"""Counter-based splittable streams (reference rng.py:1-137 semantics).

A stream is a 64-bit key derived from (master seed, path of integer tokens)
plus a draw counter; draw j is ``mix64(key + (j + 1) * G)``.  The host object
below only derives keys and tracks counters -- the population operators draw
their cells on the device (csrc/rng.cuh) from ``keys`` and ``counter``, so a
reference ``arrayneat.RngStream`` (same ``_keys`` / ``_counter`` attributes)
can be passed in its place.  The dense host draws exist for API parity and
small host-side uses (e.g. cart-pole start states).
"""

from __future__ import annotations

import numpy as np

M64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15


def _mix(z: np.ndarray) -> np.ndarray:
    z = z.astype(np.uint64, copy=True)
    with np.errstate(over="ignore"):
        z ^= z >> np.uint64(30)
        z *= np.uint64(0xBF58476D1CE4E5B9)
        z ^= z >> np.uint64(27)
        z *= np.uint64(0x94D049BB133111EB)
        z ^= z >> np.uint64(31)
    return z


def _tokens(value) -> np.ndarray:
    return np.atleast_1d(np.asarray(value)).astype(np.int64).view(np.uint64)


def _absorb(keys: np.ndarray, tokens: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        return _mix(keys ^ _mix(tokens + np.uint64(GOLDEN)))


def mix64_int(z: int) -> int:
    """splitmix64 finaliser on a Python int (same bits as ``_mix``)."""
    z &= M64
    z ^= z >> 30
    z = (z * 0xBF58476D1CE4E5B9) & M64
    z ^= z >> 27
    z = (z * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def key_of(seed: int, *path: int) -> int:
    """Key of the scalar-path stream RngStream(seed, path)."""
    k = _mix(_tokens(seed))
    for t in path:
        k = _absorb(k, _tokens(t))
    return int(k[0])


class RngStream:
    """Batched stream; ``batch_shape`` is () for one stream (rng.py:45-82)."""

    __slots__ = ("master_seed", "path", "batch_shape", "_keys", "_counter")

    def __init__(self, master_seed: int, path: tuple = ()):
        self.master_seed = int(master_seed)
        self.path = tuple(path)
        keys = _mix(_tokens(self.master_seed))
        shape: tuple[int, ...] = ()
        for tok in self.path:
            t = _tokens(tok)
            if np.ndim(tok) == 0:
                keys = _absorb(keys, t)
            else:
                keys = _absorb(keys[:, None], t[None, :]).reshape(-1)
                shape = shape + (t.size,)
        self.batch_shape = shape
        self._keys = keys
        self._counter = 0

    def child(self, *tokens: int) -> "RngStream":
        toks = tuple(int(t) for t in tokens)
        if self.batch_shape != ():
            return RngStream(self.master_seed, self.path + toks)
        # scalar stream: absorb the new tokens into this key (no re-derivation
        # of the whole path; same bits as __init__)
        k = int(self._keys.reshape(-1)[0])
        for t in toks:
            k = mix64_int(k ^ mix64_int((t & M64) + GOLDEN))
        out = RngStream.__new__(RngStream)
        out.master_seed, out.path, out.batch_shape = self.master_seed, self.path + toks, ()
        out._keys = np.array([k], dtype=np.uint64)
        out._counter = 0
        return out

    def split(self, tokens) -> "RngStream":
        tokens = np.asarray(tokens, dtype=np.int64)
        if tokens.ndim != 1:
            raise ValueError("split expects a 1-D token array")
        return RngStream(self.master_seed, self.path + (tokens,))

    # -- host draws (same tape as the device cells) --------------------------
    def _cells(self, base: int, rows, cols) -> np.ndarray:
        with np.errstate(over="ignore"):
            offs = (np.asarray(cols, dtype=np.uint64) + np.uint64(base + 1)) * np.uint64(GOLDEN)
            return _mix(self._keys[np.asarray(rows, dtype=np.int64)] + offs)

    @staticmethod
    def _unit(bits: np.ndarray) -> np.ndarray:
        return ((bits >> np.uint64(11)).astype(np.float64) + 0.5) * 2.0 ** -53

    def uniforms(self, *shape: int) -> np.ndarray:
        n = int(np.prod(shape)) if shape else 1
        b = self._counter
        self._counter += n
        rows = np.repeat(np.arange(self._keys.size), n)
        cols = np.tile(np.arange(n), self._keys.size)
        return self._unit(self._cells(b, rows, cols)).reshape(self.batch_shape + tuple(shape))

    def normals(self, *shape: int) -> np.ndarray:
        n = int(np.prod(shape)) if shape else 1
        u = self.uniforms(2 * n).reshape(-1, 2 * n)
        z = np.sqrt(-2.0 * np.log(u[:, :n])) * np.cos(2.0 * np.pi * u[:, n:])
        return z.reshape(self.batch_shape + tuple(shape))

    def uniforms_at(self, width: int, rows, cols) -> np.ndarray:
        b = self._counter
        self._counter += width
        return self._unit(self._cells(b, rows, cols))

    def normals_at(self, width: int, rows, cols) -> np.ndarray:
        b = self._counter
        self._counter += 2 * width
        cols = np.asarray(cols, dtype=np.uint64)
        u1 = self._unit(self._cells(b, rows, cols))
        u2 = self._unit(self._cells(b, rows, cols + np.uint64(width)))
        return np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)

    def __repr__(self) -> str:  # pragma: no cover
        return f"RngStream(seed={self.master_seed}, path={self.path}, batch={self.batch_shape})"
