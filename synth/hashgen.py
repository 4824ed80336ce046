"""Counter-based integer hash shared by every input generator.

This module holds NO arithmetic of the method (no argmax, no accept scan, no
padding or realignment rule).  It only turns (seed, stream, index) triples into
64-bit pseudo-random words, identically on numpy (host) and torch (any device),
so that the CPU oracle and the CUDA path can be fed bit-identical inputs:

    key(seed, stream) = splitmix64((seed << 32) ^ stream)      (host, Python int)
    h(seed, stream, i) = splitmix64(key + i  mod 2**64)

splitmix64 is the finaliser of Steele, Lea & Flood, "Fast splittable
pseudorandom number generators" (OOPSLA 2014).
"""
from __future__ import annotations

import numpy as np

M64 = (1 << 64) - 1
_C0 = 0x9E3779B97F4A7C15
_C1 = 0xBF58476D1CE4E5B9
_C2 = 0x94D049BB133111EB


def splitmix64_int(x: int) -> int:
    """Scalar splitmix64 on Python ints (exact, arbitrary precision then masked)."""
    z = (x + _C0) & M64
    z = ((z ^ (z >> 30)) * _C1) & M64
    z = ((z ^ (z >> 27)) * _C2) & M64
    return z ^ (z >> 31)


def stream_key(seed: int, stream: int) -> int:
    return splitmix64_int((((seed & 0xFFFFFFFF) << 32) ^ (stream & 0xFFFFFFFF)) & M64)


# ----------------------------------------------------------------------------- numpy
def splitmix64_np(x: np.ndarray) -> np.ndarray:
    x = x.astype(np.uint64, copy=False)
    with np.errstate(over="ignore"):
        z = x + np.uint64(_C0)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(_C1)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(_C2)
        return z ^ (z >> np.uint64(31))


def hash_np(seed: int, stream: int, idx) -> np.ndarray:
    """uint64 hash words for an index array (any shape)."""
    idx = np.asarray(idx, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return splitmix64_np(idx + np.uint64(stream_key(seed, stream)))


def uniform_np(seed: int, stream: int, idx) -> np.ndarray:
    """float64 in [0, 1) from the top 53 bits (exact)."""
    h = hash_np(seed, stream, idx)
    return (h >> np.uint64(11)).astype(np.float64) * (1.0 / (1 << 53))


# ----------------------------------------------------------------------------- torch
def _s64(c: int) -> int:
    """Unsigned 64-bit constant -> the int64 with the same bits."""
    c &= M64
    return c - (1 << 64) if c >= (1 << 63) else c


def _lsr(z, s: int):
    # logical shift right on int64 bit patterns
    return (z >> s) & ((1 << (64 - s)) - 1)


def splitmix64_torch(x):
    z = x + _s64(_C0)
    z = (z ^ _lsr(z, 30)) * _s64(_C1)
    z = (z ^ _lsr(z, 27)) * _s64(_C2)
    return z ^ _lsr(z, 31)


def hash_torch(seed: int, stream: int, idx):
    """int64 tensor holding the same 64 bits as hash_np (idx: int64 tensor)."""
    return splitmix64_torch(idx + _s64(stream_key(seed, stream)))


def to_u64_np(t) -> np.ndarray:
    """Reinterpret an int64 torch tensor's bits as numpy uint64."""
    return t.cpu().numpy().view(np.uint64)
