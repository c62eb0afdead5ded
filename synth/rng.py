"""Counter-based SplitMix64 streams for the seeded synthetic inputs.

This module holds NO arithmetic of the DG method. It is the one piece shared by
the oracle (`oracle/`) and the product binding (`paper_1805_11930_b200/`): both
receive identical input arrays from it.

Stream definition: value ``i`` of a stream with seed ``s`` is
``mix(s + (i+1)*GOLDEN)`` with the SplitMix64 finaliser ``mix``. Being counter
based, any sub-range (e.g. one rank's z-slab) can be generated on its own and is
bit-identical to the same slice of the global array.
"""
from __future__ import annotations

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64(seed: int, start: int, count: int) -> np.ndarray:
    """Raw 64-bit draws ``start .. start+count-1`` of the stream ``seed``."""
    idx = np.arange(start + 1, start + count + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + idx * GOLDEN
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        z = z ^ (z >> np.uint64(31))
    return z


def uniform_pm1(seed: int, start: int, count: int) -> np.ndarray:
    """Uniform doubles on [-1, 1): ((x >> 11) * 2^-53) * 2 - 1."""
    x = splitmix64(seed, start, count)
    return (x >> np.uint64(11)).astype(np.float64) * (2.0 ** -53) * 2.0 - 1.0


def normal(seed: int, start: int, count: int) -> np.ndarray:
    """Standard normals by Box-Muller; normal i uses draws 2i and 2i+1."""
    x = splitmix64(seed, 2 * start, 2 * count)
    u1 = ((x[0::2] >> np.uint64(11)).astype(np.float64) + 1.0) * (2.0 ** -53)  # (0, 1]
    u2 = (x[1::2] >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)          # [0, 1)
    return np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)
