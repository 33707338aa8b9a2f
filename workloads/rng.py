"""Counter-based splitmix64 streams (SURVEY.md §8d "Synthetic inputs").

Output k (k = 0, 1, ...) of stream s is the (k+1)-th output of the sequential splitmix64 generator
seeded with seed(s) = 1307*16 + s, so a vectorised draw and a sequential draw agree bit for bit.
Uniforms are (x >> 11) * 2**-53, i.e. in [0, 1) with 53 random bits.
"""
from __future__ import annotations

import numpy as np

MASTER_SEED = 1307
_GAMMA = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def stream_seed(stream: int) -> int:
    return MASTER_SEED * 16 + stream


def splitmix64(seed: int, n: int, start: int = 0) -> np.ndarray:
    """Outputs start .. start+n-1 of splitmix64(seed) as uint64."""
    with np.errstate(over="ignore"):
        k = np.arange(start + 1, start + n + 1, dtype=np.uint64)
        z = np.uint64(seed) + k * _GAMMA
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def splitmix64_scalar(seed: int, n: int) -> list[int]:
    """Sequential reference implementation (used by tests to pin the vectorised one)."""
    mask = (1 << 64) - 1
    s = seed & mask
    out = []
    for _ in range(n):
        s = (s + 0x9E3779B97F4A7C15) & mask
        z = s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & mask
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & mask
        out.append(z ^ (z >> 31))
    return out


def uniform(stream: int, n: int, start: int = 0) -> np.ndarray:
    """n uniforms in [0, 1) from stream `stream`, starting at output `start`."""
    x = splitmix64(stream_seed(stream), n, start)
    return (x >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
