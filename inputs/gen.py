"""Counter-based byte generator G(seed, j) -- host twin (numpy).

G(seed, j) = little-endian byte (j mod 8) of the k-th SplitMix64 output,
k = floor(j / 8), for a SplitMix64 stream started at state ``seed``
(Steele, Lea, Flood 2014).  The k-th output (0-based) is

    z = seed + (k + 1) * 0x9E3779B97F4A7C15          (mod 2^64)
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9
    z = (z ^ (z >> 27)) * 0x94D049BB133111EB
    z =  z ^ (z >> 31)

Because byte j depends only on (seed, j), any rank can generate its shard
[b, e) of a global buffer without generating the rest; data are therefore
identical at 1/2/4/8 GPUs.  The CUDA twin lives in ``inputs/csrc/b64gen.cu``.
"""
from __future__ import annotations

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
M1 = np.uint64(0xBF58476D1CE4E5B9)
M2 = np.uint64(0x94D049BB133111EB)


def splitmix_words(seed: int, k0: int, k1: int) -> np.ndarray:
    """SplitMix64 outputs k0 .. k1-1 (uint64)."""
    k = np.arange(k0, k1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + (k + np.uint64(1)) * GOLDEN
        z = (z ^ (z >> np.uint64(30))) * M1
        z = (z ^ (z >> np.uint64(27))) * M2
        z = z ^ (z >> np.uint64(31))
    return z


def splitmix_bytes(seed: int, begin: int, end: int) -> np.ndarray:
    """Bytes G(seed, j) for j in [begin, end) as a uint8 array."""
    if end <= begin:
        return np.zeros(0, dtype=np.uint8)
    k0, k1 = begin // 8, (end + 7) // 8
    w = splitmix_words(seed, k0, k1).astype("<u8", copy=False)
    b = w.view(np.uint8)
    off = begin - 8 * k0
    return np.ascontiguousarray(b[off: off + (end - begin)])
