"""Per-config input recipes (BASELINE.json ``configs``).

Everything here is input *shape*: sizes, seeds, message lengths, corruption
positions and corruption byte values.  Nothing here encodes or decodes.

NA191 is the set of 191 byte values that are neither one of the 64 RFC 4648
alphabet characters nor the pad '=' -- the corruption bytes of
configs 1 and 4 ("bytes drawn uniformly from the 191 non-alphabet, non-'='
byte values", BASELINE.json configs[3]).
"""
from __future__ import annotations

import math

import numpy as np

_ALPHABET_CHARS = (
    [ord("A") + i for i in range(26)]
    + [ord("a") + i for i in range(26)]
    + [ord("0") + i for i in range(10)]
    + [ord("+"), ord("/")]
)
NA191 = np.array(
    [b for b in range(256) if b not in set(_ALPHABET_CHARS) and b != ord("=")],
    dtype=np.uint8,
)
assert NA191.size == 191

# ---- C1: round trip on 2^20 random bytes (seed 0) + one corrupted copy ----
C1_N = 1 << 20
C1_SEED = 0


def c1_corruption(m: int) -> tuple[int, int]:
    """(position, byte) of the single corruption in C1's dirty copy.

    pos in [0, m-2) so the corruption never lands on the final '=='."""
    rng = np.random.default_rng(0)
    pos = int(rng.integers(0, m - 2))
    byte = int(NA191[int(rng.integers(0, 191))])
    return pos, byte


# ---- C2: 10,000 messages, log-uniform lengths in [100 B, 64 KiB] (seed 1) ----
C2_K = 10_000
C2_SEED = 1


def c2_lengths(k: int = C2_K, seed: int = C2_SEED) -> tuple[np.ndarray, np.random.Generator]:
    """Message lengths (int64) and the rng, positioned after the draw."""
    rng = np.random.default_rng(seed)
    u = rng.uniform(math.log(100), math.log(65537), size=k)
    lens = np.clip(np.floor(np.exp(u)), 100, 65536).astype(np.int64)
    return lens, rng


def offsets_from_lengths(lens: np.ndarray) -> np.ndarray:
    off = np.zeros(lens.size + 1, dtype=np.int64)
    np.cumsum(lens, out=off[1:])
    return off


def c2_injections(text_lens: np.ndarray, rng: np.random.Generator, frac: float = 0.01):
    """1% of messages get one NA191 byte: list of (msg, pos_in_msg, byte)."""
    k = text_lens.size
    nsel = max(1, int(round(frac * k)))
    msgs = np.sort(rng.choice(k, size=nsel, replace=False))
    out = []
    for i in msgs:
        L = int(text_lens[i])
        if L == 0:
            continue
        pos = int(rng.integers(0, L))
        byte = int(NA191[int(rng.integers(0, 191))])
        out.append((int(i), pos, byte))
    return out


# ---- C3: 1 GiB + 2 random bytes on one GPU (seed 2) ----
C3_N = (1 << 30) + 2
C3_SEED = 2

# ---- C4: 256 MiB of valid text = encoding of 201,326,592 seed-3 bytes ----
C4_RAW = 201_326_592
C4_M = 1 << 28
C4_SEED = 3


def c4_corruptions(m: int = C4_M, count: int = 256, seed: int = 4):
    """Positions (sorted, unique) and NA191 bytes of C4's dirty variant."""
    rng = np.random.default_rng(seed)
    pos = rng.choice(m, size=count, replace=False).astype(np.int64)
    byt = NA191[rng.integers(0, 191, size=count)]
    return pos, byt


# ---- C5: 32 GiB over 1/2/4/8 GPUs (seed 5) ----
C5_N = 1 << 35
C5_SEED = 5
