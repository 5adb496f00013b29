"""Helpers for the GPU parity tests (test infrastructure)."""
from __future__ import annotations

import numpy as np
import torch

DEV = torch.device("cuda:0")


def to_dev(x: np.ndarray, mis: int = 0, slack: int = 64) -> torch.Tensor:
    """Copy x to a fresh device buffer whose data pointer is misaligned by
    `mis` bytes from a 256-byte boundary (guard bytes around it)."""
    n = x.size
    base = torch.full((n + mis + slack,), 0xA5, dtype=torch.uint8, device=DEV)
    v = base[mis: mis + n]
    if n:
        v.copy_(torch.from_numpy(np.ascontiguousarray(x)))
    return v


def empty_dev(n: int, mis: int = 0, slack: int = 64, fill: int = 0xCC):
    base = torch.full((max(n, 0) + mis + slack,), fill, dtype=torch.uint8, device=DEV)
    return base, base[mis: mis + max(n, 0)]


def host(t: torch.Tensor) -> np.ndarray:
    return t.cpu().numpy()
