"""Sketch parameters and seeds (P/linalg.py:20-33, 116-123, 187-194).

The sketch matrices are the reference's: for slice k, Omega_k is the first
J*s_k standard normals of ``Generator(PCG64(derived_seed(seed, k)))`` in
C order, and the stage-2 matrix uses ``derived_seed(seed, K)``.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

_MASK64 = (1 << 64) - 1


@dataclass(frozen=True)
class RsvdParams:
    """Sketching parameters (P/linalg.py:20-33): ``oversampling=None`` selects
    ``min(10, min(m, n) - rank)``; ``power_iters`` extra multiplications by
    A A^T; ``seed`` the (base) PCG64 seed."""

    rank: int
    oversampling: int | None = None
    power_iters: int = 1
    seed: int = 0


def derived_seed(seed, index):
    """P/linalg.py:187-194: SeedSequence([seed & mask, index]) first uint64."""
    ss = np.random.SeedSequence([seed & _MASK64, int(index)])
    return int(ss.generate_state(1, np.uint64)[0])


def sketch_width(m, n, rank, oversampling=None):
    """P/linalg.py:116-120."""
    over = min(10, min(m, n) - rank) if oversampling is None else oversampling
    if over < 0:
        raise ValueError("oversampling must be >= 0")
    return rank + over


def padded_width(s_max):
    """Column stride of the packed sketch buffers: multiple of 8 up to 32,
    then of 32 (the sketch kernel processes 32-column groups)."""
    return ((s_max + 7) // 8) * 8 if s_max <= 32 else ((s_max + 31) // 32) * 32
