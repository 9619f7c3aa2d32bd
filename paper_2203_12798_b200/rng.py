"""Sketch-matrix (Omega) generation.

Omega_k must be bit-identical to the reference's draw (P/linalg.py:122-123):
``Generator(PCG64(derived_seed(seed, k))).standard_normal((J, s_k))``.  This
module produces them on the host with NumPy's own generator (the algorithm the
reference specifies), packed as (K, J, sp) float64 with zero padding, in
parallel over slices, and copies them to the device through pinned memory.
"""
from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

from .linalg import derived_seed

_MASK64 = (1 << 64) - 1


def _fill(out, seeds, n, widths, lo, hi):
    for k in range(lo, hi):
        g = np.random.Generator(np.random.PCG64(seeds[k] & _MASK64))
        s = widths[k]
        if s == out.shape[2]:
            g.standard_normal(out=out[k])
        else:
            out[k, :, :s] = g.standard_normal((n, s))


def omega_host(seed, n, widths, sp, threads=None, slice_ids=None):
    """Pinned host tensor (K, n, sp) with slice k's Omega in [:, :widths[k]].
    ``slice_ids`` gives the global slice index of each local slice (multi-GPU
    shards keep the reference's per-slice seeds)."""
    K = len(widths)
    ids = range(K) if slice_ids is None else slice_ids
    seeds = [derived_seed(seed, k) for k in ids]
    host = torch.zeros((K, n, sp), dtype=torch.float64, pin_memory=torch.cuda.is_available())
    arr = host.numpy()
    threads = threads or min(32, os.cpu_count() or 1)
    step = max(1, (K + threads - 1) // threads)
    if threads <= 1 or K < 2:
        _fill(arr, seeds, n, widths, 0, K)
    else:
        with ThreadPoolExecutor(max_workers=threads) as pool:
            list(pool.map(lambda lo: _fill(arr, seeds, n, widths, lo, min(K, lo + step)), range(0, K, step)))
    return host


def omega_device(seed, n, widths, sp, device, stream=None, slice_ids=None):
    host = omega_host(seed, n, widths, sp, slice_ids=slice_ids)
    return host.to(device, non_blocking=True), host


def stage2_omega(seed, rows, width):
    """Omega_2 (rows x width), one stream seeded ``seed`` (P/compress.py:109-111)."""
    g = np.random.Generator(np.random.PCG64(seed & _MASK64))
    return g.standard_normal((rows, width))
