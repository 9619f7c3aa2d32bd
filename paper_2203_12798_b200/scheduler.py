"""Slice partitioning (P/scheduler.py).

``greedy_partition`` is Alg. 4 (LPT) computed by the native library and is
bit-exact with the reference (P/scheduler.py:29-51): it is what places slices
on GPUs in the multi-GPU path.  ``resolve_threads`` keeps the reference's
validation (P/scheduler.py:69-82) so option handling is unchanged, although the
GPU path has no host worker threads.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

from . import _lib


@dataclass
class PartitionPlan:
    """Assignment of slice indices to worker sets with their row loads."""

    sets: list = field(default_factory=list)
    loads: list = field(default_factory=list)

    @property
    def workers(self):
        return len(self.sets)


def greedy_partition(row_counts, workers):
    """Longest-first greedy assignment (ties: ascending slice index, then the
    lowest set index); ``max(loads) - min(loads) <= max(row_counts)``."""
    counts = np.ascontiguousarray([int(c) for c in row_counts], dtype=np.int64)
    if counts.size < 1:
        raise ValueError("need at least one slice")
    if workers < 1:
        raise ValueError("need at least one worker")
    if (counts < 1).any():
        raise ValueError("row counts must be positive")
    K = counts.size
    order = np.empty(K, np.int64)
    owner = np.empty(K, np.int32)
    loads = np.empty(workers, np.int64)
    st = _lib.lib().dp2_greedy_partition(
        counts.ctypes.data_as(C.POINTER(C.c_int64)), K, int(workers),
        order.ctypes.data_as(C.POINTER(C.c_int64)), owner.ctypes.data_as(C.POINTER(C.c_int32)),
        loads.ctypes.data_as(C.POINTER(C.c_int64)))
    if st != _lib.DP2_OK:
        raise ValueError(_lib.lib().dp2_last_error().decode())
    sets = [[] for _ in range(workers)]
    for k in order:
        sets[owner[k]].append(int(k))
    return PartitionPlan(sets=sets, loads=[int(x) for x in loads])


def resolve_threads(threads=None):
    """Explicit argument, else DPAR2_THREADS, else cpu count (validation only)."""
    if threads is not None:
        t = int(threads)
        if t < 1:
            raise ValueError("threads must be >= 1")
        return t
    env = os.environ.get("DPAR2_THREADS")
    if env:
        t = int(env)
        if t < 1:
            raise ValueError(f"DPAR2_THREADS must be >= 1, got {env!r}")
        return t
    return os.cpu_count() or 1
