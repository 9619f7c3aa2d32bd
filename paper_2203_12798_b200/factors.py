"""Factor containers and solver options (P/factors.py:22-99).

Same fields and semantics as the reference.  Arrays are NumPy by default
(drop-in); with ``output="device"`` the solver returns CUDA tensors and Q is a
sequence of views into one packed (sum I_k x R) device tensor.
"""
from __future__ import annotations

from collections.abc import Sequence
from dataclasses import dataclass, field

import numpy as np

_MASK64 = (1 << 64) - 1


@dataclass
class SolverOptions:
    """max_iters, tol (relative change of e; 0 disables early stopping), seed,
    threads (validated only), normalize (None -> DPar2 default True)."""

    max_iters: int = 32
    tol: float = 1e-6
    seed: int = 0
    threads: int | None = None
    normalize: bool | None = None


@dataclass
class FitTrace:
    """Objective e and wall time per iteration, one-off compression time."""

    objective: list = field(default_factory=list)
    seconds: list = field(default_factory=list)
    preprocess_seconds: float = 0.0
    converged: bool = False
    compressed_float_count: int | None = None
    stage_ms: dict = field(default_factory=dict)   # per-phase device times (extra)

    @property
    def iterations(self):
        return len(self.objective)


class SliceViews(Sequence):
    """Read-only sequence of the per-slice row blocks of one packed array,
    built on access: Q_k = packed[row_off[k]:row_off[k+1]].  Making K views
    eagerly costs ~1 us each on the host (1 ms at K = 1000, 7% of a c2 fit)."""

    __slots__ = ("packed", "row_off")

    def __init__(self, packed, row_off):
        self.packed = packed
        self.row_off = np.asarray(row_off, dtype=np.int64)

    def __len__(self):
        return len(self.row_off) - 1

    def __getitem__(self, k):
        if isinstance(k, slice):
            return [self[i] for i in range(*k.indices(len(self)))]
        n = len(self)
        if k < -n or k >= n:
            raise IndexError("slice index out of range")
        k %= n
        return self.packed[int(self.row_off[k]):int(self.row_off[k + 1])]

    def __iter__(self):
        b = self.row_off.tolist()
        return (self.packed[a:z] for a, z in zip(b[:-1], b[1:]))

    def __repr__(self):
        return f"SliceViews({len(self)} slices of {tuple(self.packed.shape)})"


@dataclass
class Parafac2Factors:
    """H (R x R), V (J x R), W (K x R), per-slice Q_k (I_k x R)."""

    H: object
    V: object
    W: object
    Q: list
    Q_packed: object = None

    @property
    def rank(self):
        return self.H.shape[1]

    @property
    def num_slices(self):
        return len(self.Q)

    def slice_factor(self, k):
        """U_k = Q_k H."""
        return self.Q[k] @ self.H

    def reconstruct_slice(self, k):
        """(Q_k (H S_k)) V^T."""
        return (self.Q[k] @ (self.H * self.W[k])) @ self.V.T

    def numpy(self, q_out=None):
        """Host copy (NumPy) of device factors (``q_out``: preallocated
        destination for the packed Q)."""
        if isinstance(self.H, np.ndarray):
            return self
        qp = device_to_numpy(self.Q_packed, out=q_out)
        H, V, W = (t.cpu().numpy() for t in (self.H, self.V, self.W))
        bounds = self.Q.row_off if isinstance(self.Q, SliceViews) else np.cumsum([0] + [q.shape[0] for q in self.Q])
        return Parafac2Factors(H=H, V=V, W=W, Q=[qp[a:b] for a, b in zip(bounds[:-1], bounds[1:])], Q_packed=qp)


def prefaulted_empty(shape, dtype, threads=None):
    """np.empty whose pages are already touched (parallel zero fill): run in
    the background while the GPU finishes, it takes the first-touch page
    faults off the readback's critical path."""
    import os
    from concurrent.futures import ThreadPoolExecutor
    out = np.empty(shape, dtype=dtype)
    flat = out.reshape(-1).view(np.uint8)
    threads = threads or min(16, os.cpu_count() or 1)
    step = -(-flat.size // threads)
    with ThreadPoolExecutor(threads) as pool:
        list(pool.map(lambda a: flat[a:a + step].fill(0), range(0, flat.size, step)))
    return out


def device_to_numpy(t, out=None):
    """Large device tensor -> NumPy array at link speed (``dp2_d2h_staged``:
    chunked async D2H through a persistent pinned staging ring, each landed
    chunk copied out by a persistent host thread team while the next ones are
    in flight).  A pageable destination would go through the driver's slow
    staging path; a fresh pinned allocation costs ~0.5 ms/MB to pin -- far
    more than the copy.  ``out``: preallocated (ideally pre-faulted)
    destination."""
    import ctypes as C

    import torch

    from . import _lib
    from .tensor import stream_ptr
    src = t.contiguous()
    if out is None:
        out = np.empty(tuple(t.shape), dtype={torch.float64: np.float64, torch.float32: np.float32,
                                              torch.int64: np.int64, torch.int32: np.int32}[t.dtype])
    if not out.flags.c_contiguous or out.nbytes != src.numel() * src.element_size():
        raise ValueError("out must be a C-contiguous array of the tensor's size")
    with torch.cuda.device(src.device):
        _lib.check(_lib.lib().dp2_d2h_staged(C.c_void_p(out.ctypes.data), C.c_void_p(src.data_ptr()),
                                             src.numel() * src.element_size(),
                                             stream_ptr()), "d2h_staged")
    return out


def initial_factors(num_cols, num_slices, rank, seed=0):
    """P/factors.py:79-90: H = I, V = eye(J, R) (seeded Gaussian if J < R), W = 1."""
    h = np.eye(rank)
    if num_cols >= rank:
        v = np.eye(num_cols, rank)
    else:
        v = np.random.Generator(np.random.PCG64(seed & _MASK64)).standard_normal((num_cols, rank))
    return h, v, np.ones((num_slices, rank))


def push_col_norms(a, b):
    """P/factors.py:93-99 (host helper; the device solve fuses it)."""
    norms = np.linalg.norm(a, axis=0)
    safe = np.where(norms < 1e-300, 1.0, norms)
    return a / safe, b * safe
