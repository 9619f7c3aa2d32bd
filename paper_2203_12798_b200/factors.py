"""Factor containers and solver options (P/factors.py:22-99).

Same fields and semantics as the reference.  Arrays are NumPy by default
(drop-in); with ``output="device"`` the solver returns CUDA tensors and Q is a
list of views into one packed (sum I_k x R) device tensor.
"""
from __future__ import annotations

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

    def numpy(self):
        """Host copy (NumPy) of device factors."""
        if isinstance(self.H, np.ndarray):
            return self
        qp = self.Q_packed.cpu().numpy()
        bounds = np.cumsum([0] + [q.shape[0] for q in self.Q])
        return Parafac2Factors(H=self.H.cpu().numpy(), V=self.V.cpu().numpy(), W=self.W.cpu().numpy(),
                               Q=[qp[a:b] for a, b in zip(bounds[:-1], bounds[1:])], Q_packed=qp)


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
