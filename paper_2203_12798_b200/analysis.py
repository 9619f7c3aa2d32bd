"""Fitness of a fitted model against the raw tensor (P/analysis.py:23-45).

One streaming pass over the packed store computes both sum ||X_k||^2 and
sum ||X_k - Q_k (H * w_k) V^T||^2 (fixed-order reductions).
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib
from .compress import _vp, nseg_for, workspace
from .errors import DegenerateInputError, ShapeMismatchError
from .factors import Parafac2Factors
from .tensor import IrregularTensor, stream_ptr


def fitness(tensor: IrregularTensor, factors: Parafac2Factors, threads=None):
    """1 - sum_k ||X_k - Xhat_k||_F^2 / sum_k ||X_k||_F^2."""
    if factors.num_slices != tensor.num_slices:
        raise ShapeMismatchError(
            f"factors cover {factors.num_slices} slices, tensor has {tensor.num_slices}")
    dev = tensor.X.device
    R = factors.H.shape[1]

    def d(x):
        if isinstance(x, torch.Tensor):
            return x.to(device=dev, dtype=torch.float64).contiguous()
        return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).to(dev)

    if factors.Q_packed is not None:
        Q = d(factors.Q_packed)
    else:
        Q = d(np.concatenate([np.asarray(q) for q in factors.Q])) if not isinstance(factors.Q[0], torch.Tensor) \
            else torch.cat([q.to(dev) for q in factors.Q]).double().contiguous()
    H, V, W = d(factors.H), d(factors.V), d(factors.W)
    st, keep = tensor.store(nseg_for(tensor))
    lib = _lib.lib()
    ws = workspace(lib.dp2_fitness_workspace(C.byref(st)), dev)
    out = torch.empty(2, dtype=torch.float64, device=dev)
    _lib.check(lib.dp2_fitness(C.byref(st), _vp(Q), R, _vp(H), _vp(V), _vp(W), _vp(out), _vp(ws), ws.numel(),
                               stream_ptr()), "fitness")
    total, resid = out.cpu().tolist()
    del keep
    if total == 0.0:
        raise DegenerateInputError("fitness undefined for an all-zero tensor")
    return 1.0 - resid / total
