"""Fitness of a fitted model against the raw tensor (P/analysis.py:23-45).

One streaming pass over the packed store computes both sum ||X_k||^2 and
sum ||X_k - Q_k (H * w_k) V^T||^2 (fixed-order reductions).

Zero-pass form for device factors fresh from ``fit_dpar2``
(``output="device"``) on an fp64 tensor: with G_k = H diag(w_k) and Q_k
orthonormal,

    ||X_k - Q_k G_k V^T||^2 = ||X_k||^2 - 2 <Q_k^T X_k, G_k V^T> + ||G_k V^T||^2

and stage 1 already holds Q_k^T X_k: Q_k = A_k Pi_k with A_k = Y_k P_k and
C_k = X_k^T Y_k from the second pass, so Q_k^T X_k = Pi_k^T (C_k P_k)^T =
Pi_k^T M_k^T, M_k the slice's (signed) block of the stage-1 matrix M.  The fit
keeps M and forms M^T V (KR x R, dp2_gemm_tn) on the first call; the fitness is then R x R work per slice in
one library kernel (dp2_fitness_zero_pass), no pass over X (||X_k||^2 comes
from the tensor's stored slice norms).  Rank-deficient slices
(completed A_k columns are not Y_k P_k) and fp32 stores (M from tf32
products) use the streaming pass.
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


def _zero_pass_terms(tensor, factors, d):
    """(sum ||X_k||^2, sum residual) from the fit's M^T V (dp2_fitness_zero_pass),
    or None when it does not apply: the factors are not the device factors of
    a fit of this very tensor, or were modified since (V compared with the
    fit's private copy; Q by identity and version counter), or a slice was
    rank deficient (its completed A_k columns are not Y_k P_k)."""
    zp = getattr(factors, "_zero_pass", None)
    if not zp or zp["tensor"]() is not tensor:
        return None
    if factors.Q is not zp["Q"] or factors.Q_packed is not zp["Q_packed"] or \
            factors.Q_packed._version != zp["Q_version"]:
        return None
    R = factors.H.shape[1]
    if int(zp["rank_found"].min().item()) < R:
        return None
    V = d(factors.V)
    if not torch.equal(V, zp["V"]):  # M^T V was formed with the fit's V
        return None
    H, W = d(factors.H), d(factors.W)
    K, J = W.shape[0], V.shape[0]
    dev = V.device
    lib = _lib.lib()
    if zp.get("MtV") is None:  # M^T V (KR x R) on the first call; M is then released
        M = zp.pop("M")
        MtV = torch.empty((M.shape[1], R), dtype=torch.float64, device=dev)
        _lib.check(lib.dp2_gemm_tn(_vp(M), M.shape[0], M.shape[1], _vp(zp["V"]), R, _vp(MtV), stream_ptr()),
                   "gemm_tn")
        zp["MtV"] = MtV
    ws = workspace(lib.dp2_zero_pass_workspace(K, R), dev)
    out = torch.empty(2, dtype=torch.float64, device=dev)
    _lib.check(lib.dp2_fitness_zero_pass(_vp(zp["MtV"]), K, J, R, _vp(H), _vp(V), _vp(W), _vp(zp["polar"]),
                                         _vp(tensor.slice_sq_norms()), _vp(out), _vp(ws), ws.numel(), stream_ptr()),
               "fitness_zero_pass")
    total, resid = out.cpu().tolist()
    return total, resid


def fitness(tensor: IrregularTensor, factors: Parafac2Factors, threads=None, zero_pass=True):
    """1 - sum_k ||X_k - Xhat_k||_F^2 / sum_k ||X_k||_F^2 (``zero_pass``: use
    the fit's stage-1 data when it applies, see the module docstring)."""
    if factors.num_slices != tensor.num_slices:
        raise ShapeMismatchError(
            f"factors cover {factors.num_slices} slices, tensor has {tensor.num_slices}")
    dev = tensor.X.device
    R = factors.H.shape[1]

    def d(x):
        if isinstance(x, torch.Tensor):
            return x.to(device=dev, dtype=torch.float64).contiguous()
        return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).to(dev)

    terms = _zero_pass_terms(tensor, factors, d) if zero_pass else None
    if terms is not None:
        total, resid = terms
        if total == 0.0:
            raise DegenerateInputError("fitness undefined for an all-zero tensor")
        return 1.0 - resid / total

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
