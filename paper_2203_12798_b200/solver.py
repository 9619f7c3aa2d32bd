"""Compressed-space DPar2 solver on the GPU (P/solver.py:39-190).

``fit_dpar2(tensor, rank, opts) -> (Parafac2Factors, FitTrace)`` keeps the
reference entry point, return values, errors and stop rule.  The whole
iteration loop runs on the device (one cooperative persistent kernel for
R <= 16 and R = 20, 24, else a stream-ordered loop of per-phase kernels --
CTA Newton-Schulz rotations, Theta-stack GEMMs, single-CTA solves; the stop
rule ``prev == 0 or |prev - e| <= tol * prev`` is evaluated on the device each
iteration), so the host only launches and reads the trace at the end.

The kernel-granular functions (update_rotations, mttkrp_mode1/2/3,
update_factors, convergence_metric) mirror the reference's test-level API;
rotations are returned as their polar factors Z_k P_k^T (the only part the
reference consumes, P/solver.py:75,144,187).
"""
from __future__ import annotations

import ctypes as C
import time
import weakref
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .compress import CompressedTensor, _vp, check_status, compress, compress_async, nseg_for, omega_mismatch, workspace
from .factors import FitTrace, Parafac2Factors, SliceViews, SolverOptions, initial_factors, prefaulted_empty
from .linalg import RsvdParams
from .scheduler import resolve_threads
from .tensor import IrregularTensor, new_status, stream_ptr


def _dev(x, dev):
    if isinstance(x, torch.Tensor):
        return x.to(device=dev, dtype=torch.float64).contiguous()
    # pinned staging: a pageable host copy would wait for the whole stream
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).pin_memory().to(dev, non_blocking=True)


@dataclass
class Rotations:
    """Per-slice rotation state: ``polar[k] = Z_k P_k^T`` and
    ``theta[k] = (P_k Z_k^T) F_k`` (P/solver.py:67-78), device (K, R, R)."""

    polar: torch.Tensor
    theta: torch.Tensor

    def __len__(self):
        return self.polar.shape[0]


def _comp_args(comp: CompressedTensor):
    return comp.cores.contiguous(), comp.col_basis.contiguous(), comp.weights.contiguous()


def update_rotations(comp: CompressedTensor, h, v, w, threads=None):
    """Solve every slice's orthogonal Procrustes problem in R x R space."""
    resolve_threads(threads)
    dev = comp.cores.device
    K, J, R = comp.num_slices, comp.num_cols, comp.rank
    F, D, E = _comp_args(comp)
    H, V, W = _dev(h, dev), _dev(v, dev), _dev(w, dev)
    polar = torch.empty((K, R, R), dtype=torch.float64, device=dev)
    theta = torch.empty((K, R, R), dtype=torch.float64, device=dev)
    lib = _lib.lib()
    ws = workspace(lib.dp2_als_workspace(K, J, R), dev)
    status = new_status(dev)
    _lib.check(lib.dp2_update_rotations(_vp(F), _vp(D), _vp(E), K, J, R, _vp(H), _vp(V), _vp(W), _vp(polar),
                                        _vp(theta), _vp(ws), ws.numel(), _vp(status), stream_ptr()),
               "update_rotations")
    check_status(status, "update_rotations")
    return Rotations(polar=polar, theta=theta)


def rotated_cores(comp, rotations: Rotations, threads=None):
    return rotations.theta


def _mttkrp(mode, comp, rotations, h, v, w):
    dev = comp.cores.device
    K, J, R = comp.num_slices, comp.num_cols, comp.rank
    _, D, E = _comp_args(comp)
    H = _dev(h, dev) if h is not None else torch.zeros((R, R), dtype=torch.float64, device=dev)
    V = _dev(v, dev) if v is not None else torch.zeros((J, R), dtype=torch.float64, device=dev)
    W = _dev(w, dev) if w is not None else torch.zeros((K, R), dtype=torch.float64, device=dev)
    shape = {1: (R, R), 2: (J, R), 3: (K, R)}[mode]
    out = torch.empty(shape, dtype=torch.float64, device=dev)
    lib = _lib.lib()
    ws = workspace(lib.dp2_als_workspace(K, J, R), dev)
    _lib.check(lib.dp2_mttkrp(mode, _vp(rotations.theta), _vp(D), _vp(E), K, J, R, _vp(H), _vp(V), _vp(W),
                              _vp(out), _vp(ws), ws.numel(), stream_ptr()), f"mttkrp_mode{mode}")
    return out.cpu().numpy()


def mttkrp_mode1(comp, rotations, w, v, threads=None):
    """R x R right-hand side for the H solve (P/solver.py:81-89)."""
    return _mttkrp(1, comp, rotations, None, v, w)


def mttkrp_mode2(comp, rotations, w, h, threads=None):
    """J x R right-hand side for the V solve (P/solver.py:92-100)."""
    return _mttkrp(2, comp, rotations, h, None, w)


def mttkrp_mode3(comp, rotations, v, h, threads=None):
    """K x R right-hand side for the W solve (P/solver.py:103-111)."""
    return _mttkrp(3, comp, rotations, h, v, None)


def update_factors(comp, rotations, h, v, w, normalize=True, threads=None):
    """One Gauss-Seidel sweep over H, V, W (P/solver.py:114-130)."""
    dev = comp.cores.device
    K, J, R = comp.num_slices, comp.num_cols, comp.rank
    _, D, E = _comp_args(comp)
    H, V, W = _dev(h, dev).clone(), _dev(v, dev).clone(), _dev(w, dev).clone()
    lib = _lib.lib()
    ws = workspace(lib.dp2_als_workspace(K, J, R), dev)
    status = new_status(dev)
    _lib.check(lib.dp2_update_factors(_vp(rotations.theta), _vp(D), _vp(E), K, J, R, _vp(H), _vp(V), _vp(W),
                                      int(bool(normalize)), _vp(ws), ws.numel(), _vp(status), stream_ptr()),
               "update_factors")
    check_status(status, "update_factors")
    return H.cpu().numpy(), V.cpu().numpy(), W.cpu().numpy()


def convergence_metric(comp, rotations, h, v, w, threads=None):
    """e = sum_k ||Theta_k E D^T - H S_k V^T||_F^2 (P/solver.py:133-149)."""
    dev = comp.cores.device
    K, J, R = comp.num_slices, comp.num_cols, comp.rank
    _, D, E = _comp_args(comp)
    H, V, W = _dev(h, dev), _dev(v, dev), _dev(w, dev)
    out = torch.empty(1, dtype=torch.float64, device=dev)
    lib = _lib.lib()
    ws = workspace(lib.dp2_als_workspace(K, J, R), dev)
    _lib.check(lib.dp2_convergence_metric(_vp(rotations.theta), _vp(D), _vp(E), K, J, R, _vp(H), _vp(V), _vp(W),
                                          _vp(out), _vp(ws), ws.numel(), stream_ptr()), "convergence_metric")
    return float(out.item())


def run_als(comp: CompressedTensor, h, v, w, max_iters, tol, normalize, use_graph=True):
    """Device iteration loop; returns (H, V, W, polar, trace list, seconds list)."""
    launched = _als_launch(comp, h, v, w, max_iters, tol, normalize, use_graph)
    return _als_collect(launched)


def _als_launch(comp: CompressedTensor, h, v, w, max_iters, tol, normalize, use_graph=True):
    """Enqueue the ALS loop; returns device outputs plus pinned readback slots
    filled by non-blocking copies (read them after a stream synchronise)."""
    dev = comp.cores.device
    K, J, R = comp.num_slices, comp.num_cols, comp.rank
    F, D, E = _comp_args(comp)
    H, V, W = _dev(h, dev).clone(), _dev(v, dev).clone(), _dev(w, dev).clone()
    polar = torch.empty((K, R, R), dtype=torch.float64, device=dev)
    trace = torch.zeros(max_iters, dtype=torch.float64, device=dev)
    tstamp = torch.zeros(max_iters + 1, dtype=torch.int64, device=dev)
    iters = torch.zeros(1, dtype=torch.int32, device=dev)
    lib = _lib.lib()
    ws = workspace(lib.dp2_als_workspace(K, J, R), dev)
    status = new_status(dev)
    _lib.check(lib.dp2_als_run(_vp(F), _vp(D), _vp(E), K, J, R, _vp(H), _vp(V), _vp(W), _vp(polar), max_iters,
                               float(tol), int(bool(normalize)), _vp(trace), _vp(tstamp), _vp(iters),
                               int(bool(use_graph)), _vp(ws), ws.numel(), _vp(status), stream_ptr()), "als_run")
    host = {}
    for name, t in (("iters", iters), ("trace", trace), ("tstamp", tstamp), ("status", status)):
        host[name] = torch.empty(tuple(t.shape), dtype=t.dtype, pin_memory=True)
        host[name].copy_(t, non_blocking=True)
    return H, V, W, polar, host


def _als_collect(launched, synced=False):
    H, V, W, polar, host = launched
    if not synced:
        torch.cuda.current_stream().synchronize()
    check_status(host["status"], "fit_dpar2")
    n = int(host["iters"].numpy()[0])
    tr = host["trace"].numpy()[:n].tolist()
    secs = (np.diff(host["tstamp"].numpy()[:n + 1]) * 1e-9).tolist()
    return H, V, W, polar, tr, secs


def assemble_q(tensor: IrregularTensor, comp: CompressedTensor, polar, nseg=None):
    """Q_k = A_k (Z_k P_k^T), packed (sum I_k x R) (P/solver.py:186-189)."""
    dev = comp.A.device
    nseg = nseg or nseg_for(tensor)
    st, keep = tensor.store(nseg)
    Q = torch.empty_like(comp.A)
    if comp.a_signs is None:
        _lib.check(_lib.lib().dp2_assemble_q(C.byref(st), _vp(comp.A), comp.rank, _vp(polar), _vp(Q), stream_ptr()),
                   "assemble_q")
    else:  # A held up to column signs (compress_async(defer_signs=True)): folded into Pi_k
        _lib.check(_lib.lib().dp2_assemble_q_signed(C.byref(st), _vp(comp.A), comp.rank, _vp(comp.a_signs),
                                                    _vp(polar), _vp(Q), stream_ptr()), "assemble_q")
    del keep
    return Q


def fit_dpar2(tensor, rank, opts: SolverOptions | None = None, output="numpy", timings=None, use_graph=False,
              _exact_omega=False):
    """Compress once, then alternate rotations and factor sweeps in R x R space.

    Returns ``(factors, trace)`` like P/solver.py:152-190.  ``output="device"``
    keeps the factors on the GPU (CUDA tensors, Q as views of one packed
    tensor); the default returns NumPy arrays like the reference.
    """
    opts = opts or SolverOptions()
    if opts.max_iters < 1:
        raise ValueError("max_iters must be >= 1")
    resolve_threads(opts.threads)
    normalize = bool(opts.normalize) if opts.normalize is not None else True
    if not isinstance(tensor, IrregularTensor):
        tensor = IrregularTensor(tensor)
    # one host synchronisation per fit (besides the Omega tail readback): the
    # compression status, ALS outputs and Q assembly are all enqueued first
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    started = time.perf_counter()
    ev0.record()
    comp, cstatus = compress_async(tensor, rank, rsvd=RsvdParams(rank=rank, seed=opts.seed), timings=timings,
                                   exact_omega=_exact_omega, defer_signs=True)
    ev1.record()
    cstatus_h = torch.empty(tuple(cstatus.shape), dtype=cstatus.dtype, pin_memory=True)
    cstatus_h.copy_(cstatus, non_blocking=True)
    host_pre = time.perf_counter() - started
    h, v, w = initial_factors(tensor.num_cols, tensor.num_slices, rank, opts.seed)
    launched = _als_launch(comp, h, v, w, opts.max_iters, opts.tol, normalize, use_graph=use_graph)
    Q = assemble_q(tensor, comp, launched[3])
    zero_pass = None
    if tensor.dtype == "f64" and output == "device":
        # the stage-1 M is kept for the fitness without a pass over X
        # (analysis.py: M^T V is formed on the first fitness call); the fit's
        # V is kept as a private copy so later edits of factors.V are seen
        zero_pass = dict(M=comp._stage1_M, V=launched[1].clone(), polar=launched[3], rank_found=comp.rank_found,
                         tensor=weakref.ref(tensor))
    comp._stage1_M = None
    q_host = None
    if output == "numpy":
        # while the GPU finishes: allocate + pre-touch Q's NumPy destination
        from concurrent.futures import ThreadPoolExecutor
        q_host = ThreadPoolExecutor(1).submit(prefaulted_empty, tuple(Q.shape), np.float64)
    torch.cuda.current_stream().synchronize()
    tensor._upload_keep = None  # the stream waited for the whole upload before stage 1 finished
    check_status(cstatus_h, "compress")
    if omega_mismatch(comp):  # speculative Omega differed from the reference's: redo exactly
        return fit_dpar2(tensor, rank, opts, output, timings, use_graph, _exact_omega=True)
    H, V, W, polar, tr, secs = _als_collect(launched, synced=True)
    trace = FitTrace(preprocess_seconds=max(host_pre, ev0.elapsed_time(ev1) * 1e-3),
                     compressed_float_count=comp.float_count())
    trace.objective = tr
    trace.seconds = secs
    if len(tr) >= 2:
        prev, e = tr[-2], tr[-1]
        trace.converged = bool(prev == 0.0 or abs(prev - e) <= opts.tol * prev)
    bounds = tensor.row_off_host
    factors = Parafac2Factors(H=H, V=V, W=W, Q=SliceViews(Q, bounds), Q_packed=Q)
    if output == "numpy":
        # staged D2H (device_to_numpy): a fresh pinned destination per fit
        # costs ~0.5 ms/MB to pin, far more than the copy
        factors = factors.numpy(q_out=q_host.result())
    if zero_pass is not None:  # valid while these very factor objects are unmodified
        zero_pass.update(Q=factors.Q, Q_packed=factors.Q_packed, Q_version=factors.Q_packed._version)
    factors._zero_pass = zero_pass
    return factors, trace
