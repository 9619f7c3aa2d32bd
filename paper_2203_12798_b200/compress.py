"""Two-stage compression on the GPU (P/compress.py:34-119).

``compress`` keeps the reference signature and semantics: rank checks with the
same messages, per-slice sketch seeds ``derived_seed(seed, k)``, M in slice
order, stage-2 seed ``derived_seed(seed, K)``; ``plan`` / ``threads`` are
accepted (they never change values in the reference either).
"""
from __future__ import annotations

import ctypes as C
import os
import time
from dataclasses import dataclass, replace

import numpy as np
import torch

from . import _lib
from .errors import NumericFailure, RankTooLargeError
from .linalg import RsvdParams, derived_seed, padded_width, sketch_width
from .rng import (omega_device, omega_device_finish, omega_device_launch, stage2_omega,  # noqa: F401
                  stage2_omega_finish, stage2_omega_launch)
from .scheduler import resolve_threads
from .tensor import IrregularTensor, new_status, sm_count, stream_ptr


def _vp(t):
    return C.c_void_p(t.data_ptr()) if t is not None else C.c_void_p(0)


def workspace(nbytes, dev):
    return torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=dev)


@dataclass
class CompressedTensor:
    """A_k (I_k x R, column-orthonormal), D (J x R), E (R), F (KR x R).

    Device tensors; ``slice_bases`` are views into the packed A buffer.
    """

    rank: int
    A: torch.Tensor            # (sum I_k, R) packed slice bases
    row_off: np.ndarray        # (K+1,)
    col_basis: torch.Tensor    # D
    weights: torch.Tensor      # E
    cores: torch.Tensor        # F
    rank_found: torch.Tensor | None = None
    # fit-internal compressions (compress_async(defer_signs=True)): A is held
    # up to column signs, A_k(reference) = A_k diag(a_signs[k]); assemble_q
    # folds them into the polar factors.  None: A is the reference's A.
    a_signs: torch.Tensor | None = None

    @property
    def num_slices(self):
        return len(self.row_off) - 1

    @property
    def num_cols(self):
        return self.col_basis.shape[0]

    @property
    def row_counts(self):
        return [int(b - a) for a, b in zip(self.row_off[:-1], self.row_off[1:])]

    @property
    def slice_bases(self):
        return [self.A[a:b] for a, b in zip(self.row_off[:-1], self.row_off[1:])]

    def core_block(self, k):
        r = self.rank
        return self.cores[k * r:(k + 1) * r]

    def core_stack(self):
        return self.cores.reshape(self.num_slices, self.rank, self.rank)

    def float_count(self):
        """sum(I_k) R + K R^2 + J R + R (P/compress.py:65-72)."""
        return int(self.A.numel() + self.cores.numel() + self.col_basis.numel() + self.weights.numel())

    def numpy(self):
        a = self.A.cpu().numpy()
        return dict(slice_bases=[a[x:y] for x, y in zip(self.row_off[:-1], self.row_off[1:])],
                    col_basis=self.col_basis.cpu().numpy(), weights=self.weights.cpu().numpy(),
                    cores=self.cores.cpu().numpy())


_FP32_ENGINES = {"tf32": 0, "fp32": 1, "fp64": 2}


def set_fp32_products(mode):
    """Arithmetic of the stage-1 sketch products for fp32-storage tensors:
    ``"fp64"`` (default; fp64 DMMA products on the exactly upcast values where
    the warp-specialised pass applies, J <= 1024, else ``"fp32"``), ``"fp32"``
    (FFMA products, fp32 accumulation within a tile, fp64 across tiles -- the
    fp32 mode of BASELINE.json) or ``"tf32"`` (opt-in speed mode: single-pass
    tf32 products on the tcgen05 tensor cores, ~5e-4 relative product error;
    J <= 1024, above 512 on CTA pairs splitting the columns).
    Returns the previous mode."""
    if mode not in _FP32_ENGINES:
        raise ValueError(f"fp32 product mode must be one of {sorted(_FP32_ENGINES)}, got {mode!r}")
    prev = int(_lib.lib().dp2_set_sketch_engine(_FP32_ENGINES[mode]))
    return {v: k for k, v in _FP32_ENGINES.items()}.get(prev, "fp64")


def nseg_for(tensor: IrregularTensor):
    """Persistent segments of the streaming passes (dp2_stream_segments): one
    CTA per SM for the f64 DMMA and f32 tensor-core passes, two for the f32
    FFMA pass."""
    return int(_lib.lib().dp2_stream_segments(0 if tensor.dtype == "f64" else 1, tensor.num_cols, sm_count()))


def check_status(status, what):
    s = status.cpu().tolist()
    if s[0] != _lib.INT64_MAX:
        from .errors import NonFiniteInputError
        raise NonFiniteInputError(f"slice {s[0]} contains non-finite values")
    if s[3] != _lib.INT64_MAX:
        raise NumericFailure("SVD did not converge", slice_index=int(s[3]))
    return s


def check_rank(tensor: IrregularTensor, rank, slice_ids=None):
    """Rank checks and messages of P/compress.py:84-90."""
    if rank < 1:
        raise RankTooLargeError(f"rank must be >= 1, got {rank}")
    if rank > tensor.num_cols:
        raise RankTooLargeError(f"rank {rank} exceeds column count {tensor.num_cols}")
    rows = np.asarray(tensor.row_counts)
    short = np.nonzero(rows < rank)[0]
    if short.size:
        k = int(short[0])
        ids = range(tensor.num_slices) if slice_ids is None else slice_ids
        raise RankTooLargeError(f"rank {rank} exceeds row count {int(rows[k])} of slice {list(ids)[k]}")
    if rank > 56:
        raise RankTooLargeError(f"rank {rank} exceeds the device limit of 56")
    jmax = 1588 if tensor.dtype == "f64" else 3176  # two 8-row X tiles of the generic pass in 200 KB
    if tensor.num_cols > jmax:
        raise ValueError(f"column count {tensor.num_cols} exceeds the device limit of {jmax} for {tensor.dtype} "
                         f"storage")


def stage2_params(base: RsvdParams, stage2, rank, K, J):
    second = stage2 if stage2 is not None else base
    second = replace(second, rank=rank, seed=derived_seed(second.seed, K))
    return second, sketch_width(J, K * rank, rank, second.oversampling)


def sketch_widths(row_counts, J, rank, oversampling):
    """linalg.sketch_width for every slice at once (list of ints)."""
    m = np.minimum(np.asarray(row_counts, dtype=np.int64), J)
    if oversampling is None:
        over = np.minimum(10, m - rank)
    else:
        over = np.full(m.shape, oversampling)
    if (over < 0).any():
        raise ValueError("oversampling must be >= 0")
    return (rank + over).tolist()


def _stage1_setup(tensor, rank, oversampling, dev):
    """(widths, sp, device widths) for ``tensor`` at ``rank`` -- cached on the
    tensor (its row counts are immutable), so repeated fits skip the host work
    before the first launch."""
    cache = tensor.__dict__.setdefault("_s1_setup", {})
    key = (rank, oversampling)
    if key not in cache:
        from .tensor import to_device_async
        widths = np.asarray(sketch_widths(tensor.row_counts, tensor.num_cols, rank, oversampling), dtype=np.int32)
        sp = padded_width(int(widths.max()))
        if sp > 256:
            raise ValueError(f"sketch width rank + oversampling = {int(widths.max())} exceeds the device limit of 256")
        cache[key] = (widths, sp, to_device_async(widths, torch.int32, dev))
    return cache[key]


def _uses_tc(sub, sp):
    st, keep = sub.store(nseg_for(sub))
    return bool(_lib.lib().dp2_sketch_uses_tc(C.byref(st), sp))


def run_stage1(tensor: IrregularTensor, rank, base: RsvdParams, slice_ids=None, timings=None, status=None,
               speculative=False, a_signs=None, omega_pre=None):
    """Stage 1 on the device for the tensor's slices (global ids ``slice_ids``
    select the per-slice seeds in a multi-GPU shard).  Returns A (sum I_k x R),
    M (J x K_local R, local slice order) and the per-slice numerical ranks
    (plus, with ``speculative``, the Omega replay check future or None --
    rng.omega_device).  With ``a_signs`` (device K x rank) A is returned up to
    its column signs, which go to ``a_signs`` (dp2_stage1_signs).
    ``omega_pre``: an already enqueued exact Omega (rng.omega_device_launch),
    finished here after the outputs are allocated."""
    J, K = tensor.num_cols, tensor.num_slices
    dev = tensor.X.device
    widths, sp, s_dev = _stage1_setup(tensor, rank, base.oversampling, dev)
    t0 = time.perf_counter()
    rstats = {}
    check = None
    if omega_pre is None:
        if speculative and _uses_tc(tensor, sp):
            omega, check = omega_device(base.seed, J, widths, sp, dev, slice_ids=slice_ids, speculative=True,
                                        s_dev=s_dev)
        else:
            omega = omega_device(base.seed, J, widths, sp, dev, slice_ids=slice_ids, stats=rstats, s_dev=s_dev)
    A = torch.empty((int(tensor.row_off_host[-1]), rank), dtype=torch.float64, device=dev)
    M = torch.empty((J, K * rank), dtype=torch.float64, device=dev)
    rank_found = torch.empty(K, dtype=torch.int32, device=dev)
    status = new_status(dev) if status is None else status
    prep = _stage1_prep(tensor, sp, rank)
    if omega_pre is not None:  # the generator ran while the host got here
        omega = omega_device_finish(omega_pre, stats=rstats)
    t_omega = time.perf_counter() - t0
    tm = _stage1_call(tensor, rank, omega, s_dev, sp, A, M, rank_found, status, timings is not None, a_signs,
                      base.power_iters, prep=prep)
    if timings is not None:
        timings.update(rstats)
        timings.update(omega_host_s=t_omega, stage1_sketch1_ms=tm[0], stage1_orth_ms=tm[1],
                       stage1_sketch2_ms=tm[2], stage1_factor_ms=tm[3], stage1_signs_ms=tm[4],
                       stage1_ms=tm[5], sp=sp, nseg=nseg_for(tensor), npieces=int(tensor.store(nseg_for(tensor))[0].npieces))
    if speculative:
        return A, M, rank_found, status, check
    return A, M, rank_found, status


def _stage1_prep(tensor, sp, rank):
    """(store, keepalive, workspace) of a dp2_stage1 call."""
    st, keep = tensor.store(nseg_for(tensor))
    ws = workspace(_lib.lib().dp2_stage1_workspace(C.byref(st), sp, rank), tensor.X.device)
    return st, keep, ws


def _stage1_call(tensor, rank, omega, s_dev, sp, A, M, rank_found, status, timed=False, a_signs=None,
                 power_iters=1, prep=None):
    """One dp2_stage1 call over ``tensor``'s slices (omega / s_dev / outputs
    already sliced to them); returns the phase timings when ``timed``."""
    st, keep, ws = prep if prep is not None else _stage1_prep(tensor, sp, rank)
    lib = _lib.lib()
    tm = (C.c_float * 8)() if timed else None
    if power_iters != 1:
        _lib.check(lib.dp2_stage1_power(C.byref(st), _vp(omega), _vp(s_dev), sp, rank, max(0, int(power_iters)),
                                        _vp(A), _vp(M), _vp(rank_found), _vp(a_signs), _vp(ws), ws.numel(),
                                        _vp(status), tm, stream_ptr()), "stage1")
    elif a_signs is None:
        _lib.check(lib.dp2_stage1(C.byref(st), _vp(omega), _vp(s_dev), sp, rank, _vp(A), _vp(M), _vp(rank_found),
                                  _vp(ws), ws.numel(), _vp(status), tm, stream_ptr()), "stage1")
    else:
        _lib.check(lib.dp2_stage1_signs(C.byref(st), _vp(omega), _vp(s_dev), sp, rank, _vp(A), _vp(M),
                                        _vp(rank_found), _vp(a_signs), _vp(ws), ws.numel(), _vp(status), tm,
                                        stream_ptr()), "stage1")
    del keep, ws
    return tm


# status words holding a (min) slice index (INT64_MAX = none) and counters;
# slices, not index lists (a list index would copy from pageable memory,
# which synchronises the stream)
_ST_INDEX = (slice(0, 1), slice(2, 4))
_ST_COUNT = (slice(1, 2), slice(4, 8))


def run_stage1_chunked(tensor: IrregularTensor, rank, base: RsvdParams, timings=None, speculative=False,
                       slice_ids=None, a_signs=None):
    """Stage 1 overlapped with the tensor's chunked upload: Omega for all
    slices first (independent of X), then per upload chunk of whole slices the
    compute stream waits for that chunk's copy event (device-side) and runs
    stage 1 on a view of its slices with their global seeds, writing straight
    into the full A / rank buffers (M block copied into place).  Per-chunk
    status words merge with the slice offset."""
    J, K = tensor.num_cols, tensor.num_slices
    rows = tensor.row_counts
    dev = tensor.X.device
    widths, sp, s_dev = _stage1_setup(tensor, rank, base.oversampling, dev)
    off = tensor.row_off_host
    bounds = [k1 for k1, _ in tensor._upload_events]
    subs, k0 = [], 0
    for k1 in bounds:  # chunk views (host-side plans only; no device waits yet)
        r0, r1 = int(off[k0]), int(off[k1])
        subs.append((k0, k1, IrregularTensor.from_packed(tensor.X[r0:r1], rows[k0:k1], J, dtype=tensor.dtype,
                                                         check=False)))
        k0 = k1
    t0 = time.perf_counter()
    rstats = {}
    check = None
    if speculative and _uses_tc(subs[0][2], sp):
        omega, check = omega_device(base.seed, J, widths, sp, dev, slice_ids=slice_ids, speculative=True,
                                    s_dev=s_dev)
    else:
        omega = omega_device(base.seed, J, widths, sp, dev, slice_ids=slice_ids, stats=rstats, s_dev=s_dev)
    t_omega = time.perf_counter() - t0
    A = torch.empty((int(off[-1]), rank), dtype=torch.float64, device=dev)
    M = torch.empty((J, K * rank), dtype=torch.float64, device=dev)
    rank_found = torch.empty(K, dtype=torch.int32, device=dev)
    status = new_status(dev)
    for k0, k1, sub in subs:
        tensor.wait_upload(k1)
        r0, r1 = int(off[k0]), int(off[k1])
        Mc = torch.empty((J, (k1 - k0) * rank), dtype=torch.float64, device=dev)
        st_c = new_status(dev)
        _stage1_call(sub, rank, omega[k0:k1], s_dev[k0:k1], sp, A[r0:r1], Mc, rank_found[k0:k1], st_c,
                     a_signs=None if a_signs is None else a_signs[k0:k1], power_iters=base.power_iters)
        M[:, k0 * rank:k1 * rank].copy_(Mc)
        for sl in _ST_INDEX:
            idx = st_c[sl]
            torch.minimum(status[sl], torch.where(idx == _lib.INT64_MAX, idx, idx + k0), out=status[sl])
        for sl in _ST_COUNT:
            status[sl] += st_c[sl]
    tensor.wait_upload()
    if timings is not None:
        timings.update(rstats)
        timings.update(omega_host_s=t_omega, stage1_chunks=len(bounds), sp=sp)
    if speculative:
        return A, M, rank_found, status, check
    return A, M, rank_found, status


def run_stage2(M, J, KR, rank, seed2, s2, om2, status, timings=None, power_iters=1):
    """Stage 2 (P/compress.py:109-111) on the device: D, E, F.

    A sketch wider than M's short side (s2 > min(J, KR), e.g. an explicit
    oversampling on few slices) spans range(M) with its first min(J, KR)
    columns already (almost surely, and exactly what the reference's
    Householder QR of the rank-deficient Y then keeps), so the device runs on
    those columns of the reference's Omega_2 -- the same D, E, F."""
    dev = M.device
    lib = _lib.lib()
    om2 = om2 if isinstance(om2, torch.Tensor) else torch.from_numpy(om2)
    if om2.device.type == "cpu" and not om2.is_pinned():
        om2 = om2.pin_memory()
    om2 = om2.to(dev, non_blocking=True)
    cap = int(min(J, KR))
    if s2 > cap >= rank:
        om2 = om2[:, :cap].contiguous()
        s2 = cap
    if s2 > 150:
        raise ValueError(f"stage-2 sketch width {s2} exceeds the device limit of 150")
    D = torch.empty((J, rank), dtype=torch.float64, device=dev)
    E = torch.empty(rank, dtype=torch.float64, device=dev)
    F = torch.empty((KR, rank), dtype=torch.float64, device=dev)
    ws2 = workspace(lib.dp2_stage2_workspace(J, KR, s2, rank), dev)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)] if timings is not None else None
    if ev:
        ev[0].record()
    _lib.check(lib.dp2_stage2_power(_vp(M), J, KR, _vp(om2), s2, rank, max(0, int(power_iters)), _vp(D), _vp(E),
                                    _vp(F), _vp(ws2), ws2.numel(), _vp(status), stream_ptr()), "stage2")
    if ev:
        ev[1].record()
        torch.cuda.synchronize()
        timings.update(stage2_ms=ev[0].elapsed_time(ev[1]), s2=s2)
    return D, E, F


def compress(tensor: IrregularTensor, rank, rsvd: RsvdParams | None = None, stage2: RsvdParams | None = None,
             plan=None, threads=None, timings=None):
    """Compress ``tensor`` at ``rank`` with two randomized-SVD stages."""
    comp, status = compress_async(tensor, rank, rsvd, stage2, plan, threads, timings)
    check_status(status, "compress")
    if omega_mismatch(comp):
        comp, status = compress_async(tensor, rank, rsvd, stage2, plan, threads, timings, exact_omega=True)
        check_status(status, "compress")
    return comp


def omega_mismatch(comp):
    """True when the speculative (tensor-core path) Omega of ``comp`` turned
    out to differ from the reference's (an acceptance decision of the
    ziggurat tail, practically never): the caller recomputes exactly."""
    chk = getattr(comp, "_omega_check", None)
    return chk is not None and bool(chk.result()["omega_mismatch"])


_OMEGA2_HOST = os.environ.get("DP2_OMEGA2_HOST", "0") not in ("", "0")


def compress_async(tensor: IrregularTensor, rank, rsvd: RsvdParams | None = None, stage2: RsvdParams | None = None,
                   plan=None, threads=None, timings=None, exact_omega=False, defer_signs=False):
    """``compress`` without the host synchronisation of its status check:
    returns (CompressedTensor, device status block); the caller checks the
    status (check_status) once its later work is enqueued.  ``defer_signs``
    (fit-internal): A is left up to its column signs (``comp.a_signs``)."""
    if not isinstance(tensor, IrregularTensor):
        tensor = IrregularTensor(tensor)
    checked = tensor.__dict__.setdefault("_rank_ok", set())
    if rank not in checked:
        check_rank(tensor, rank)
        checked.add(rank)
    resolve_threads(threads)
    base = rsvd if rsvd is not None else RsvdParams(rank=rank)
    J, K = tensor.num_cols, tensor.num_slices
    spec = not exact_omega
    chunked = len(tensor._upload_events) > 1
    pre = None
    if not chunked:  # the critical path starts with stage 1's Omega: enqueue it first
        widths, sp, s_dev = _stage1_setup(tensor, rank, base.oversampling, tensor.X.device)
        if not (spec and _uses_tc(tensor, sp)):
            pre = omega_device_launch(base.seed, J, widths, sp, tensor.X.device, s_dev=s_dev)
    second, s2 = stage2_params(base, stage2, rank, K, J)
    # DP2_OMEGA2_HOST=1: draw Omega_2 with NumPy while stage 1 runs (A/B knob)
    om2h = None if _OMEGA2_HOST else stage2_omega_launch(second.seed, K * rank, s2, tensor.X.device)
    a_signs = torch.empty((K, rank), dtype=torch.float64, device=tensor.X.device) if defer_signs else None
    if chunked:
        res = run_stage1_chunked(tensor, rank, base, timings=timings, speculative=spec, a_signs=a_signs)
    else:
        res = run_stage1(tensor, rank, base, timings=timings, speculative=spec, a_signs=a_signs, omega_pre=pre)
    A, M, rank_found, status = res[:4]
    check = res[4] if len(res) > 4 else None
    # stage-2 Omega (one stream, P/compress.py:109-111): generated on the
    # device ahead of stage 1; its few tail draws are replayed and patched
    # now, while stage 1 runs
    om2 = stage2_omega(second.seed, K * rank, s2) if om2h is None else stage2_omega_finish(om2h)
    D, E, F = run_stage2(M, J, K * rank, rank, second.seed, s2, om2, status, timings=timings,
                         power_iters=second.power_iters)
    comp = CompressedTensor(rank=rank, A=A, row_off=tensor.row_off_host.copy(), col_basis=D, weights=E,
                            cores=F, rank_found=rank_found, a_signs=a_signs)
    comp._omega_check = check
    if defer_signs:  # fit-internal: fit_dpar2 takes V^T M for the zero-pass fitness
        comp._stage1_M = M
    return comp, status


def reconstruct_slice(comp: CompressedTensor, k):
    """A_k (F_k (diag(E) D^T)) (P/compress.py:122-127)."""
    if not 0 <= k < comp.num_slices:
        raise IndexError(f"slice index {k} out of range [0, {comp.num_slices})")
    small = comp.core_block(k) @ (comp.weights[:, None] * comp.col_basis.T)
    return comp.slice_bases[k] @ small


def as_numpy_compressed(comp: CompressedTensor):
    """Host NumPy copy laid out like the reference's CompressedTensor fields."""
    return comp.numpy()
