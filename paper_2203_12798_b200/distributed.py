"""Multi-GPU DPar2: slices sharded over ranks (one process per GPU).

* Placement: ``greedy_partition(row_counts, world)`` -- the reference's Alg. 4
  (P/scheduler.py:29-51), bit-exact -- assigns slices to ranks; each rank keeps
  its slices in ascending global order.
* Stage 1: local, no communication; the per-slice sketch seeds use the
  GLOBAL slice index (derived_seed(seed, k), P/compress.py:96-103), so every
  slice gets exactly the reference's Omega_k wherever it lives.
* Stage 2: M (J x KR) must be in global slice order (P/compress.py:108).  Each
  rank scatters its J x R blocks into a zero J x KR buffer and one allreduce
  (sum) assembles M exactly -- every entry has a single nonzero contributor, so
  the sum is exact -- then stage 2 runs replicated (identical inputs, identical
  outputs on every rank).
* ALS (default ``als="replicated"``): after stage 2 every rank holds the full
  compressed tensor (D, E and all K R x R cores F_k -- K R^2 doubles, tiny),
  so each rank runs the single-GPU persistent ALS loop on all of it: no
  per-iteration communication at all; Q is then assembled for the local
  slices only (their A_k and polar factors).  ``als="sharded"`` keeps the
  phase-split variant: D, E, H, V replicated, F rows / W rows / rotations
  local, three allreduces of tiny buffers (2 R^2, 2 R^2, 1 doubles) per
  iteration between the phases of ``dp2_als_phase``.

The driver (``ShardedALS``) only sequences phases and collectives; the phase
compute is a pluggable ``ops`` object (the C ABI on the GPU; the gloo tests on
CPU substitute a NumPy emulation to check the sharded decomposition).
"""
from __future__ import annotations

import ctypes as C
import time

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from .scheduler import greedy_partition


def shard_slices(row_counts, world):
    """Per-rank global slice ids (LPT placement, ascending within a rank)."""
    plan = greedy_partition(row_counts, world)
    return [sorted(s) for s in plan.sets], plan.loads


def assemble_m(M_local, local_ids, K, R, group=None, cols=None):
    """Exact J x KR M in global slice order from each rank's J x K_local R blocks
    (``cols``: the device column index of the local blocks, see ``m_columns``)."""
    J = M_local.shape[0]
    full = torch.zeros((J, K * R), dtype=M_local.dtype, device=M_local.device)
    if len(local_ids):
        if cols is None:
            cols = m_columns(local_ids, R, M_local.device)
        full[:, cols] = M_local
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(full, group=group)
    return full


def m_columns(local_ids, R, device):
    """Device index of the local slices' columns of M (rows of F): k R + r.
    Built from pinned memory (a pageable copy would synchronise the stream)."""
    from .tensor import to_device_async
    ids = np.asarray(local_ids, dtype=np.int64)
    cols = (ids[:, None] * R + np.arange(R, dtype=np.int64)[None, :]).reshape(-1)
    if torch.device(device).type != "cuda":
        return torch.from_numpy(cols)
    return to_device_async(cols, torch.int64, device)


def local_rows(F, local_ids, R):
    """Rows of F (KR x R) belonging to the local slices, in local order."""
    idx = (torch.as_tensor(local_ids, device=F.device)[:, None] * R +
           torch.arange(R, device=F.device)[None, :]).reshape(-1)
    return F.index_select(0, idx).contiguous()


def replicated_als(F, D, E, K, J, R, h, v, w, max_iters, tol, normalize):
    """The single-GPU ALS loop (``dp2_als_run``: one cooperative launch for
    R <= 16) on the FULL compressed tensor (global K); returns device H, V, W
    (K x R), polar (K x R x R), trace, tstamp, iters, status."""
    from .tensor import new_status, stream_ptr, to_device_async
    dev = D.device
    lib = _lib.lib()
    H = to_device_async(np.ascontiguousarray(h), torch.float64, dev)
    V = to_device_async(np.ascontiguousarray(v), torch.float64, dev)
    W = to_device_async(np.ascontiguousarray(w), torch.float64, dev)
    polar = torch.empty((K, R, R), dtype=torch.float64, device=dev)
    trace = torch.zeros(max_iters, dtype=torch.float64, device=dev)
    tstamp = torch.zeros(max_iters + 1, dtype=torch.int64, device=dev)
    iters = torch.zeros(1, dtype=torch.int32, device=dev)
    ws = torch.empty(max(256, int(lib.dp2_als_workspace(K, J, R))), dtype=torch.uint8, device=dev)
    status = new_status(dev)
    vp = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
    _lib.check(lib.dp2_als_run(vp(F), vp(D), vp(E), K, J, R, vp(H), vp(V), vp(W), vp(polar), max_iters, float(tol),
                               int(bool(normalize)), vp(trace), vp(tstamp), vp(iters), 0, vp(ws), ws.numel(),
                               vp(status), stream_ptr()), "als_run")
    return H, V, W, polar, trace, tstamp, iters, status


class ShardedALS:
    """Phase sequencer: per iteration three allreduces of R x R sized partials."""

    def __init__(self, ops, allreduce):
        self.ops, self.allreduce = ops, allreduce

    def run(self, max_iters):
        self.ops.phase(0)
        for it in range(max_iters):
            red = self.allreduce(self.ops.phase(1, it=it))
            self.ops.phase(2, it=it, red_in=red)
            red = self.allreduce(self.ops.phase(3, it=it))
            self.ops.phase(4, it=it, red_in=red)
            red = self.allreduce(self.ops.phase(5, it=it))
            self.ops.phase(6, it=it, red_in=red)


class GpuAlsOps:
    """``dp2_als_phase`` on the local slices."""

    def __init__(self, F_local, D, E, H, V, W_local, J, R, max_iters, tol, normalize):
        dev = D.device
        self.F, self.D, self.E, self.H, self.V, self.W = F_local, D, E, H, V, W_local
        self.K, self.J, self.R = W_local.shape[0], J, R
        self.tol, self.normalize = float(tol), int(bool(normalize))
        self.polar = torch.empty((self.K, R, R), dtype=torch.float64, device=dev)
        self.trace = torch.zeros(max_iters, dtype=torch.float64, device=dev)
        self.tstamp = torch.zeros(max_iters + 1, dtype=torch.int64, device=dev)
        self.iters = torch.zeros(1, dtype=torch.int32, device=dev)
        self.red = torch.zeros(2 * R * R, dtype=torch.float64, device=dev)
        self.ws = torch.empty(max(256, int(_lib.lib().dp2_als_workspace(self.K, J, R))), dtype=torch.uint8,
                              device=dev)
        from .tensor import new_status
        self.status = new_status(dev)

    def phase(self, ph, it=0, red_in=None):
        from .tensor import stream_ptr
        vp = lambda t: C.c_void_p(t.data_ptr()) if t is not None else C.c_void_p(0)  # noqa: E731
        n = 2 * self.R * self.R if ph in (1, 3) else 1
        out = self.red[:n] if ph in (1, 3, 5) else None
        _lib.check(_lib.lib().dp2_als_phase(
            ph, vp(self.F), vp(self.D), vp(self.E), self.K, self.J, self.R, vp(self.H), vp(self.V), vp(self.W),
            vp(self.polar), it, self.tol, self.normalize, vp(self.trace), vp(self.tstamp), vp(self.iters),
            vp(red_in), vp(out), vp(self.ws), self.ws.numel(), vp(self.status),
            stream_ptr()), f"als_phase{ph}")
        return out.clone() if out is not None else None


def nccl_allreduce(group=None):
    def f(t):
        if dist.is_initialized() and dist.get_world_size(group) > 1:
            dist.all_reduce(t, group=group)
        return t
    return f


class DistributedFit:
    """This rank's shard of a synthetic BASELINE-model tensor, fitted jointly
    with the other ranks (bench.py's N > 1 path)."""

    def __init__(self, cfg, seed, rank, world, host_slices=None):
        """``host_slices``: this rank's slices (``synth.generate(cfg, seed,
        slices=shard)``) to upload; default: draw them on the device."""
        from . import synth
        from .tensor import IrregularTensor
        rows_all, _, _ = synth.shared_factors(cfg, seed)
        shards, loads = shard_slices(rows_all, world)
        self.local_ids = shards[rank]
        self.rank, self.world, self.cfg, self.seed = rank, world, cfg, seed
        if host_slices is not None:
            up = IrregularTensor(host_slices, dtype=cfg.dtype)
            up.wait_upload()
            rows = up.row_counts
            self.tensor = IrregularTensor.from_packed(up.X, rows, cfg.cols, dtype=cfg.dtype)
        else:
            X, rows, _, _ = synth.generate_device(cfg, seed, slices=self.local_ids)
            self.tensor = IrregularTensor.from_packed(X, rows, cfg.cols)
        self.local_rows = int(sum(rows))
        self.total_rows = int(sum(rows_all))
        self.total_entries = self.total_rows * cfg.cols
        self.K = cfg.num_slices
        self.loads = loads

    def fit(self, R, opts, timings=None, als="replicated", tensor=None, _exact_omega=False):
        """Fit the whole tensor with this rank's slices from ``tensor`` (default:
        the device-resident shard; a host-backed ``IrregularTensor`` of the same
        slices is uploaded in chunks overlapped with stage 1, as in
        ``fit_dpar2``).  Like ``fit_dpar2`` the fit is enqueued without host
        synchronisation (speculative stage-1 Omega, index tensors from pinned
        memory) and synchronises once at the end; a speculative-Omega mismatch
        on ANY rank (agreed by one allreduce) makes every rank redo exactly."""
        from .compress import check_status, run_stage1, run_stage1_chunked, run_stage2, stage2_params
        from .factors import FitTrace, Parafac2Factors, SliceViews, initial_factors
        from .linalg import RsvdParams
        from .rng import stage2_omega_finish, stage2_omega_launch
        from .solver import assemble_q
        from .tensor import to_device_async
        t = self.tensor if tensor is None else tensor
        J, K = t.num_cols, self.K
        dev = t.X.device
        if getattr(self, "_dev_index", None) is None or self._dev_index[0] != (R, dev):
            self._dev_index = ((R, dev), m_columns(self.local_ids, R, dev),
                               to_device_async(np.asarray(self.local_ids, dtype=np.int64), torch.int64, dev))
        _, cols, ids = self._dev_index
        base = RsvdParams(rank=R, seed=opts.seed)
        second, s2 = stage2_params(base, None, R, K, J)
        started = time.perf_counter()
        om2h = stage2_omega_launch(second.seed, K * R, s2, dev)  # replicated on every rank, ahead of stage 1
        spec = not _exact_omega
        a_signs = torch.empty((t.num_slices, R), dtype=torch.float64, device=dev)  # folded into Q's Pi_k
        if len(t._upload_events) > 1:
            res = run_stage1_chunked(t, R, base, timings=timings, speculative=spec, slice_ids=self.local_ids,
                                     a_signs=a_signs)
        else:
            res = run_stage1(t, R, base, slice_ids=self.local_ids, timings=timings, speculative=spec,
                             a_signs=a_signs)
        A, M_local, rank_found, status = res[:4]
        check = res[4] if len(res) > 4 else None
        om2 = stage2_omega_finish(om2h)  # tail replay + patch, while stage 1 runs
        M = assemble_m(M_local, self.local_ids, K, R, cols=cols)
        D, E, F = run_stage2(M, J, K * R, R, second.seed, s2, om2, status, timings=timings)
        normalize = bool(opts.normalize) if opts.normalize is not None else True
        if als == "replicated":
            h, v, w = initial_factors(J, K, R, opts.seed)
            H, V, W, polar, trace, tstamp, iters, st_als = replicated_als(
                F, D, E, K, J, R, h, v, w, opts.max_iters, opts.tol, normalize)
            polar_local = polar.index_select(0, ids)
            W_out = W.index_select(0, ids)
        else:
            h, v, w = initial_factors(J, len(self.local_ids), R, opts.seed)
            H, V = torch.from_numpy(h).to(dev), torch.from_numpy(v).to(dev)
            W = torch.from_numpy(w).to(dev)
            ops = GpuAlsOps(local_rows(F, self.local_ids, R), D, E, H, V, W, J, R, opts.max_iters, opts.tol,
                            normalize)
            ShardedALS(ops, nccl_allreduce()).run(opts.max_iters)
            st_als = ops.status
            H, V, W_out, polar_local = ops.H, ops.V, ops.W, ops.polar
            trace, tstamp, iters = ops.trace, ops.tstamp, ops.iters
        from .compress import CompressedTensor
        comp = CompressedTensor(rank=R, A=A, row_off=t.row_off_host.copy(), col_basis=D, weights=E, cores=F,
                                a_signs=a_signs)
        Q = assemble_q(t, comp, polar_local.contiguous())
        torch.cuda.current_stream().synchronize()
        t._upload_keep = None
        mismatch = bool(check.result()["omega_mismatch"]) if check is not None else False
        if dist.is_initialized() and dist.get_world_size() > 1:
            flag = torch.tensor([int(mismatch)], dtype=torch.int32, device=dev)
            dist.all_reduce(flag, op=dist.ReduceOp.MAX)
            mismatch = bool(flag.item())
        if mismatch:
            return self.fit(R, opts, timings, als, tensor, _exact_omega=True)
        check_status(status, "compress")
        check_status(st_als, "fit_dpar2")
        pre = time.perf_counter() - started
        n = int(iters.item())
        tr = FitTrace(objective=trace[:n].cpu().tolist(),
                      seconds=list(np.diff(tstamp[:n + 1].cpu().numpy()) * 1e-9), preprocess_seconds=pre,
                      compressed_float_count=self.total_rows * R + K * R * R + J * R + R)
        if n >= 2:
            prev, e = tr.objective[-2], tr.objective[-1]
            tr.converged = bool(prev == 0.0 or abs(prev - e) <= opts.tol * prev)
        bounds = t.row_off_host
        factors = Parafac2Factors(H=H, V=V, W=W_out, Q=SliceViews(Q, bounds), Q_packed=Q)
        return factors, tr
