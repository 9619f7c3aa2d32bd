"""Multi-GPU DPar2: slices sharded over ranks (one process per GPU).

* Placement: ``greedy_partition(row_counts, world)`` -- the reference's Alg. 4
  (P/scheduler.py:29-51), bit-exact -- assigns slices to ranks; each rank keeps
  its slices in ascending global order.
* Stage 1: local, no communication; the per-slice sketch seeds use the
  GLOBAL slice index (derived_seed(seed, k), P/compress.py:96-103), so every
  slice gets exactly the reference's Omega_k wherever it lives.
* Stage 2: M (J x KR) must be in global slice order (P/compress.py:108).  One
  all-gather of every rank's J x K_local R block (padded to the largest
  shard) and a column permutation assemble it exactly (each rank sends 1/world
  of M instead of allreducing a zero-padded J x KR buffer); stage 2 then runs
  replicated (identical inputs, identical outputs on every rank).
* ALS, ``als="auto"`` (default) picks by a measured cost model:
  - ``"replicated"``: every rank holds the whole compressed tensor (D, E and
    the K R x R cores -- tiny), so it runs the single-GPU persistent loop on
    all of it with no per-iteration communication, then assembles Q for its
    own slices (the winner at c2 scale: the persistent loop takes ~1.9 ms for
    K = 1000);
  - ``"sharded"``: D, E, H, V replicated; F rows, W rows and rotations local;
    per iteration three allreduces of R x R sized partials between the phases
    of ``dp2_als_phase`` (P/solver.py:81-111 and 133-149 are K-reductions),
    the whole 32-iteration phase + NCCL sequence captured once in a CUDA graph
    and replayed (the winner when K / world is large, e.g. c5: K = 20 000).

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


def gather_plan(shards, R, device):
    """(block width, column permutation) of the all-gather M assembly: rank r
    sends its J x K_r R block padded to ``width`` columns; global column
    k R + c of M is column perm[k R + c] of the gathered J x (world width)."""
    width = max(len(s) for s in shards) * R
    K = sum(len(s) for s in shards)
    perm = np.empty(K * R, dtype=np.int64)
    for r, ids in enumerate(shards):
        for li, k in enumerate(ids):
            perm[k * R:(k + 1) * R] = r * width + li * R + np.arange(R)
    if torch.device(device).type != "cuda":
        return width, torch.from_numpy(perm)
    from .tensor import to_device_async
    return width, to_device_async(perm, torch.int64, device)


def assemble_m(M_local, local_ids, K, R, group=None, shards=None, plan=None):
    """Exact J x KR M in global slice order from each rank's J x K_local R
    block: one all-gather (blocks padded to the largest shard) and a column
    permutation.  ``shards``: every rank's global slice ids (needed for
    world > 1); ``plan``: a cached ``gather_plan``."""
    J = M_local.shape[0]
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if world == 1:
        if list(local_ids) == list(range(K)):
            return M_local
        full = torch.zeros((J, K * R), dtype=M_local.dtype, device=M_local.device)
        full[:, m_columns(local_ids, R, M_local.device)] = M_local
        return full
    width, perm = plan if plan is not None else gather_plan(shards, R, M_local.device)
    send = M_local
    if send.shape[1] != width:
        send = torch.zeros((J, width), dtype=M_local.dtype, device=M_local.device)
        send[:, :M_local.shape[1]] = M_local
    send = send.contiguous()
    buf = torch.empty((world * J, width), dtype=M_local.dtype, device=M_local.device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(buf, send, group=group)
    else:
        dist.all_gather(list(buf.view(world, J, width).unbind(0)), send, group=group)
    return buf.view(world, J, width).permute(1, 0, 2).reshape(J, world * width).index_select(1, perm)


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


class GraphedShardedALS:
    """The sharded loop with static buffers, captured once (all phases of all
    iterations plus the NCCL allreduces between them) into a CUDA graph and
    replayed per fit: no per-phase host launches.  Falls back to eager
    sequencing if the capture is refused (e.g. a backend without graph-safe
    collectives)."""

    def __init__(self, K_local, J, R, max_iters, tol, normalize, dev, allreduce):
        f64 = dict(dtype=torch.float64, device=dev)
        self.F = torch.zeros((K_local * R, R), **f64)
        self.D = torch.zeros((J, R), **f64)
        self.E = torch.zeros(R, **f64)
        self.H = torch.zeros((R, R), **f64)
        self.V = torch.zeros((J, R), **f64)
        self.W = torch.zeros((K_local, R), **f64)
        self.ops = GpuAlsOps(self.F, self.D, self.E, self.H, self.V, self.W, J, R, max_iters, tol, normalize)
        self.allreduce, self.max_iters = allreduce, max_iters
        self.graph = None
        self.captured = False

    def run(self, F_local, D, E, H, V, W):
        from .tensor import new_status
        for dst, src in ((self.F, F_local), (self.D, D), (self.E, E), (self.H, H), (self.V, V), (self.W, W)):
            dst.copy_(src)
        self.ops.status.copy_(new_status(self.F.device))
        if self.graph is None:
            try:
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    ShardedALS(self.ops, self.allreduce).run(self.max_iters)
                self.graph, self.captured = g, True
            except Exception:  # capture refused: eager from now on
                self.graph = False
        if self.graph:
            self.graph.replay()
        else:
            ShardedALS(self.ops, self.allreduce).run(self.max_iters)
        return self.ops


def als_policy(K, world, J, R, nccl_us=16.0):
    """'replicated' or 'sharded' by the cost model of DESIGN.md §7, measured on
    one B200 for 32 iterations at J = 1000 (tools/scratch/als_scale.py,
    shard_cost.py): the persistent replicated loop costs ~0.9 ms + 0.9 us per
    slice (K = 1000: 1.9 ms, 20 000: 18.8 ms); the graph-captured sharded
    phase loop ~4 ms + 1.9 us per local slice (125: 5.8 ms, 2 500: 12.0 ms)
    plus 96 allreduces of R x R partials (~16 us each, NCCL small-message
    floor).  c2 (K = 1000) stays replicated at any world size; c5 (K = 20 000)
    shards from 4 GPUs up."""
    if world <= 1:
        return "replicated"
    if R > 16:  # the persistent loop covers R <= 16; beyond it both use the phase kernels
        return "sharded"
    t_rep = 0.9 + 0.9e-3 * K
    k_local = -(-K // world)
    t_shard = 4.0 + 1.9e-3 * k_local + 32 * 3 * nccl_us * 1e-3
    return "sharded" if t_shard < t_rep else "replicated"


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
        self.shards = shards
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

    def fit(self, R, opts, timings=None, als="auto", tensor=None, _exact_omega=False):
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
        if getattr(self, "_gather", None) is None or self._gather[0] != (R, dev):
            self._gather = ((R, dev), gather_plan(self.shards, R, dev))
        M = assemble_m(M_local, self.local_ids, K, R, shards=self.shards, plan=self._gather[1])
        D, E, F = run_stage2(M, J, K * R, R, second.seed, s2, om2, status, timings=timings)
        normalize = bool(opts.normalize) if opts.normalize is not None else True
        if als == "auto":
            als = als_policy(K, self.world, J, R)
        self.last_als = als
        if als == "replicated":
            h, v, w = initial_factors(J, K, R, opts.seed)
            H, V, W, polar, trace, tstamp, iters, st_als = replicated_als(
                F, D, E, K, J, R, h, v, w, opts.max_iters, opts.tol, normalize)
            polar_local = polar.index_select(0, ids)
            W_out = W.index_select(0, ids)
        else:
            h, v, w = initial_factors(J, len(self.local_ids), R, opts.seed)
            key = (len(self.local_ids), J, R, opts.max_iters, float(opts.tol), normalize, dev)
            if getattr(self, "_als_graph", None) is None or self._als_graph[0] != key:
                self._als_graph = (key, GraphedShardedALS(len(self.local_ids), J, R, opts.max_iters, opts.tol,
                                                          normalize, dev, nccl_allreduce()))
            if getattr(self, "_ids_f", None) is None or self._ids_f[0] != (R, dev):
                self._ids_f = ((R, dev), (torch.as_tensor(self.local_ids, device=dev)[:, None] * R +
                                          torch.arange(R, device=dev)[None, :]).reshape(-1))
            to = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev, non_blocking=False)  # noqa: E731
            ops = self._als_graph[1].run(F.index_select(0, self._ids_f[1]), D, E, to(h), to(v), to(w))
            # the graph's static buffers are reused by the next fit: copy the results out
            st_als = ops.status.clone()
            H, V, W_out, polar_local = ops.H.clone(), ops.V.clone(), ops.W.clone(), ops.polar.clone()
            trace, tstamp, iters = ops.trace.clone(), ops.tstamp.clone(), ops.iters.clone()
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
