"""Irregular dense tensor held in a packed HBM store (P/tensor.py:34-80).

All K slices (I_k x J) live in ONE device buffer of shape (sum I_k, ldx):
slice k is rows [row_off[k], row_off[k+1]).  ``ldx`` pads rows to 16 bytes
(padding columns are zero) so every row is a whole number of 16-byte
``cp.async`` chunks.  Construction mirrors the reference's validation order and
messages (2-D, non-empty, consistent J, finite).  Host slices upload
asynchronously in chunks of whole slices on a copy stream (one event per
chunk, so stage 1 can start on the first chunks while the rest is in flight)
and the finiteness scan runs on host threads over the same memory meanwhile;
device inputs are scanned on the device.  Squared norms are computed lazily.

``dtype='f64'`` is the reference's float64 container; ``dtype='f32'`` is the
optional fp32 mode (the reference sees the same values upcast exactly).
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib
from .errors import NonFiniteInputError, ShapeMismatchError

_TORCH = {"f64": torch.float64, "f32": torch.float32}
_NP = {"f64": np.float64, "f32": np.float32}


def _ldx_for(J, dtype):
    per = 2 if dtype == "f64" else 4
    return ((J + per - 1) // per) * per


def device():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2203_12798_b200 needs a CUDA device (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr(dev=None):
    """Raw handle of the current CUDA stream of ``dev`` (default: the current
    device; torch's C accessor: no Stream object per call -- a fit passes it a
    dozen times on its enqueue path)."""
    index = torch.cuda.current_device() if dev is None else torch.device(dev).index
    if index is None:
        index = torch.cuda.current_device()
    return C.c_void_p(torch._C._cuda_getCurrentRawStream(index))


_COPY_STREAMS = {}
UPLOAD_CHUNKS = 6          # upload chunks of whole slices (stage 1 overlaps all but the last)
UPLOAD_MIN_CHUNK = 64 << 20


def copy_stream(dev):
    """Per-device stream for host->device uploads."""
    key = dev.index if dev.index is not None else torch.cuda.current_device()
    if key not in _COPY_STREAMS:
        _COPY_STREAMS[key] = torch.cuda.Stream(device=dev)
    return _COPY_STREAMS[key]


def sm_count():
    return torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count


def _coalesce_pinned(arrs, J, tdt):
    """Merge runs of row-adjacent, contiguous pinned host tensors that view one
    storage (e.g. slices cut from one pinned buffer) into single tensors, so
    the upload is one large async copy per run instead of one per slice."""
    out, run, run_rows, end = [], None, 0, None
    for a in arrs:
        ok = (isinstance(a, torch.Tensor) and a.device.type == "cpu" and a.dtype == tdt and a.is_contiguous()
              and a.shape[1] == J and a.is_pinned())
        if ok and run is not None and a.untyped_storage().data_ptr() == run.untyped_storage().data_ptr() \
                and a.data_ptr() == end:
            run_rows += a.shape[0]
            end = a.data_ptr() + a.numel() * a.element_size()
            continue
        if run is not None:
            out.append(torch.empty(0, dtype=tdt).set_(run.untyped_storage(), run.storage_offset(), (run_rows, J),
                                                      (J, 1)))
            run = None
        if ok:
            run, run_rows, end = a, a.shape[0], a.data_ptr() + a.numel() * a.element_size()
        else:
            out.append(a)
    if run is not None:
        out.append(torch.empty(0, dtype=tdt).set_(run.untyped_storage(), run.storage_offset(), (run_rows, J), (J, 1)))
    return out


class IrregularTensor:
    """K dense slices (I_k x J) sharing the column count J, packed on the GPU."""

    def __init__(self, slices, dtype="f64"):
        if dtype not in _TORCH:
            raise ValueError(f"dtype must be 'f64' or 'f32', got {dtype!r}")
        # a reference container (P/tensor.py:34-80) passes through the CLI seam
        # (P/cli.py:45, 113-121): take its slices
        if not isinstance(slices, (list, tuple)) and hasattr(slices, "slices"):
            slices = list(slices.slices)
        if len(slices) < 1:
            raise ShapeMismatchError("tensor needs at least one slice")
        cols = None
        arrs = []
        for k, x in enumerate(slices):
            if isinstance(x, torch.Tensor):
                shape = tuple(x.shape)
            else:
                x = np.asarray(x)
                shape = x.shape
            if len(shape) != 2:
                raise ShapeMismatchError(f"slice {k} must be 2-D, got ndim={len(shape)}")
            if shape[0] < 1 or shape[1] < 1:
                raise ShapeMismatchError(f"slice {k} has empty shape {shape}")
            if cols is None:
                cols = shape[1]
            elif shape[1] != cols:
                raise ShapeMismatchError(
                    f"inconsistent column counts: slice 0 has {cols}, slice {k} has {shape[1]}")
            arrs.append(x)
        self.dtype = dtype
        self._J = int(cols)
        self._rows = [int(a.shape[0]) for a in arrs]
        self._host = None if any(isinstance(a, torch.Tensor) for a in arrs) else arrs
        self._upload_events = []
        self._upload_keep = None
        if all(not (isinstance(a, torch.Tensor) and a.device.type != "cpu") for a in arrs):
            self._upload_host(arrs)
        else:
            self._upload(arrs)
            self._stats()

    # ------------------------------------------------------------ construction
    @classmethod
    def from_packed(cls, packed, row_counts, num_cols, dtype=None, check=True):
        """Wrap an existing device buffer (sum I_k, ldx) without copying."""
        self = cls.__new__(cls)
        self.dtype = dtype or ("f64" if packed.dtype == torch.float64 else "f32")
        self._J = int(num_cols)
        self._rows = [int(r) for r in row_counts]
        self._host = None
        self.X = packed
        self.ldx = packed.shape[1]
        self._upload_events = []
        self._upload_keep = None
        self._finish_layout()
        if check:
            self._stats()
        return self

    @classmethod
    def plan_only(cls, row_counts, dev):
        """Row layout and piece plans of a tensor whose values are absent (e.g.
        the slice bases of a loaded compressed tensor): consumers that only
        walk rows by pieces (assemble_q) take its store; X is a one-row
        16-byte placeholder broadcast over the rows and never read."""
        X = torch.zeros((1, 2), dtype=torch.float64, device=dev).expand(int(sum(row_counts)), 2)
        return cls.from_packed(X, row_counts, 1, dtype="f64", check=False)

    def _finish_layout(self):
        dev = self.X.device
        off = np.zeros(len(self._rows) + 1, np.int64)
        np.cumsum(self._rows, out=off[1:])
        self.row_off_host = off
        self.row_off = to_device_async(off, torch.int64, dev)
        self._plans = {}
        self._sqnorm = None

    def _upload(self, arrs):
        dev = device()
        J = self._J
        self.ldx = _ldx_for(J, self.dtype)
        total = int(sum(self._rows))
        tdt = _TORCH[self.dtype]
        self.X = torch.zeros((total, self.ldx), dtype=tdt, device=dev) if self.ldx != J else \
            torch.empty((total, J), dtype=tdt, device=dev)
        r = 0
        for a in _coalesce_pinned(arrs, J, tdt):
            n = a.shape[0]
            if isinstance(a, torch.Tensor):
                # pinned host tensors go straight into the packed buffer (async H2D)
                src = a if (a.device.type == "cpu" and a.dtype == tdt) else a.to(device=dev, dtype=tdt)
            else:
                src = torch.from_numpy(np.ascontiguousarray(a, dtype=_NP[self.dtype]))
            if self.ldx == J:
                self.X[r:r + n].copy_(src, non_blocking=True)
            else:
                self.X[r:r + n, :J].copy_(src, non_blocking=True)
            r += n
        self._finish_layout()

    def _upload_host(self, arrs):
        """Host slices: chunked async H2D on the copy stream (pinned sources
        are DMA'd directly; pageable ones are staged by the driver) with an
        event per chunk of whole slices, and the reference's isfinite check
        (P/tensor.py:61) on host threads while the copies are in flight."""
        dev = device()
        J = self._J
        self.ldx = _ldx_for(J, self.dtype)
        tdt, ndt = _TORCH[self.dtype], _NP[self.dtype]
        srcs = []
        for a in arrs:
            if isinstance(a, torch.Tensor):
                t = a if a.dtype == tdt else a.to(tdt)
            else:
                t = torch.from_numpy(np.asarray(a, dtype=ndt))
            if t.stride(1) != 1:
                t = t.contiguous()
            srcs.append(t)
        total = int(sum(self._rows))
        self.X = torch.zeros((total, self.ldx), dtype=tdt, device=dev) if self.ldx != J else \
            torch.empty((total, J), dtype=tdt, device=dev)
        self._finish_layout()
        cs = copy_stream(dev)
        cs.wait_stream(torch.cuda.current_stream())  # the allocation / zero fill above
        off = self.row_off_host
        esz = torch.empty(0, dtype=tdt).element_size()
        K = len(srcs)
        events = []
        target = max(UPLOAD_MIN_CHUNK, -(-total * J * esz // UPLOAD_CHUNKS))
        with torch.cuda.stream(cs):
            k0 = 0
            while k0 < K:
                k1, nbytes = k0, 0
                while k1 < K and (k1 == k0 or nbytes < target):
                    nbytes += self._rows[k1] * J * esz
                    k1 += 1
                self._copy_run(srcs, k0, k1, off, J)
                ev = torch.cuda.Event()
                ev.record(cs)
                events.append((k1, ev))
                k0 = k1
        self._upload_events = events
        self._upload_keep = srcs
        # host isfinite scan over the same memory, concurrent with the DMA
        ptrs = np.fromiter((t.data_ptr() for t in srcs), dtype=np.uint64, count=K)
        rows = np.asarray(self._rows, dtype=np.int64)
        lds = np.fromiter((t.stride(0) for t in srcs), dtype=np.int64, count=K)
        bad = C.c_int64(0)
        _lib.check(_lib.lib().dp2_host_first_nonfinite(
            C.c_void_p(ptrs.ctypes.data), C.c_void_p(rows.ctypes.data), C.c_void_p(lds.ctypes.data), K, J,
            _lib.DP2_F64 if self.dtype == "f64" else _lib.DP2_F32, 0, C.byref(bad)), "host_first_nonfinite")
        if bad.value != _lib.INT64_MAX:
            cs.synchronize()
            raise NonFiniteInputError(f"slice {bad.value} contains non-finite values")

    def _copy_run(self, srcs, k0, k1, off, J):
        """Copy slices [k0, k1) into X: one copy per run of slices that are
        row-contiguous views of one storage, else one per slice."""
        k = k0
        while k < k1:
            t = srcs[k]
            e = k + 1
            if t.is_contiguous():
                end = t.data_ptr() + t.numel() * t.element_size()
                base = t.untyped_storage().data_ptr()
                while e < k1 and srcs[e].is_contiguous() and srcs[e].data_ptr() == end and \
                        srcs[e].untyped_storage().data_ptr() == base:
                    end = srcs[e].data_ptr() + srcs[e].numel() * srcs[e].element_size()
                    e += 1
            r0, r1 = int(off[k]), int(off[e])
            if e - k > 1:
                src = torch.empty(0, dtype=t.dtype).set_(t.untyped_storage(), t.storage_offset(), (r1 - r0, J),
                                                        (J, 1))
            else:
                src = t
            dst = self.X[r0:r1] if self.ldx == J else self.X[r0:r1, :J]
            dst.copy_(src, non_blocking=True)
            k = e

    def wait_upload(self, k_end=None):
        """Make the current stream wait (device-side, no host sync) for the
        upload of slices [0, k_end) -- all of it by default."""
        if not self._upload_events:
            return
        cur = torch.cuda.current_stream()
        if k_end is None:
            cur.wait_event(self._upload_events[-1][1])
            self._upload_events = []
            return
        for k1, ev in self._upload_events:
            if k1 >= k_end:
                cur.wait_event(ev)
                return

    def _stats(self):
        self.wait_upload()
        dev = self.X.device
        sq = torch.empty(self.num_slices, dtype=torch.float64, device=dev)
        status = new_status(dev)
        st, keep = self.store(1)
        _lib.check(_lib.lib().dp2_slice_stats(C.byref(st), C.c_void_p(sq.data_ptr()),
                                              C.c_void_p(status.data_ptr()), stream_ptr()), "slice_stats")
        s = status.cpu()
        bad = int(s[0])
        if bad != _lib.INT64_MAX:
            raise NonFiniteInputError(f"slice {bad} contains non-finite values")
        self._sqnorm = sq
        del keep

    # ------------------------------------------------------------ plan
    def store(self, nseg):
        """(dp2_store, keepalive) for a streaming plan with ``nseg`` segments."""
        if nseg not in self._plans:
            K = self.num_slices
            cap = _lib.lib().dp2_piece_capacity(K, nseg)
            ps = np.empty(cap, np.int32)
            pr0 = np.empty(cap, np.int64)
            prs = np.empty(cap, np.int32)
            sb = np.empty(nseg + 1, np.int32)
            sl = np.empty(K + 1, np.int32)
            npc = C.c_int64(0)
            P = C.POINTER
            _lib.check(_lib.lib().dp2_plan_pieces(
                self.row_off_host.ctypes.data_as(P(C.c_int64)), K, nseg, ps.ctypes.data_as(P(C.c_int32)),
                pr0.ctypes.data_as(P(C.c_int64)), prs.ctypes.data_as(P(C.c_int32)),
                sb.ctypes.data_as(P(C.c_int32)), sl.ctypes.data_as(P(C.c_int32)), C.byref(npc)), "plan_pieces")
            n = npc.value
            dev = self.X.device
            arrays = dict(piece_slice=to_device_async(ps[:n], torch.int32, dev),
                          piece_row0=to_device_async(pr0[:n], torch.int64, dev),
                          piece_rows=to_device_async(prs[:n], torch.int32, dev),
                          seg_begin=to_device_async(sb, torch.int32, dev),
                          slice_piece=to_device_async(sl, torch.int32, dev))
            self._plans[nseg] = (n, arrays, dict(piece_slice=ps[:n].copy(), slice_piece=sl.copy()))
        n, arrays, _ = self._plans[nseg]
        self.wait_upload()
        st = _lib.Store()
        st.X = self.X.data_ptr()
        st.dtype = _lib.DP2_F64 if self.dtype == "f64" else _lib.DP2_F32
        st.nseg = nseg
        st.ldx = self.ldx
        st.J = self._J
        st.K = self.num_slices
        st.total_rows = int(self.row_off_host[-1])
        st.npieces = n
        st.row_off = self.row_off.data_ptr()
        for name, t in arrays.items():
            setattr(st, name, t.data_ptr())
        return st, (self.X, self.row_off, arrays)

    def plan_host(self, nseg):
        self.store(nseg)
        return self._plans[nseg][2]

    # ------------------------------------------------------------ reference surface
    @property
    def num_slices(self):
        return len(self._rows)

    @property
    def num_cols(self):
        return self._J

    @property
    def row_counts(self):
        return list(self._rows)

    @property
    def slices(self):
        """Host float64 views of the slices (the reference's ``slices``)."""
        if self._host is None:
            self.wait_upload()
            x = self.X[:, :self._J].double().cpu().numpy()
            self._host = [x[a:b] for a, b in zip(self.row_off_host[:-1], self.row_off_host[1:])]
        return [np.asarray(a, dtype=np.float64) for a in self._host]

    def total_sq_norm(self):
        return float(self.slice_sq_norms().sum().item())

    def slice_sq_norms(self):
        if self._sqnorm is None:
            self._stats()
        return self._sqnorm


_STATUS_TEMPLATE = {}


def new_status(dev):
    """Fresh device status block (index words INT64_MAX, counters 0): one
    device-to-device clone of a cached template (no host copy, so no implicit
    stream synchronisation)."""
    key = str(dev)
    tpl = _STATUS_TEMPLATE.get(key)
    if tpl is None:
        tpl = torch.zeros(_lib.STATUS_WORDS, dtype=torch.int64, device=dev)
        tpl[0:1].fill_(_lib.INT64_MAX)
        tpl[2:4].fill_(_lib.INT64_MAX)
        _STATUS_TEMPLATE[key] = tpl
    return tpl.clone()


_SMALL_KEEP = []          # (pinned source, completion event) of small uploads
_SMALL_KEEP_MAX = 256


def to_device_async(values, dtype, dev):
    """Small host list/array -> device without an implicit synchronisation:
    staged in pinned memory and copied by a kernel that reads it through the
    UVA mapping (dp2_copy_h2d_small), so the upload neither synchronises the
    stream (pageable copies do) nor waits behind bulk uploads queued on a copy
    engine.  The pinned source is kept alive until an event recorded after the
    copy has completed."""
    src = torch.as_tensor(np.asarray(values), dtype=dtype).pin_memory()
    out = torch.empty(tuple(src.shape), dtype=dtype, device=dev)
    nbytes = src.numel() * src.element_size()
    if nbytes:
        # launched (and ordered) on dev's current stream, under dev's context
        with torch.cuda.device(out.device):
            _lib.check(_lib.lib().dp2_copy_h2d_small(C.c_void_p(out.data_ptr()), C.c_void_p(src.data_ptr()),
                                                      nbytes, stream_ptr(out.device)), "copy_h2d_small")
            ev = torch.cuda.Event()
            ev.record(torch.cuda.current_stream(out.device))
        _SMALL_KEEP.append((src, ev))
        if len(_SMALL_KEEP) > _SMALL_KEEP_MAX:
            _SMALL_KEEP[:] = [(t, e) for t, e in _SMALL_KEEP if not e.query()]
    return out