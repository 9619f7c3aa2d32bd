"""Irregular dense tensor held in a packed HBM store (P/tensor.py:34-80).

All K slices (I_k x J) live in ONE device buffer of shape (sum I_k, ldx):
slice k is rows [row_off[k], row_off[k+1]).  ``ldx`` pads rows to 16 bytes
(padding columns are zero) so every row is a whole number of 16-byte
``cp.async`` chunks.  Construction mirrors the reference's validation order and
messages (2-D, non-empty, consistent J, finite) -- the finiteness scan and the
per-slice squared norms run on the device in one pass.

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


def stream_ptr():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


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
        self._finish_layout()
        if check:
            self._stats()
        return self

    def _finish_layout(self):
        dev = self.X.device
        off = np.zeros(len(self._rows) + 1, np.int64)
        np.cumsum(self._rows, out=off[1:])
        self.row_off_host = off
        self.row_off = torch.from_numpy(off).to(dev)
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

    def _stats(self):
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
            arrays = dict(piece_slice=torch.from_numpy(ps[:n].copy()).to(dev),
                          piece_row0=torch.from_numpy(pr0[:n].copy()).to(dev),
                          piece_rows=torch.from_numpy(prs[:n].copy()).to(dev),
                          seg_begin=torch.from_numpy(sb).to(dev), slice_piece=torch.from_numpy(sl).to(dev))
            self._plans[nseg] = (n, arrays, dict(piece_slice=ps[:n].copy(), slice_piece=sl.copy()))
        n, arrays, _ = self._plans[nseg]
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
            x = self.X[:, :self._J].double().cpu().numpy()
            self._host = [x[a:b] for a, b in zip(self.row_off_host[:-1], self.row_off_host[1:])]
        return [np.asarray(a, dtype=np.float64) for a in self._host]

    def total_sq_norm(self):
        return float(self._sqnorm.sum().item()) if self._sqnorm is not None else float(
            (self.X.double() ** 2).sum().item())

    def slice_sq_norms(self):
        return self._sqnorm


def new_status(dev):
    # device-side fills: no host copy, so no implicit stream synchronisation
    st = torch.zeros(_lib.STATUS_WORDS, dtype=torch.int64, device=dev)
    st[0:1].fill_(_lib.INT64_MAX)
    st[2:4].fill_(_lib.INT64_MAX)
    return st


def to_device_async(values, dtype, dev):
    """Small host list/array -> device without an implicit synchronisation
    (pageable host copies wait for the stream; pinned ones are async)."""
    return torch.as_tensor(np.asarray(values), dtype=dtype).pin_memory().to(dev, non_blocking=True)
