"""IRT1 / IRC1 archives straight to and from the device store.

Formats (restated from the reference; all payloads little-endian float64,
row-major):

* IRT1 (irregular tensor, ``P/tensor.py:172-212``):
  ``b"IRT1" | u32 K | u32 J | K x ( u32 I_k | X_k )``
* IRC1 (compressed tensor, ``P/compress.py:13-18,130-179``):
  ``b"IRC1" | u32 K | u32 J | u32 R | D (J x R) | E (R) | F (KR x R) |
  K x ( u32 I_k | A_k (I_k x R) )``

The host-side parsers (``read_irt1`` / ``read_irc1``) validate exactly what the
reference's loaders validate, with the same ``ArchiveFormatError`` messages, and
never copy payloads: ``read_irt1`` returns zero-copy views into a read-only
memory map, which ``load_archive`` hands to ``IrregularTensor`` -- the chunked
copy-stream upload with the finiteness scan on host threads (tensor.py), so a
large archive streams from the page cache to HBM without an intermediate
packed host copy.  The writers produce byte-identical files to the
reference's ``save_archive`` / ``save_compressed`` for the same arrays.

``fit_compressed`` runs the compressed-space ALS on a loaded IRC1 archive
(compress once, fit many times), the same device loop as ``fit_dpar2``.
"""
from __future__ import annotations

import mmap
import os
import struct
from pathlib import Path

import numpy as np

from .errors import ArchiveFormatError, NonFiniteInputError

IRT1 = b"IRT1"
IRC1 = b"IRC1"
_F8 = np.dtype("<f8")


def _map(path):
    """Read-only memory map of ``path`` (an empty file maps to b"")."""
    with open(path, "rb") as fh:
        size = os.fstat(fh.fileno()).st_size
        if size == 0:
            return b""
        return mmap.mmap(fh.fileno(), 0, access=mmap.ACCESS_READ)


# ------------------------------------------------------------------ IRT1
def read_irt1(path):
    """Parse an IRT1 archive (checks and messages of P/tensor.py:182-206).

    Returns ``(slices, buf)``: per-slice float64 views into the memory map
    ``buf`` (keep it alive as long as the views are used)."""
    data = _map(path)
    n = len(data)
    if n < 4 or data[:4] != IRT1:
        raise ArchiveFormatError(f"{path}: bad magic, not an IRT1 archive")
    off = 4
    if n < off + 8:
        raise ArchiveFormatError(f"{path}: truncated header")
    num_slices, cols = struct.unpack_from("<II", data, off)
    off += 8
    if num_slices < 1 or cols < 1:
        raise ArchiveFormatError(f"{path}: invalid dimensions K={num_slices}, J={cols}")
    slices = []
    for k in range(num_slices):
        if n < off + 4:
            raise ArchiveFormatError(f"{path}: truncated at slice {k} header")
        (rows,) = struct.unpack_from("<I", data, off)
        off += 4
        if rows < 1:
            raise ArchiveFormatError(f"{path}: slice {k} has zero rows")
        nbytes = rows * cols * 8
        if n < off + nbytes:
            raise ArchiveFormatError(f"{path}: truncated payload in slice {k}")
        slices.append(np.frombuffer(data, dtype=_F8, count=rows * cols, offset=off).reshape(rows, cols))
        off += nbytes
    if off != n:
        raise ArchiveFormatError(f"{path}: {n - off} trailing bytes after last slice")
    return slices, data


def write_irt1(slices, path):
    """IRT1 from host arrays (P/tensor.py:172-179 layout)."""
    cols = int(np.shape(slices[0])[1])
    with open(path, "wb") as fh:
        fh.write(IRT1)
        fh.write(struct.pack("<II", len(slices), cols))
        for x in slices:
            fh.write(struct.pack("<I", int(np.shape(x)[0])))
            fh.write(np.ascontiguousarray(x, dtype=_F8).tobytes())


def load_archive(path, dtype="f64"):
    """``IrregularTensor`` from an IRT1 archive (P/tensor.py:182-212): the
    slices stream from the memory map to the device store; a non-finite value
    raises ``ArchiveFormatError`` naming the archive and the slice."""
    import warnings

    from .tensor import IrregularTensor
    slices, buf = read_irt1(path)
    try:
        with warnings.catch_warnings():  # read-only mapped views are only read
            warnings.filterwarnings("ignore", message="The given NumPy array is not writable")
            t = IrregularTensor(slices, dtype=dtype)
    except NonFiniteInputError as exc:
        raise ArchiveFormatError(f"{path}: {exc}") from exc
    t._archive_map = buf  # the upload may still read the mapped pages
    return t


def save_archive(tensor, path, chunk_rows=1 << 16):
    """Write ``tensor`` (device store, fp64 or fp32 values -- fp32 widens
    exactly) as IRT1; round-trips bit-exactly through ``load_archive``."""
    import torch
    J, K = tensor.num_cols, tensor.num_slices
    off = tensor.row_off_host
    with open(path, "wb") as fh:
        fh.write(IRT1)
        fh.write(struct.pack("<II", K, J))
        for k in range(K):
            r0, r1 = int(off[k]), int(off[k + 1])
            fh.write(struct.pack("<I", r1 - r0))
            for a in range(r0, r1, chunk_rows):
                b = min(r1, a + chunk_rows)
                blk = tensor.X[a:b, :J].to(torch.float64).cpu().numpy()
                fh.write(np.ascontiguousarray(blk, dtype=_F8).tobytes())


# ------------------------------------------------------------------ IRC1
def read_irc1(path):
    """Parse an IRC1 archive (checks and messages of P/compress.py:147-179).
    Returns ``(rank, D, E, F, bases)`` as float64 views into the memory map."""
    data = _map(path)
    n = len(data)
    if n < 4 or data[:4] != IRC1:
        raise ArchiveFormatError(f"{path}: bad magic, not an IRC1 archive")
    off = 4
    if n < off + 12:
        raise ArchiveFormatError(f"{path}: truncated header")
    num_slices, cols, rank = struct.unpack_from("<III", data, off)
    off += 12
    if num_slices < 1 or cols < 1 or rank < 1:
        raise ArchiveFormatError(f"{path}: invalid dimensions")

    def take(count, shape):
        nonlocal off
        nbytes = count * 8
        if n < off + nbytes:
            raise ArchiveFormatError(f"{path}: truncated payload")
        arr = np.frombuffer(data, dtype=_F8, count=count, offset=off).reshape(shape)
        off += nbytes
        return arr

    D = take(cols * rank, (cols, rank))
    E = take(rank, (rank,))
    F = take(num_slices * rank * rank, (num_slices * rank, rank))
    bases = []
    for k in range(num_slices):
        if n < off + 4:
            raise ArchiveFormatError(f"{path}: truncated at slice {k}")
        (rows,) = struct.unpack_from("<I", data, off)
        off += 4
        bases.append(take(rows * rank, (rows, rank)))
    if off != n:
        raise ArchiveFormatError(f"{path}: trailing bytes")
    return rank, D, E, F, bases


def write_irc1(rank, D, E, F, bases, path):
    """IRC1 from host arrays (P/compress.py:133-142 layout)."""
    with open(path, "wb") as fh:
        fh.write(IRC1)
        fh.write(struct.pack("<III", len(bases), int(np.shape(D)[0]), int(rank)))
        for arr in (D, E, F):
            fh.write(np.ascontiguousarray(arr, dtype=_F8).tobytes())
        for a in bases:
            fh.write(struct.pack("<I", int(np.shape(a)[0])))
            fh.write(np.ascontiguousarray(a, dtype=_F8).tobytes())


def save_compressed(comp, path):
    """Write a device ``CompressedTensor`` as IRC1 (A with its column signs
    applied when the compression deferred them)."""
    import torch
    A = comp.A
    if comp.a_signs is not None:
        rows = torch.as_tensor(np.diff(comp.row_off), device=A.device)
        A = A * comp.a_signs.repeat_interleave(rows, dim=0)
    A_h = A.cpu().numpy()
    off = comp.row_off
    bases = [A_h[int(off[k]):int(off[k + 1])] for k in range(comp.num_slices)]
    write_irc1(comp.rank, comp.col_basis.cpu().numpy(), comp.weights.cpu().numpy(), comp.cores.cpu().numpy(),
               bases, path)


def load_compressed(path):
    """Device ``CompressedTensor`` from an IRC1 archive (P/compress.py:145-179)."""
    import torch

    from .compress import CompressedTensor
    from .tensor import device
    rank, D, E, F, bases = read_irc1(path)
    dev = device()
    rows = np.array([b.shape[0] for b in bases], np.int64)
    row_off = np.zeros(len(bases) + 1, np.int64)
    np.cumsum(rows, out=row_off[1:])
    A = torch.empty((int(row_off[-1]), rank), dtype=torch.float64)
    for k, b in enumerate(bases):
        A[int(row_off[k]):int(row_off[k + 1])] = torch.from_numpy(np.array(b))
    t = lambda a: torch.from_numpy(np.array(a)).to(dev)  # noqa: E731
    return CompressedTensor(rank=rank, A=A.to(dev), row_off=row_off, col_basis=t(D), weights=t(E), cores=t(F))


def fit_compressed(comp, opts=None, output="numpy"):
    """The compressed-space ALS of ``fit_dpar2`` (P/solver.py:167-190) on an
    already compressed tensor (e.g. ``load_compressed``): returns
    ``(factors, trace)`` with Q_k = A_k Z_k P_k^T."""
    import time

    import torch

    from .factors import FitTrace, Parafac2Factors, SliceViews, SolverOptions, initial_factors
    from .solver import _als_collect, _als_launch, assemble_q
    from .tensor import IrregularTensor
    opts = opts or SolverOptions()
    if opts.max_iters < 1:
        raise ValueError("max_iters must be >= 1")
    normalize = bool(opts.normalize) if opts.normalize is not None else True
    K, J, R = comp.num_slices, comp.num_cols, comp.rank
    started = time.perf_counter()
    h, v, w = initial_factors(J, K, R, opts.seed)
    launched = _als_launch(comp, h, v, w, opts.max_iters, opts.tol, normalize)
    # the piece plan of the slices' rows (assemble_q walks A by pieces)
    rows_view = IrregularTensor.plan_only(np.diff(comp.row_off), comp.A.device)
    Q = assemble_q(rows_view, comp, launched[3])
    H, V, W, polar, tr, secs = _als_collect(launched)
    trace = FitTrace(preprocess_seconds=time.perf_counter() - started, compressed_float_count=comp.float_count())
    trace.objective = tr
    trace.seconds = secs
    if len(tr) >= 2:
        prev, e = tr[-2], tr[-1]
        trace.converged = bool(prev == 0.0 or abs(prev - e) <= opts.tol * prev)
    factors = Parafac2Factors(H=H, V=V, W=W, Q=SliceViews(Q, comp.row_off), Q_packed=Q)
    if output == "numpy":
        factors = factors.numpy()
    torch.cuda.current_stream().synchronize()
    return factors, trace
