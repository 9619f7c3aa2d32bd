"""Sketch-matrix (Omega) generation.

Omega_k must be bit-identical to the reference's draw (P/linalg.py:122-123):
``Generator(PCG64(derived_seed(seed, k))).standard_normal((J, s_k))``.

``omega_device`` (the product path) runs the native generator
(csrc/dp2_rng.cu: SeedSequence -> PCG64 -> 256-layer ziggurat, one thread per
slice) and then replays the rare layer-0 tail draws on the host with NumPy's
log1p -- the only step whose last bit depends on the libm -- patching those
entries, so the result is byte-identical to NumPy.  ``omega_host`` draws the
same matrices with NumPy itself (used for stage 2's single stream, overlapped
with stage 1, and as the test reference).
"""
from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

from .linalg import derived_seed

_MASK64 = (1 << 64) - 1


def _fill(out, seeds, n, widths, lo, hi):
    for k in range(lo, hi):
        g = np.random.Generator(np.random.PCG64(seeds[k] & _MASK64))
        s = widths[k]
        if s == out.shape[2]:
            g.standard_normal(out=out[k])
        else:
            out[k, :, :s] = g.standard_normal((n, s))


def omega_host(seed, n, widths, sp, threads=None, slice_ids=None):
    """Pinned host tensor (K, n, sp) with slice k's Omega in [:, :widths[k]].
    ``slice_ids`` gives the global slice index of each local slice (multi-GPU
    shards keep the reference's per-slice seeds)."""
    K = len(widths)
    ids = range(K) if slice_ids is None else slice_ids
    seeds = [derived_seed(seed, k) for k in ids]
    host = torch.zeros((K, n, sp), dtype=torch.float64, pin_memory=torch.cuda.is_available())
    arr = host.numpy()
    threads = threads or min(32, os.cpu_count() or 1)
    step = max(1, (K + threads - 1) // threads)
    if threads <= 1 or K < 2:
        _fill(arr, seeds, n, widths, 0, K)
    else:
        with ThreadPoolExecutor(max_workers=threads) as pool:
            list(pool.map(lambda lo: _fill(arr, seeds, n, widths, lo, min(K, lo + step)), range(0, K, step)))
    return host


_REC = np.dtype([("slice", "<i8"), ("index", "<i8"), ("attempts", "<i4"), ("negative", "<i4"),
                 ("u", "<f8", (8,))])
_ZIG_R = 3.6541528853610087963519472518
_ZIG_INV_R = 0.27366123732975827203338247596


_REPLAY_POOL = None
_SCRATCH = {}


def _scratch(device, K, cap):
    """Device tail-record buffers and their pinned readback copies, reused
    across calls (two alternating sets per shape, so a speculative replay
    still reading one set is never overwritten)."""
    key = (str(device), K, cap)
    sets = _SCRATCH.get(key)
    if sets is None:
        def one():
            return {"recs": torch.empty((cap, _REC.itemsize), dtype=torch.uint8, device=device),
                    "nrec": torch.zeros(1, dtype=torch.int32, device=device),
                    "redo": torch.zeros(K, dtype=torch.int32, device=device),
                    "nrec_h": torch.empty(1, dtype=torch.int32, pin_memory=True),
                    "redo_h": torch.empty(K, dtype=torch.int32, pin_memory=True),
                    "recs_h": torch.empty((cap, _REC.itemsize), dtype=torch.uint8, pin_memory=True),
                    "busy": None}
        sets = _SCRATCH[key] = [one(), one(), 0]
    sets[2] ^= 1
    cur = sets[sets[2]]
    if cur["busy"] is not None:
        cur["busy"].result()  # its replay must be done reading the pinned copies
        cur["busy"] = None
    return cur


def _replay_check(ev, nrec_h, redo_h_t, recs_h, cap):
    """Background half of a speculative omega_device: wait for the records,
    replay them with libm's log1p and report whether any acceptance decision
    (or a record overflow / device redo flag) differs from the reference's."""
    import ctypes as C

    from . import _lib
    ev.synchronize()
    count = int(nrec_h[0])
    mismatch = count > cap or bool(redo_h_t.numpy().any())
    if count and not mismatch:
        r = recs_h[:count].numpy().view(_REC).reshape(-1)
        vals = np.empty(r.size)
        okv = np.empty(r.size, dtype=np.int32)
        _lib.check(_lib.lib().dp2_omega_replay(C.c_void_p(r.ctypes.data), r.size,
                                               vals.ctypes.data_as(C.POINTER(C.c_double)),
                                               okv.ctypes.data_as(C.POINTER(C.c_int32))), "omega_replay")
        mismatch = not bool(okv.all())
    return {"omega_tail_events": count, "omega_mismatch": mismatch}


def omega_device(seed, n, widths, sp, device, slice_ids=None, stats=None, speculative=False, s_dev=None):
    """Device tensor (K, n, sp) of the reference's Omega_k (byte-exact).

    ``speculative=True`` (for consumers that round Omega to tf32, the fp32
    tensor-core sketch): no host synchronisation -- the device's own tail
    values (its log1p may differ from libm's in the last bit, which tf32
    rounding absorbs) are used as they are, and the libm replay runs on a
    background thread; returns ``(omega, future)`` whose result reports
    ``omega_mismatch`` (an acceptance decision differing from the reference's,
    practically never: the caller then recomputes with the exact path)."""
    h = omega_device_launch(seed, n, widths, sp, device, slice_ids=slice_ids, s_dev=s_dev)
    if speculative:
        global _REPLAY_POOL
        if _REPLAY_POOL is None:
            from concurrent.futures import ThreadPoolExecutor
            _REPLAY_POOL = ThreadPoolExecutor(1)
        bufs = h["bufs"]
        fut = _REPLAY_POOL.submit(_replay_check, h["ev"], bufs["nrec_h"], bufs["redo_h"], bufs["recs_h"], h["cap"])
        bufs["busy"] = fut
        return h["out"], fut
    return omega_device_finish(h, stats=stats)


def omega_device_launch(seed, n, widths, sp, device, slice_ids=None, s_dev=None):
    """First half of the exact ``omega_device``: enqueue the generator and the
    readback of its tail records on the current stream, record an event, and
    return a handle for ``omega_device_finish`` -- the host is free (and the
    stream can take more work) until the records are needed."""
    import ctypes as C

    from . import _lib
    K = len(widths)
    out = torch.empty((K, n, sp), dtype=torch.float64, device=device)
    from .tensor import stream_ptr, to_device_async
    if s_dev is None:
        s_dev = to_device_async(list(widths), torch.int32, device)
    ids = None if slice_ids is None else to_device_async(list(slice_ids), torch.int64, device)
    cap = max(4096, 8 * K + n * int(np.max(widths)) * K // 1000)
    bufs = _scratch(device, K, cap)
    recs, nrec, redo = bufs["recs"], bufs["nrec"], bufs["redo"]  # zeroed by dp2_omega_generate
    vp = lambda t: C.c_void_p(t.data_ptr()) if t is not None else C.c_void_p(0)  # noqa: E731
    _lib.check(_lib.lib().dp2_omega_generate(C.c_uint64(seed & _MASK64), K, n, vp(s_dev), sp, vp(ids), vp(out),
                                             vp(recs), cap, vp(nrec), vp(redo),
                                             stream_ptr()), "omega")
    # one readback: record count, per-slice redo flags and the records
    bufs["nrec_h"].copy_(nrec, non_blocking=True)
    bufs["redo_h"].copy_(redo, non_blocking=True)
    bufs["recs_h"].copy_(recs, non_blocking=True)
    ev = torch.cuda.Event()
    ev.record()
    return dict(out=out, ev=ev, bufs=bufs, cap=cap, seed=seed, n=n, widths=widths, sp=sp, slice_ids=slice_ids,
                keep=(s_dev, ids))


def omega_device_finish(h, stats=None):
    """Second half of the exact ``omega_device``: wait for the tail records
    only (the handle's event, not the stream), replay each attempt with the C
    library's log1p -- the function the reference sampler calls (npy_log1p);
    NumPy's np.log1p ufunc may use a SIMD implementation with different
    rounding -- and scatter the exact values into Omega on the stream
    (dp2_omega_patch).  Slices whose acceptance decision differs, or a record
    overflow, are regenerated with NumPy (never expected)."""
    import ctypes as C

    from . import _lib
    from .tensor import stream_ptr
    out, bufs, cap, widths, n, sp = h["out"], h["bufs"], h["cap"], h["widths"], h["n"], h["sp"]
    K = len(widths)
    h["ev"].synchronize()
    nrec_h, redo_h_t, recs_h = bufs["nrec_h"], bufs["redo_h"], bufs["recs_h"]
    count = int(nrec_h[0])
    redo_h = redo_h_t.numpy().copy()
    if count > cap:
        redo_h[:] = 1  # record overflow: regenerate everything on the host (never expected)
    patched = 0
    if count and count <= cap:
        w32 = widths if isinstance(widths, np.ndarray) and widths.dtype == np.int32 else \
            np.ascontiguousarray(widths, dtype=np.int32)
        npatch = C.c_int32(0)
        _lib.check(_lib.lib().dp2_omega_patch(C.c_void_p(recs_h.data_ptr()), count, n,
                                              C.c_void_p(w32.ctypes.data), sp, C.c_void_p(out.data_ptr()),
                                              C.c_void_p(redo_h.ctypes.data), C.byref(npatch), stream_ptr()),
                   "omega_patch")
        patched = int(npatch.value)
    bad = np.nonzero(redo_h)[0]
    if bad.size:
        slice_ids = h["slice_ids"]
        ids_h = list(range(K)) if slice_ids is None else list(slice_ids)
        host = omega_host(h["seed"], n, [widths[k] for k in bad], sp, slice_ids=[ids_h[k] for k in bad])
        out[torch.from_numpy(bad).to(out.device)] = host.to(out.device)
    if stats is not None:
        stats.update(omega_tail_events=count, omega_patched=patched, omega_host_regenerated=int(bad.size))
    return out


def stage2_omega(seed, rows, width):
    """Omega_2 (rows x width), one stream seeded ``seed`` (P/compress.py:109-111)."""
    g = np.random.Generator(np.random.PCG64(seed & _MASK64))
    return g.standard_normal((rows, width))


def stage2_omega_launch(seed, rows, width, device):
    """Enqueue Omega_2 on the device (``dp2_omega_generate_stream``: the one
    stream split into segments parsed in parallel, stitched exactly) and the
    readback of its tail records; ``stage2_omega_finish`` completes it.
    Launched ahead of stage 1, it leaves the host free while stage 1 runs."""
    return _stage2_omega_enqueue(seed, rows, width, device, torch.cuda.current_stream(device))


_WIDTH_DEV = {}


def _stage2_omega_enqueue(seed, rows, width, device, main):
    import ctypes as C

    from . import _lib
    from .tensor import stream_ptr, to_device_async
    out = torch.empty((rows, width), dtype=torch.float64, device=device)
    key = (str(device), int(width))
    w_dev = _WIDTH_DEV.get(key)
    if w_dev is None:  # the width as a device int32, uploaded once per (device, width)
        w_dev = _WIDTH_DEV[key] = to_device_async(np.array([width], np.int32), torch.int32, device)
    cap = max(4096, rows * width // 1000)
    bufs = _scratch(device, 1, cap)
    vp = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
    _lib.check(_lib.lib().dp2_omega_generate_stream(C.c_uint64(seed & _MASK64), rows, width, vp(w_dev), vp(out),
                                                    vp(bufs["recs"]), cap, vp(bufs["nrec"]), vp(bufs["redo"]),
                                                    stream_ptr()),
               "omega_stream")
    bufs["nrec_h"].copy_(bufs["nrec"], non_blocking=True)
    bufs["redo_h"].copy_(bufs["redo"], non_blocking=True)
    bufs["recs_h"].copy_(bufs["recs"], non_blocking=True)
    ev = torch.cuda.Event()
    ev.record()
    return dict(out=out, ev=ev, bufs=bufs, cap=cap, seed=seed, rows=rows, width=width, keep=w_dev, main=main)


def stage2_omega_finish(h, stats=None):
    """Wait for Omega_2's records only (its event, not the stream), replay
    the tail draws with libm log1p (dp2_omega_replay) and patch the device
    matrix in place (stream-ordered): byte-exact with ``stage2_omega``.  A
    record overflow or a differing acceptance decision regenerates it with
    NumPy (never expected)."""
    import ctypes as C

    from . import _lib
    from .tensor import to_device_async
    h["ev"].synchronize()
    bufs, out, cap = h["bufs"], h["out"], h["cap"]
    count = int(bufs["nrec_h"].numpy()[0])
    redo = count > cap or bool(bufs["redo_h"].numpy()[0])
    if count and not redo:
        r = bufs["recs_h"][:count].numpy().view(_REC).reshape(-1)
        vals = np.empty(r.size)
        okv = np.empty(r.size, dtype=np.int32)
        _lib.check(_lib.lib().dp2_omega_replay(C.c_void_p(r.ctypes.data), r.size,
                                               vals.ctypes.data_as(C.POINTER(C.c_double)),
                                               okv.ctypes.data_as(C.POINTER(C.c_int32))), "omega_replay")
        if okv.all():
            idx = to_device_async(np.ascontiguousarray(r["index"]), torch.int64, out.device)
            out.view(-1).index_copy_(0, idx, to_device_async(vals, torch.float64, out.device))
        else:
            redo = True
    if redo:
        out.copy_(torch.from_numpy(stage2_omega(h["seed"], h["rows"], h["width"])))
    if stats is not None:
        stats.update(omega2_tail_events=count, omega2_host_regenerated=int(redo))
    return out
