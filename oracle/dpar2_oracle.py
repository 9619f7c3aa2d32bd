"""CPU oracle for the DPar2 hot path -- TEST INFRASTRUCTURE ONLY.

A plain-NumPy restatement of the reference algorithm (``dpar2`` package,
``/root/reference/pkg/src/dpar2``), written independently so it can run on the
GPU box where the reference is absent.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline / ``--impl
reference`` legs may import this module; the product package
(``paper_2203_12798_b200``) never does.

Pinning: ``oracle/make_golden.py`` runs the real reference in the build
container and checks this restatement against it (bit-exact on the
compressed factors and the fit for every golden case); the reference's outputs
are committed as fixtures under ``tests/golden/``.

Every function cites the reference lines it restates.  ``P/`` below is
``/root/reference/pkg/src/dpar2/``.
"""
from __future__ import annotations

import os
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

MASK64 = (1 << 64) - 1


class OracleError(Exception):
    """Raised where the reference raises one of its DecompositionError types."""


# --------------------------------------------------------------------------
# seeds, sketch matrices, partition
# --------------------------------------------------------------------------
def derived_seed(seed, index):
    """P/linalg.py:187-194 -- SeedSequence([seed, index]) -> first uint64."""
    words = np.random.SeedSequence([seed & MASK64, int(index)]).generate_state(1, np.uint64)
    return int(words[0])


def sketch_width(m, n, rank, oversampling=None):
    """P/linalg.py:116-120 -- s = rank + (oversampling or min(10, min(m,n)-rank))."""
    over = min(10, min(m, n) - rank) if oversampling is None else oversampling
    if over < 0:
        raise ValueError("oversampling must be >= 0")
    return rank + over


def omega(seed, n, s):
    """P/linalg.py:122-123 -- PCG64(seed) standard normals, C-order (n, s)."""
    return np.random.Generator(np.random.PCG64(seed & MASK64)).standard_normal((n, s))


def greedy_partition(row_counts, workers):
    """P/scheduler.py:29-51 -- LPT: visit by (-count, index), lightest set wins
    (lowest set index on ties).  Returns (sets, loads)."""
    counts = [int(c) for c in row_counts]
    if not counts or workers < 1 or min(counts) < 1:
        raise ValueError("bad partition input")
    sets = [[] for _ in range(workers)]
    loads = [0] * workers
    for k in sorted(range(len(counts)), key=lambda i: (-counts[i], i)):
        t = int(np.argmin(loads))  # argmin returns the first minimum
        sets[t].append(k)
        loads[t] += counts[k]
    return sets, loads


def _slice_map(fn, n, threads, groups=None):
    """P/scheduler.py:85-122 -- slot-per-slice map over worker-owned groups
    (contiguous chunks by default, P/scheduler.py:54-66); results in slice
    order."""
    if threads <= 1 or n <= 1:
        return [fn(k) for k in range(n)]
    if groups is None:
        parts = min(threads, n)
        base, extra = divmod(n, parts)
        bounds = np.cumsum([0] + [base + (1 if i < extra else 0) for i in range(parts)])
        groups = [range(int(a), int(b)) for a, b in zip(bounds[:-1], bounds[1:])]
    out = [None] * n

    def run(group):
        for k in group:
            out[k] = fn(k)

    with ThreadPoolExecutor(max_workers=min(threads, len(groups))) as pool:
        list(pool.map(run, groups))
    return out


# --------------------------------------------------------------------------
# dense kernels
# --------------------------------------------------------------------------
def fix_signs(u, v):
    """P/linalg.py:62-70 -- largest-|.| entry of each u column made >= 0
    (argmax ties -> first index); v columns flip with u."""
    pick = np.abs(u).argmax(axis=0)
    neg = u[pick, np.arange(u.shape[1])] < 0.0
    u[:, neg] = -u[:, neg]
    v[:, neg] = -v[:, neg]
    return u, v


def truncated_svd(a, rank):
    """P/linalg.py:73-94 -- gesdd, keep ``rank`` triplets, sign rule."""
    a = np.asarray(a, dtype=np.float64)
    if rank < 1 or rank > min(a.shape):
        raise OracleError(f"rank {rank} invalid for shape {a.shape}")
    u, s, vt = np.linalg.svd(a, full_matrices=False)
    u = np.ascontiguousarray(u[:, :rank])
    v = np.ascontiguousarray(vt[:rank].T)
    u, v = fix_signs(u, v)
    return u, np.ascontiguousarray(s[:rank]), v


def randomized_svd(a, rank, seed, oversampling=None, power_iters=1):
    """P/linalg.py:97-132 -- Y = (A A^T)^q A Omega, Householder QR, exact SVD
    of Q^T A, U = Q U~, sign rule again on U."""
    a = np.asarray(a, dtype=np.float64)
    if not np.isfinite(a).all():
        raise OracleError("non-finite input")
    m, n = a.shape
    if rank < 1 or rank > min(m, n):
        raise OracleError(f"rank {rank} invalid for shape {a.shape}")
    om = omega(seed, n, sketch_width(m, n, rank, oversampling))
    y = a @ om
    for _ in range(power_iters):
        y = a @ (a.T @ y)
    q, _ = np.linalg.qr(y)
    ub, s, v = truncated_svd(q.T @ a, rank)
    u, v = fix_signs(q @ ub, v)
    return u, s, v


def pinv_small(a):
    """P/linalg.py:135-151 -- SVD pseudoinverse, cutoff max(shape)*s0*1e-12."""
    a = np.asarray(a, dtype=np.float64)
    u, s, vt = np.linalg.svd(a, full_matrices=False)
    if s.size == 0 or s[0] == 0.0:
        return np.zeros((a.shape[1], a.shape[0]))
    inv = np.zeros_like(s)
    np.divide(1.0, s, out=inv, where=s > max(a.shape) * s[0] * 1e-12)
    return (vt.T * inv) @ u.T


def push_col_norms(a, b):
    """P/factors.py:93-99 -- unit-norm columns of a, norms into b (<1e-300 kept)."""
    n = np.linalg.norm(a, axis=0)
    n = np.where(n < 1e-300, 1.0, n)
    return a / n, b * n


def initial_factors(num_cols, num_slices, rank, seed=0):
    """P/factors.py:79-90 -- H = I, V = eye(J, R) (Gaussian if J < R), W = 1."""
    if num_cols >= rank:
        v = np.eye(num_cols, rank)
    else:
        v = np.random.Generator(np.random.PCG64(seed & MASK64)).standard_normal((num_cols, rank))
    return np.eye(rank), v, np.ones((num_slices, rank))


# --------------------------------------------------------------------------
# two-stage compression
# --------------------------------------------------------------------------
class Compressed:
    """Mirror of P/compress.py:34-72 (A_k list, D, E, F stacked KR x R)."""

    def __init__(self, rank, bases, d, e, f):
        self.rank, self.bases, self.D, self.E, self.F = rank, bases, d, e, f

    def block(self, k):
        return self.F[k * self.rank:(k + 1) * self.rank]

    @property
    def K(self):
        return len(self.bases)

    def float_count(self):
        return sum(a.size for a in self.bases) + self.F.size + self.D.size + self.E.size


def compress(slices, rank, seed=0, oversampling=None, power_iters=1,
             stage2_oversampling="same", threads=1, keep_stage1=False):
    """P/compress.py:75-119 -- rank checks, per-slice rSVD with
    derived_seed(seed, k), M = [V_k S_k] in slice order, stage-2 rSVD with
    derived_seed(seed, K)."""
    cols = slices[0].shape[1]
    if rank < 1 or rank > cols:
        raise OracleError(f"rank {rank} exceeds column count {cols}")
    for k, x in enumerate(slices):
        if rank > x.shape[0]:
            raise OracleError(f"rank {rank} exceeds row count {x.shape[0]} of slice {k}")

    def one(k):
        return randomized_svd(slices[k], rank, derived_seed(seed, k), oversampling, power_iters)

    # slices owned per worker by the Alg. 4 LPT plan (P/compress.py:93-94, 105)
    groups = greedy_partition([x.shape[0] for x in slices], threads)[0] if threads > 1 else None
    trips = _slice_map(one, len(slices), threads, groups=groups)
    merged = np.concatenate([v * s for (_, s, v) in trips], axis=1)
    over2 = oversampling if stage2_oversampling == "same" else stage2_oversampling
    d, e, f = randomized_svd(merged, rank, derived_seed(seed, len(slices)), over2, power_iters)
    comp = Compressed(rank, [t[0] for t in trips], d, e, np.ascontiguousarray(f))
    if keep_stage1:
        comp.stage1 = trips
        comp.M = merged
    return comp


# --------------------------------------------------------------------------
# compressed-space ALS (P/solver.py)
# --------------------------------------------------------------------------
def core_cols(comp, v):
    """P/solver.py:51 -- E * (D^T V)."""
    return comp.E[:, None] * (comp.D.T @ v)


def update_rotations(comp, h, v, w, threads=1):
    """P/solver.py:48-64 -- T_k = (F_k cc) * w_k @ H^T, SVD -> (Z_k, P_k)."""
    cc = core_cols(comp, v)
    ht = h.T

    def rot(k):
        t = ((comp.block(k) @ cc) * w[k]) @ ht
        z, sig, p = truncated_svd(t, comp.rank)
        return z, p, sig

    return _slice_map(rot, comp.K, threads)


def rotated_cores(comp, rots, threads=1):
    """P/solver.py:67-78 -- Theta_k = (P_k Z_k^T) F_k, stacked (K, R, R)."""
    return np.stack(_slice_map(lambda k: (rots[k][1] @ rots[k][0].T) @ comp.block(k), comp.K, threads))


def mttkrp_mode1(comp, rots, w, v, threads=1):
    """P/solver.py:81-89 (Lemma 1)."""
    th = rotated_cores(comp, rots, threads)
    cc = core_cols(comp, v)
    return np.einsum("rij,jr->ir", np.einsum("kr,kij->rij", w, th), cc)


def mttkrp_mode2(comp, rots, w, h, threads=1):
    """P/solver.py:92-100 (Lemma 2)."""
    th = rotated_cores(comp, rots, threads)
    summed = np.einsum("kr,kar->ar", w, np.einsum("kba,br->kar", th, h))
    return comp.D @ (comp.E[:, None] * summed)


def mttkrp_mode3(comp, rots, v, h, threads=1):
    """P/solver.py:103-111 (Lemma 3)."""
    th = rotated_cores(comp, rots, threads)
    cc = core_cols(comp, v)
    return np.einsum("ir,kir->kr", h, np.einsum("kij,jr->kir", th, cc))


def update_factors(comp, rots, h, v, w, normalize=True, threads=1):
    """P/solver.py:114-130 -- Gauss-Seidel H, V, W sweep with pinv solves."""
    h = mttkrp_mode1(comp, rots, w, v, threads) @ pinv_small((w.T @ w) * (v.T @ v))
    if normalize:
        h, w = push_col_norms(h, w)
    v = mttkrp_mode2(comp, rots, w, h, threads) @ pinv_small((w.T @ w) * (h.T @ h))
    if normalize:
        v, w = push_col_norms(v, w)
    w = mttkrp_mode3(comp, rots, v, h, threads) @ pinv_small((v.T @ v) * (h.T @ h))
    return h, v, w


def convergence_metric(comp, rots, h, v, w, threads=1):
    """P/solver.py:133-149 -- sum_k ||Theta_k E D^T - (H*w_k) V^T||^2,
    reduced in ascending slice order."""
    basis = comp.E[:, None] * comp.D.T
    vt = v.T

    def residual(k):
        z, p, _ = rots[k]
        buf = ((p @ z.T) @ comp.block(k)) @ basis
        buf -= (h * w[k]) @ vt
        return float(np.dot(buf.ravel(), buf.ravel()))

    return float(np.add.reduce(np.asarray(_slice_map(residual, comp.K, threads))))


def fit_dpar2(slices, rank, max_iters=32, tol=1e-6, seed=0, normalize=True,
              oversampling=None, threads=1, comp=None, timings=None, als_threads=1):
    """P/solver.py:152-190 -- compress once, iterate, stop on
    ``prev == 0 or |prev - e| <= tol * prev``; Q_k = A_k Z_k P_k^T from the
    last iteration.  ``oversampling`` replays the config-4 harness (the
    reference's fit_dpar2 pins it to the default).  ``threads`` are the
    compression's slice threads, ``als_threads`` the per-slice maps of the
    iterations (the reference uses one resolved count for both,
    P/solver.py:162-189; values never depend on either)."""
    if max_iters < 1:
        raise ValueError("max_iters must be >= 1")
    t0 = time.perf_counter()
    if comp is None:
        comp = compress(slices, rank, seed=seed, oversampling=oversampling, threads=threads)
    t1 = time.perf_counter()
    h, v, w = initial_factors(slices[0].shape[1], len(slices), rank, seed)
    trace, seconds, converged, prev, rots = [], [], False, None, None
    for _ in range(max_iters):
        tick = time.perf_counter()
        rots = update_rotations(comp, h, v, w, threads=als_threads)
        h, v, w = update_factors(comp, rots, h, v, w, normalize=normalize, threads=als_threads)
        e = convergence_metric(comp, rots, h, v, w, threads=als_threads)
        trace.append(e)
        seconds.append(time.perf_counter() - tick)
        if prev is not None and (prev == 0.0 or abs(prev - e) <= tol * prev):
            converged = True
            break
        prev = e
    q = _slice_map(lambda k: comp.bases[k] @ (rots[k][0] @ rots[k][1].T), comp.K, als_threads)
    if timings is not None:
        timings.update(preprocess=t1 - t0, iterations=sum(seconds), total=time.perf_counter() - t0)
    return dict(H=h, V=v, W=w, Q=q, objective=trace, seconds=seconds, converged=converged,
                compressed_float_count=comp.float_count(), comp=comp)


def fitness(slices, h, v, w, q):
    """P/analysis.py:23-45 -- 1 - sum ||X_k - Q_k (H*w_k) V^T||^2 / sum ||X_k||^2."""
    tot, res = [], []
    for k, x in enumerate(slices):
        d = x - (q[k] @ (h * w[k])) @ v.T
        tot.append(float(np.dot(x.ravel(), x.ravel())))
        res.append(float(np.dot(d.ravel(), d.ravel())))
    total = float(np.add.reduce(np.asarray(tot)))
    if total == 0.0:
        raise OracleError("fitness undefined for an all-zero tensor")
    return 1.0 - float(np.add.reduce(np.asarray(res))) / total


def cpu_threads():
    return os.cpu_count() or 1
