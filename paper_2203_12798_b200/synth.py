"""Seeded synthetic PARAFAC2 tensors with the BASELINE.json generative model.

    H ~ N(0,1) (R x R),  V ~ N(0,1) (J x R)
    Q_k = qr(N(0,1) I_k x R),  S_k = diag(U(0.5, 1.5)^R)
    X_k = Q_k H S_k V^T + eta * ||signal_k||_F / sqrt(I_k J) * N(0,1)

Per-slice randomness comes from ``SeedSequence([seed, 1, k])`` so any subset
of slices (a multi-GPU shard, a bounded CPU-baseline sample) regenerates
bit-identically on its own; row counts, H and V come from
``SeedSequence([seed, 0])``.  This replaces the reference's own generator
(P/tensor.py:128-169), whose model differs from the benchmark's.
"""
from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class SynthConfig:
    name: str
    num_slices: int
    cols: int
    rows: tuple          # ("uniform", lo, hi) or ("lognormal", mu, sigma, lo, hi)
    rank: int = 10
    noise: float = 0.1
    dtype: str = "f64"


CONFIGS = {
    "c1": SynthConfig("c1", 100, 100, ("uniform", 200, 1000)),
    "c2": SynthConfig("c2", 1000, 512, ("uniform", 500, 4000)),
    "c2f32": SynthConfig("c2f32", 1000, 512, ("uniform", 500, 4000), dtype="f32"),
    "c3": SynthConfig("c3", 10000, 256, ("lognormal", 7.0, 1.0, 50, 60000), dtype="f32"),
    "c4": SynthConfig("c4", 1000, 512, ("uniform", 500, 4000)),
    "c5": SynthConfig("c5", 20000, 1000, ("uniform", 1000, 7000), noise=0.05, dtype="f32"),
}


def _shared_stream(seed):
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, 0])))


def row_counts(cfg: SynthConfig, seed=0):
    rng = _shared_stream(seed)
    kind = cfg.rows[0]
    if kind == "uniform":
        rows = rng.integers(cfg.rows[1], cfg.rows[2] + 1, size=cfg.num_slices)
    elif kind == "lognormal":
        _, mu, sigma, lo, hi = cfg.rows
        rows = np.clip(np.round(rng.lognormal(mu, sigma, size=cfg.num_slices)), lo, hi)
    else:
        raise ValueError(f"unknown row law {kind!r}")
    return [int(r) for r in rows], rng


def shared_factors(cfg: SynthConfig, seed=0):
    rows, rng = row_counts(cfg, seed)
    h = rng.standard_normal((cfg.rank, cfg.rank))
    v = rng.standard_normal((cfg.cols, cfg.rank))
    return rows, h, v


def make_slice(cfg: SynthConfig, seed, k, rows_k, h, v):
    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, 1, k])))
    q, _ = np.linalg.qr(rng.standard_normal((rows_k, cfg.rank)))
    s = rng.uniform(0.5, 1.5, cfg.rank)
    signal = (q @ (h * s)) @ v.T
    noise = rng.standard_normal(signal.shape)
    x = signal + (cfg.noise * np.linalg.norm(signal) / np.sqrt(signal.size)) * noise
    return x.astype(np.float32 if cfg.dtype == "f32" else np.float64)


def generate(cfg: SynthConfig, seed=0, slices=None, threads=None):
    """Host slices (list of C-contiguous arrays) for ``cfg``; ``slices``
    restricts generation to a subset of slice indices (in the given order)."""
    rows, h, v = shared_factors(cfg, seed)
    idx = range(cfg.num_slices) if slices is None else list(slices)
    fn = lambda k: make_slice(cfg, seed, k, rows[k], h, v)  # noqa: E731
    threads = threads or 1
    if threads <= 1:
        return [fn(k) for k in idx]
    with ThreadPoolExecutor(max_workers=threads) as pool:
        return list(pool.map(fn, idx))


def scaled(cfg: SynthConfig, **kw):
    """A copy of ``cfg`` with fields replaced (e.g. fewer slices for tests)."""
    d = cfg.__dict__.copy()
    d.update(kw)
    return SynthConfig(**d)


def generate_device(cfg: SynthConfig, seed=0, device="cuda", slices=None):
    """Same generative model drawn with torch's CUDA generator (for the large
    benchmark configs, where host generation would dominate the run).
    Returns (packed X (sum I_k x J) on ``device``, row counts, H, V).  Row
    counts, H and V are the host draws above, so slice shapes match
    ``generate``; the per-slice Gaussians differ (different RNG)."""
    import torch

    rows, h, v = shared_factors(cfg, seed)
    idx = list(range(cfg.num_slices)) if slices is None else list(slices)
    rows = [rows[k] for k in idx]
    tdt = torch.float32 if cfg.dtype == "f32" else torch.float64
    g = torch.Generator(device=device)
    g.manual_seed(int(np.random.SeedSequence([seed, 2]).generate_state(1, np.uint64)[0]) & ((1 << 63) - 1))
    H = torch.from_numpy(h).to(device)
    V = torch.from_numpy(v).to(device)
    X = torch.empty((int(sum(rows)), cfg.cols), dtype=tdt, device=device)
    r0 = 0
    for n in rows:
        q, _ = torch.linalg.qr(torch.randn((n, cfg.rank), generator=g, device=device, dtype=torch.float64))
        s = torch.rand(cfg.rank, generator=g, device=device, dtype=torch.float64) + 0.5
        signal = (q @ (H * s)) @ V.T
        noise = torch.randn(signal.shape, generator=g, device=device, dtype=torch.float64)
        scale = cfg.noise * torch.linalg.norm(signal) / float(np.sqrt(signal.numel()))
        X[r0:r0 + n] = (signal + scale * noise).to(tdt)
        r0 += n
    return X, rows, h, v
