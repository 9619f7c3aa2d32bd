"""Parity at the benchmarked scale: every BASELINE.json config (or the K-subset
named below) through the CUDA path against the CPU oracle on the SAME input.

* c2 in full (K=1000, J=512, I_k ~ U{500..4000}, 1.18e9 entries) in fp64 (the
  configuration ``bench.py`` measures), in the fp32 mode (fp32 storage; fp64
  DMMA sketch products on the upcast values by default, fp32 FFMA products
  via ``set_fp32_products("fp32")``) and in the opt-in tf32 mode (single-pass
  tf32 products on
  the tcgen05 tensor cores, ``set_fp32_products("tf32")``, bench.py's
  labelled sub-record);
* c3: a 240-slice K-subset of the heavy-tailed tensor (lognormal I_k, random
  slice order) that contains its largest slices (>= 20 000 rows), fp32;
* c4: the c2 tensor at R = 20 and R = 50 with oversampling p = R through the
  replay harness of BASELINE.md section 3 (``compress(rsvd=RsvdParams(R,
  oversampling=R))`` then the loop of P/solver.py:170-190): s = 2R = 40 / 100
  takes the stage-1 sp > 32 branch, stage 2 runs at s2 = 2R and the ALS at
  R > 16;
* c5-shaped: K=96 slices with J=1000, I_k ~ U{1000..7000}, noise 0.05, fp32.

Tolerances are BASELINE.json's north star: fp64 -- fitness within 1e-6
absolute, H/V/W and U_k = Q_k H within 1e-5 relative (max-abs error over
max-abs value after per-column sign alignment); fp32 mode -- 1e-3 for both.
The oracle runs on the fp32 values upcast exactly.
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

FP64 = dict(fit=1e-6, factor=1e-5)
FP32 = dict(fit=1e-3, factor=1e-3)


def rel_signed(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    s = np.sign(np.sum(a * b, axis=0))
    s[s == 0] = 1.0
    return float(np.abs(a * s - b).max() / max(np.abs(b).max(), 1e-300))


def _threads():
    return os.cpu_count() or 1


def _oracle_fit(xs, R, iters, oversampling=None):
    from threadpoolctl import threadpool_limits

    from oracle import dpar2_oracle as orc
    x64 = [np.asarray(x, dtype=np.float64) for x in xs]
    with threadpool_limits(limits=1):  # slice threads, single-threaded BLAS (BASELINE.md setting A)
        comp = orc.compress(x64, R, seed=0, oversampling=oversampling, threads=_threads())
    o = orc.fit_dpar2(x64, R, iters, 0.0, 0, comp=comp)
    o["fitness"] = orc.fitness(x64, o["H"], o["V"], o["W"], o["Q"])
    return o


def _device_fit(xs, R, iters, dtype, oversampling=None):
    import paper_2203_12798_b200 as dp
    t = dp.IrregularTensor(xs, dtype=dtype)
    opts = dp.SolverOptions(max_iters=iters, tol=0.0, seed=0)
    if oversampling is None:
        f, tr = dp.fit_dpar2(t, R, opts)
    else:  # replay harness: compress with p = R, then the fit loop on it
        comp = dp.compress(t, R, rsvd=dp.RsvdParams(rank=R, oversampling=oversampling, seed=0))
        f, tr = dp.fit_compressed(comp, opts)
    fit = dp.fitness(t, f, zero_pass=False)
    return f, tr, fit


def _compare(xs, R, iters, dtype, tol, oversampling=None):
    f, tr, fit = _device_fit(xs, R, iters, dtype, oversampling)
    o = _oracle_fit(xs, R, iters, oversampling)
    assert tr.iterations == len(o["objective"]) == iters
    assert abs(fit - o["fitness"]) <= tol["fit"], (fit, o["fitness"])
    errs = {k: rel_signed(getattr(f, k), o[k]) for k in ("H", "V", "W")}
    U = np.concatenate([np.asarray(q) @ f.H for q in f.Q])
    Uo = np.concatenate([q @ o["H"] for q in o["Q"]])
    errs["U"] = rel_signed(U, Uo)
    errs["objective"] = float(np.max(np.abs(np.asarray(tr.objective) - o["objective"]) / np.asarray(o["objective"])))
    bad = {k: v for k, v in errs.items() if k != "objective" and v > tol["factor"]}
    assert not bad, (bad, errs, fit, o["fitness"])
    return errs, fit, o["fitness"]


@pytest.fixture(scope="module")
def c2_host():
    from paper_2203_12798_b200 import synth
    return synth.generate(synth.CONFIGS["c2"], 0, threads=_threads())


def test_c2_full_fp64(c2_host):
    errs, fit, fit_o = _compare(c2_host, 10, 32, "f64", FP64)
    print(f"c2 fp64: fitness {fit:.10f} oracle {fit_o:.10f}; errors {errs}")


def test_c2_full_fp32_mode(c2_host):
    xs = [x.astype(np.float32) for x in c2_host]
    errs, fit, fit_o = _compare(xs, 10, 32, "f32", FP32)
    print(f"c2 fp32: fitness {fit:.10f} oracle {fit_o:.10f}; errors {errs}")


def test_c2_full_fp32_ffma_products(c2_host):
    import paper_2203_12798_b200 as dp
    xs = [x.astype(np.float32) for x in c2_host]
    prev = dp.set_fp32_products("fp32")
    try:
        errs, fit, fit_o = _compare(xs, 10, 32, "f32", FP32)
    finally:
        dp.set_fp32_products(prev)
    print(f"c2 fp32 (FFMA products): fitness {fit:.10f} oracle {fit_o:.10f}; errors {errs}")


def test_c2_full_tf32_mode(c2_host):
    import paper_2203_12798_b200 as dp
    xs = [x.astype(np.float32) for x in c2_host]
    prev = dp.set_fp32_products("tf32")
    try:
        errs, fit, fit_o = _compare(xs, 10, 32, "f32", FP32)
    finally:
        dp.set_fp32_products(prev)
    print(f"c2 tf32: fitness {fit:.10f} oracle {fit_o:.10f}; errors {errs}")


@pytest.mark.parametrize("R", [20, 30, 40, 50])
def test_c4_rank_sweep_oversampling_equals_rank(c2_host, R):
    errs, fit, fit_o = _compare(c2_host, R, 32, "f64", FP64, oversampling=R)
    print(f"c4 R={R}: fitness {fit:.10f} oracle {fit_o:.10f}; errors {errs}")


def test_c3_heavy_tailed_subset_fp32():
    from paper_2203_12798_b200 import synth
    cfg = synth.CONFIGS["c3"]
    rows, _ = synth.row_counts(cfg, 0)
    rows = np.asarray(rows)
    rng = np.random.default_rng(3)
    big = np.argsort(-rows, kind="stable")[:6]
    rest = rng.choice(np.setdiff1d(np.arange(cfg.num_slices), big), size=234, replace=False)
    idx = rng.permutation(np.concatenate([big, rest]))  # random order, not by size
    assert rows[idx].max() >= 20000 and rows[idx].min() <= 200
    xs = synth.generate(cfg, 0, slices=idx, threads=_threads())
    errs, fit, fit_o = _compare(xs, 10, 32, "f32", FP32)
    print(f"c3 subset ({len(idx)} slices, max I_k {rows[idx].max()}): fitness {fit:.8f} oracle {fit_o:.8f}; {errs}")


def test_c5_shaped_subset_fp32():
    from paper_2203_12798_b200 import synth
    cfg = synth.scaled(synth.CONFIGS["c5"], num_slices=96)
    xs = synth.generate(cfg, 0, threads=_threads())
    errs, fit, fit_o = _compare(xs, 10, 32, "f32", FP32)
    print(f"c5 subset (K=96, J=1000): fitness {fit:.8f} oracle {fit_o:.8f}; {errs}")


def test_c5_shaped_subset_tf32_mode():
    """J = 1000 in the opt-in tf32 mode: the tcgen05 pass on a CTA pair (J split)."""
    import paper_2203_12798_b200 as dp
    from paper_2203_12798_b200 import synth
    cfg = synth.scaled(synth.CONFIGS["c5"], num_slices=96)
    xs = synth.generate(cfg, 0, threads=_threads())
    prev = dp.set_fp32_products("tf32")
    try:
        errs, fit, fit_o = _compare(xs, 10, 32, "f32", FP32)
    finally:
        dp.set_fp32_products(prev)
    print(f"c5 subset tf32 (K=96, J=1000): fitness {fit:.8f} oracle {fit_o:.8f}; {errs}")


def test_c5_shaped_subset_fp64():
    """The J = 1000 shape through the fp64 path (DMMA pass at J > 512)."""
    from paper_2203_12798_b200 import synth
    cfg = synth.scaled(synth.CONFIGS["c5"], num_slices=48, dtype="f64")
    xs = synth.generate(cfg, 0, threads=_threads())
    errs, fit, fit_o = _compare(xs, 10, 32, "f64", FP64)
    print(f"c5 subset fp64 (K=48, J=1000): fitness {fit:.10f} oracle {fit_o:.10f}; {errs}")
