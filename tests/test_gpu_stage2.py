"""Stage 2 (P/compress.py:108-111: the randomized SVD of M = [V_k S_k]) on the
library's own DMMA kernels, against the oracle's compress on the same input:
D (J x R) and F (KR x R) sign-aligned within 1e-7, E within 1e-9 relative
(the c1 golden bounds), and D^T D = I.  Shapes: c2 (J=512, KR=10^4, s2=20),
c4-like p = R = 50 (s2 = 100 -> five 24-column groups), the c5 width J=1000,
and a noiseless planted rank-R tensor with s2 > R (the orthonormalisation of
a rank-deficient Y2)."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def rel_signed(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    s = np.sign(np.sum(a * b, axis=0))
    s[s == 0] = 1.0
    return float(np.abs(a * s - b).max() / max(np.abs(b).max(), 1e-300))


def _check(xs, R, oversampling=None, tol_d=1e-7, tol_e=1e-9):
    from threadpoolctl import threadpool_limits

    import paper_2203_12798_b200 as dp
    from oracle import dpar2_oracle as orc
    t = dp.IrregularTensor(xs)
    rsvd = dp.RsvdParams(rank=R, oversampling=oversampling, seed=0)
    comp = dp.compress(t, R, rsvd=rsvd)
    with threadpool_limits(limits=1):
        o = orc.compress([np.asarray(x, np.float64) for x in xs], R, seed=0, oversampling=oversampling,
                         threads=os.cpu_count() or 1)
    D, E, F = comp.col_basis.cpu().numpy(), comp.weights.cpu().numpy(), comp.cores.cpu().numpy()
    assert np.abs(D.T @ D - np.eye(R)).max() <= 1e-10
    assert float(np.abs(E - o.E).max() / o.E.max()) <= tol_e
    assert rel_signed(D, o.D) <= tol_d, rel_signed(D, o.D)
    # F's columns flip with D's (the sign rule is applied to D)
    sg = np.sign(np.sum(D * o.D, axis=0))
    assert float(np.abs(F * sg - o.F).max() / np.abs(o.F).max()) <= tol_d


def test_stage2_c2_shape():
    from paper_2203_12798_b200 import synth
    cfg = synth.scaled(synth.CONFIGS["c2"], num_slices=400)
    _check(synth.generate(cfg, 0, threads=os.cpu_count()), 10)


def test_stage2_wide_sketch_p_equals_r():
    from paper_2203_12798_b200 import synth
    cfg = synth.scaled(synth.CONFIGS["c2"], num_slices=200, rank=50)
    _check(synth.generate(cfg, 0, threads=os.cpu_count()), 50, oversampling=50)


def test_stage2_c5_width():
    from paper_2203_12798_b200 import synth
    cfg = synth.scaled(synth.CONFIGS["c5"], num_slices=40, dtype="f64")
    _check(synth.generate(cfg, 0, threads=os.cpu_count()), 10)


def test_stage2_noiseless_rank_deficient_y2():
    """Exact rank-R data, s2 = R + 10 > R: Y2 = M M^T M Omega2 has numerical
    rank R; Q2 must still be orthonormal and D, E, F match the reference."""
    from paper_2203_12798_b200 import synth
    cfg = synth.scaled(synth.CONFIGS["c1"], num_slices=60, noise=0.0, rank=6)
    _check(synth.generate(cfg, 1), 6, tol_d=1e-6, tol_e=1e-8)


@pytest.mark.parametrize("q,tol", [(0, 1e-6), (2, 1e-6), (3, 1e-3)])
def test_compress_power_iters_match_oracle(q, tol):
    """RsvdParams.power_iters != 1 (P/linalg.py:124-126) through both stages:
    the stage-1 bases, D, E and F match the oracle's compress(power_iters=q).
    The reference forms (X X^T)^q X Omega without re-orthonormalising, so its
    weakest sketch directions lose accuracy as kappa^(2q+1); ours
    re-orthonormalises each iteration (the same range in exact arithmetic).
    At q = 3 the two therefore agree only to the reference's own rounding on
    the weakest column (~4e-4 measured); q <= 2 to 1e-6."""
    import paper_2203_12798_b200 as dp
    from oracle import dpar2_oracle as orc
    from paper_2203_12798_b200 import synth
    cfg = synth.scaled(synth.CONFIGS["c1"], num_slices=30)
    xs = synth.generate(cfg, 2)
    comp = dp.compress(dp.IrregularTensor(xs), 10, rsvd=dp.RsvdParams(rank=10, power_iters=q, seed=0))
    o = orc.compress(xs, 10, seed=0, power_iters=q)
    A = comp.A.cpu().numpy()
    Ao = np.concatenate(o.bases)
    assert rel_signed(A, Ao) <= tol, rel_signed(A, Ao)
    assert float(np.abs(comp.weights.cpu().numpy() - o.E).max() / o.E.max()) <= tol * 1e-2
    assert rel_signed(comp.col_basis.cpu().numpy(), o.D) <= tol


def test_wide_stage1_sketch_above_128_columns():
    """s = R + p > 128 (sp = 160): the large-sketch stage-1 path (the CC T
    product over more than 128 columns, one pass over Y for A and the sign
    candidates) against the oracle's per-slice rSVD: U_k sign-exact (the
    reference's sign rule) within 1e-7, and D / E / F (s2 = 142 < K R)."""
    import paper_2203_12798_b200 as dp
    from oracle import dpar2_oracle as orc
    rng = np.random.default_rng(11)
    R, p, J = 12, 130, 200
    xs = [rng.standard_normal((int(m), J)) @ np.diag(np.linspace(2.0, 0.5, J)) for m in rng.integers(160, 260, size=16)]
    t = dp.IrregularTensor(xs)
    comp = dp.compress(t, R, rsvd=dp.RsvdParams(rank=R, oversampling=p, seed=0))
    o = orc.compress(xs, R, seed=0, oversampling=p, keep_stage1=True)
    for k in range(len(xs)):
        A = comp.slice_bases[k].cpu().numpy()
        U = o.stage1[k][0]
        assert float(np.abs(A - U).max()) <= 1e-7, k
    _check(xs, R, oversampling=p)


def test_stage2_sketch_wider_than_m():
    """s2 = R + p > K R (few slices, explicit oversampling): Y2 = M Omega_2 is
    rank deficient; the result is the reference's (range(M) either way)."""
    rng = np.random.default_rng(12)
    xs = [rng.standard_normal((int(m), 120)) for m in rng.integers(90, 140, size=5)]
    _check(xs, 8, oversampling=60)  # s2 = 68 > K R = 40
    ys = [rng.standard_normal((int(m), 200)) for m in rng.integers(160, 260, size=6)]
    _check(ys, 12, oversampling=130)  # s2 = 142 > K R = 72 (D^T D was 43 off the identity before the cap)
