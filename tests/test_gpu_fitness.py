"""Zero-pass fitness (analysis.py, dp2_fitness_zero_pass; SURVEY §8(f) 3,
P/analysis.py:23-45): for device factors fresh from a fit, equal to the
streaming pass over X to rounding and to the oracle within the fitness
tolerance; every case it does not cover -- NumPy factors, fp32 stores,
another tensor, rank-deficient slices, factors edited in place or replaced
after the fit -- falls back to the pass."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_zero_pass_fitness_matches_streaming_pass_and_oracle(seed):
    import paper_2203_12798_b200 as dp
    from paper_2203_12798_b200.analysis import _zero_pass_terms
    from oracle import dpar2_oracle as orc
    rng = np.random.default_rng(seed)
    J, R = int(rng.integers(20, 80)), int(rng.integers(2, 9))
    u = rng.standard_normal((J, R))
    xs = [rng.standard_normal((int(m), R)) @ u.T + 0.2 * rng.standard_normal((int(m), J))
          for m in rng.integers(R + 1, 300, size=int(rng.integers(3, 30)))]
    t = dp.IrregularTensor(xs)
    f, _ = dp.fit_dpar2(t, R, dp.SolverOptions(max_iters=12, tol=0.0, seed=seed), output="device")
    assert _zero_pass_terms(t, f, lambda x: x.cuda() if hasattr(x, "cuda") else
                            __import__("torch").from_numpy(np.asarray(x)).cuda()) is not None
    fz = dp.fitness(t, f)
    fp = dp.fitness(t, f, zero_pass=False)
    assert abs(fz - fp) <= 1e-12
    o = orc.fit_dpar2(xs, R, 12, 0.0, seed)
    assert abs(fz - orc.fitness(xs, o["H"], o["V"], o["W"], o["Q"])) <= 1e-6


def test_zero_pass_fitness_fallbacks():
    import torch
    import paper_2203_12798_b200 as dp
    from paper_2203_12798_b200.analysis import _zero_pass_terms
    rng = np.random.default_rng(5)
    xs = [rng.standard_normal((int(m), 25)) for m in rng.integers(10, 90, size=8)]
    d = lambda x: x if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(x)).cuda()  # noqa
    # fp32 store: M comes from fp32 (or tf32) products -> the streaming pass
    t32 = dp.IrregularTensor([x.astype(np.float32) for x in xs], dtype="f32")
    f32, _ = dp.fit_dpar2(t32, 4, dp.SolverOptions(max_iters=5, tol=0.0), output="device")
    assert _zero_pass_terms(t32, f32, d) is None
    # a different tensor, or changed V -> the streaming pass
    t = dp.IrregularTensor(xs)
    f, _ = dp.fit_dpar2(t, 4, dp.SolverOptions(max_iters=5, tol=0.0), output="device")
    assert _zero_pass_terms(t, f, d) is not None
    assert _zero_pass_terms(dp.IrregularTensor(xs), f, d) is None
    # NumPy factors: the streaming pass
    fn, _ = dp.fit_dpar2(t, 4, dp.SolverOptions(max_iters=5, tol=0.0))
    assert _zero_pass_terms(t, fn, d) is None
    # in-place edits of the fit's own device tensors: V and Q
    f.V.mul_(1.5)
    assert _zero_pass_terms(t, f, d) is None
    assert dp.fitness(t, f) == dp.fitness(t, f, zero_pass=False)
    f.V.copy_(f._zero_pass["V"])
    assert _zero_pass_terms(t, f, d) is not None
    f.Q_packed[:3].neg_()
    assert _zero_pass_terms(t, f, d) is None
    assert dp.fitness(t, f) == dp.fitness(t, f, zero_pass=False)
    g = dp.Parafac2Factors(H=f.H, V=f.V * 1.5, W=f.W, Q=f.Q, Q_packed=f.Q_packed)
    g._zero_pass = f._zero_pass
    assert _zero_pass_terms(t, g, d) is None
    assert dp.fitness(t, g) == dp.fitness(t, g, zero_pass=False)
    # a rank-deficient slice (completed A_k columns) -> the streaming pass
    ys = [x.copy() for x in xs]
    ys[3] = np.outer(rng.standard_normal(40), rng.standard_normal(25))
    td = dp.IrregularTensor(ys)
    fd, _ = dp.fit_dpar2(td, 4, dp.SolverOptions(max_iters=5, tol=0.0), output="device")
    assert _zero_pass_terms(td, fd, d) is None
    assert dp.fitness(td, fd) == dp.fitness(td, fd, zero_pass=False)
