"""One stage-1 streaming pass (dp2_stream_pass) against NumPy, per piece.

The pass computes, for every piece p of the streaming plan (segment x slice),
Z_p = X_p^T (X_p B_k) -- the two products of P/linalg.py:124-127 -- plus the
Y rows, G_p = Y_p^T Y_p and the per-piece sum of squares.  Both fp32 engines
are checked: the tcgen05 tf32 tensor-core pass (tolerance: tf32 products,
relative 2e-3 of the block norm) and the FFMA pass (fp32, 1e-5).
"""
import ctypes as C

import numpy as np
import pytest
import torch

import paper_2203_12798_b200 as dp
from paper_2203_12798_b200 import _lib

pytestmark = pytest.mark.gpu


def _vp(t):
    return C.c_void_p(t.data_ptr()) if t is not None else C.c_void_p(0)


def run_pass(slices, J, sp, nseg, engine, seed=0, want_y=True, want_g=True, want_sq=True):
    packed = torch.from_numpy(np.concatenate(slices).astype(np.float32)).cuda()
    ldx = (J + 3) // 4 * 4
    if ldx != J:
        packed = torch.nn.functional.pad(packed, (0, ldx - J))
    t = dp.IrregularTensor.from_packed(packed, [s.shape[0] for s in slices], J, check=False)
    K = len(slices)
    rng = np.random.default_rng(seed + 7)
    B = rng.standard_normal((K, J, sp))
    st, keep = t.store(nseg)
    plan = t.plan_host(nseg)
    n = len(plan["piece_slice"])
    dev = t.X.device
    Bd = torch.from_numpy(B).to(dev)
    out = torch.full((n, J, sp), np.nan, dtype=torch.float64, device=dev)
    total = int(t.row_off_host[-1])
    y = torch.full((total, sp), np.nan, dtype=torch.float64, device=dev) if want_y else None
    g = torch.full((n, sp, sp), np.nan, dtype=torch.float64, device=dev) if want_g else None
    sq = torch.full((n,), np.nan, dtype=torch.float64, device=dev) if want_sq else None
    status = dp.tensor.new_status(dev)
    prev = _lib.lib().dp2_set_sketch_engine(engine)
    try:
        _lib.check(_lib.lib().dp2_stream_pass(C.byref(st), _vp(Bd), sp, _vp(out), _vp(y), _vp(g), _vp(sq),
                                              _vp(status), C.c_void_p(torch.cuda.current_stream().cuda_stream)),
                   "stream_pass")
        torch.cuda.synchronize()
    finally:
        _lib.lib().dp2_set_sketch_engine(prev)
    # host-side piece geometry
    ps = plan["piece_slice"]
    row0 = keep[2]["piece_row0"].cpu().numpy()
    prow = keep[2]["piece_rows"].cpu().numpy()
    X = t.X.cpu().numpy()[:, :J].astype(np.float64)
    res = dict(out=out.cpu().numpy(), y=None if y is None else y.cpu().numpy(),
               g=None if g is None else g.cpu().numpy(), sq=None if sq is None else sq.cpu().numpy(),
               status=status.cpu().numpy())
    return X, B, ps, row0, prow, res


def rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


SHAPES = [
    # (row counts, J, sp, nseg)
    ([130, 64, 1, 200, 77], 128, 24, 3),
    ([300, 500, 257], 512, 24, 4),
    ([90, 33, 400], 100, 8, 2),
    ([256, 129], 300, 32, 3),
    ([700] * 6, 512, 16, 5),
    # J > 512: the tensor-core pass splits the columns across a CTA pair
    # (cluster of 2, Y partials exchanged through distributed shared memory);
    # odd nseg leaves the last pair one segment
    ([300, 500, 257, 64], 1000, 24, 5),
    ([700, 700, 700], 1024, 16, 4),
    ([130, 1, 77, 260], 600, 8, 3),
    ([400, 900], 520, 32, 6),
]


@pytest.mark.parametrize("engine", [0, 1], ids=["tcgen05", "ffma"])
@pytest.mark.parametrize("case", range(len(SHAPES)))
def test_stream_pass_matches_numpy(engine, case):
    rows, J, sp, nseg = SHAPES[case]
    if engine == 0 and sp == 32 and J > 256:
        pass  # ineligible for the tensor-core plan -> FFMA; still must match
    rng = np.random.default_rng(case)
    slices = [rng.standard_normal((m, J)) + 0.5 for m in rows]
    X, B, ps, row0, prow, res = run_pass(slices, J, sp, nseg, engine)
    tol = 2e-3 if engine == 0 else 1e-5
    for p in range(len(ps)):
        Xp = X[row0[p]:row0[p] + prow[p]]
        Yp = Xp @ B[ps[p]]
        Zp = Xp.T @ Yp
        assert rel(res["out"][p], Zp) < tol, (p, rel(res["out"][p], Zp))
        assert rel(res["y"][row0[p]:row0[p] + prow[p]], Yp) < tol, p
        assert rel(res["g"][p], Yp.T @ Yp) < 2 * tol, p
        # tensor-core pass: fp32 partials of 32 squares, fp64 across them
        assert abs(res["sq"][p] - np.sum(Xp * Xp)) <= (1e-6 if engine == 0 else 1e-9) * np.sum(Xp * Xp), p
    assert res["status"][0] == _lib.INT64_MAX


@pytest.mark.parametrize("J", [600, 1000, 1024])
def test_stream_pass_tc_pair_eligible(J):
    """512 < J <= 1024 runs the tcgen05 CTA-pair pass (not a fallback) in the tf32 mode."""
    import ctypes as C
    slices = [np.ones((70, J), np.float32)]
    t = dp.IrregularTensor.from_packed(torch.from_numpy(np.concatenate(slices)).cuda(), [70], J, check=False)
    st, keep = t.store(4)
    prev = _lib.lib().dp2_set_sketch_engine(0)
    try:
        assert _lib.lib().dp2_sketch_uses_tc(C.byref(st), 24) == 1
    finally:
        _lib.lib().dp2_set_sketch_engine(prev)


def test_stream_pass_tc_pair_flags_nonfinite():
    rng = np.random.default_rng(4)
    slices = [rng.standard_normal((m, 1000)) for m in (100, 150, 80)]
    slices[2][40, 900] = np.nan  # in the second CTA's column half
    *_, res = run_pass(slices, 1000, 24, 3, 0)
    assert res["status"][0] == 2


def test_stream_pass_tc_flags_nonfinite():
    rng = np.random.default_rng(3)
    slices = [rng.standard_normal((m, 128)) for m in (100, 150, 80)]
    slices[1][17, 5] = np.inf
    *_, res = run_pass(slices, 128, 24, 2, 0)
    assert res["status"][0] == 1
