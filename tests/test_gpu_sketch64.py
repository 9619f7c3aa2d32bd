"""The warp-specialised fp64 DMMA streaming pass (csrc/dp2_sketch64.cu) against
NumPy, per piece: Z_p = X_p^T (X_p B_k), the Y rows and G_p = Y_p^T Y_p
(P/linalg.py:124-127 fused).  fp64 storage (the default pass of fp64 tensors)
and fp32 storage with fp64 products (engine 2, exactly upcast values).  The
pass computes in fp64: tolerance 1e-12 relative to the block norm.
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


def run_pass(slices, J, sp, nseg, dtype, want_y=True, want_g=True, seed=0):
    npdt = np.float64 if dtype == "f64" else np.float32
    packed = torch.from_numpy(np.concatenate(slices).astype(npdt)).cuda()
    align = 2 if dtype == "f64" else 4
    ldx = (J + align - 1) // align * align
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
    status = dp.tensor.new_status(dev)
    prev = _lib.lib().dp2_set_sketch_engine(2)  # fp32 storage -> fp64 products (fp64 storage always)
    try:
        kind = _lib.lib().dp2_sketch_kind(C.byref(st), sp, 0, int(want_g))
        _lib.check(_lib.lib().dp2_stream_pass(
            C.byref(st), _vp(Bd), sp, _vp(out), _vp(y), _vp(g), C.c_void_p(0), _vp(status),
            C.c_void_p(torch.cuda.current_stream().cuda_stream)), "stream_pass")
        torch.cuda.synchronize()
    finally:
        _lib.lib().dp2_set_sketch_engine(prev)
    ps = plan["piece_slice"]
    row0 = keep[2]["piece_row0"].cpu().numpy()
    prow = keep[2]["piece_rows"].cpu().numpy()
    X = t.X.cpu().numpy()[:, :J].astype(np.float64)
    res = dict(out=out.cpu().numpy(), y=None if y is None else y.cpu().numpy(),
               g=None if g is None else g.cpu().numpy(), status=status.cpu().numpy(), kind=kind)
    return X, B, ps, row0, prow, res


def rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


SHAPES = [
    # (row counts, J, sp, nseg, want_g)
    ([130, 64, 1, 200, 77], 128, 24, 3, True),   # 1-row slice, partial tiles, pieces across segments
    ([300, 500, 257], 512, 24, 4, True),          # the c2 width
    ([90, 33, 400], 100, 8, 2, True),             # J padded to 128, one column block
    ([256, 129], 300, 32, 3, False),              # sp = 32: two column groups (G elsewhere)
    ([700] * 6, 512, 16, 5, True),
    ([41, 600, 999], 512, 128, 7, False),         # c4-like (s = 2R = 100 -> sp 128): six groups
    ([3000, 17], 256, 24, 148, True),             # many more segments than rows per segment (16-row tiles)
    ([300, 77, 1200], 1000, 24, 4, False),        # the c5 width: one column block per CTA group (G elsewhere)
]


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("case", range(len(SHAPES)))
def test_sketch64_matches_numpy(dtype, case):
    rows, J, sp, nseg, want_g = SHAPES[case]
    rng = np.random.default_rng(case)
    slices = [rng.standard_normal((m, J)) + 0.5 for m in rows]
    if dtype == "f32":
        slices = [s.astype(np.float32) for s in slices]
    X, B, ps, row0, prow, res = run_pass(slices, J, sp, nseg, dtype, want_g=want_g)
    assert res["kind"] == 3, "the DMMA pass did not run (ineligible shape?)"
    for p in range(len(ps)):
        Xp = X[row0[p]:row0[p] + prow[p]]
        Yp = Xp @ B[ps[p]]
        Zp = Xp.T @ Yp
        assert rel(res["out"][p], Zp) < 1e-12, (p, rel(res["out"][p], Zp))
        assert rel(res["y"][row0[p]:row0[p] + prow[p]], Yp) < 1e-12, p
        if want_g:
            assert rel(res["g"][p], Yp.T @ Yp) < 1e-12, p
    assert res["status"][0] == _lib.INT64_MAX


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_sketch64_flags_lowest_nonfinite_slice(dtype):
    rng = np.random.default_rng(3)
    slices = [rng.standard_normal((m, 128)) for m in (100, 150, 80, 60)]
    slices[2][17, 5] = np.nan
    slices[3][1, 100] = np.inf
    if dtype == "f32":
        slices = [s.astype(np.float32) for s in slices]
    *_, res = run_pass(slices, 128, 24, 3, dtype)
    assert res["status"][0] == 2


@pytest.mark.parametrize("J,sp", [(128, 24), (600, 8)])
def test_sketch64_fp32_widening_is_exact_on_denormals_and_zeros(J, sp):
    """fp32 storage is upcast inside the pass -- with integer instructions when
    NT > 1 (csrc/dp2_sketch64.cu widen) -- and must equal the exact value for
    +-0, denormals and the smallest / largest normals (P/tensor.py: the oracle
    sees the fp32 values upcast exactly)."""
    rng = np.random.default_rng(11)
    tiny = np.float32(1.1754944e-38)  # FLT_MIN
    pool = np.array([0.0, -0.0, 1.4e-45, -1.4e-45, 7e-42, -3e-40, 5.8e-39, tiny, -tiny, 2.5e-38, -9e-38],
                    dtype=np.float32)
    slices = [pool[rng.integers(0, len(pool), size=(m, J))] for m in (150, 37, 260)]
    X, B, ps, row0, prow, res = run_pass(slices, J, sp, 3, "f32", want_g=False)
    assert res["kind"] == 3
    for p in range(len(ps)):
        Xp = X[row0[p]:row0[p] + prow[p]]
        Yp = Xp @ B[ps[p]]
        assert rel(res["y"][row0[p]:row0[p] + prow[p]], Yp) < 1e-12, p
        assert rel(res["out"][p], Xp.T @ Yp) < 1e-12, p
    big = [np.where(rng.random((90, J)) < 0.5, np.float32(3.4028235e38), np.float32(-1.7e38)).astype(np.float32)]
    X, B, ps, row0, prow, res = run_pass(big, J, sp, 2, "f32", want_g=False)
    for p in range(len(ps)):
        Xp = X[row0[p]:row0[p] + prow[p]]
        assert rel(res["y"][row0[p]:row0[p] + prow[p]], Xp @ B[ps[p]]) < 1e-12, p
    assert res["status"][0] == _lib.INT64_MAX


def test_sketch64_cta_pairs_match_numpy():
    """The CTA-pair (thread-block cluster) variant of the pass, DP2_S64_PAIRS=1:
    each CTA of a pair owns half of J, the Y partials cross over DSMEM.  Run in
    a subprocess (the switch is read once per process)."""
    import subprocess
    import sys
    code = ("import sys; sys.path.insert(0, 'tests'); import test_gpu_sketch64 as T; "
            "[T.test_sketch64_matches_numpy(d, c) for d in ('f64', 'f32') for c in (1, 4, 6)]; "
            "T.test_sketch64_flags_lowest_nonfinite_slice('f64')")
    env = dict(__import__("os").environ, DP2_S64_PAIRS="1")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
