"""IRT1 / IRC1 through the device store: archives written by the reference
load into the same fit as in-memory slices; device tensors and compressions
save back byte-identically / exactly; a loaded IRC1 archive fits without
recompressing (fit_compressed)."""
import json
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

IO = Path(__file__).resolve().parent / "golden" / "io"


def test_load_archive_fit_matches_in_memory(tmp_path):
    import paper_2203_12798_b200 as dp
    from paper_2203_12798_b200 import archive
    slices, _ = archive.read_irt1(IO / "small.irt1")
    xs = [np.array(x) for x in slices]
    t = dp.load_archive(IO / "small.irt1")
    opts = dp.SolverOptions(max_iters=8, tol=0.0, seed=1)
    f, tr = dp.fit_dpar2(t, 3, opts)
    g, tr2 = dp.fit_dpar2(dp.IrregularTensor(xs), 3, opts)
    for key in ("H", "V", "W"):
        assert getattr(f, key).tobytes() == getattr(g, key).tobytes(), key
    assert tr.objective == tr2.objective
    dp.save_archive(t, tmp_path / "back.irt1")
    assert (tmp_path / "back.irt1").read_bytes() == (IO / "small.irt1").read_bytes()
    t32 = dp.load_archive(IO / "small.irt1", dtype="f32")
    assert t32.dtype == "f32" and t32.num_slices == len(xs)


def test_load_archive_nonfinite_message(tmp_path):
    import paper_2203_12798_b200 as dp
    from oracle.make_golden_io import corruptions
    expected = json.loads((IO / "errors.json").read_text())["irt1_nonfinite"]
    irt1, irc1 = (IO / "small.irt1").read_bytes(), (IO / "small.irc1").read_bytes()
    data = dict((n, d) for n, _, d in corruptions(irt1, irc1))["irt1_nonfinite"]
    p = tmp_path / "nan.irt1"
    p.write_bytes(data)
    with pytest.raises(dp.ArchiveFormatError) as ei:
        dp.load_archive(p)
    assert str(ei.value) == expected.replace("{path}", str(p))


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_compressed_round_trip_and_fit_compressed(tmp_path, dtype):
    import torch
    import paper_2203_12798_b200 as dp
    from paper_2203_12798_b200 import archive
    from paper_2203_12798_b200.compress import reconstruct_slice
    rng = np.random.default_rng(9)
    xs = [rng.standard_normal((int(m), 30)) for m in rng.integers(20, 200, size=15)]
    t = dp.IrregularTensor(xs, dtype=dtype)
    R = 5
    comp = dp.compress(t, R, rsvd=dp.RsvdParams(rank=R, seed=2))  # fit_dpar2 compresses with opts.seed
    dp.save_compressed(comp, tmp_path / "c.irc1")
    rank, D, E, F, bases = archive.read_irc1(tmp_path / "c.irc1")
    assert rank == R
    assert np.array_equal(D, comp.col_basis.cpu().numpy()) and np.array_equal(E, comp.weights.cpu().numpy())
    assert np.array_equal(F, comp.cores.cpu().numpy())
    assert np.array_equal(np.concatenate(bases), comp.A.cpu().numpy())
    back = dp.load_compressed(tmp_path / "c.irc1")
    for k in (0, 7, 14):
        assert torch.equal(reconstruct_slice(back, k), reconstruct_slice(comp, k))
    # compress once, fit from the archive: the same ALS as fit_dpar2 on the same compression
    opts = dp.SolverOptions(max_iters=10, tol=0.0, seed=2)
    f, tr = dp.fit_compressed(back, opts)
    g, tr2 = dp.fit_dpar2(t, R, dp.SolverOptions(max_iters=10, tol=0.0, seed=2))
    assert tr.objective == tr2.objective
    for key in ("H", "V", "W"):
        assert np.array_equal(getattr(f, key), getattr(g, key)), key
    assert np.array_equal(np.concatenate(f.Q), np.concatenate(g.Q))


def test_fit_compressed_from_reference_irc1():
    """The reference's own IRC1 archive fits on the device like the oracle's
    ALS on the same compressed arrays (P/solver.py:167-190)."""
    import paper_2203_12798_b200 as dp
    from oracle import dpar2_oracle as orc
    from paper_2203_12798_b200 import archive
    from test_gpu_parity import rel_signed
    comp = dp.load_compressed(IO / "small.irc1")
    f, tr = dp.fit_compressed(comp, dp.SolverOptions(max_iters=6, tol=0.0, seed=0))
    rank, D, E, F, bases = archive.read_irc1(IO / "small.irc1")
    slices, _ = archive.read_irt1(IO / "small.irt1")
    oc = orc.Compressed(rank, [np.array(b) for b in bases], np.array(D), np.array(E), np.array(F))
    o = orc.fit_dpar2([np.array(x) for x in slices], rank, max_iters=6, tol=0.0, seed=0, comp=oc)
    assert len(tr.objective) == len(o["objective"])
    assert max(abs(a - b) / max(abs(b), 1e-300) for a, b in zip(tr.objective, o["objective"])) <= 1e-6
    for key in ("H", "V", "W"):
        assert rel_signed(getattr(f, key), o[key]) <= 1e-5, key
    for q, qo in zip(f.Q, o["Q"]):
        assert rel_signed(q, qo) <= 1e-5
