"""IRT1 / IRC1 host parsing and writing against the reference's own files
(tests/golden/io, written by oracle/make_golden_io.py with the reference's
save_archive / save_compressed) -- CPU only."""
import json
import sys
from pathlib import Path

import numpy as np
import pytest

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle.make_golden_io import corruptions  # noqa: E402  (the same corrupted variants)
from paper_2203_12798_b200 import archive  # noqa: E402
from paper_2203_12798_b200.errors import ArchiveFormatError  # noqa: E402

IO = Path(__file__).resolve().parent / "golden" / "io"


def _arrays():
    z = np.load(IO / "arrays.npz")
    rows, X = z["rows"], z["X"]
    J = X.size // int(rows.sum())
    xs, off = [], 0
    for r in rows:
        xs.append(X[off:off + r * J].reshape(r, J))
        off += r * J
    A = z["A"]
    bases, off = [], 0
    for r in rows:
        bases.append(A[off:off + r])
        off += r
    return xs, z, bases


def test_read_irt1_matches_reference_arrays():
    xs, _, _ = _arrays()
    slices, _ = archive.read_irt1(IO / "small.irt1")
    assert len(slices) == len(xs)
    for a, b in zip(slices, xs):
        assert a.tobytes() == b.tobytes()


def test_write_irt1_byte_identical(tmp_path):
    xs, _, _ = _arrays()
    archive.write_irt1(xs, tmp_path / "x.irt1")
    assert (tmp_path / "x.irt1").read_bytes() == (IO / "small.irt1").read_bytes()


def test_read_write_irc1_matches_reference(tmp_path):
    _, z, bases = _arrays()
    rank, D, E, F, got = archive.read_irc1(IO / "small.irc1")
    assert rank == int(z["rank"])
    assert D.tobytes() == z["D"].tobytes() and E.tobytes() == z["E"].tobytes() and F.tobytes() == z["F"].tobytes()
    for a, b in zip(got, bases):
        assert a.tobytes() == b.tobytes()
    archive.write_irc1(rank, D, E, F, got, tmp_path / "c.irc1")
    assert (tmp_path / "c.irc1").read_bytes() == (IO / "small.irc1").read_bytes()


def test_corrupt_archives_raise_reference_messages(tmp_path):
    """Every structural corruption raises ArchiveFormatError with the
    reference's message (the non-finite case needs the device upload: GPU test)."""
    expected = json.loads((IO / "errors.json").read_text())
    irt1, irc1 = (IO / "small.irt1").read_bytes(), (IO / "small.irc1").read_bytes()
    for name, kind, data in corruptions(irt1, irc1):
        if name == "irt1_nonfinite":
            continue
        p = tmp_path / name
        p.write_bytes(data)
        with pytest.raises(ArchiveFormatError) as ei:
            (archive.read_irt1 if kind == "irt1" else archive.read_irc1)(p)
        assert str(ei.value) == expected[name].replace("{path}", str(p)), name
