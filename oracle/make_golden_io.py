"""IRT1 / IRC1 fixtures from the REAL reference (test infrastructure only).

    python oracle/make_golden_io.py

Writes tests/golden/io/: an IRT1 archive and an IRC1 archive produced by the
reference's own ``save_archive`` / ``save_compressed`` (P/tensor.py:172-179,
P/compress.py:133-142), the arrays they hold (``arrays.npz``, as the
reference's loaders return them), and ``errors.json``: for a set of corrupted
variants (built here and rebuilt identically by the tests), the
``ArchiveFormatError`` message the reference's loader raises, with the path
replaced by ``{path}``.
"""
from __future__ import annotations

import json
import os
import sys
import tempfile
from pathlib import Path

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
REF = Path("/root/reference/pkg/src")
OUT = ROOT / "tests" / "golden" / "io"


def corruptions(irt1: bytes, irc1: bytes):
    """(name, kind, bytes) variants; tests/test_archive.py rebuilds the same."""
    bad_rows = bytearray(irt1)
    bad_rows[12:16] = (0).to_bytes(4, "little")  # slice 0 rows = 0
    bad_dims = bytearray(irt1)
    bad_dims[4:8] = (0).to_bytes(4, "little")    # K = 0
    nan = bytearray(irt1)
    nan[16 + 8 * 3:16 + 8 * 4] = np.array([np.nan], "<f8").tobytes()  # slice 0, entry 3
    return [
        ("irt1_magic", "irt1", b"XRT1" + irt1[4:]),
        ("irt1_empty", "irt1", b""),
        ("irt1_header", "irt1", irt1[:9]),
        ("irt1_dims", "irt1", bytes(bad_dims)),
        ("irt1_zero_rows", "irt1", bytes(bad_rows)),
        ("irt1_slice_header", "irt1", irt1[:12]),
        ("irt1_payload", "irt1", irt1[:40]),
        ("irt1_trailing", "irt1", irt1 + b"\x00\x01\x02"),
        ("irt1_nonfinite", "irt1", bytes(nan)),
        ("irc1_magic", "irc1", b"IRT1" + irc1[4:]),
        ("irc1_header", "irc1", irc1[:10]),
        ("irc1_dims", "irc1", irc1[:8] + (0).to_bytes(4, "little") + irc1[12:]),
        ("irc1_payload", "irc1", irc1[:30]),
        ("irc1_trailing", "irc1", irc1 + b"\x00"),
    ]


def main():
    sys.path.insert(0, str(REF))
    import dpar2  # the reference (only here: the tests import corruptions() without it)
    from dpar2.errors import ArchiveFormatError
    OUT.mkdir(parents=True, exist_ok=True)
    rng = np.random.default_rng(2203)
    slices = [rng.standard_normal((int(m), 7)) for m in (5, 9, 3, 12)]
    t = dpar2.IrregularTensor(slices)
    dpar2.save_archive(t, OUT / "small.irt1")
    comp = dpar2.compress(t, 3, dpar2.RsvdParams(rank=3, seed=11))
    dpar2.save_compressed(comp, OUT / "small.irc1")
    t2 = dpar2.load_archive(OUT / "small.irt1")
    c2 = dpar2.load_compressed(OUT / "small.irc1")
    np.savez(OUT / "arrays.npz", rows=np.array([x.shape[0] for x in t2.slices]),
             X=np.concatenate([x.ravel() for x in t2.slices]), D=c2.col_basis, E=c2.weights, F=c2.cores,
             A=np.concatenate(c2.slice_bases), rank=c2.rank)
    irt1, irc1 = (OUT / "small.irt1").read_bytes(), (OUT / "small.irc1").read_bytes()
    errors = {}
    with tempfile.TemporaryDirectory() as d:
        for name, kind, data in corruptions(irt1, irc1):
            p = Path(d) / name
            p.write_bytes(data)
            try:
                (dpar2.load_archive if kind == "irt1" else dpar2.load_compressed)(p)
                errors[name] = None
            except ArchiveFormatError as exc:
                errors[name] = str(exc).replace(str(p), "{path}")
    (OUT / "errors.json").write_text(json.dumps(errors, indent=1) + "\n")
    print(json.dumps(errors, indent=1))


if __name__ == "__main__":
    main()
