"""The drop-in seam of the reference CLI (P/cli.py:45: ``_run_method`` calls
the module global ``fit_dpar2``, which R/pkg/tests/test_cli.py:156-163
monkeypatches).  Runs where the reference is importable (this build
container); skipped elsewhere.

CPU half (no GPU): the reference's ``dpar2 generate`` + ``dpar2 decompose``
end to end with ``cli.fit_dpar2`` swapped for a function that returns OUR
containers (paper_2203_12798_b200.Parafac2Factors / FitTrace, filled from the
pinned oracle's fit): the reference's report writer, ``save_factors`` and
``analysis.fitness`` consume them unchanged.  GPU half: the swapped-in
function is our ``fit_dpar2`` itself, called with the reference's own
IrregularTensor and SolverOptions objects.
"""
import json
import sys
from pathlib import Path

import numpy as np
import pytest

REF = Path("/root/reference/pkg/src")
pytestmark = pytest.mark.skipif(not REF.exists(), reason="reference package not present")


@pytest.fixture()
def ref_cli(monkeypatch):
    monkeypatch.syspath_prepend(str(REF))
    for m in [m for m in sys.modules if m == "dpar2" or m.startswith("dpar2.")]:
        monkeypatch.delitem(sys.modules, m)
    from dpar2 import cli
    return cli


def _oracle_fit_as_ours(tensor, rank, opts):
    """Our containers around the oracle's fit of the reference tensor."""
    import paper_2203_12798_b200 as dp
    from oracle import dpar2_oracle as orc
    o = orc.fit_dpar2(list(tensor.slices), rank, opts.max_iters, opts.tol, opts.seed)
    tr = dp.FitTrace(objective=list(o["objective"]), seconds=list(o["seconds"]),
                     preprocess_seconds=0.0, compressed_float_count=o["compressed_float_count"])
    tr.converged = o["converged"]
    return dp.Parafac2Factors(H=o["H"], V=o["V"], W=o["W"], Q=list(o["Q"])), tr


def _run(cli, tmp_path, fit):
    tmp_path.mkdir(parents=True, exist_ok=True)
    arch = tmp_path / "t.irt"
    assert cli.main(["generate", "--I", "40", "--J", "12", "--K", "6", "--rank", "3", "--seed", "1",
                     "--out", str(arch)]) == 0
    cli.fit_dpar2 = fit
    out = tmp_path / "factors"
    rep = tmp_path / "report.csv"
    rc = cli.main(["decompose", str(arch), "--rank", "3", "--max-iters", "8", "--tol", "0", "--seed", "0",
                   "--out-factors", str(out), "--out-report", str(rep), "--report-fitness"])
    return rc, out, rep


def test_reference_cli_consumes_our_containers(ref_cli, tmp_path):
    rc, out, rep = _run(ref_cli, tmp_path, _oracle_fit_as_ours)
    assert rc == 0
    man = json.loads((out / "manifest.json").read_text())
    assert man["rank"] == 3 and man["num_slices"] == 6
    assert (out / "U_0005.csv").exists() and rep.read_text().count("\n") >= 9


@pytest.mark.gpu
def test_reference_cli_drives_b200_fit(ref_cli, tmp_path):
    """``cli.fit_dpar2 = paper_2203_12798_b200.fit_dpar2``: the CLI's own
    tensor / options objects go in, its writers take our factors; the written
    H matches the reference's own run within the fp64 tolerance."""
    import paper_2203_12798_b200 as dp
    ref_fit = ref_cli.fit_dpar2
    rc, out, _ = _run(ref_cli, tmp_path / "b200", dp.fit_dpar2)
    assert rc == 0
    rc2, out2, _ = _run(ref_cli, tmp_path / "ref", ref_fit)
    assert rc2 == 0
    h, h2 = (np.loadtxt(d / "H.csv", delimiter=",") for d in (out, out2))
    s = np.sign(np.sum(h * h2, axis=0))
    assert float(np.abs(h * s - h2).max() / np.abs(h2).max()) <= 1e-5
