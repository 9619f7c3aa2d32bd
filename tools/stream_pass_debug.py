"""Print per-output errors of one streaming pass vs NumPy (both engines)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
import numpy as np  # noqa: E402

from test_gpu_stream_pass import SHAPES, rel, run_pass  # noqa: E402

for case, (rows, J, sp, nseg) in enumerate(SHAPES):
    for engine in (0, 1):
        rng = np.random.default_rng(case)
        slices = [rng.standard_normal((m, J)) + 0.5 for m in rows]
        X, B, ps, row0, prow, res = run_pass(slices, J, sp, nseg, engine)
        eo, ey, eg, es = [], [], [], []
        for p in range(len(ps)):
            Xp = X[row0[p]:row0[p] + prow[p]]
            Yp = Xp @ B[ps[p]]
            eo.append(rel(res["out"][p], Xp.T @ Yp))
            ey.append(rel(res["y"][row0[p]:row0[p] + prow[p]], Yp))
            eg.append(rel(res["g"][p], Yp.T @ Yp))
            es.append(abs(res["sq"][p] - np.sum(Xp * Xp)) / np.sum(Xp * Xp))
        print(f"case {case} engine {engine} pieces {len(ps)} out {max(eo):.2e} y {max(ey):.2e} "
              f"g {max(eg):.2e} sq {max(es):.2e} status0 {res['status'][0]}", flush=True)
        if engine == 0 and case == 0:
            p = 0
            Xp = X[row0[p]:row0[p] + prow[p]]
            Yp = Xp @ B[ps[p]]
            print(" y[0,:6] got", np.round(res["y"][row0[p], :6], 4), "want", np.round(Yp[0, :6], 4))
            print(" y[20,:6] got", np.round(res["y"][row0[p] + 20, :6], 4), "want", np.round(Yp[20, :6], 4))
            Z = Xp.T @ Yp
            print(" z[0,:6] got", np.round(res["out"][p][0, :6], 3), "want", np.round(Z[0, :6], 3))
            print(" z[40,:6] got", np.round(res["out"][p][40, :6], 3), "want", np.round(Z[40, :6], 3))
            print(" per-row y err (first 70 rows):", np.round(np.abs(res["y"][row0[p]:row0[p] + 70] - Yp[:70]).max(axis=1), 2).tolist())
