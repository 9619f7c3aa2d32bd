"""Tensor-core (tcgen05 tf32) vs FFMA fp32 streaming pass: stage-1 outputs,
fit, and pass timings on the same device tensor.

    python tools/tc_check.py [--config c2] [--slices 200] [--iters 32]
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2203_12798_b200 as dp  # noqa: E402
from paper_2203_12798_b200 import _lib, synth  # noqa: E402


def run(t, R, engine, iters):
    _lib.lib().dp2_set_sketch_engine(engine)
    tm = {}
    comp = dp.compress(t, R, timings=tm)
    torch.cuda.synchronize()
    tm = {}
    comp = dp.compress(t, R, timings=tm)
    opts = dp.SolverOptions(max_iters=iters, tol=0.0, seed=0)
    f, tr = dp.fit_dpar2(t, R, opts, output="device")
    fit = dp.fitness(t, f)
    return comp, tm, tr.objective, fit


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--slices", type=int, default=200)
    ap.add_argument("--iters", type=int, default=32)
    args = ap.parse_args()
    cfg = synth.scaled(synth.CONFIGS[args.config], dtype="f32", num_slices=args.slices)
    X, rows, _, _ = synth.generate_device(cfg, 0)
    t = dp.IrregularTensor.from_packed(X, rows, cfg.cols)
    R = cfg.rank
    c1, tm1, o1, f1 = run(t, R, 1, args.iters)
    c0, tm0, o0, f0 = run(t, R, 0, args.iters)
    A1, A0 = c1.A.cpu().numpy(), c0.A.cpu().numpy()
    sgn = np.sign(np.sum(A1 * A0, axis=0))
    out = {
        "A_max_abs": float(np.abs(A0 * sgn - A1).max()),
        "D_rel": float(np.abs(np.abs(c0.col_basis.cpu().numpy()) - np.abs(c1.col_basis.cpu().numpy())).max()),
        "E_rel": float(np.max(np.abs(c0.weights.cpu().numpy() - c1.weights.cpu().numpy()) /
                              np.abs(c1.weights.cpu().numpy()))),
        "fit_ffma": float(f1), "fit_tc": float(f0), "fit_diff": float(abs(f0 - f1)),
        "obj_rel": float(abs(o0[-1] - o1[-1]) / abs(o1[-1])),
        "timings_ffma": {k: v for k, v in tm1.items() if k.endswith("_ms")},
        "timings_tc": {k: v for k, v in tm0.items() if k.endswith("_ms")},
    }
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
