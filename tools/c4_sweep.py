"""BASELINE config 4: the rank sweep on the c2 tensor (K=1000, J=512,
I_k ~ U{500..4000}, fp64), R in {10, 20, 30, 40, 50} with oversampling p = R
(the replay harness: compress(rsvd=RsvdParams(R, oversampling=R)) then the
fit loop, P/solver.py:170-190), 32 iterations; stage 1 and the per-iteration
ALS timed separately (CUDA events / device timestamps), plus the oracle's
fitness on the same tensor for R = 10 and 20 (CPU time permitting).

    python tools/c4_sweep.py [--ranks 10,20,30,40,50] [--out profiles/r2_c4_sweep.json]
"""
import argparse
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2203_12798_b200 as dp  # noqa: E402
from paper_2203_12798_b200 import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ranks", default="10,20,30,40,50")
    ap.add_argument("--out", default=None)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    cfg = synth.CONFIGS["c4"]
    xs = synth.generate(cfg, 0, threads=os.cpu_count())
    up = dp.IrregularTensor(xs)
    up.wait_upload()
    t = dp.IrregularTensor.from_packed(up.X, up.row_counts, cfg.cols)
    entries = int(sum(x.shape[0] for x in xs)) * cfg.cols
    out = {"config": "c4: c2 tensor (K=1000, J=512, I_k~U{500..4000}, fp64), p = R, 32 iterations, tol 0",
           "entries": entries, "ranks": {}}
    opts = dp.SolverOptions(max_iters=32, tol=0.0, seed=0)
    for R in [int(r) for r in a.ranks.split(",")]:
        rsvd = dp.RsvdParams(rank=R, oversampling=R, seed=0)
        rec = []
        for rep in range(a.reps + 1):
            tm = {}
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            comp = dp.compress(t, R, rsvd=rsvd, timings=tm)
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            f, tr = dp.fit_compressed(comp, opts, output="device")
            torch.cuda.synchronize()
            t2 = time.perf_counter()
            if rep:
                rec.append(dict(stage1_ms=tm["stage1_ms"], sketch_pass_ms=[tm["stage1_sketch1_ms"],
                                                                          tm["stage1_sketch2_ms"]],
                                stage2_ms=tm["stage2_ms"], compress_wall_ms=(t1 - t0) * 1e3,
                                als_per_iter_us=float(np.mean(tr.seconds)) * 1e6,
                                fit_compressed_wall_ms=(t2 - t1) * 1e3, sp=tm["sp"]))
        fit = dp.fitness(t, f, zero_pass=False)
        med = {k: float(np.median([r[k] for r in rec])) for k in rec[0] if k not in ("sketch_pass_ms", "sp")}
        med["sketch_pass_ms"] = [float(np.median([r["sketch_pass_ms"][i] for r in rec])) for i in (0, 1)]
        med["sp"] = rec[0]["sp"]
        med["fitness"] = fit
        # stage-1 roofline: F1 = 8 s sum(I_k) J at the measured DMMA peak
        s = 2 * R
        peak = json.loads((Path(__file__).resolve().parents[1] / "profiles" / "r2_compute_peaks.json").read_text())[
            "dmma_f64_tflops"]
        med["stage1_T_roof_ms"] = 8.0 * s * entries / (peak * 1e12) * 1e3
        med["stage1_roofline_achieved"] = med["stage1_T_roof_ms"] / med["stage1_ms"]
        out["ranks"][R] = med
        print(R, json.dumps(med), flush=True)
    if a.out:
        Path(a.out).write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
