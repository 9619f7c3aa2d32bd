"""Warm per-phase ALS timings via the phase API (CUDA events around each phase).

    python tools/als_phase_timing.py [--config c2] [--iters 32]
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2203_12798_b200 as dp  # noqa: E402
from paper_2203_12798_b200 import distributed as D_, synth  # noqa: E402
from paper_2203_12798_b200.factors import initial_factors  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--iters", type=int, default=32)
    ap.add_argument("--dtype", default="f32")
    args = ap.parse_args()
    cfg = synth.scaled(synth.CONFIGS[args.config], dtype=args.dtype)
    X, rows, _, _ = synth.generate_device(cfg, 0)
    t = dp.IrregularTensor.from_packed(X, rows, cfg.cols)
    comp = dp.compress(t, cfg.rank)
    K, J, R = t.num_slices, t.num_cols, cfg.rank
    h, v, w = initial_factors(J, K, R)
    dev = comp.cores.device
    ops = D_.GpuAlsOps(comp.cores, comp.col_basis, comp.weights, torch.from_numpy(h).to(dev),
                       torch.from_numpy(v).to(dev), torch.from_numpy(w).to(dev), J, R, args.iters, 0.0, True)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(8)]
    times = np.zeros((args.iters, 6))
    ops.phase(0)
    for it in range(args.iters):
        ev[0].record()
        red = ops.phase(1, it=it)
        ev[1].record()
        ops.phase(2, it=it, red_in=red)
        ev[2].record()
        red = ops.phase(3, it=it)
        ev[3].record()
        ops.phase(4, it=it, red_in=red)
        ev[4].record()
        red = ops.phase(5, it=it)
        ev[5].record()
        ops.phase(6, it=it, red_in=red)
        ev[6].record()
        torch.cuda.synchronize()
        times[it] = [ev[i].elapsed_time(ev[i + 1]) * 1e3 for i in range(6)]
    names = ["rotate+red", "solve_h", "mode2+red", "solve_v", "mode3+metric+red", "finish"]
    out = {n: {"first_us": float(times[0, i]), "mean_us_after_first": float(times[1:, i].mean())}
           for i, n in enumerate(names)}
    out["total_mean_us"] = float(times[1:].sum(axis=1).mean())
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
