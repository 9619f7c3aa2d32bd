"""One warm c4 fit (compress with oversampling p = R, then the ALS) inside an
NVTX range "dp2_fit", for ncu launch lists of the large-rank paths.

    python tools/profile_c4.py --rank 50 [--slices 1000] [--iters 4]
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2203_12798_b200 as dp  # noqa: E402
from paper_2203_12798_b200 import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rank", type=int, default=50)
    ap.add_argument("--slices", type=int, default=1000)
    ap.add_argument("--iters", type=int, default=4)
    a = ap.parse_args()
    cfg = synth.scaled(synth.CONFIGS["c4"], num_slices=a.slices)
    X, rows, _, _ = synth.generate_device(cfg, 0)
    t = dp.IrregularTensor.from_packed(X, rows, cfg.cols)
    R = a.rank
    rsvd = dp.RsvdParams(rank=R, oversampling=R, seed=0)
    opts = dp.SolverOptions(max_iters=a.iters, tol=0.0, seed=0)
    for rep in range(2):
        torch.cuda.synchronize()
        if rep:
            torch.cuda.nvtx.range_push("dp2_fit")
        comp = dp.compress(t, R, rsvd=rsvd)
        dp.fit_compressed(comp, opts, output="device")
        torch.cuda.synchronize()
        if rep:
            torch.cuda.nvtx.range_pop()


if __name__ == "__main__":
    main()
