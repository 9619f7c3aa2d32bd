"""One warm fit_dpar2 step inside an NVTX range "dp2_fit" (for ncu --nvtx
--nvtx-include dp2_fit/ launch lists without the data generation).

    python tools/profile_fit.py [--config c2] [--dtype f32] [--iters 32]
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
    ap.add_argument("--config", default="c2")
    ap.add_argument("--dtype", default="f32")
    ap.add_argument("--iters", type=int, default=32)
    a = ap.parse_args()
    cfg = synth.scaled(synth.CONFIGS[a.config], dtype=a.dtype)
    X, rows, _, _ = synth.generate_device(cfg, 0)
    t = dp.IrregularTensor.from_packed(X, rows, cfg.cols)
    opts = dp.SolverOptions(max_iters=a.iters, tol=0.0, seed=0)
    dp.fit_dpar2(t, cfg.rank, opts, output="device")  # warm-up
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_push("dp2_fit")
    dp.fit_dpar2(t, cfg.rank, opts, output="device")
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()


if __name__ == "__main__":
    main()
