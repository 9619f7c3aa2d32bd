"""Per-phase device time of the persistent ALS loop (c2 fp32 workload).

Runs fit-equivalent ALS with DP2_ALS_STAMPS=1, reads CTA 0's globaltimer
stamps from the ALS workspace (dp2_als_stamp_offset) and prints the median
duration of each phase over the warm iterations:
  rotate | bar1 | red_h | pinv_h | rest_h | mode2 | bar2 | red_v | rest_v | mode3 | bar3+e
"""
import importlib
import os
import sys
from pathlib import Path

os.environ["DP2_ALS_STAMPS"] = "1"
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2203_12798_b200 as dp  # noqa: E402
from paper_2203_12798_b200 import _lib, synth  # noqa: E402
from paper_2203_12798_b200.factors import initial_factors  # noqa: E402
from paper_2203_12798_b200.linalg import RsvdParams  # noqa: E402

solver = importlib.import_module("paper_2203_12798_b200.solver")
cm = importlib.import_module("paper_2203_12798_b200.compress")
name = sys.argv[1] if len(sys.argv) > 1 else "c2"
cfg = synth.scaled(synth.CONFIGS[name], dtype="f32")
X, rows, _, _ = synth.generate_device(cfg, 0)
t = dp.IrregularTensor.from_packed(X, rows, cfg.cols)
R = cfg.rank
comp = cm.compress(t, R, rsvd=RsvdParams(rank=R, seed=0))
captured = {}
orig = solver.workspace


def grab(nbytes, dev):
    captured["ws"] = orig(nbytes, dev).zero_()
    return captured["ws"]


solver.workspace = grab
names = ["rotate", "bar1", "red_h", "pinv_h", "rest_h", "mode2", "bar2", "red_v", "rest_v", "mode3", "bar3+e"]
order = [0, 1, 2, 8, 9, 3, 4, 5, 10, 6, 7]  # stamp slots in time order
for rep in range(3):
    h, v, w = initial_factors(t.num_cols, t.num_slices, R, 0)
    H, V, W, polar, tr, secs = solver.run_als(comp, h, v, w, 32, 0.0, True, use_graph=False)
    off = _lib.lib().dp2_als_stamp_offset(t.num_slices, t.num_cols, R)
    raw = captured["ws"][off:off + 64 * 16 * 8].view(torch.int64).cpu().numpy().reshape(64, 16)[:len(tr)]
    if rep == 2 and os.environ.get("DP2_ALS_DBGQ"):
        q = np.median(raw[1:, 11:16], axis=0)
        print("rotate per-warp maxima (cycles): setup %d jacobi %d epilogue %d sweeps %d total %d" % tuple(q))
    st = raw[:, order]
    nxt = np.concatenate([st[1:, 0], [st[-1, -1] + int(np.median(np.diff(st[:, 0])) - np.median(st[:, -1] - st[:, 0]))]])
    d = np.diff(np.concatenate([st, nxt[:, None]], axis=1), axis=1) * 1e-3
    med = np.median(d[1:], axis=0)
    print("iter us %.1f | " % med.sum() + " ".join(f"{n} {m:.1f}" for n, m in zip(names, med)),
          "| first iter %.1f" % d[0].sum())
