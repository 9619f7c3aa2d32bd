"""Phases of the e2e step (host slices -> fit -> NumPy), c2 fp32."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2203_12798_b200 as dp  # noqa: E402
from paper_2203_12798_b200 import synth  # noqa: E402

cfg = synth.scaled(synth.CONFIGS["c2"], dtype="f32")
X, rows, _, _ = synth.generate_device(cfg, 0)
host = torch.empty(tuple(X.shape), dtype=X.dtype, pin_memory=True)
host.copy_(X)
off = np.concatenate([[0], np.cumsum(rows)])
views = [host[a:b, :cfg.cols] for a, b in zip(off[:-1], off[1:])]
dev_buf = torch.empty_like(X)
opts = dp.SolverOptions(max_iters=32, tol=0.0, seed=0)
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dev_buf.copy_(host, non_blocking=True)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    t = dp.IrregularTensor(views, dtype="f32")  # returns with the upload still in flight
    t2 = time.perf_counter()
    f, tr = dp.fit_dpar2(t, cfg.rank, opts, output="device")
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    fn = f.numpy()
    t4 = time.perf_counter()
    print(f"one-copy H2D {1e3*(t1-t0):.1f} ms ({X.numel()*4/(t1-t0)/1e9:.1f} GB/s) | IrregularTensor(views) "
          f"{1e3*(t2-t1):.1f} | fit(device) {1e3*(t3-t2):.1f} | factors->numpy {1e3*(t4-t3):.1f}")
