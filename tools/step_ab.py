"""A/B of the bench step: device-event time over K steps with/without timings."""
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
t = dp.IrregularTensor.from_packed(X, rows, cfg.cols)
opts = dp.SolverOptions(max_iters=32, tol=0.0, seed=0)


def run(K, with_t, output="device"):
    for _ in range(3):
        dp.fit_dpar2(t, cfg.rank, opts, output=output, timings={} if with_t else None)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w0 = time.perf_counter()
    a.record()
    for _ in range(K):
        f, tr = dp.fit_dpar2(t, cfg.rank, opts, output=output, timings={} if with_t else None)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / K, (time.perf_counter() - w0) * 1e3 / K


for with_t in (False, True, False, True):
    print("timings" if with_t else "plain  ", "device-ms/step %.2f wall-ms/step %.2f" % run(5, with_t))
print("numpy output", "device-ms/step %.2f wall-ms/step %.2f" % run(5, False, "numpy"))
