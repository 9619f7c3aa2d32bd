"""Wall-clock phases of one warm fit_dpar2 step (synchronised), c2 fp32."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2203_12798_b200 as dp  # noqa: E402
import importlib  # noqa: E402
from paper_2203_12798_b200 import synth  # noqa: E402
cmod = importlib.import_module("paper_2203_12798_b200.compress")
solver = importlib.import_module("paper_2203_12798_b200.solver")
from paper_2203_12798_b200.factors import initial_factors  # noqa: E402
from paper_2203_12798_b200.linalg import RsvdParams  # noqa: E402

cfg = synth.scaled(synth.CONFIGS["c2"], dtype="f32")
X, rows, _, _ = synth.generate_device(cfg, 0)
t = dp.IrregularTensor.from_packed(X, rows, cfg.cols)
R = cfg.rank
opts = dp.SolverOptions(max_iters=32, tol=0.0, seed=0)
for rep in range(4):
    tm = {}
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    comp = cmod.compress(t, R, rsvd=RsvdParams(rank=R, seed=0), timings=tm)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    h, v, w = initial_factors(t.num_cols, t.num_slices, R, 0)
    t2 = time.perf_counter()
    H, V, W, polar, tr, secs = solver.run_als(comp, h, v, w, 32, 0.0, True, use_graph=True)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    Q = solver.assemble_q(t, comp, polar)
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    f, trc = dp.fit_dpar2(t, R, opts, output="device")
    torch.cuda.synchronize()
    t5 = time.perf_counter()
    print(f"compress {1e3*(t1-t0):.2f} (stage1 {tm.get('stage1_ms',0):.2f} stage2 {tm.get('stage2_ms',0):.2f} "
          f"omega {1e3*tm.get('omega_host_s',0):.2f}) init {1e3*(t2-t1):.2f} als {1e3*(t3-t2):.2f} "
          f"(iters {1e3*sum(secs):.2f}) q {1e3*(t4-t3):.2f} | fit_dpar2 {1e3*(t5-t4):.2f} ms")
