"""Per-config timings on one B200 for the BASELINE.json configs other than the
bench headline (c2): c1 (fp64, full), c3 (fp32, full: K=10 000, J=256,
lognormal I_k, 4.6e9 entries), and the per-GPU share of c5 at 8 GPUs (fp32,
K=2 500 of the 20 000 slices, J=1000: the LPT shard one rank fits, ~1e10
entries / 40 GB).  Tensors are drawn on the device (synth.generate_device:
same shapes and row counts as the host generator; parity on these configs is
covered by tests/test_gpu_scale_parity.py on K-subsets).

    python tools/config_sweep.py [--configs c1,c3,c5shard] [--out profiles/r2_config_sweep.json]
"""
import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2203_12798_b200 as dp  # noqa: E402
from paper_2203_12798_b200 import synth  # noqa: E402


def workload(name):
    if name == "c1":
        return synth.CONFIGS["c1"], None
    if name == "c3":
        return synth.CONFIGS["c3"], None
    if name == "c5shard":  # rank 0's LPT shard of c5 at 8 GPUs
        cfg = synth.CONFIGS["c5"]
        from paper_2203_12798_b200.distributed import shard_slices
        rows, _, _ = synth.shared_factors(cfg, 0)
        return cfg, shard_slices(rows, 8)[0][0]
    raise ValueError(name)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c1,c3,c5shard")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--out", default=None)
    ap.add_argument("--fp32-products", default=None, choices=["fp64", "fp32", "tf32"],
                    help="products of fp32-storage tensors (default: the library default, fp64 DMMA)")
    a = ap.parse_args()
    if a.fp32_products:
        dp.set_fp32_products(a.fp32_products)
    out = {}
    for name in a.configs.split(","):
        cfg, ids = workload(name)
        t0 = time.perf_counter()
        X, rows, _, _ = synth.generate_device(cfg, 0, slices=ids)
        t = dp.IrregularTensor.from_packed(X, rows, cfg.cols, dtype=cfg.dtype)
        gen_s = time.perf_counter() - t0
        opts = dp.SolverOptions(max_iters=32, tol=0.0, seed=0)
        dp.fit_dpar2(t, cfg.rank, opts, output="device")
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record()
        for _ in range(a.reps):
            dp.fit_dpar2(t, cfg.rank, opts, output="device")
        ev[1].record()
        torch.cuda.synchronize()
        ms = ev[0].elapsed_time(ev[1]) / a.reps
        tm = {}
        f, tr = dp.fit_dpar2(t, cfg.rank, opts, output="device", timings=tm)
        entries = int(sum(rows)) * cfg.cols
        rec = dict(workload=f"{name}: K={len(rows)}, J={cfg.cols}, storage {cfg.dtype}, R={cfg.rank}, 32 iterations",
                   entries=entries, ms_per_fit=ms, entries_per_s=entries / (ms * 1e-3),
                   stage1_ms=tm["stage1_ms"], sketch_pass_ms=[tm["stage1_sketch1_ms"], tm["stage1_sketch2_ms"]],
                   stage2_ms=tm["stage2_ms"], als_per_iter_us=float(np.mean(tr.seconds)) * 1e6,
                   fitness=dp.fitness(t, f), generation_s=gen_s,
                   fp32_products=a.fp32_products or "default")
        w = 8 if cfg.dtype == "f64" else 4
        rec["pass_hbm_gbs"] = [entries * w / (ms_ * 1e-3) / 1e9 for ms_ in rec["sketch_pass_ms"]]
        out[name] = rec
        print(name, json.dumps(rec), flush=True)
        del t, X, f
        torch.cuda.empty_cache()
    if a.out:
        Path(a.out).write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
