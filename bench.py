"""DPar2 hot-path benchmark (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c2] [--dtype f32|f64] [--iters 32]

A *step* is one full ``fit_dpar2`` of the workload: stage-1 randomized SVD of
every slice, stage 2, 32 ALS iterations (tol = 0, so every iteration runs) and
the final Q assembly.  ``value`` is tensor entries (sum I_k * J) fitted per
second with the tensor resident in HBM; ``e2e`` is the same metric through the
public API from pinned HOST buffers (H2D of X and the sketch matrices, D2H of
H, V, W, Q and the trace inside the timed region).  ``--impl reference`` times
the reference algorithm on the host cores (the CPU oracle port, all threads)
on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

METRIC = "DPar2 fit throughput: stage-1 rSVD of all slices + stage 2 + 32 ALS iterations + Q"
UNIT = "entries/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2")
    ap.add_argument("--dtype", default="f32", choices=["f32", "f64"])
    ap.add_argument("--iters", type=int, default=32)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--cpu-sample", type=int, default=64, help="slices in the CPU-baseline sample")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--also-f64", action="store_true", help="add a c2 fp64 sub-measurement")
    ap.add_argument("--dist-path", action="store_true",
                    help="use the multi-rank (sharded stage 1 + NCCL) path even at world size 1")
    return ap.parse_args()


def workload(args):
    from paper_2203_12798_b200 import synth
    cfg = synth.scaled(synth.CONFIGS[args.config], dtype=args.dtype)
    return cfg


def workload_desc(cfg, iters):
    rows = cfg.rows
    return (f"{cfg.name}: K={cfg.num_slices}, J={cfg.cols}, I_k~{rows[0]}{tuple(rows[1:])}, R={cfg.rank}, "
            f"noise={cfg.noise}, {iters} ALS iters, tol=0, seed 0, storage {cfg.dtype}")


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.rows, self.proc, self.index = [], None, index

    def start(self):
        if os.environ.get("DP2_BENCH_CLOCK_MS") == "0":
            self.proc = None
            return
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", os.environ.get("DP2_BENCH_CLOCK_MS", "20")], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append((time.monotonic(), [x.strip() for x in line.split(",")]))

    def mark(self):
        """Start of the timed window (the sampler itself starts before warm-up so
        nvidia-smi's NVML start-up never lands inside the timed region)."""
        self.t0 = time.monotonic()

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        t1 = time.monotonic() + 0.05
        time.sleep(0.1)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:  # pragma: no cover
            self.proc.kill()
        t0 = getattr(self, "t0", 0.0)
        good = [r for t, r in self.rows if len(r) >= 8 and t0 <= t <= t1]
        if not good:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"], "samples": 0}
        sm = [float(r[0]) for r in good if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in good if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in good for i in range(4) if r[4 + i].lower().startswith("active")})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(good)}


# ---------------------------------------------------------------- reference arm
def cpu_fit_sample(xs, rank, iters, threads):
    """Reference algorithm (oracle port) on a host sample; returns seconds."""
    from oracle import dpar2_oracle as orc
    from threadpoolctl import threadpool_limits
    # slice-parallel compress with single-threaded BLAS (the reference's best
    # setting for compress, BASELINE.md setting A); the tiny ALS ops run serially
    with threadpool_limits(limits=1):
        t0 = time.perf_counter()
        comp = orc.compress(xs, rank, seed=0, threads=threads)
        o = orc.fit_dpar2(xs, rank, iters, 0.0, 0, comp=comp)
        dt = time.perf_counter() - t0
    return dt, o


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return  # rank 0 alone measures the host reference
    from paper_2203_12798_b200 import synth
    cfg = workload(args)
    S = min(args.cpu_sample, cfg.num_slices)
    threads = os.cpu_count() or 1
    xs = synth.generate(cfg, args.seed, slices=range(S), threads=threads)
    xs = [x.astype(np.float64) for x in xs]   # the reference's float64 container
    entries = sum(x.size for x in xs)
    for _ in range(args.warmup):
        cpu_fit_sample(xs, cfg.rank, args.iters, threads)
    times = [cpu_fit_sample(xs, cfg.rank, args.iters, threads)[0] for _ in range(args.steps)]
    t = float(np.mean(times))
    value = entries / t
    sample = f"first {S} slices of {cfg.name} ({entries} entries), full fit (compress + {args.iters} iters)"
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (BASELINE.json model)",
        "config": {"workload": workload_desc(cfg, args.iters), "sample_slices": S},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(line)


# ---------------------------------------------------------------- our arm
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    sharded = world > 1 or args.dist_path
    if sharded:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29531")
        os.environ.setdefault("RANK", str(rank))
        os.environ.setdefault("WORLD_SIZE", str(world))
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2203_12798_b200 as dp
    from paper_2203_12798_b200 import _lib, synth
    from paper_2203_12798_b200.solver import fit_dpar2

    cfg = workload(args)
    opts = dp.SolverOptions(max_iters=args.iters, tol=0.0, seed=args.seed)
    if sharded:
        from paper_2203_12798_b200.distributed import DistributedFit
        runner = DistributedFit(cfg, args.seed, rank, world)
        tensor = runner.tensor
        total_entries = runner.total_entries

        def step(timings=None):
            return runner.fit(cfg.rank, opts, timings=timings)
    else:
        X, rows, _, _ = synth.generate_device(cfg, args.seed)
        tensor = dp.IrregularTensor.from_packed(X, rows, cfg.cols)
        total_entries = int(sum(rows)) * cfg.cols

        def step(timings=None):
            return fit_dpar2(tensor, cfg.rank, opts, output="device", timings=timings)

    def barrier():
        if sharded:
            dist.barrier()
        torch.cuda.synchronize()

    clocks = ClockSampler(local)
    clocks.start()
    for _ in range(args.warmup):
        step()
    barrier()
    clocks.mark()
    _lib.lib().dp2_launch_count(1)
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    phase = []
    barrier()
    start.record()
    for _ in range(args.steps):
        f, tr = step()
    stop.record()
    barrier()
    launches = int(_lib.lib().dp2_launch_count(1))
    clk = clocks.stop()
    # per-phase breakdown from one extra, untimed step (its timing events
    # synchronise mid-fit, which the timed steps must not do)
    tm = {}
    f, tr = step(timings=tm)
    phase.append((tm, tr))
    barrier()
    ms = start.elapsed_time(stop) / args.steps
    if sharded:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = total_entries / (ms * 1e-3)

    # ---- roofline of the dominant kernel (the streaming sketch pass)
    tms = [p[0] for p in phase]
    s1 = float(np.mean([t["stage1_sketch1_ms"] for t in tms]))
    s2 = float(np.mean([t["stage1_sketch2_ms"] for t in tms]))
    sp = tms[0]["sp"]
    elem = 4 if cfg.dtype == "f32" else 8
    N_rows = runner.local_rows if sharded else int(tensor.row_off_host[-1])
    K_loc = tensor.num_slices
    x_bytes = N_rows * cfg.cols * elem
    # algorithmic bytes of one streaming pass (X once per pass
    # plus the per-slice B and the pass outputs).  The fp32 tensor-core pass
    # (J <= 512) reads B as a pre-tiled tf32 image and stores Y rows in fp32;
    # the fp64 DMMA / FFMA passes read B and write Y in fp64.
    tc = cfg.dtype == "f32" and cfg.cols <= 512 and sp <= 32
    jp = -(-cfg.cols // 128) * 128
    b_bytes = K_loc * (jp if tc else cfg.cols) * sp * (4 if tc else 8)
    part_bytes = int(tms[0].get("npieces", K_loc)) * cfg.cols * sp * 8  # fp64 per-piece partials
    alg_pass1 = x_bytes + b_bytes + part_bytes
    alg_pass2 = alg_pass1 + N_rows * sp * (4 if tc else 8)
    avg_launch_ms = (s1 + s2) / 2
    achieved = (alg_pass1 + alg_pass2) / 2 / (avg_launch_ms * 1e-3) / 1e9
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() \
        else {"hbm_gbs": 6650.0}
    peak = float(peaks.get("hbm_gbs", 6650.0))
    flops_launch = 4.0 * N_rows * cfg.cols * sp  # two skinny GEMMs per pass over the padded sketch width
    kernel_name = ("tcs::sketch_tc_kernel (stage-1 streaming pass: tcgen05 kind::tf32, TMA ring, X^T in TMEM)"
                   if tc else "sketch_kernel (stage-1 streaming pass, %s)" % ("fp64 DMMA m8n8k4" if cfg.dtype == "f64"
                                                                               else "fp32 FFMA"))
    traffic = None
    prof = ROOT / "profiles" / "sketch_traffic.json"
    if prof.exists():
        try:
            traffic = json.loads(prof.read_text()).get(f"{cfg.name}_{cfg.dtype}")
        except Exception:
            traffic = None
    tr0 = phase[-1][1]
    stage1_ms = float(np.mean([t["stage1_ms"] for t in tms]))
    stage2_ms = float(np.mean([t["stage2_ms"] for t in tms]))
    als_s = float(np.mean([sum(p[1].seconds) for p in phase]))
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None,
        "dtype": (f"{cfg.dtype} X; stage-1 sketch products tf32 on tcgen05 (fp32 accumulate, fp64 partials); "
                  "f64 factorizations, stage 2, ALS" if tc else
                  f"{cfg.dtype} X; f64 compute (stage-1 DMMA m8n8k4), f64 stage 2 / ALS"),
        "data": "synthetic (BASELINE.json model, generated on device)",
        "config": {"workload": workload_desc(cfg, args.iters), "entries": total_entries,
                   "parallelism": f"slice-sharded dp{world} (LPT)" if sharded else "single GPU",
                   "l2": "inputs larger than L2 (X %.1f GB >> 126 MB)" % (x_bytes / 1e9)},
        "gpu_launches": launches,
        "clocks": clk,
        "roofline": {"bound": "hbm", "kernel": kernel_name, "achieved": achieved,
                     "peak": peak, "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                     "alg_bytes_per_launch": (alg_pass1 + alg_pass2) / 2, "avg_launch_ms": avg_launch_ms,
                     "pass_frac": [alg_pass1 / (s1 * 1e-3) / 1e9 / peak, alg_pass2 / (s2 * 1e-3) / 1e9 / peak],
                     ("tf32_tflops_achieved" if tc else "fp64_tflops_achieved"):
                         flops_launch / (avg_launch_ms * 1e-3) / 1e12,
                     "traffic_source": "profiles/sketch_traffic.json (ncu dram__bytes_read+write per launch)",
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured)"},
        "breakdown_ms": {"stage1": stage1_ms, "sketch_pass1": s1, "sketch_pass2": s2,
                         "orth": float(np.mean([t["stage1_orth_ms"] for t in tms])),
                         "factor": float(np.mean([t["stage1_factor_ms"] for t in tms])),
                         "signs_A": float(np.mean([t["stage1_signs_ms"] for t in tms])),
                         "stage2": stage2_ms, "als_total": als_s * 1e3,
                         "als_per_iter_us": als_s * 1e6 / max(1, tr0.iterations),
                         "omega_host": float(np.mean([t["omega_host_s"] for t in tms])) * 1e3},
    }
    # ---- end-to-end through the public API from pinned host buffers
    if not args.no_e2e:
        line["e2e"] = e2e_sharded(runner, cfg, opts, args) if sharded else e2e(tensor, cfg, opts, args)
    if not args.no_cpu and rank == 0 and world == 1:
        line["cpu_baseline"] = cpu_baseline(tensor, cfg, args)
    if args.also_f64 and world == 1:
        line["f64"] = f64_sub(args, opts)
    if rank == 0:
        emit(line)
    if sharded:
        dist.destroy_process_group()


def e2e(tensor, cfg, opts, args):
    import torch
    import paper_2203_12798_b200 as dp
    host = torch.empty(tuple(tensor.X.shape), dtype=tensor.X.dtype, pin_memory=True)
    host.copy_(tensor.X)
    views = [host[a:b, :cfg.cols] for a, b in zip(tensor.row_off_host[:-1], tensor.row_off_host[1:])]
    R = cfg.rank
    steps = max(1, min(args.steps, 3))
    times = []
    for i in range(steps + 1):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        t = dp.IrregularTensor(views, dtype=cfg.dtype)
        f, tr = dp.fit_dpar2(t, R, opts)          # NumPy factors back on the host
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if i > 0:
            times.append(dt)
        del t
    N = int(tensor.row_off_host[-1])
    elem = 4 if cfg.dtype == "f32" else 8
    from paper_2203_12798_b200.linalg import padded_width
    sp = padded_width(cfg.rank + 10)
    h2d = N * cfg.cols * elem + tensor.num_slices * cfg.cols * sp * 8 + tensor.num_slices * 10 * cfg.rank * 8
    d2h = (N * R + R * R + cfg.cols * R + tensor.num_slices * R + args.iters * 2) * 8
    sec = float(np.mean(times))
    return {"value": N * cfg.cols / sec, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "seconds_per_step": sec, "steps": steps,
            "timing": "wall clock around IrregularTensor(pinned host slices) + fit_dpar2 -> NumPy, synced"}


def e2e_sharded(runner, cfg, opts, args):
    """End to end at N ranks: every rank builds an IrregularTensor over its own
    pinned host slices, fits jointly (stage-1 upload inside the timed region),
    and copies its factors (its Q slices, H, V, its W rows) back to NumPy.
    The step time is the max over ranks."""
    import torch
    import torch.distributed as dist
    import paper_2203_12798_b200 as dp
    tensor = runner.tensor
    host = torch.empty(tuple(tensor.X.shape), dtype=tensor.X.dtype, pin_memory=True)
    host.copy_(tensor.X)
    views = [host[a:b, :cfg.cols] for a, b in zip(tensor.row_off_host[:-1], tensor.row_off_host[1:])]
    R = cfg.rank
    steps = max(1, min(args.steps, 3))
    times = []
    for i in range(steps + 1):
        dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        t = dp.IrregularTensor(views, dtype=cfg.dtype)
        f, tr = runner.fit(R, opts, tensor=t)
        f.numpy()
        torch.cuda.synchronize()
        dt = torch.tensor([time.perf_counter() - t0], device="cuda")
        dist.all_reduce(dt, op=dist.ReduceOp.MAX)
        if i > 0:
            times.append(float(dt.item()))
        del t
    N = runner.local_rows
    K = runner.K
    elem = 4 if cfg.dtype == "f32" else 8
    from paper_2203_12798_b200.linalg import padded_width
    sp = padded_width(cfg.rank + 10)
    # per rank: its X slices + Omega for them; replicated stage-2 Omega
    h2d = N * cfg.cols * elem + len(runner.local_ids) * cfg.cols * sp * 8 + K * 10 * R * 8
    d2h = (N * R + R * R + cfg.cols * R + len(runner.local_ids) * R + args.iters * 2) * 8
    sec = float(np.mean(times))
    return {"value": runner.total_entries / sec, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "seconds_per_step": sec, "steps": steps, "per_rank_bytes": True,
            "timing": "wall clock, max over ranks, around IrregularTensor(pinned host shard) + joint fit -> NumPy"}


def cpu_baseline(tensor, cfg, args):
    S = min(args.cpu_sample, tensor.num_slices)
    xs_all = tensor.X[: int(tensor.row_off_host[S]), :cfg.cols].double().cpu().numpy()
    xs = [xs_all[a:b] for a, b in zip(tensor.row_off_host[:S], tensor.row_off_host[1:S + 1])]
    entries = sum(x.size for x in xs)
    threads = os.cpu_count() or 1
    dt, _ = cpu_fit_sample(xs, cfg.rank, args.iters, threads)
    return {"value": entries / dt, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"first {S} slices of the same device-generated {cfg.name} tensor ({entries} entries), "
                      f"full fit (compress + {args.iters} iters), {dt:.2f} s"}


def f64_sub(args, opts):
    import torch
    import paper_2203_12798_b200 as dp
    from paper_2203_12798_b200 import synth
    from paper_2203_12798_b200.solver import fit_dpar2
    cfg = synth.scaled(synth.CONFIGS[args.config], dtype="f64")
    X, rows, _, _ = synth.generate_device(cfg, args.seed)
    t = dp.IrregularTensor.from_packed(X, rows, cfg.cols)
    for _ in range(2):
        fit_dpar2(t, cfg.rank, opts, output="device")
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    tms = []
    a.record()
    for _ in range(args.steps):
        tm = {}
        fit_dpar2(t, cfg.rank, opts, output="device", timings=tm)
        tms.append(tm)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / args.steps
    entries = int(sum(rows)) * cfg.cols
    return {"value": entries / (ms * 1e-3), "ms_per_step": ms,
            "stage1_ms": float(np.mean([t["stage1_ms"] for t in tms])),
            "sketch_pass_ms": float(np.mean([(t["stage1_sketch1_ms"] + t["stage1_sketch2_ms"]) / 2 for t in tms]))}


_JSON_OUT = None


def emit(line):
    """The one JSON line, on the real stdout."""
    out = _JSON_OUT if _JSON_OUT is not None else sys.stdout
    print(json.dumps(line), file=out, flush=True)


if __name__ == "__main__":
    # stdout carries exactly one JSON line: anything else written to fd 1 by
    # libraries (NCCL's version banner, warnings) goes to stderr instead
    sys.stdout.flush()
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    main()
