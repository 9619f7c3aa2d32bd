"""DPar2 hot-path benchmark (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c2] [--dtype f64|f32] [--iters 32]

A *step* is one full ``fit_dpar2`` of the workload (BASELINE.json config c2
by default: K=1000, J=512, I_k ~ U{500..4000}, R=10, 32 ALS iterations,
tol=0, fp64): stage-1 randomized SVD of every slice, stage 2, the iterations
and the final Q.  ``value`` is tensor entries (sum I_k * J) fitted per second
with the tensor resident in HBM; ``e2e`` is the same metric through the public
API from pinned HOST slices (upload of X, the fit, NumPy factors back, all in
the timed region).

Both arms fit the SAME host tensor: ``synth.generate`` (BASELINE.json's
generative model, per-slice seeded) on all host cores.  ``--impl reference``
times the reference algorithm on the host (the CPU oracle port, pinned
bit-exact to the reference; BASELINE.md section 3 settings A and B), full
workload per step.  Our arm also checks its fit against that oracle on the
same tensor (``parity``) and reports the opt-in tf32 tensor-core mode as a
labelled sub-record (``tf32_mode``).
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
FP64_TOL = dict(fit=1e-6, factor=1e-5)   # BASELINE.json north star, fp64 mode
FP32_TOL = dict(fit=1e-3, factor=1e-3)   # fp32 / tf32 modes


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2")
    ap.add_argument("--dtype", default="f64", choices=["f32", "f64"])
    ap.add_argument("--iters", type=int, default=32)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true", help="skip the oracle run (parity + cpu_baseline)")
    ap.add_argument("--no-tf32", action="store_true", help="skip the tf32-mode sub-record")
    ap.add_argument("--dist-path", action="store_true",
                    help="use the multi-rank (sharded stage 1 + NCCL) path even at world size 1")
    return ap.parse_args()


def workload(args):
    from paper_2203_12798_b200 import synth
    return synth.scaled(synth.CONFIGS[args.config], dtype=args.dtype)


def workload_desc(cfg, iters):
    rows = cfg.rows
    return (f"{cfg.name}: K={cfg.num_slices}, J={cfg.cols}, I_k~{rows[0]}{tuple(rows[1:])}, R={cfg.rank}, "
            f"noise={cfg.noise}, {iters} ALS iters, tol=0, seed 0, storage {cfg.dtype}")


def host_tensor(cfg, seed, slices=None):
    """The benchmark tensor on the host (list of C-contiguous slices)."""
    from paper_2203_12798_b200 import synth
    return synth.generate(cfg, seed, slices=slices, threads=os.cpu_count() or 1)


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
                 "-lms", os.environ.get("DP2_BENCH_CLOCK_MS", "20")], stdout=subprocess.PIPE,
                stderr=subprocess.DEVNULL, text=True)
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


# ---------------------------------------------------------------- the reference algorithm on the host
def blas_info():
    try:
        from threadpoolctl import threadpool_info
        return [{k: d.get(k) for k in ("internal_api", "version", "num_threads", "threading_layer")}
                for d in threadpool_info()]
    except Exception as e:  # pragma: no cover
        return [repr(e)]


def oracle_fit(xs, rank, iters, setting):
    """One full fit of the reference algorithm (oracle port, P/solver.py:152-190)
    on host slices under a BASELINE.md section-3 thread setting:
      "A": slice threads = nproc, BLAS 1 thread (compress and iterations);
      "B": slice threads = 1, BLAS nproc threads;
      "best": A for the compression, B for the iterations (each phase's best).
    Returns (result dict, {compress_s, als_s, total_s})."""
    from threadpoolctl import threadpool_limits

    from oracle import dpar2_oracle as orc
    n = os.cpu_count() or 1
    comp_threads, comp_blas = (n, 1) if setting in ("A", "best") else (1, n)
    als_threads, als_blas = (n, 1) if setting == "A" else (1, n)
    t0 = time.perf_counter()
    with threadpool_limits(limits=comp_blas, user_api="blas"):
        comp = orc.compress(xs, rank, seed=0, threads=comp_threads)
    t1 = time.perf_counter()
    with threadpool_limits(limits=als_blas, user_api="blas"):
        o = orc.fit_dpar2(xs, rank, iters, 0.0, 0, comp=comp, als_threads=als_threads)
    t2 = time.perf_counter()
    return o, {"compress_s": t1 - t0, "als_s": t2 - t1, "total_s": t2 - t0}


def run_reference(args):
    if int(os.environ.get("RANK", "0")) != 0:
        return  # rank 0 alone measures the host reference
    cfg = workload(args)
    xs = [x.astype(np.float64) for x in host_tensor(cfg, args.seed)]  # the reference's float64 container
    entries = sum(x.size for x in xs)
    n = os.cpu_count() or 1
    # warm-up doubles as the A / B calibration (full fits), then the per-phase best
    calib = {}
    for i in range(max(args.warmup, 2)):
        setting = "A" if i == 0 else "B" if i == 1 else "best"
        calib.setdefault(setting, oracle_fit(xs, cfg.rank, args.iters, setting)[1])
    times, phases = [], []
    for _ in range(args.steps):
        _, tm = oracle_fit(xs, cfg.rank, args.iters, "best")
        times.append(tm["total_s"])
        phases.append(tm)
    t = float(np.mean(times))
    value = entries / t
    best = {k: float(np.mean([p[k] for p in phases])) for k in ("compress_s", "als_s", "total_s")}
    sample = (f"full {cfg.name} ({entries} entries) per step: compress + {args.iters} iterations; "
              f"setting 'best' = A (slice threads={n}, BLAS 1) for compress, B (slice threads 1, BLAS {n}) "
              f"for the iterations")
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (BASELINE.json model, host-generated, identical to our arm's tensor)",
        "config": {"workload": workload_desc(cfg, args.iters), "entries": entries, "same_config": True},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": n, "kind": "port", "sample": sample},
        "settings": {"A": calib.get("A"), "B": calib.get("B"), "best": best},
        "host": {"nproc": n, "numpy": np.__version__, "blas": blas_info()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(line)


def rel_signed(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    s = np.sign(np.sum(a * b, axis=0))
    s[s == 0] = 1.0
    return float(np.abs(a * s - b).max() / max(np.abs(b).max(), 1e-300))


def parity_vs_oracle(f, fit, o, tol):
    """Our fit vs the oracle's on the same tensor (north-star tolerances)."""
    from oracle import dpar2_oracle as orc  # noqa: F401  (checker only)
    errs = {k: rel_signed(np.asarray(getattr(f, k)), o[k]) for k in ("H", "V", "W")}
    U = np.concatenate([np.asarray(q) @ np.asarray(f.H) for q in f.Q])
    Uo = np.concatenate([q @ o["H"] for q in o["Q"]])
    errs["U"] = rel_signed(U, Uo)
    d_fit = abs(fit - o["fitness"])
    ok = d_fit <= tol["fit"] and max(errs.values()) <= tol["factor"]
    return {"fitness": fit, "fitness_oracle": o["fitness"], "abs_fitness_diff": d_fit,
            "factor_rel_err": errs, "tolerance": tol, "pass": bool(ok)}


# ---------------------------------------------------------------- our arm
def load_peaks():
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() \
        else {}
    cp = ROOT / "profiles" / "r2_compute_peaks.json"
    comp = json.loads(cp.read_text()) if cp.exists() else {}
    return float(peaks.get("hbm_gbs", 6544.3)), comp


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
    xs = None
    if sharded:
        from paper_2203_12798_b200.distributed import DistributedFit, shard_slices
        rows_all, _, _ = synth.shared_factors(cfg, args.seed)
        local_ids = shard_slices(rows_all, world)[0][rank]
        xs_local = host_tensor(cfg, args.seed, slices=local_ids)
        runner = DistributedFit(cfg, args.seed, rank, world, host_slices=xs_local)
        tensor = runner.tensor
        total_entries = runner.total_entries

        def step(timings=None):
            return runner.fit(cfg.rank, opts, timings=timings)
    else:
        xs = host_tensor(cfg, args.seed)
        up = dp.IrregularTensor(xs, dtype=cfg.dtype)   # chunked upload + host isfinite check
        up.wait_upload()
        tensor = dp.IrregularTensor.from_packed(up.X, up.row_counts, cfg.cols, dtype=cfg.dtype)  # HBM-resident
        total_entries = int(sum(x.shape[0] for x in xs)) * cfg.cols

        def step(timings=None):
            return fit_dpar2(tensor, cfg.rank, opts, output="device", timings=timings)

    def barrier():
        if sharded:
            dist.barrier()
        torch.cuda.synchronize()

    clocks = ClockSampler(local)
    clocks.start()
    for _ in range(max(args.warmup, 3)):
        step()
    barrier()
    clocks.mark()
    _lib.lib().dp2_launch_count(1)
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    start.record()
    for _ in range(args.steps):
        f, tr = step()
    stop.record()
    barrier()
    launches = int(_lib.lib().dp2_launch_count(1))
    clk = clocks.stop()
    ms = start.elapsed_time(stop) / args.steps
    multi = None
    if sharded:
        own = ms
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        multi = multi_gpu_record(runner, cfg, world, own)
    value = total_entries / (ms * 1e-3)
    # per-phase breakdown from one extra, untimed step (its timing events
    # synchronise mid-fit, which the timed steps must not do)
    tm = {}
    f, tr = step(timings=tm)
    barrier()

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": cfg.dtype,
        "data": "synthetic (BASELINE.json model, host-generated per-slice seeded; the reference arm fits the same "
                "tensor)",
        "config": {"workload": workload_desc(cfg, args.iters), "entries": total_entries,
                   "parallelism": f"slice-sharded dp{world} (LPT)" if sharded else "single GPU",
                   "l2": "inputs larger than L2 (X %.1f GB >> 126 MB)" % (total_entries * (
                       8 if cfg.dtype == "f64" else 4) / 1e9),
                   "precision": ("fp64 storage and arithmetic (DMMA / DFMA), the reference's precision"
                                 if cfg.dtype == "f64" else "fp32 storage, fp64 sketch products on the exactly "
                                 "upcast values (DMMA), fp64 factorizations / stage 2 / ALS")},
        "gpu_launches": launches,
        "clocks": clk,
    }
    if multi is not None:
        line["multi_gpu"] = multi
    line.update(roofline_fields(tm, tr, tensor, cfg, sharded, runner if sharded else None))
    if not args.no_e2e:
        line["e2e"] = e2e_sharded(runner, cfg, opts, args) if sharded else e2e(xs, cfg, opts, args)
    if rank == 0 and world == 1 and not sharded:
        f_np = f.numpy() if hasattr(f, "numpy") else f
        fit = dp.fitness(tensor, f, zero_pass=False)
        if not args.no_cpu:
            x64 = [x.astype(np.float64) for x in xs] if cfg.dtype != "f64" else xs
            o, otm = oracle_fit(x64, cfg.rank, args.iters, "best")
            from oracle import dpar2_oracle as orc
            o["fitness"] = orc.fitness(x64, o["H"], o["V"], o["W"], o["Q"])
            line["parity"] = parity_vs_oracle(f_np, fit, o, FP64_TOL if cfg.dtype == "f64" else FP32_TOL)
            n = os.cpu_count() or 1
            line["cpu_baseline"] = {
                "value": total_entries / otm["total_s"], "unit": UNIT, "cores": n, "kind": "port",
                "sample": f"the full {cfg.name} tensor of this run (fp64), one fit: compress {otm['compress_s']:.2f} s "
                          f"(slice threads {n}, BLAS 1) + {args.iters} iterations {otm['als_s']:.2f} s "
                          f"(slice threads 1, BLAS {n})"}
        if not args.no_tf32 and cfg.dtype == "f64":
            line["tf32_mode"] = tf32_sub(xs, cfg, opts, args, o if not args.no_cpu else None)
    if rank == 0:
        emit(line)
    if sharded:
        dist.destroy_process_group()


def multi_gpu_record(runner, cfg, world, own_ms):
    """N > 1: the ALS split the fit used, measured NCCL costs on this box
    (one R x R-partials allreduce and the M all-gather, CUDA events, after the
    timed region), NCCL time per iteration, and every rank's own step time
    (its share of the max-over-ranks clock)."""
    import torch
    import torch.distributed as dist
    from paper_2203_12798_b200 import distributed as D_
    R, J, K = cfg.rank, cfg.cols, cfg.num_slices
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    part = torch.zeros(2 * R * R, dtype=torch.float64, device="cuda")
    for _ in range(3):
        dist.all_reduce(part)
    dist.barrier()
    ev[0].record()
    for _ in range(32):
        dist.all_reduce(part)
    ev[1].record()
    width = max(len(s) for s in runner.shards) * R
    send = torch.zeros((J, width), dtype=torch.float64, device="cuda")
    buf = torch.empty((world * J, width), dtype=torch.float64, device="cuda")
    dist.all_gather_into_tensor(buf, send)
    dist.barrier()
    ev[2].record()
    dist.all_gather_into_tensor(buf, send)
    ev[3].record()
    torch.cuda.synchronize()
    ar_us = ev[0].elapsed_time(ev[1]) * 1e3 / 32
    ag_ms = ev[2].elapsed_time(ev[3])
    rank_ms = [torch.zeros(1, device="cuda") for _ in range(world)]
    dist.all_gather(rank_ms, torch.tensor([own_ms], device="cuda"))
    als = getattr(runner, "last_als", "replicated")
    return {"als": als, "als_policy": "distributed.als_policy (DESIGN.md 7)",
            "nccl_allreduce_us": ar_us, "nccl_ms_per_iter": (3 * ar_us * 1e-3) if als == "sharded" else 0.0,
            "m_allgather_ms": ag_ms, "m_allgather_bytes_per_rank": J * width * 8,
            "rank_ms_per_step": [float(x.item()) for x in rank_ms],
            "rank_rows": [int(x) for x in runner.loads]}


def roofline_fields(tm, tr, tensor, cfg, sharded, runner):
    """Roofline of the dominant kernel (the stage-1 streaming sketch pass) and
    of stage 1 as a whole, with measured peaks."""
    hbm, comp = load_peaks()
    sp = int(tm["sp"])
    s = cfg.rank + 10                     # algorithmic sketch width (R + min(10, .))
    w = 8 if cfg.dtype == "f64" else 4
    N = runner.local_rows if sharded else int(tensor.row_off_host[-1])
    K = tensor.num_slices
    J = cfg.cols
    p1, p2 = float(tm["stage1_sketch1_ms"]), float(tm["stage1_sketch2_ms"])
    avg_ms = (p1 + p2) / 2
    engine = tm.get("sketch_engine", "")
    flops_launch = 4.0 * N * J * s       # Y = X B and Z = X^T Y: 2 * 2 * N * J * s algorithmic flops
    bytes_launch = w * N * J + 8.0 * K * J * s  # X once + B (Omega or Q_Z)
    if cfg.dtype == "f64":
        peak = float(comp.get("dmma_f64_tflops", 36.9))
        kernel = {"bound": "tensor", "kernel": f"stage-1 streaming sketch pass ({engine or 'fp64 DMMA'})",
                  "achieved": flops_launch / (avg_ms * 1e-3) / 1e12, "peak": peak, "unit": "TFLOP/s",
                  "peak_source": "profiles/r2_compute_peaks.json dmma_f64_tflops (measured, DMMA.8x8x4 on all SMs)"}
    else:
        kernel = {"bound": "hbm", "kernel": f"stage-1 streaming sketch pass ({engine or 'fp32 FFMA'})",
                  "achieved": bytes_launch / (avg_ms * 1e-3) / 1e9, "peak": hbm, "unit": "GB/s",
                  "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured)"}
    kernel["frac"] = kernel["achieved"] / kernel["peak"]
    kernel["traffic"] = None
    prof = ROOT / "profiles" / "sketch_traffic.json"
    if prof.exists():
        try:
            kernel["traffic"] = json.loads(prof.read_text()).get(f"{cfg.name}_{cfg.dtype}")
        except Exception:
            pass
    kernel.update({"avg_launch_ms": avg_ms, "pass_ms": [p1, p2], "alg_flops_per_launch": flops_launch,
                   "alg_bytes_per_launch": bytes_launch, "hbm_gbs_achieved": bytes_launch / (avg_ms * 1e-3) / 1e9,
                   "units": f"one launch = one pass over all {N} rows x {J} columns (4 s flops and w bytes per "
                            f"entry, s = {s}, w = {w}; padded width sp = {sp})",
                   "traffic_source": "profiles/sketch_traffic.json (ncu dram__bytes_read+write per launch)"})
    # stage 1 as a whole: T_roof = max(B1 / HBM, F1 / P_peak)
    F1 = 8.0 * s * N * J
    B1 = w * N * J + w * (K * J * s + N * cfg.rank)
    p_peak = float(comp.get("dmma_f64_tflops", 36.9) if cfg.dtype == "f64" else comp.get("ffma_f32_tflops", 71.9))
    t_roof = max(B1 / (hbm * 1e9), F1 / (p_peak * 1e12)) * 1e3
    stage1_ms = float(tm["stage1_ms"])
    stage1 = {"T_roof_ms": t_roof, "stage1_ms": stage1_ms, "achieved": t_roof / stage1_ms,
              "F1_flops": F1, "B1_bytes": B1, "peak_tflops": p_peak, "hbm_gbs": hbm,
              "bound": "fp64 tensor (DMMA)" if cfg.dtype == "f64" and F1 / (p_peak * 1e12) > B1 / (hbm * 1e9)
              else ("FP32 FFMA" if F1 / (p_peak * 1e12) > B1 / (hbm * 1e9) else "hbm"),
              "passes_over_X": 2}
    als_s = float(sum(tr.seconds))
    breakdown = {"stage1": stage1_ms, "sketch_pass1": p1, "sketch_pass2": p2,
                 "orth": float(tm["stage1_orth_ms"]), "factor": float(tm["stage1_factor_ms"]),
                 "signs_A": float(tm["stage1_signs_ms"]), "stage2": float(tm["stage2_ms"]),
                 "als_total": als_s * 1e3, "als_per_iter_us": als_s * 1e6 / max(1, tr.iterations),
                 "omega_host": float(tm.get("omega_host_s", 0.0)) * 1e3}
    return {"roofline": kernel, "stage1_roofline": stage1, "breakdown_ms": breakdown}


def e2e(xs, cfg, opts, args):
    """Pinned host slices -> IrregularTensor (upload inside the timed region)
    -> fit_dpar2 -> NumPy factors, wall clock, synchronised."""
    import torch
    import paper_2203_12798_b200 as dp
    tdt = torch.float64 if cfg.dtype == "f64" else torch.float32
    N = sum(x.shape[0] for x in xs)
    host = torch.empty((N, cfg.cols), dtype=tdt, pin_memory=True)
    off, views = 0, []
    for x in xs:
        host[off:off + x.shape[0]] = torch.from_numpy(x)
        views.append(host[off:off + x.shape[0]])
        off += x.shape[0]
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
    K = len(xs)
    elem = 8 if cfg.dtype == "f64" else 4
    # copied per step: X, the row counts (the sketch matrices are generated on the device)
    h2d = N * cfg.cols * elem + (K + 1) * 8
    d2h = (N * R + R * R + cfg.cols * R + K * R + 2 * args.iters) * 8
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
    elem = 4 if cfg.dtype == "f32" else 8
    h2d = N * cfg.cols * elem + (len(runner.local_ids) + 1) * 8
    d2h = (N * R + R * R + cfg.cols * R + len(runner.local_ids) * R + args.iters * 2) * 8
    sec = float(np.mean(times))
    return {"value": runner.total_entries / sec, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "seconds_per_step": sec, "steps": steps, "per_rank_bytes": True,
            "timing": "wall clock, max over ranks, around IrregularTensor(pinned host shard) + joint fit -> NumPy"}


def tf32_sub(xs, cfg, opts, args, o64):
    """The opt-in tf32 mode (fp32 storage, single-pass tf32 sketch products on
    the tcgen05 tensor cores) on the same tensor cast to fp32: step time,
    its HBM roofline, and parity against the oracle on the upcast values."""
    import torch
    import paper_2203_12798_b200 as dp
    from paper_2203_12798_b200.solver import fit_dpar2
    x32 = [x.astype(np.float32) for x in xs]
    t = dp.IrregularTensor(x32, dtype="f32")
    prev = dp.set_fp32_products("tf32")
    try:
        for _ in range(3):
            fit_dpar2(t, cfg.rank, opts, output="device")
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(args.steps):
            f, tr = fit_dpar2(t, cfg.rank, opts, output="device")
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / args.steps
        tm = {}
        f, tr = fit_dpar2(t, cfg.rank, opts, output="device", timings=tm)
    finally:
        dp.set_fp32_products(prev)
    N = sum(x.shape[0] for x in xs)
    entries = N * cfg.cols
    hbm, _ = load_peaks()
    K, J, s = len(xs), cfg.cols, cfg.rank + 10
    avg = (tm["stage1_sketch1_ms"] + tm["stage1_sketch2_ms"]) / 2
    alg = 4.0 * N * J + 8.0 * K * J * s
    out = {"label": "opt-in tf32 mode: fp32 storage, single-pass tf32 sketch products on tcgen05 "
                    "(fp32 accumulate, fp64 partials), fp64 factorizations / stage 2 / ALS",
           "value": entries / (ms * 1e-3), "unit": UNIT, "ms_per_step": ms,
           "stage1_ms": tm["stage1_ms"], "sketch_pass_ms": [tm["stage1_sketch1_ms"], tm["stage1_sketch2_ms"]],
           "roofline": {"bound": "hbm", "achieved": alg / (avg * 1e-3) / 1e9, "peak": hbm, "unit": "GB/s",
                        "frac": alg / (avg * 1e-3) / 1e9 / hbm,
                        "kernel": "tcs::sketch_tc_kernel (tcgen05 kind::tf32, TMA ring, X^T in TMEM)"}}
    if o64 is not None:
        from oracle import dpar2_oracle as orc
        x64 = [x.astype(np.float64) for x in x32]
        o, _ = oracle_fit(x64, cfg.rank, args.iters, "best")
        o["fitness"] = orc.fitness(x64, o["H"], o["V"], o["W"], o["Q"])
        fit = dp.fitness(t, f, zero_pass=False)
        out["parity"] = parity_vs_oracle(f.numpy(), fit, o, FP32_TOL)
    return out


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
