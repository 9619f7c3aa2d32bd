"""Device idle gaps inside consecutive warm fit_dpar2 steps (c2, --dtype f32 or f64): kernel
intervals from torch.profiler (CUPTI), gaps > 5 us listed with the kernels
around them -- where the host, not the GPU, sets the pace.

    python tools/gap_probe.py [--steps 3]
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_2203_12798_b200 as dp  # noqa: E402
from paper_2203_12798_b200 import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--stack", action="store_true", help="list the host calls inside the largest gap")
    ap.add_argument("--dtype", default="f32")
    ap.add_argument("--timeline", action="store_true", help="print the device events of the last step with the idle gap before each")
    a = ap.parse_args()
    cfg = synth.scaled(synth.CONFIGS["c2"], dtype=a.dtype)
    X, rows, _, _ = synth.generate_device(cfg, 0)
    t = dp.IrregularTensor.from_packed(X, rows, cfg.cols)
    opts = dp.SolverOptions(max_iters=32, tol=0.0, seed=0)
    for _ in range(3):
        dp.fit_dpar2(t, cfg.rank, opts, output="device")
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU], with_stack=a.stack) as prof:
        for _ in range(a.steps):
            dp.fit_dpar2(t, cfg.rank, opts, output="device")
        torch.cuda.synchronize()
    ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    ev.sort(key=lambda e: e.time_range.start)
    span = ev[-1].time_range.end - ev[0].time_range.start
    busy = 0.0
    gaps = []
    end = ev[0].time_range.start
    prev = None
    for e in ev:
        s0, s1 = e.time_range.start, e.time_range.end
        if s0 > end:
            gaps.append((s0 - end, prev, e.name))
        busy += max(0.0, s1 - max(s0, end))
        end = max(end, s1)
        prev = e.name
    print(f"span {span / a.steps:.1f} us/step, busy {busy / a.steps:.1f} us/step, "
          f"idle {(span - busy) / a.steps:.1f} us/step over {a.steps} steps")
    agg = {}
    for g, p, n in gaps:
        key = (str(p)[:50], str(n)[:50])
        agg[key] = agg.get(key, 0.0) + g
    for (p, n), g in sorted(agg.items(), key=lambda kv: -kv[1])[:25]:
        if g / a.steps > 5:
            print(f"{g / a.steps:9.1f} us/step  after {p:50s} before {n}")
    if a.timeline:
        n_per = len(ev) // a.steps
        last = ev[-n_per:]
        t0 = last[0].time_range.start
        prev_end = t0
        for e in last:
            gap = e.time_range.start - prev_end
            print(f"{e.time_range.start - t0:9.1f} +{max(0.0, gap):7.1f} {e.time_range.end - e.time_range.start:8.1f}  {e.name[:70]}")
            prev_end = max(prev_end, e.time_range.end)
    if a.stack:  # host events overlapping the largest single gap
        big = max(range(len(ev) - 1), key=lambda i: ev[i + 1].time_range.start - ev[i].time_range.end)
        g0, g1 = ev[big].time_range.end, ev[big + 1].time_range.start
        cpu = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CPU
               and e.time_range.end > g0 - 50 and e.time_range.start < g1]
        cpu.sort(key=lambda e: e.time_range.start)
        print(f"largest gap {g1 - g0:.1f} us; host events in it:")
        for e in cpu[:120]:
            print(f"  {e.time_range.start - g0:9.1f} {e.time_range.end - e.time_range.start:8.1f}  {e.name[:90]}")


if __name__ == "__main__":
    main()
