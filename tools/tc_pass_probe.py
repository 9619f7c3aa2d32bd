"""Time the fp32-storage streaming pass alone (dp2_stream_pass, pass-1 form:
Z partials only) on a device-drawn BASELINE tensor, per product engine:

    python tools/tc_pass_probe.py [--config c5shard|c2|c3] [--engine 0] [--reps 5]

DP2_TC_DEBUG=1 adds the tensor-core pass's per-role barrier-wait means.
"""
import argparse
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2203_12798_b200 as dp  # noqa: E402
from paper_2203_12798_b200 import _lib, synth  # noqa: E402
from paper_2203_12798_b200.compress import nseg_for  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5shard")
    ap.add_argument("--engine", type=int, default=0)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--sp", type=int, default=24)
    a = ap.parse_args()
    ids = None
    if a.config == "c5shard":
        cfg = synth.CONFIGS["c5"]
        from paper_2203_12798_b200.distributed import shard_slices
        rows, _, _ = synth.shared_factors(cfg, 0)
        ids = shard_slices(rows, 8)[0][0]
    else:
        cfg = synth.CONFIGS[a.config]
    cfg = synth.scaled(cfg, dtype="f32") if cfg.dtype != "f32" else cfg
    X, rows, _, _ = synth.generate_device(cfg, 0, slices=ids)
    t = dp.IrregularTensor.from_packed(X, rows, cfg.cols, dtype="f32")
    nseg = nseg_for(t)
    st, keep = t.store(nseg)
    n = len(t.plan_host(nseg)["piece_slice"])
    K, J, sp = len(rows), cfg.cols, a.sp
    B = torch.randn(K, J, sp, dtype=torch.float64, device="cuda")
    out = torch.empty(n, J, sp, dtype=torch.float64, device="cuda")
    status = dp.tensor.new_status(X.device)
    prev = _lib.lib().dp2_set_sketch_engine(a.engine)
    uses_tc = _lib.lib().dp2_sketch_uses_tc(C.byref(st), sp)
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)

    def run():
        _lib.check(_lib.lib().dp2_stream_pass(C.byref(st), C.c_void_p(B.data_ptr()), sp, C.c_void_p(out.data_ptr()),
                                              None, None, None, C.c_void_p(status.data_ptr()), s), "stream_pass")
    run()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    for _ in range(a.reps):
        run()
    ev[1].record()
    torch.cuda.synchronize()
    _lib.lib().dp2_set_sketch_engine(prev)
    ms = ev[0].elapsed_time(ev[1]) / a.reps
    entries = int(sum(rows)) * J
    print(f"{a.config}: K={K} J={J} entries={entries:.3e} nseg={nseg} pieces={n} engine={a.engine} tc={uses_tc} "
          f"pass {ms:.3f} ms = {entries * 4 / ms / 1e6:.0f} GB/s (incl. B image)")


if __name__ == "__main__":
    main()
