"""Text summary of one kernel in an ``ncu --set full`` report (.ncu-rep): the
metrics a roofline argument needs (duration, DRAM bytes and throughput, pipe
utilisation, issue activity, warp-stall breakdown, shared-memory conflicts).

    python tools/ncu_full_summary.py report.ncu-rep [--title T] > profiles/<name>.txt
"""
import argparse
import csv
import io
import subprocess

KEYS = [
    ("gpu__time_duration.sum", "duration (ms)"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__bytes_read.sum.per_second", "DRAM read rate"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput % of peak"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe active % (DMMA/HMMA/UTC)"),
    ("sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active", "DMMA subpipe %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 (DFMA) pipe active %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe active %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active % (occupancy)"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "smem load bank conflicts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "smem store bank conflicts"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
    ("launch__registers_per_thread", "registers / thread"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem / CTA"),
    ("launch__grid_size", "grid size"),
    ("launch__block_size", "block size"),
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--title", default="")
    a = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", a.rep, "--page", "raw", "--csv"], capture_output=True).stdout
    rows = list(csv.reader(io.StringIO(raw.decode("utf-8", "replace"))))
    h, units, v = rows[0], rows[1], rows[2]
    col = {n: i for i, n in enumerate(h)}
    print(f"# {a.title or a.rep}")
    print(f"kernel: {v[col['Kernel Name']] if 'Kernel Name' in col else '?'}")
    for k, label in KEYS:
        if k in col:
            print(f"{label:42s} {v[col[k]]:>18s} {units[col[k]]}")
    stalls = [(n, float(v[i] or 0)) for n, i in col.items()
              if n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("_per_issue_active.ratio")]
    stalls.sort(key=lambda x: -x[1])
    print("warp stalls per issued instruction (top):")
    for n, x in stalls[:10]:
        print(f"  {n.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''):28s}"
              f" {x:8.3f}")


if __name__ == "__main__":
    main()
