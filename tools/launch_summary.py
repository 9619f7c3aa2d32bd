"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list.

    python tools/launch_summary.py launches.csv [--last-from KERNEL] [--metric NAME]

--last-from keeps only the launches from the last launch of KERNEL onward
(e.g. omega_kernel: the last fit of a bench run, without data generation).
"""
import argparse
import collections
import csv


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("path")
    ap.add_argument("--last-from", default=None)
    ap.add_argument("--metric", default="gpu__time_duration.sum")
    ap.add_argument("--top", type=int, default=40)
    a = ap.parse_args()
    rows = list(csv.reader(l for l in open(a.path) if not l.startswith("==")))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hi]
    ki, vi, mi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    recs = [(r[ki], float(r[vi].replace(",", ""))) for r in rows[hi + 1:] if len(r) > vi and r[mi] == a.metric]
    if a.last_from:
        starts = [i for i, (n, _) in enumerate(recs) if a.last_from in n]
        if starts:
            recs = recs[starts[-1]:]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for name, v in recs:
        key = name.split("(")[0][:72]
        agg[key][0] += 1
        agg[key][1] += v
    total = sum(v[1] for v in agg.values())
    print(f"{'total_ms':>9} {'share':>6} {'launches':>8} {'us/launch':>10}  kernel")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:a.top]:
        print(f"{t / 1e6:9.3f} {100 * t / total:5.1f}% {n:8d} {t / n / 1e3:10.1f}  {k}")
    print(f"# total {total / 1e6:.3f} ms over {sum(v[0] for v in agg.values())} launches")


if __name__ == "__main__":
    main()
