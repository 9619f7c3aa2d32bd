"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list."""
import collections
import csv
import sys


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hi]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0][:72]
        agg[name][0] += 1
        agg[name][1] += float(r[vi].replace(",", ""))
    total = sum(v[1] for v in agg.values())
    print(f"{'total_ms':>9} {'share':>6} {'launches':>8} {'us/launch':>10}  kernel")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        print(f"{t / 1e6:9.3f} {100 * t / total:5.1f}% {n:8d} {t / n / 1e3:10.1f}  {k}")
    print(f"# total {total / 1e6:.3f} ms")


if __name__ == "__main__":
    main(sys.argv[1])
