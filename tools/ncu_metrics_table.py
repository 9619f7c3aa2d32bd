"""Per-kernel table from an ncu ``--metrics ... --csv`` launch list (one row per
kernel x metric): mean of each metric per kernel name.

    python tools/ncu_metrics_table.py launches.csv
"""
import csv
import sys
from collections import defaultdict


def main(path):
    rows = list(csv.reader(l for l in open(path) if not l.startswith("==")))
    h = rows[0]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    d = defaultdict(lambda: defaultdict(list))
    for r in rows[1:]:
        if len(r) > vi:
            d[r[ki].split("(")[0]][r[mi]].append(float(r[vi].replace(",", "")))
    metrics = sorted({m for v in d.values() for m in v})
    print("kernel".ljust(40) + "".join(m[:28].rjust(30) for m in metrics) + "  n")
    for k, v in d.items():
        print(k[:40].ljust(40) + "".join(
            (f"{sum(v[m]) / len(v[m]):.1f}" if v[m] else "-").rjust(30) for m in metrics) + f"  {len(v[metrics[0]])}")


if __name__ == "__main__":
    main(sys.argv[1])
