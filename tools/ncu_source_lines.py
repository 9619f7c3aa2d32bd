"""Aggregate an ncu ``--page source --print-source cuda,sass --csv`` export by
CUDA source line: instructions executed and stall samples per line.

    ncu -i rep --page source --csv --kernel-name regex:K --print-source cuda,sass > k.csv
    python tools/ncu_source_lines.py k.csv [top]
"""
import csv
import sys
from collections import defaultdict


def main(path, top=30):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if r[:2] == ["Line No", "Source"])
    h = rows[hdr]
    ie, ss = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    stall_cols = [i for i, n in enumerate(h) if n.startswith("stall_") and "Not Issued" not in n]
    inst, samp, src = defaultdict(float), defaultdict(float), {}
    stalls = defaultdict(lambda: defaultdict(float))
    line, fname = None, rows[0][1].rsplit("/", 1)[-1] if rows[0][:1] == ["File Path"] else ""
    for r in rows[hdr + 1:]:
        if r[:1] == ["File Path"]:
            fname, line = r[1].rsplit("/", 1)[-1], None
            continue
        if len(r) < 3:
            continue
        if r[0]:
            line = (fname, int(r[0])) if r[0].isdigit() else None
            src[line] = r[1]
        if line is None or len(r) <= ie or not r[ie]:
            continue
        try:
            inst[line] += float(r[ie])
            samp[line] += float(r[ss] or 0)
            for c in stall_cols:
                stalls[line][h[c]] += float(r[c] or 0)
        except ValueError:
            pass
    tot_i, tot_s = sum(inst.values()), sum(samp.values())
    print(f"total inst {tot_i:.0f}  samples {tot_s:.0f}")
    for ln in sorted(samp, key=lambda k: -samp[k])[:top]:
        top_st = sorted(stalls[ln].items(), key=lambda kv: -kv[1])[:2]
        st = " ".join(f"{k[6:]}={v:.0f}" for k, v in top_st if v)
        print(f"{ln[0][:14]:>14s}:{ln[1]:<5d} samp {samp[ln]:5.0f} ({100 * samp[ln] / max(tot_s, 1):4.1f}%) inst {inst[ln]:8.0f}  {st:30s} "
              f"{src.get(ln, '').strip()[:70]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
