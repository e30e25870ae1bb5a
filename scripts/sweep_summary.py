"""Summarise scripts/sweep.py's cfg5 CSV: per dtype a table of speedup over cuBLAS (step time) per
size (rows) and N:M / L (columns), '*' where the paper-derived target 0.7 M/N is met, and the kernel
roofline fraction range.  Usage: sweep_summary.py sweep.csv"""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.DictReader(l for l in open(sys.argv[1]) if not l.startswith("#"))]
by = defaultdict(dict)
cols = defaultdict(set)
for r in rows:
    key = f'{r["N"]}:{r["M"]} L{r["L"]}'
    by[(r["dtype"], int(r["m"]))][key] = r
    cols[r["dtype"]].add((-int(r["N"]), int(r["L"]), key))
for dt in sorted({d for d, _ in by}):
    keys = [k for _, _, k in sorted(cols[dt])]
    print(f"== {dt}: speedup vs cuBLAS dense of the same dtype (step), * = meets 0.7 M/N")
    print("size   " + " ".join(f"{k:>13s}" for k in keys))
    hits = tot = 0
    fr = []
    for (d, s) in sorted(k for k in by if k[0] == dt):
        cells = []
        for k in keys:
            r = by[(d, s)].get(k)
            if not r:
                cells.append(f"{'-':>13s}")
                continue
            sp, tg = float(r["speedup_vs_cublas"]), float(r["target"])
            hit = sp >= tg
            hits += hit
            tot += 1
            fr.append(float(r["roofline_frac"]))
            cells.append(f"{sp:12.2f}{'*' if hit else ' '}")
        print(f"{s:<6d} " + " ".join(cells))
    print(f"   targets met: {hits} / {tot}; kernel roofline fraction {min(fr):.3f} .. {max(fr):.3f}\n")
