"""Summarise scripts/llama_dataset.py's CSV: per dtype and sparsity, mean / min / max speedup over
cuBLAS and the share of the 100 points that reach the paper-derived target 0.7 M/N."""
import csv, sys, statistics
from collections import defaultdict
rows = list(csv.DictReader(open(sys.argv[1])))
g = defaultdict(list)
for r in rows:
    g[(r["dtype"], f'{r["N"]}:{r["M"]}')].append(r)
print("dtype  N:M   points  speedup mean  min    max    >= target  eff TFLOP/s mean")
for (dt, nm), rs in sorted(g.items()):
    sp = [float(r["speedup"]) for r in rs]
    hit = sum(float(r["speedup"]) >= float(r["target"]) for r in rs)
    tf = statistics.fmean(float(r["tflops_eff"]) for r in rs)
    print(f"{dt:5s}  {nm:5s} {len(rs):6d}  {statistics.fmean(sp):12.2f}  {min(sp):5.2f}  {max(sp):5.2f}  "
          f"{hit:4d}/{len(rs):<4d}   {tf:8.1f}")
