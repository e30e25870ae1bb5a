"""Summarise scripts/paper_protocol.py's CSVs (v123 and af studies): the step-wise table at 4096^3
and, per (matrix, dtype, sparsity), the selector's kernel rate, the best variant and the selector's
loss to it.  Usage: protocol_summary.py v123.csv af.csv"""
import sys
from collections import defaultdict


def rows(path):
    """paper_protocol.py writes variant names with commas unquoted: the last six fields are fixed."""
    out = []
    lines = open(path).read().splitlines()
    hdr = lines[0].split(",")
    for line in lines[1:]:
        f = line.split(",")
        if len(f) < len(hdr):
            continue
        fixed = f[:8] + [",".join(f[8:len(f) - 6])] + f[len(f) - 6:]
        r = dict(zip(hdr, fixed))
        if r.get("kernel_tflops"):
            out.append(r)
    return out


v123, af = rows(sys.argv[1]), rows(sys.argv[2])
print("## step-wise study at m = n = k = 4096 (P:700-720): kernel TFLOP/s, efficiency, speedup over cuBLAS dense")
print(f"{'sparsity':>9s} {'variant':32s} {'TFLOP/s':>8s} {'eff':>6s} {'x cuBLAS':>9s}")
for r in v123:
    sparsity = 100.0 * (1 - int(r["N"]) / int(r["M"]))
    print(f"{sparsity:8.1f}% {r['dtype'] + ' ' + r['variant']:32s} {float(r['kernel_tflops']):8.1f} "
          f"{float(r['efficiency']):6.3f} {float(r['speedup_vs_cublas']):9.3f}")
print()
print("## blocking study A-F (P:646-660): selector vs the best variant per (matrix, dtype, sparsity)")
g = defaultdict(dict)
for r in af:
    g[(r["dtype"], r["matrix"], r["m"], r["n"], r["k"], r["N"], r["M"])][r["variant"]] = r
within3 = total = 0
for key in sorted(g):
    dt, mat, m, n, k, N, M = key
    v = g[key]
    sel = v.get("selector")
    if not sel:
        continue
    best_name, best = max(v.items(), key=lambda x: float(x[1]["kernel_tflops"]))
    loss = float(best["kernel_tflops"]) / float(sel["kernel_tflops"]) - 1.0
    total += 1
    within3 += loss <= 0.03
    sparsity = 100.0 * (1 - int(N) / int(M))
    print(f"{dt:5s} {mat} ({m}x{n}x{k}) {sparsity:5.1f}%: selector {float(sel['kernel_tflops']):8.1f} TF "
          f"({float(sel['speedup_vs_cublas']):.2f}x cuBLAS), best '{best_name}' {float(best['kernel_tflops']):8.1f} TF, "
          f"selector within {100 * loss:5.1f} %")
print(f"\nselector within 3 % of the best variant at {within3} / {total} points")
