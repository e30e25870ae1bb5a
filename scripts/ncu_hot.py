"""Top SASS instructions by warp-stall samples from an ncu report: ncu_hot.py rep [n]"""
import csv, subprocess, sys, io
rep = sys.argv[1]; n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ia, isrc = hdr.index('Address'), hdr.index('Source')
iw, ie = hdr.index('Warp Stall Sampling (All Samples)'), hdr.index('Instructions Executed')
data = [(r[ia], r[isrc], int(r[iw] or 0), int(r[ie] or 0)) for r in rows[2:] if len(r) > ie]
tot = sum(d[2] for d in data)
print("total samples", tot)
for i, (a, s, w, e) in enumerate(data):
    pass
top = sorted(range(len(data)), key=lambda i: -data[i][2])[:n]
for i in sorted(top):
    a, s, w, e = data[i]
    print(f"{i:5d} {w:6d} {100*w/tot:5.1f}% {e:10d} {s[:95]}")
