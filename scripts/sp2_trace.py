"""Per-stage %globaltimer trace of the CTA-pair slot kernel (NM_SP_DBG=64, cluster 0, stages < 64):
hop latencies of the stage hand-off (owner copies issued -> relay sees the peer's full barrier ->
leader MMA warp sees full -> commit -> owners of stage g+4 see their empty barrier).
Usage: sp2_trace.py [m n k N M L]  (env SP2_DBG: extra NM_SP_DBG bits, e.g. 27 skeleton, 1024 spin)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2503_01253_b200 import nmspmm, synth
m, n, k, N, M, L = [int(x) for x in (sys.argv[1:] or [4096, 4096, 4096, 16, 32, 32])]
A = torch.from_numpy(synth.uniform((m, k), 1, 1)).cuda().bfloat16()
B = torch.from_numpy(synth.uniform((k, n), 2, 2)).cuda().bfloat16()
PW = nmspmm.nm_prepack(nmspmm.nm_compress(B, N, M, L))
C = torch.zeros(m, n, device="cuda", dtype=torch.bfloat16)
for extra in [int(x) for x in os.environ.get("SP2_DBGS", "0 27 1024 3072 1051 128").split()]:
    os.environ["NM_SP_DBG"] = str(64 | extra)
    for _ in range(3):
        C.zero_()
        nmspmm.nm_spmm_prepacked(A, PW, out=C)
    torch.cuda.synchronize()
    t = C.view(torch.int64).flatten()[:64 * 16].cpu().numpy().reshape(64, 16).astype(np.float64)
    g = np.arange(4, 60)
    def d(a, b, off=0):
        x = t[g + off, b] - t[g, a]
        return np.median(x), np.percentile(x, 90)
    per = np.median(np.diff(t[4:60, 10]))
    rows = [("peer issued -> relay saw full", 6, 8, 0), ("leader issued -> MMA saw full", 2, 10, 0),
            ("relay saw -> MMA saw full", 8, 10, 0), ("MMA saw full -> committed", 10, 11, 0),
            ("commit -> leader owner(g+4) woke", 11, 1, 4), ("commit -> peer owner(g+4) woke", 11, 5, 4),
            ("leader owner woke -> issued", 1, 2, 0), ("peer owner woke -> issued", 5, 6, 0)]
    print(f"NM_SP_DBG={64 | extra}: stage period (MMA saw full) median {per:.0f} ns")
    for name, a, b, off in rows:
        med, p90 = d(a, b, off)
        print(f"   {name:36s} median {med:7.0f} ns  p90 {p90:7.0f} ns")
