"""Per-stage clock64 trace of CTA (0,0) of spmm_tc_sp_kernel (NM_SP_DBG=64|mask).
Columns: producer before/after empty wait, after issue; MMA before/after full wait, after commit."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2503_01253_b200 import nmspmm, synth
m, n, k, N, M, L = 4096, 4096, 4096, 16, 32, 32
A = torch.from_numpy(synth.uniform((m, k), 1, 1)).cuda().bfloat16()
B = torch.from_numpy(synth.uniform((k, n), 2, 2)).cuda().bfloat16()
W = nmspmm.nm_compress(B, N, M, L)
PW = nmspmm.nm_prepack(W)
for mask in [int(x) for x in os.environ.get("SP_MASKS", "0 27").split()]:
    os.environ["NM_SP_DBG"] = str(64 | mask)
    C = torch.zeros(m, n, device="cuda", dtype=torch.bfloat16)
    for _ in range(2):
        nmspmm.nm_spmm_prepacked(A, PW, out=C)
    torch.cuda.synchronize()
    ts = C.view(-1).view(torch.int64)[: 8 * 100].view(100, 8).cpu().tolist()
    base = ts[0][0]
    print(f"mask {mask}")
    prev = None
    for st, r in enumerate(ts):
        if r[0] == 0 and r[6] == 0 and st > 0:
            break
        rel = [x - base if x else -1 for x in r[:8]]
        d = (r[4] - prev) if prev else 0
        prev = r[4]
        print(st, rel, "mma-step", d)
