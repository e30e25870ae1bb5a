"""Per-stage clock64 trace of cluster (0,0) of spmm_tc_sp2_kernel (NM_SP_PAIR=1, NM_SP_DBG=64).
Leader: gather before/after empty wait, after issue, MMA after full wait, after commit;
peer: same gather columns + relay after local full wait.  (clock64 is per SM: compare within a CTA.)"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["NM_SP_PAIR"] = "1"
import torch
from paper_2503_01253_b200 import nmspmm, synth
m, n, k, N, M, L = 4096, 4096, 4096, 16, 32, 32
A = torch.from_numpy(synth.uniform((m, k), 1, 1)).cuda().bfloat16()
B = torch.from_numpy(synth.uniform((k, n), 2, 2)).cuda().bfloat16()
W = nmspmm.nm_compress(B, N, M, L)
PW = nmspmm.nm_prepack(W)
os.environ["NM_SP_DBG"] = "64"
C = torch.zeros(m, n, device="cuda", dtype=torch.bfloat16)
for _ in range(2):
    nmspmm.nm_spmm_prepacked(A, PW, out=C)
torch.cuda.synchronize()
ts = C.view(-1).view(torch.int64)[: 16 * 80].view(80, 16).cpu().tolist()
b0, b1 = ts[0][0], ts[0][8]
for st, r in enumerate(ts[:75]):
    print(st, "L", [x - b0 if x else -1 for x in r[0:5]], "P", [x - b1 if x else -1 for x in r[8:11]], r[13] - b1 if r[13] else -1)
