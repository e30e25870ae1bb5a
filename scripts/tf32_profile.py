"""cfg2 on the tf32 sparse-tensor-core path, prepacked weight, 6 launches (for one ncu capture)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2503_01253_b200 import nmspmm, synth
m, n, k, N, M, L = 4096, 4096, 4096, 16, 32, 32
A = torch.from_numpy(synth.uniform((m, k), 1, synth.TID_A)).cuda()
W = nmspmm.nm_compress(torch.from_numpy(synth.uniform((k, n), 2, synth.TID_B)).cuda(), N, M, L)
PW = nmspmm.nm_prepack(W, math="tf32_tc")
C = torch.empty(m, n, device="cuda")
for _ in range(6):
    nmspmm.nm_spmm_prepacked(A, PW, out=C)
torch.cuda.synchronize()
print("done")
