"""bf16 slot kernel on one shape, prepacked weight, 4 launches (for one ncu capture).
Usage: prof_sp.py [m n k N M L]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2503_01253_b200 import nmspmm, synth
m, n, k, N, M, L = [int(x) for x in (sys.argv[1:] or [4096, 4096, 4096, 16, 32, 32])]
A = torch.from_numpy(synth.bf16grid((m, k), 1, synth.TID_A)).cuda().bfloat16()
W = nmspmm.nm_compress(torch.from_numpy(synth.bf16grid((k, n), 2, synth.TID_B)).cuda().bfloat16(), N, M, L)
PW = nmspmm.nm_prepack(W)
C = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
for _ in range(4):
    nmspmm.nm_spmm_prepacked(A, PW, out=C)
torch.cuda.synchronize()
print("done", PW.buf.numel())
