"""Timing ablation of spmm_tc_pair_kernel stages (NM_TC_DBG mask; outputs are garbage
when a stage is skipped).  Usage: tc_ablate.py [m n k N M L]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2503_01253_b200 import nmspmm, synth
m, n, k, N, M, L = [int(x) for x in (sys.argv[1:] or [4096, 4096, 4096, 16, 32, 32])]
A = torch.from_numpy(synth.uniform((m, k), 1, 1)).cuda().bfloat16()
B = torch.from_numpy(synth.uniform((k, n), 2, 2)).cuda().bfloat16()
W = nmspmm.nm_compress(B, N, M, L)
PW = nmspmm.nm_prepack(W)
C = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
flops = 2.0 * m * n * (k // M * N)
names = {0: "full", 1: "no gather", 2: "no MMA", 4: "no repack", 3: "loader+ctl only", 5: "MMA+TMA only",
         6: "gather only", 7: "TMA/sync skeleton", 15: "skel, B TMA only", 23: "skel, A TMA only", 31: "sync only"}
for dbg in [0, 1, 2, 4, 3, 5, 6, 7, 15, 23, 31]:
    os.environ["NM_TC_DBG"] = str(dbg)
    for _ in range(3):
        nmspmm.nm_spmm_prepacked(A, PW, out=C)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(20):
        nmspmm.nm_spmm_prepacked(A, PW, out=C)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(f"dbg={dbg} {names[dbg]:20s} {ms*1e3:8.1f} us  {flops/ms/1e9:8.1f} TFLOP/s-equiv", flush=True)
