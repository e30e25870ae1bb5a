"""Timing ablation of spmm_tc_sp_kernel (NM_SP_DBG mask; outputs are garbage when a
stage is skipped).  Kernel time from nm_profile (CUDA events around the SpMM launch).
Usage: sp_ablate.py [m n k N M L]"""
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
names = {0: "full", 1: "no gather", 2: "no MMA", 3: "no gather, no MMA", 8: "no C stores",
         11: "no gather/MMA/stores", 16: "no weights", 27: "sync skeleton", 155: "skeleton, arrive not commit",
         131: "no gather/MMA, arrive", 19: "no gather/MMA/weights", 147: "no g/MMA/w, arrive",
         283: "skeleton, warp arrivals", 411: "skel, warp arr, plain empty", 17: "MMA only (no gather/weights)",
         512: "no stages (fixed costs)", 18: "no MMA, no weights", 9: "no gather, no C stores"}
lib = nmspmm.lib()
import ctypes
for dbg in [int(x) for x in os.environ.get('SP_DBGS', '0 1 2 3 8 11 16 27 155 131').split()]:
    os.environ["NM_SP_DBG"] = str(dbg)
    for _ in range(3):
        nmspmm.nm_spmm_prepacked(A, PW, out=C)
    torch.cuda.synchronize()
    lib.nm_profile_begin()
    for _ in range(20):
        nmspmm.nm_spmm_prepacked(A, PW, out=C)
    torch.cuda.synchronize()
    ms, cnt, la = ctypes.c_double(), ctypes.c_int64(), ctypes.c_int64()
    lib.nm_profile_end(ctypes.byref(ms), ctypes.byref(cnt), ctypes.byref(la))
    kms = ms.value / max(cnt.value, 1)
    print(f"dbg={dbg} {names.get(dbg, str(dbg)):28s} kernel {kms*1e3:8.1f} us  {flops/kms/1e9:8.1f} TFLOP/s-equiv", flush=True)
