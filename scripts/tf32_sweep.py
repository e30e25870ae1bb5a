"""tf32 slot kernel: token tile NT and column halves H sweep (NM_SP_NT / NM_SP_H), kernel events."""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2503_01253_b200 import nmspmm, synth
lib = nmspmm.lib()
for (m, n, k, N, M, L) in [(4096, 4096, 4096, 16, 32, 32), (2048, 11008, 4096, 8, 32, 32), (2048, 22016, 8192, 4, 32, 32)]:
    A = torch.from_numpy(synth.uniform((m, k), 1, 1)).cuda()
    W = nmspmm.nm_compress(torch.from_numpy(synth.uniform((k, n), 2, 2)).cuda(), N, M, L)
    C = torch.empty(m, n, device="cuda")
    flops = 2.0 * m * n * (k // M * N)
    for h, nts in (("1", ["256", "192", "128"]), ("2", ["160", "176", "192", "208", "224", "128"])):
        os.environ["NM_SP_H"] = h
        PW = nmspmm.nm_prepack(W, math="tf32_tc")
        for nt in nts:
            os.environ["NM_SP_NT"] = nt
            for _ in range(3):
                nmspmm.nm_spmm_prepacked(A, PW, out=C)
            torch.cuda.synchronize()
            lib.nm_profile_begin()
            for _ in range(10):
                nmspmm.nm_spmm_prepacked(A, PW, out=C)
            torch.cuda.synchronize()
            ms, cnt, la = ctypes.c_double(), ctypes.c_int64(), ctypes.c_int64()
            lib.nm_profile_end(ctypes.byref(ms), ctypes.byref(cnt), ctypes.byref(la))
            kms = ms.value / max(cnt.value, 1)
            print(f"{m}x{n}x{k} {N}:{M} H={h} NT={nt}: {kms*1e3:8.1f} us {flops/kms/1e9:7.1f} TFLOP/s", flush=True)
        os.environ.pop("NM_SP_NT")
    os.environ.pop("NM_SP_H")
