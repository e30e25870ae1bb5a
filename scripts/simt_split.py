"""SIMT fp32 on per-rank column shards of cfg2 / cfg4 (n / G columns): automatic k-split of a
sub-wave grid vs none (NM_SIMT_SPLIT=1)."""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2503_01253_b200 import nmspmm, synth
lib = nmspmm.lib()
for (m, n, k, N, M, L) in [(4096, 512, 4096, 16, 32, 32), (4096, 1024, 4096, 16, 32, 32), (4096, 2048, 4096, 16, 32, 32),
                           (2048, 1376, 4096, 8, 32, 32), (2048, 2752, 8192, 4, 32, 32)]:
    A = torch.from_numpy(synth.uniform((m, k), 1, 1)).cuda()
    B = torch.from_numpy(synth.uniform((k, n), 2, 2)).cuda()
    W = nmspmm.nm_compress(B, N, M, L)
    C = torch.empty(m, n, device="cuda")
    flops = 2.0 * m * n * (k // M * N)
    for sp in ["auto", "1"]:
        if sp == "1":
            os.environ["NM_SIMT_SPLIT"] = "1"
        for _ in range(3):
            nmspmm.nm_spmm(A, W, out=C)
        torch.cuda.synchronize()
        lib.nm_profile_begin()
        for _ in range(10):
            nmspmm.nm_spmm(A, W, out=C)
        torch.cuda.synchronize()
        ms, cnt, la = ctypes.c_double(), ctypes.c_int64(), ctypes.c_int64()
        lib.nm_profile_end(ctypes.byref(ms), ctypes.byref(cnt), ctypes.byref(la))
        kms = ms.value / max(cnt.value, 1)
        print(f"{m}x{n}x{k} {N}:{M} split={sp}: kernel {kms*1e3:8.1f} us  {flops/kms/1e9:6.2f} TFLOP/s", flush=True)
        os.environ.pop("NM_SIMT_SPLIT", None)
