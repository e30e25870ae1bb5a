"""fp32 operands: SIMT (the paper's fp32 semantics) vs the tf32 sparse-tensor-core slot kernel,
kernel time by CUDA events (nm_profile) on the BASELINE shapes."""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2503_01253_b200 import nmspmm, synth
lib = nmspmm.lib()
for (m, n, k, N, M, L) in [(4096, 4096, 4096, 16, 32, 32), (2048, 11008, 4096, 12, 32, 32),
                           (2048, 11008, 4096, 8, 32, 32), (2048, 22016, 8192, 4, 32, 32), (2048, 13824, 5120, 4, 32, 32),
                           (8192, 8192, 8192, 16, 32, 32)]:
    A = torch.from_numpy(synth.uniform((m, k), 1, 1)).cuda()
    B = torch.from_numpy(synth.uniform((k, n), 2, 2)).cuda()
    W = nmspmm.nm_compress(B, N, M, L)
    C = torch.empty(m, n, device="cuda")
    flops = 2.0 * m * n * (k // M * N)
    for math in ("f32_simt", "tf32_tc"):
        for _ in range(3):
            nmspmm.nm_spmm(A, W, out=C, math=math)
        torch.cuda.synchronize()
        lib.nm_profile_begin()
        for _ in range(10):
            nmspmm.nm_spmm(A, W, out=C, math=math)
        torch.cuda.synchronize()
        ms, cnt, la = ctypes.c_double(), ctypes.c_int64(), ctypes.c_int64()
        lib.nm_profile_end(ctypes.byref(ms), ctypes.byref(cnt), ctypes.byref(la))
        kms = ms.value / max(cnt.value, 1)
        print(f"{m}x{n}x{k} {N}:{M} {math:9s}: kernel {kms*1e3:8.1f} us  {flops/kms/1e9:7.2f} TFLOP/s", flush=True)
