"""fp32 SIMT kernel time vs the grouped-raster height NM_SIMT_GROUP (row tiles per group) on the
headline and LLaMA shapes (nm_profile kernel events, 10 launches after 3 warm-ups, L2 not flushed)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2503_01253_b200 import nmspmm, synth
lib = nmspmm.lib()


def kt(fn):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    lib.nm_profile_begin()
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    ms, c, la = ctypes.c_double(), ctypes.c_int64(), ctypes.c_int64()
    lib.nm_profile_end(ctypes.byref(ms), ctypes.byref(c), ctypes.byref(la))
    return ms.value / c.value * 1e3


for (m, n, k, N, M, L) in [(4096, 4096, 4096, 16, 32, 32), (2048, 11008, 4096, 8, 32, 32), (2048, 22016, 8192, 4, 32, 32),
                           (8192, 8192, 8192, 16, 32, 32)]:
    A = torch.from_numpy(synth.uniform((m, k), 1, 1)).cuda()
    W = nmspmm.nm_compress(torch.from_numpy(synth.uniform((k, n), 2, 2)).cuda(), N, M, L)
    C = torch.empty(m, n, device="cuda")
    out = []
    for g in ("2", "4", "8", "16", "32"):
        os.environ["NM_SIMT_GROUP"] = g
        out.append(f"g{g} {kt(lambda: nmspmm.nm_spmm(A, W, out=C, math='f32_simt')):7.1f}")
    os.environ.pop("NM_SIMT_GROUP")
    print(f"{m}x{n}x{k} {N}:{M}: " + "  ".join(out), flush=True)
