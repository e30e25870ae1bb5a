"""fp32 SIMT kernel time with the 64- and 128-row tiles (NM_SIMT_BM) and the selector's choice, on
the shapes that pin simt_row_tile (tests/test_abi_cpu.py ROW_TILE_MEASURED).  Kernel events via
nm_profile, 10 launches after 3 warm-ups."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2503_01253_b200 import nmspmm, synth
lib = nmspmm.lib()
SHAPES = [(1024, 1024, 1024, 16, 32, 32), (1024, 1024, 1024, 4, 32, 32), (256, 13824, 5120, 4, 32, 32),
          (2048, 1376, 4096, 8, 32, 32), (256, 256, 256, 2, 4, 4), (256, 22016, 8192, 4, 32, 32),
          (2048, 2752, 8192, 4, 32, 32), (2048, 2048, 2048, 16, 32, 32), (256, 4096, 4096, 8, 32, 32),
          (256, 4096, 11008, 8, 32, 32), (256, 8192, 8192, 8, 32, 32), (4096, 512, 4096, 16, 32, 32),
          (256, 12288, 4096, 8, 32, 32), (512, 6656, 6656, 8, 32, 32), (256, 4096, 4096, 16, 32, 32),
          (512, 5120, 5120, 8, 32, 32), (256, 5120, 5120, 8, 32, 32)]


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


for (m, n, k, N, M, L) in SHAPES:
    A = torch.from_numpy(synth.uniform((m, k), 1, 1)).cuda()
    W = nmspmm.nm_compress(torch.from_numpy(synth.uniform((k, n), 2, 2)).cuda(), N, M, L)
    C = torch.empty(m, n, device="cuda")
    r = {}
    for bm in ("64", "128", None):
        if bm:
            os.environ["NM_SIMT_BM"] = bm
        else:
            os.environ.pop("NM_SIMT_BM", None)
        r[bm or "sel"] = kt(lambda: nmspmm.nm_spmm(A, W, out=C, math="f32_simt"))
    sel = nmspmm.nm_plan_query(m, n, k, N, M, L, torch.float32)["bm"]
    best = "64" if r["64"] < r["128"] else "128"
    print(f"{m}x{n}x{k} {N}:{M} L{L}: 64 {r['64']:7.1f}  128 {r['128']:7.1f}  selector bm {sel} ({r['sel']:7.1f} us)"
          f"  {'ok' if str(sel) == best or abs(r['64'] - r['128']) < 0.03 * min(r['64'], r['128']) else 'MISS'}", flush=True)
