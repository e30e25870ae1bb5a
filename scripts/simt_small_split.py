import ctypes, os, sys
sys.path.insert(0, '/root/repo')
import torch
from paper_2503_01253_b200 import nmspmm, synth
lib = nmspmm.lib()
def kt(fn):
    for _ in range(3): fn()
    torch.cuda.synchronize(); lib.nm_profile_begin()
    for _ in range(10): fn()
    torch.cuda.synchronize()
    ms, c, la = ctypes.c_double(), ctypes.c_int64(), ctypes.c_int64()
    lib.nm_profile_end(ctypes.byref(ms), ctypes.byref(c), ctypes.byref(la)); return ms.value / c.value * 1e3
for (m,n,k,N,M,L) in [(1024,1024,1024,16,32,32),(1024,1024,1024,8,32,32),(1024,1024,1024,4,32,32),(512,512,512,16,32,32),(256,256,256,2,4,4),(2048,2048,2048,16,32,32),(1024,2048,2048,16,32,32),(512,1024,1024,16,32,32)]:
    A = torch.from_numpy(synth.uniform((m, k), 1, 1)).cuda()
    W = nmspmm.nm_compress(torch.from_numpy(synth.uniform((k, n), 2, 2)).cuda(), N, M, L)
    C = torch.empty(m, n, device="cuda")
    out = []
    for bm in ("64", "128"):
        for sp in (None, "2", "3", "4"):
            os.environ["NM_SIMT_BM"] = bm
            if sp: os.environ["NM_SIMT_SPLIT"] = sp
            else: os.environ.pop("NM_SIMT_SPLIT", None)
            t = kt(lambda: nmspmm.nm_spmm(A, W, out=C, math="f32_simt"))
            out.append(f"bm{bm}/S{sp or 'auto'} {t:6.1f}")
    os.environ.pop("NM_SIMT_BM"); os.environ.pop("NM_SIMT_SPLIT", None)
    tsel = kt(lambda: nmspmm.nm_spmm(A, W, out=C, math="f32_simt"))
    print(f"{m}x{n}x{k} {N}:{M} L{L}: sel {tsel:6.1f} | " + "  ".join(out), flush=True)
