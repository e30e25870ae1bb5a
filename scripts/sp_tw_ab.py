"""A/B of the bf16 slot kernel by an environment switch (SP_ENV, default NM_SP_TW: weights in TMEM,
the round-2 study; NM_SP_PERSIST: the persistent form), per token tile NT, on the BASELINE shapes.  Kernel time from nm_profile (CUDA events around the
SpMM launch, 20 launches after 3 warm-ups); C of every variant is compared with the TW=0 default
(bit-identical expected: same slots, same MMA K order) and with cuBLAS on the decompressed weight.
Usage: sp_tw_ab.py [m n k N M L ...] (groups of six), SP_NTS="0 192 176 160" (0 = selector)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2503_01253_b200 import nmspmm, synth

args = [int(x) for x in sys.argv[1:]]
shapes = [tuple(args[i:i + 6]) for i in range(0, len(args), 6)] or [
    (4096, 4096, 4096, 16, 32, 32), (2048, 11008, 4096, 12, 32, 32), (2048, 11008, 4096, 8, 32, 32),
    (2048, 22016, 8192, 4, 32, 32), (256, 22016, 8192, 4, 32, 32), (8192, 8192, 8192, 16, 32, 32),
    (1024, 1024, 1024, 16, 32, 32)]
nts = [int(x) for x in os.environ.get("SP_NTS", "0").split()]
lib = nmspmm.lib()


def ktime(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    lib.nm_profile_begin()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    ms, cnt, la = ctypes.c_double(), ctypes.c_int64(), ctypes.c_int64()
    lib.nm_profile_end(ctypes.byref(ms), ctypes.byref(cnt), ctypes.byref(la))
    return ms.value / max(cnt.value, 1) * 1e3


def etime(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3


for (m, n, k, N, M, L) in shapes:
    A = torch.from_numpy(synth.uniform((m, k), 1, 1)).cuda().bfloat16()
    B = torch.from_numpy(synth.uniform((k, n), 2, 2)).cuda().bfloat16()
    W = nmspmm.nm_compress(B, N, M, L)
    PW = nmspmm.nm_prepack(W)
    Bd = nmspmm.nm_decompress(W)
    ref = (A.float() @ Bd.float())
    t_cub = etime(lambda: torch.matmul(A, B))
    flops = 2.0 * m * n * (k // M * N)
    base = None
    for tw in (0, 1):
        os.environ[os.environ.get("SP_ENV", "NM_SP_TW")] = str(tw)
        for nt in nts:
            if nt:
                os.environ["NM_SP_NT"] = str(nt)
            else:
                os.environ.pop("NM_SP_NT", None)
            C = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
            try:
                t = ktime(lambda: nmspmm.nm_spmm_prepacked(A, PW, out=C))
            except Exception as ex:  # unsupported (H, NT)
                print(f"{m}x{n}x{k} {N}:{M} L{L} tw={tw} nt={nt}: {ex}", flush=True)
                continue
            nmspmm.nm_spmm_prepacked(A, PW, out=C)
            torch.cuda.synchronize()
            err = ((C.float() - ref).norm() / ref.norm()).item()
            same = "" if base is None else (" bit-identical" if torch.equal(C, base) else
                                             f" DIFFERS from tw=0 (max {(C.float() - base.float()).abs().max().item():.3g})")
            if base is None:
                base = C.clone()
            print(f"{m}x{n}x{k} {N}:{M} L{L} tw={tw} nt={nt or 'sel'}: kernel {t:7.1f} us  {flops / t / 1e6:7.1f} TFLOP/s  "
                  f"{t_cub / t:5.2f}x cuBLAS ({t_cub:.1f} us)  rel_err {err:.2e}{same}", flush=True)
    os.environ.pop("NM_SP_NT", None)
    os.environ.pop(os.environ.get("SP_ENV", "NM_SP_TW"), None)
