"""bf16 operands with L the slot kernel cannot take (cfg5's L = 4, and L = 8): the fp32 SIMT kernel
on exact fp32 copies (kernel 5, default) vs the one-thread-per-element generic kernel
(NM_BF16_SIMT=0), per-call time of nm_spmm (CUDA events, conversions included) and cuBLAS bf16 on
the dense shape.  Usage: bf16_simt_time.py [sizes...] (default 1024 2048 4096)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2503_01253_b200 import nmspmm, synth

sizes = [int(x) for x in sys.argv[1:]] or [1024, 2048, 4096]


def etime(fn, reps=10):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3


print("# m=n=k, N:M, L, kernel: SIMT-bf16 (default) / generic (NM_BF16_SIMT=0) us, TFLOP/s (kept MACs), x cuBLAS bf16")
for s in sizes:
    for N, L in [(16, 4), (8, 4), (4, 4), (16, 8)]:
        M = 32
        A = torch.from_numpy(synth.uniform((s, s), 1, 1)).cuda().bfloat16()
        B = torch.from_numpy(synth.uniform((s, s), 2, 2)).cuda().bfloat16()
        W = nmspmm.nm_compress(B, N, M, L)
        C = torch.empty(s, s, device="cuda", dtype=torch.bfloat16)
        flops = 2.0 * s * s * (s // M * N)
        tc = etime(lambda: torch.matmul(A, B))
        out = []
        for simt in ("1", "0"):
            os.environ["NM_BF16_SIMT"] = simt
            kid = nmspmm.nm_plan_query(s, s, s, N, M, L, torch.bfloat16)["kernel"]
            if simt == "0" and s > 2048:
                out.append("generic skipped")
                continue
            t = etime(lambda: nmspmm.nm_spmm(A, W, out=C), reps=3 if simt == "0" else 10)
            out.append(f"kernel {kid}: {t:9.1f} us {flops / t / 1e6:6.1f} TFLOP/s {tc / t:5.2f}x")
        os.environ.pop("NM_BF16_SIMT", None)
        print(f"{s} {N}:{M} L{L}: " + " | ".join(out) + f"  (cuBLAS {tc:.1f} us)", flush=True)
