"""Time nm_prepack (slot packing + images) for the BASELINE configs."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2503_01253_b200 import nmspmm, synth
for (m, n, k, N, M, L) in [(4096, 4096, 4096, 16, 32, 32), (2048, 11008, 4096, 12, 32, 32), (2048, 22016, 8192, 4, 32, 32)]:
    B = torch.from_numpy(synth.uniform((k, n), 2, 2)).cuda().bfloat16()
    W = nmspmm.nm_compress(B, N, M, L)
    PW = nmspmm.nm_prepack(W)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        PW = nmspmm.nm_prepack(W)
    torch.cuda.synchronize()
    print(f"prepack {m}x{n}x{k} {N}:{M} L={L}: {(time.perf_counter() - t0) / 3 * 1e3:.2f} ms", flush=True)
