"""Exact prepacked-weight bytes (nm_prepack_size, kind 2 bf16 / kind 3 tf32) vs the compressed
weight B' at the BASELINE shapes (the verdict's footprint check: <= 2.2x B')."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2503_01253_b200 import nmspmm
print("config,dtype,k,n,N:M,B'_MB,prepacked_MB,ratio")
for name in ["cfg2", "cfg3_62", "cfg3_75", "cfg4_13b", "cfg4_13b_sq", "cfg4_65b_sq", "cfg4_65b"]:
    m, n, k, N, M, L = bench.CONFIGS[name]
    for dt, math in ((torch.bfloat16, "auto"), (torch.float32, "tf32_tc")):
        _, Bd, W = bench.make_inputs((256, n, k, N, M, L), dt, "cuda")
        PW = nmspmm.nm_prepack(W, math=math)
        bp = W.values.numel() * W.values.element_size() + W.idx.numel()
        pb = PW.buf.numel()
        print(f"{name},{'bf16' if dt == torch.bfloat16 else 'tf32'},{k},{n},{N}:{M},{bp / 1e6:.1f},{pb / 1e6:.1f},{pb / bp:.2f}", flush=True)
        del Bd, W, PW
        torch.cuda.empty_cache()
