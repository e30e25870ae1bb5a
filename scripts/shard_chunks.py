"""Per-rank compute of the column-sharded layer (ShardedNmLinear.local) on one GPU: one rank's
shard of G in {2, 4, 8} for cfg2 / cfg3-75 % / cfg4-65B, its rows in c in {1, 2, 4} slices (the
NCCL overlap of SURVEY 8(f)1 computes slice i+1 while slice i is gathered).  Prints the summed
kernel time per step, so the cost of slicing can be weighed against the all-gather it hides
(floor (G-1)/G x m n e / ~770 GB/s).  Usage: shard_chunks.py [f32|bf16]."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2503_01253_b200 import nmspmm, sharded, synth

dt = torch.bfloat16 if (sys.argv[1:] or ["f32"])[0] == "bf16" else torch.float32
lib = nmspmm.lib()
cfgs = {"cfg2": (4096, 4096, 4096, 16, 32, 32), "cfg3_75": (2048, 11008, 4096, 8, 32, 32),
        "cfg4_65b": (2048, 22016, 8192, 4, 32, 32)}


def ktime(fn, reps=10):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    lib.nm_profile_begin()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    ms, cnt, la = ctypes.c_double(), ctypes.c_int64(), ctypes.c_int64()
    lib.nm_profile_end(ctypes.byref(ms), ctypes.byref(cnt), ctypes.byref(la))
    return ms.value / reps * 1e3, a.elapsed_time(b) / reps * 1e3


gen = synth.uniform if dt == torch.float32 else synth.bf16grid
print(f"# {dt}: per-rank kernel time (sum over slices) / step time, us; all-gather floor at 770 GB/s")
for name, (m, n, k, N, M, L) in cfgs.items():
    A = torch.from_numpy(gen((m, k), 1, 1)).cuda().to(dt)
    B = torch.from_numpy(gen((k, n), 2, 2)).cuda().to(dt)
    W = nmspmm.nm_compress(B, N, M, L)
    for G in (2, 4, 8):
        v, d = sharded.shard_weight(W.values, W.idx, L, N, 0, G)
        Ws = nmspmm.NmWeight(v, d, k, N, M, L)
        PW = nmspmm.nm_prepack(Ws) if dt == torch.bfloat16 else None
        nr = v.shape[1]
        out = []
        for c in (1, 2, 4):
            rc = -(-m // c)
            rc = -(-rc // 128) * 128 if c > 1 else m

            def step():
                for r0 in range(0, m, rc):
                    Ai = A[r0:min(m, r0 + rc)]
                    if PW is not None:
                        nmspmm.nm_spmm_prepacked(Ai, PW)
                    else:
                        nmspmm.nm_spmm(Ai, Ws)
            kt, st = ktime(step)
            out.append(f"c={c}: {kt:7.1f} / {st:7.1f}")
        ag = (G - 1) / G * m * n * A.element_size() / 770e9 * 1e6
        print(f"{name} G={G} shard {m}x{nr}x{k}: " + "  ".join(out) + f"  | all-gather floor {ag:6.1f} us", flush=True)
