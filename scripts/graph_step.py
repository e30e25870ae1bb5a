"""The bench step (nm_spmm_prepacked / nm_spmm) eager vs replayed from a CUDA graph captured once
(torch.cuda.graph on the current stream: the library's pool allocations, memsets and launches
become graph nodes), CUDA events per step with the L2 flush between steps, as in bench.py.
Checks that the replayed C equals the eager C.  Usage: graph_step.py [f32|bf16|bf16at]."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2503_01253_b200 import nmspmm, synth

mode = (sys.argv[1:] or ["bf16"])[0]
dt = torch.float32 if mode == "f32" else torch.bfloat16
m = n = k = 4096
N, M, L = 16, 32, 32
gen = synth.uniform if dt == torch.float32 else synth.bf16grid
A = torch.from_numpy(gen((m, k), 1, 1)).cuda().to(dt)
B = torch.from_numpy(gen((k, n), 2, 2)).cuda().to(dt)
W = nmspmm.nm_compress(B, N, M, L)
C = torch.empty(m, n, device="cuda", dtype=dt)
if mode == "f32":
    step = lambda: nmspmm.nm_spmm(A, W, out=C, math="f32_simt")  # noqa: E731
elif mode == "bf16at":
    At = A.t().contiguous()
    PW = nmspmm.nm_prepack(W)
    step = lambda: nmspmm.nm_spmm_prepacked_at(At, PW, out=C)  # noqa: E731
else:
    PW = nmspmm.nm_prepack(W)
    step = lambda: nmspmm.nm_spmm_prepacked(A, PW, out=C)  # noqa: E731
flush_buf = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")


def timed(fn, steps=20, warmup=3):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for s, e in ev:
        flush_buf.fill_(1.0)
        s.record()
        fn()
        e.record()
    torch.cuda.synchronize()
    return statistics.median([s.elapsed_time(e) for s, e in ev]) * 1e3


t_eager = timed(step)
step()
torch.cuda.synchronize()
ref = C.clone()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    for _ in range(3):
        step()
torch.cuda.current_stream().wait_stream(s)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    step()
C.zero_()
g.replay()
torch.cuda.synchronize()
same = torch.equal(C, ref)
t_graph = timed(g.replay)
print(f"{mode} cfg2: eager step {t_eager:.1f} us, graph replay {t_graph:.1f} us, C identical: {same}")
