"""Small-shape anomaly probe: kernel time with and without the L2 flush between steps, and
back-to-back (no host gap), for fp32 SIMT / bf16 slot kernels and cuBLAS at 1024^3 16:32."""
import os, sys, statistics, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2503_01253_b200 import nmspmm
flush_buf = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
def ev_time(fn, reps, flush=None):
    out = []
    for _ in range(reps):
        if flush: flush()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        out.append(a.elapsed_time(b) * 1e3)
    return statistics.median(out)
for dt in (torch.float32, torch.bfloat16):
    cfg = (1024, 1024, 1024, 16, 32, 32)
    A, Bd, W = bench.make_inputs(cfg, dt, "cuda")
    C = torch.empty(1024, 1024, dtype=dt, device="cuda")
    step = bench.make_step(A, W, C, dt, None)
    for _ in range(5): step()
    for name, fl in (("flush(fill 256MB)", lambda: flush_buf.fill_(1.0)), ("no flush", None)):
        nmspmm.nm_profile_begin()
        t = ev_time(step, 20, fl)
        k_ms, k_cnt, _ = nmspmm.nm_profile_end()
        td = ev_time(lambda: torch.mm(A, Bd, out=C), 20, fl)
        print(f"{dt} {name:18s}: step {t:7.1f} us kernel {k_ms / max(1, k_cnt) * 1e3:7.1f} us  cuBLAS {td:7.1f} us", flush=True)
    # back to back: 20 steps between one pair of events
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20): step()
    b.record(); torch.cuda.synchronize()
    print(f"{dt} back-to-back: {a.elapsed_time(b) * 1e3 / 20:7.1f} us/step", flush=True)
