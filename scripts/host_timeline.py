"""CUPTI timeline (torch.profiler) of one nm_spmm_host call: copies and kernels per stream with
start / end in us relative to the first event.  Usage: host_timeline.py [m n k N M L] [f32|bf16]."""
import json, os, sys, tempfile
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import profile, ProfilerActivity
from paper_2503_01253_b200 import nmspmm, synth
args = sys.argv[1:]
dt = torch.bfloat16 if args and args[-1] == "bf16" else torch.float32
nums = [int(x) for x in args if x.isdigit()] or [4096, 4096, 4096, 16, 32, 32]
m, n, k, N, M, L = nums
A = torch.from_numpy(synth.uniform((m, k), 1, 1)).to(dt)
B = torch.from_numpy(synth.uniform((k, n), 2, 2)).to(dt).cuda()
W = nmspmm.nm_compress(B, N, M, L)
Ah, Vh, Dh = A.pin_memory(), W.values.cpu().pin_memory(), W.idx.cpu().pin_memory()
Ch = torch.empty(m, n, dtype=dt).pin_memory()
run = nmspmm.HostSpmm(m, n, k, N, M, L, ab_dtype=dt, math="f32_simt" if dt == torch.float32 else "auto")
for _ in range(3):
    run(Ah, Vh, Dh, Ch)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    run(Ah, Vh, Dh, Ch)
    torch.cuda.synchronize()
f = tempfile.mktemp(suffix=".json")
prof.export_chrome_trace(f)
ev = [e for e in json.load(open(f))["traceEvents"] if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
t0 = min(e["ts"] for e in ev)
for e in sorted(ev, key=lambda e: e["ts"]):
    print(f"{e['cat']:10s} stream {e['args'].get('stream', '?'):>4} {e['ts'] - t0:9.1f} .. {e['ts'] + e['dur'] - t0:9.1f} us  "
          f"{e['name'][:60]}  {e['args'].get('bytes', '')}")
print(f"span {max(e['ts'] + e['dur'] for e in ev) - t0:.1f} us")
