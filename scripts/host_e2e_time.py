"""nm_spmm_host end to end (pinned host A/B'/D in, C out) with 1..8 row chunks (NM_HOST_CHUNKS);
DT=bf16 runs the bf16 sparse-TC path (per-call prepack, then the chunks)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2503_01253_b200 import nmspmm, synth
for (m, n, k, N, M, L) in [(4096, 4096, 4096, 16, 32, 32), (2048, 22016, 8192, 4, 32, 32)]:
    dt = torch.bfloat16 if os.environ.get("DT") == "bf16" else torch.float32
    gen = synth.bf16grid if dt == torch.bfloat16 else synth.uniform
    A = torch.from_numpy(gen((m, k), 1, 1)).to(dt).pin_memory()
    W = nmspmm.nm_compress(torch.from_numpy(gen((k, n), 2, 2)).cuda().to(dt), N, M, L)
    V, D = W.values.cpu().pin_memory(), W.idx.cpu().pin_memory()
    C = torch.empty(m, n, dtype=dt).pin_memory()
    flops = 2.0 * m * n * (k // M * N)
    for ch in ["0", "1", "4", "6", "8"]:
        os.environ["NM_HOST_CHUNKS"] = ch
        run = nmspmm.HostSpmm(m, n, k, N, M, L, ab_dtype=dt)
        for _ in range(2):
            run(A, V, D, C)
        ts = []
        for _ in range(5):
            t0 = time.perf_counter(); run(A, V, D, C); ts.append(time.perf_counter() - t0)
        t = sorted(ts)[2]
        print(f"{m}x{n}x{k} {N}:{M} chunks={ch if ch != '0' else 'auto'}: {t*1e3:7.2f} ms  {flops/t/1e12:6.2f} TFLOP/s e2e ({dt})", flush=True)
