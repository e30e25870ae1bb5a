"""fp32 SIMT row tile 64 vs 128 (NM_SIMT_BM) at sub-wave / small / full shapes: kernel us (L2 flushed)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
flush_buf = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
flush = lambda: flush_buf.fill_(1.0)
shapes = [(4096, 512, 4096, 16, 32, 32), (2048, 1376, 4096, 8, 32, 32), (2048, 2752, 8192, 4, 32, 32),
          (1024, 1024, 1024, 16, 32, 32), (1024, 1024, 1024, 4, 32, 32), (2048, 2048, 2048, 16, 32, 32),
          (2048, 2048, 2048, 4, 32, 32), (256, 13824, 5120, 4, 32, 32), (256, 22016, 8192, 4, 32, 32),
          (512, 2048, 2048, 16, 32, 32), (256, 256, 256, 2, 4, 4), (4096, 4096, 4096, 16, 32, 32)]
for cfg in shapes:
    for bm in ("auto", "128", "64"):
        os.environ.pop("NM_SIMT_BM", None)
        if bm != "auto": os.environ["NM_SIMT_BM"] = bm
        r, _ = bench.measure_config(cfg, torch.float32, 10, 3, flush, with_cublas=False)
        print(f"{cfg} bm={bm}: kernel {r['kernel_ms']*1e3:8.1f} us {r['kernel_tflops']:6.2f} TF", flush=True)
    os.environ.pop("NM_SIMT_BM", None)
