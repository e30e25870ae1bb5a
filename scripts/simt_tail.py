"""fp32 SIMT tail handling: kernel time at partial-wave / sub-wave shapes with the stream-K schedule
(auto), data-parallel only (NM_SIMT_SK=0) and forced stream-K CTA counts, L2 flushed between steps."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
flush_buf = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
flush = lambda: flush_buf.fill_(1.0)
shapes = [(2048, 5120, 5120, 4, 32, 32), (256, 22016, 8192, 4, 32, 32), (256, 13824, 5120, 4, 32, 32),
          (4096, 512, 4096, 16, 32, 32), (2048, 1376, 4096, 8, 32, 32), (2048, 2752, 8192, 4, 32, 32),
          (2048, 13824, 5120, 4, 32, 32), (4096, 4096, 4096, 16, 32, 32), (2048, 11008, 4096, 8, 32, 32),
          (1024, 1024, 1024, 16, 32, 32), (1024, 1024, 1024, 4, 32, 32), (2048, 2048, 2048, 16, 32, 32),
          (2048, 2048, 2048, 4, 32, 32)]
for cfg in shapes:
    for sp in os.environ.get("SKS", "auto off 148 222 296").split():
        os.environ.pop("NM_SIMT_SK", None); os.environ.pop("NM_SIMT_SK_CTAS", None)
        if sp == "off": os.environ["NM_SIMT_SK"] = "0"
        elif sp != "auto": os.environ["NM_SIMT_SK_CTAS"] = sp
        r, _ = bench.measure_config(cfg, torch.float32, 10, 3, flush, with_cublas=False)
        print(f"{cfg} sk={sp}: kernel {r['kernel_ms']*1e3:8.1f} us {r['kernel_tflops']:6.2f} TF", flush=True)
    os.environ.pop("NM_SIMT_SK", None); os.environ.pop("NM_SIMT_SK_CTAS", None)
