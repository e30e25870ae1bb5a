"""bf16 slot kernel: kernel time of sub-wave / partial-wave shapes under NM_SP_SPLIT (parts per split
tile) and NM_SP_TAIL=0 (no split), prepacked weights, L2 flushed between steps -- the data for the
slot kernel's split rule."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
flush_buf = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
flush = lambda: flush_buf.fill_(1.0)
shapes = [(1024, 1024, 1024, 16, 32, 32), (1024, 1024, 1024, 4, 32, 32), (2048, 2048, 2048, 16, 32, 32),
          (4096, 512, 4096, 16, 32, 32), (2048, 1376, 4096, 8, 32, 32), (2048, 2752, 8192, 4, 32, 32),
          (256, 22016, 8192, 4, 32, 32), (256, 13824, 5120, 4, 32, 32), (2048, 5120, 5120, 4, 32, 32),
          (4096, 4096, 4096, 16, 32, 32), (2048, 11008, 4096, 12, 32, 32)]
for cfg in shapes:
    for sp in os.environ.get("SPS", "auto off 2 3 4 6").split():
        os.environ.pop("NM_SP_SPLIT", None); os.environ.pop("NM_SP_TAIL", None)
        if sp == "off": os.environ["NM_SP_TAIL"] = "0"
        elif sp != "auto": os.environ["NM_SP_SPLIT"] = sp
        r, _ = bench.measure_config(cfg, torch.bfloat16, 10, 3, flush, with_cublas=False)
        print(f"{cfg} split={sp}: kernel {r['kernel_ms']*1e3:8.1f} us {r['kernel_tflops']:7.1f} TF", flush=True)
    os.environ.pop("NM_SP_SPLIT", None); os.environ.pop("NM_SP_TAIL", None)
