"""A/B kernel times of the fp32 SIMT path for one library build (NM_LIB_PATH selects it):
BASELINE shapes + multi-GPU shard shapes + small shapes, L2 flushed between steps."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
flush_buf = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
flush = lambda: flush_buf.fill_(1.0)
tag = os.environ.get("AB_TAG", "new")
shapes = [(4096, 4096, 4096, 16, 32, 32), (2048, 11008, 4096, 8, 32, 32), (2048, 22016, 8192, 4, 32, 32),
          (2048, 5120, 5120, 4, 32, 32), (256, 22016, 8192, 4, 32, 32), (4096, 512, 4096, 16, 32, 32),
          (2048, 1376, 4096, 8, 32, 32), (2048, 2752, 8192, 4, 32, 32), (1024, 1024, 1024, 16, 32, 32),
          (2048, 2048, 2048, 16, 32, 32)]
for cfg in shapes:
    r, _ = bench.measure_config(cfg, torch.float32, 10, 3, flush, with_cublas=False)
    print(f"{tag} {os.environ.get('NM_SIMT_SK', 'auto')} {cfg}: kernel {r['kernel_ms']*1e3:8.1f} us {r['kernel_tflops']:6.2f} TF", flush=True)
