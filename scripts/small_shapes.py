"""Small-shape probe: kernel and step times of nm_spmm at m=n=k in {1024, 2048} (fp32 SIMT, bf16
slot kernel) under NM_SIMT_SPLIT / NM_SP_SPLIT variants, L2 flushed between steps.
Usage: small_shapes.py [dtype=f32|bf16] [sizes...]"""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
dt = {"f32": torch.float32, "bf16": torch.bfloat16}[sys.argv[1] if len(sys.argv) > 1 else "f32"]
sizes = [int(x) for x in sys.argv[2:]] or [1024, 2048]
flush_buf = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
flush = lambda: flush_buf.fill_(1.0)
var = "NM_SIMT_SPLIT" if dt == torch.float32 else "NM_SP_SPLIT"
for s in sizes:
    for N in (16, 4):
        for sp in os.environ.get("SPLITS", "auto 1 2 4").split():
            if sp == "auto":
                os.environ.pop(var, None)
            else:
                os.environ[var] = sp
            r, _ = bench.measure_config((s, s, s, N, 32, 32), dt, 20, 3, flush, with_cublas=(sp == "auto"))
            print(f"{s}^3 {N}:32 {var}={sp}: step {r['ms']*1e3:7.1f} us kernel {r['kernel_ms']*1e3:7.1f} us "
                  f"({r['kernel_tflops']:.1f} TF) launches/step {r['launches_per_step']:.0f}"
                  + (f"  cuBLAS {r['cublas_ms']*1e3:.1f} us speedup {r['speedup_vs_cublas']:.2f} (target {r['target_speedup']:.2f})" if 'cublas_ms' in r else ""), flush=True)
    os.environ.pop(var, None)
