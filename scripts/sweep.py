"""cfg5 sweep (BASELINE.json): m = n = k in {1024 ... 16384} x N:M in {16,12,8,4}:32 x L in {4, 32, 64},
fp32 (CUDA-core kernel) and bf16 (sparse-tensor-core kernel), each vs cuBLAS dense GEMM of the
same shape and dtype on the same GPU.  Prints one CSV row per point (effective TFLOP/s = kept MACs,
step = one nm_spmm / nm_spmm_prepacked incl. the per-call A transpose, kernel = the SpMM launch).
Usage: sweep.py [sizes...]  (default 1024 2048 4096 8192 16384); SWEEP_DT=f32,bf16 (default) or tf32
(fp32 operands on the tf32 sparse-TC kernel; its cuBLAS column is then the TF32 dense GEMM)."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2503_01253_b200 import nmspmm

sizes = [int(x) for x in sys.argv[1:]] or [1024, 2048, 4096, 8192, 16384]
peaks, _ = bench.load_peaks()
flush_buf = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
flush = lambda: flush_buf.fill_(1.0)
print("dtype,m,n,k,N,M,L,kernel_id,step_ms,step_tflops,kernel_tflops,roofline_frac,cublas_tflops,speedup_vs_cublas,target", flush=True)
DTS = {"f32": (torch.float32, None), "bf16": (torch.bfloat16, None), "tf32": (torch.float32, "tf32_tc")}
for name in os.environ.get("SWEEP_DT", "f32,bf16").split(","):
    dt, math = DTS[name]
    for s in sizes:
        cub = None
        for N in (16, 12, 8, 4):
            for L in (4, 32, 64):
                if math and L == 4:
                    continue  # the tf32 tensor-core path needs L >= 16 (bf16 L = 4 runs the SIMT kernel, id 5)
                cfg = (s, s, s, N, 32, L)
                steps = 3 if s >= 8192 else 5
                try:
                    r, _ = bench.measure_config(cfg, dt, steps, 2, flush, with_cublas=cub is None, math=math)
                except Exception as e:  # noqa: BLE001 -- report and continue the sweep
                    print(f"# {cfg} {dt}: {e}", flush=True)
                    continue
                if cub is None:
                    cub = r["cublas_tf32_dense_tflops"] if math else r["cublas_dense_tflops"]
                peak = (peaks.get("bf16_tflops", 1590.0) / 2 if math else
                        bench.fp32_alu_peak_tflops(peaks.get("sm_max_mhz", 1965.0)) if dt == torch.float32
                        else peaks.get("bf16_tflops", 1590.0))
                speed = (r["tflops"] * 32 / N) / cub  # = t_cublas / t_step
                print(f"{name},{s},{s},{s},{N},32,{L},{r['plan']['kernel']},{r['ms']:.4f},"
                      f"{r['tflops']:.2f},{r['kernel_tflops']:.2f},{r['kernel_tflops'] / peak:.4f},{cub:.1f},{speed:.3f},"
                      f"{0.7 * 32 / N:.2f}", flush=True)
                torch.cuda.empty_cache()
