"""The paper's evaluation protocol on B200, synthetic weights:
  * study=v123  -- the step-wise study (Fig. step_wise) at m = n = k = 4096, sparsity
                   0 % (N = M = 32) / 50 / 62.5 / 75 / 87.5 %, fp32: V1 = hierarchical blocking,
                   A gathered straight from the TMA-staged [m][k] panel (NM_SIMT_MODE=0); V2 = + the
                   sparsity-aware footprint reduction, only the tile's col_info rows of A^T loaded
                   (mode 2); V3 = + latency hiding, the software-pipelined index -> gather ->
                   FFMA2 chain on the TMA-staged A^T panel (mode 1, the default; Listing 4);
                   and cuBLAS SGEMM (dense, all sparsities);
                   bf16: the slot kernel vs cuBLAS bf16 at the same points;
  * study=af    -- the blocking study (P:646-660 Table matrix_sizes): matrices A-F x the
                   same 5 sparsities x kernel variants: fp32 'selector' (default schedule with the
                   wave-model split), 'no-split' (one CTA per tile), mode 0; bf16 'selector',
                   H = 1 / H = 2 column halves, token tiles NT = 128 / 192 / 256; cuBLAS at 0 %.
Kernel time = nm_profile CUDA events around the SpMM launch (median of 10, L2 flushed between
steps); efficiency = kernel TFLOP/s (kept MACs) / the path's peak (FP32 FFMA 74.45, bf16 measured).
Usage: paper_protocol.py v123|af  -> CSV on stdout."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench

peaks, _ = bench.load_peaks()
P_F32 = bench.fp32_alu_peak_tflops(peaks.get("sm_max_mhz", 1965.0))
P_BF16 = peaks.get("bf16_tflops", 1610.0)
flush_buf = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
flush = lambda: flush_buf.fill_(1.0)
SP = [(32, 32), (16, 32), (12, 32), (8, 32), (4, 32)]
ENVS = ["NM_SIMT_MODE", "NM_SIMT_SPLIT", "NM_SP_H", "NM_SP_NT"]


def run(cfg, dt, env, cublas):
    for e in ENVS:
        os.environ.pop(e, None)
    os.environ.update(env)
    try:
        r, _ = bench.measure_config(cfg, dt, 10, 3, flush, with_cublas=cublas)
    except Exception as ex:  # noqa: BLE001 -- a variant that does not apply is reported, not fatal
        return None, str(ex).splitlines()[0][:80]
    finally:
        for e in ENVS:
            os.environ.pop(e, None)
    return r, None


study = sys.argv[1] if len(sys.argv) > 1 else "v123"
print("study,matrix,dtype,m,n,k,N,M,variant,kernel_us,kernel_tflops,efficiency,cublas_dense_tflops,speedup_vs_cublas,note", flush=True)
if study == "v123":
    mats = {"4096^3": (4096, 4096, 4096)}
    F32V = {"V1 (mode 0)": {"NM_SIMT_MODE": "0"}, "V2 (mode 2, packed)": {"NM_SIMT_MODE": "2"},
            "V3 (mode 1, default)": {}}
    BF16V = {"slot kernel (default)": {}}
else:
    mats = {"A": (512, 512, 512), "B": (512, 1024, 1024), "C": (512, 2048, 2048), "D": (1024, 2048, 2048),
            "E": (2048, 4096, 4096), "F": (4096, 4096, 4096)}
    F32V = {"selector": {}, "no-split": {"NM_SIMT_SPLIT": "1"}, "A straight from [m][k] panels (mode 0)": {"NM_SIMT_MODE": "0"}}
    BF16V = {"selector": {}, "H=1": {"NM_SP_H": "1"}, "H=2": {"NM_SP_H": "2"}, "H=2 NT=128": {"NM_SP_H": "2", "NM_SP_NT": "128"},
             "H=1 NT=128": {"NM_SP_H": "1", "NM_SP_NT": "128"}, "H=1 NT=192": {"NM_SP_H": "1", "NM_SP_NT": "192"}}
for label, (m, n, k) in mats.items():
    for dt, variants, peak in ((torch.float32, F32V, P_F32), (torch.bfloat16, BF16V, P_BF16)):
        for (N, M) in SP:
            cub = None
            for vi, (vname, env) in enumerate(variants.items()):
                r, err = run((m, n, k, N, M, 32), dt, env, cublas=(vi == 0))
                if r is None:
                    print(f"{study},{label},{'f32' if dt == torch.float32 else 'bf16'},{m},{n},{k},{N},{M},{vname},,,,,,{err}", flush=True)
                    continue
                if vi == 0:
                    cub = r["cublas_dense_tflops"]
                sp = r["kernel_tflops"] * M / N / cub  # t_cublas / t_kernel
                print(f"{study},{label},{'f32' if dt == torch.float32 else 'bf16'},{m},{n},{k},{N},{M},{vname},"
                      f"{r['kernel_ms'] * 1e3:.1f},{r['kernel_tflops']:.2f},{r['kernel_tflops'] / peak:.4f},{cub:.1f},{sp:.3f},"
                      f"kernel {r['plan']['kernel']}", flush=True)
