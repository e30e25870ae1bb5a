#!/usr/bin/env python
"""bench.py -- effective TFLOPS of the vector-wise N:M SpMM hot path on B200.

Contract (driver): `python bench.py --gpus N --steps K --warmup W` prints ONE
JSON line on rank 0.  A "step" is one pass of the hot path over one batch:
  N = 1 : nm_spmm(A, B', D) -> C  (one launch of our kernel);
  N > 1 : column-sharded: each rank runs nm_spmm on its slice of
          the column groups, C is assembled with an NCCL all-gather and our
          unshard kernel (strong scaling: the problem size is fixed);
          `--exchange p2p` instead fuses the assembly into the SpMM epilogue
          (peer stores over CUDA IPC / NVLink + a flag barrier).
Variants (not the headline): the other BASELINE configs in fp32 and bf16, and
tf32 (fp32 operands on the tf32 sparse tensor cores, also timed against
cuBLAS with TF32 tensor cores).
Metric (BASELINE.json): effective TFLOPS = 2*m*n*w / t, w = k*N/M (kept MACs
only), plus speedup over cuBLAS dense GEMM of the same shape and dtype
on the same GPU.  Inputs are resident in HBM when the timed region starts;
L2 is flushed (256 MiB write) between timed steps, outside the CUDA events.

`--impl reference` times the CPU oracle (oracle/, the only other place this
file executes it) on a bounded row sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (m, n, k, N, M, L)   -- BASELINE.json configs
    "cfg1": (256, 256, 256, 2, 4, 4),
    "cfg2": (4096, 4096, 4096, 16, 32, 32),
    "cfg3_62": (2048, 11008, 4096, 12, 32, 32),
    "cfg3_75": (2048, 11008, 4096, 8, 32, 32),
    "cfg4_13b": (2048, 13824, 5120, 4, 32, 32),
    "cfg4_13b_sq": (2048, 5120, 5120, 4, 32, 32),
    "cfg4_65b_sq": (2048, 8192, 8192, 4, 32, 32),
    "cfg4_65b": (2048, 22016, 8192, 4, 32, 32),
    # m = 256 tokens is the bf16 HBM-bound point of the 87.5 % regime
    "cfg4_65b_m256": (256, 22016, 8192, 4, 32, 32),
    "cfg4_13b_m256": (256, 13824, 5120, 4, 32, 32),
    # one rank's column shard of the 8-GPU split (ceil(q/8) groups of L): kernel-only
    # scaling = T_kernel(full) / (8 T_kernel(shard)), reported beside the full config's variant
    "cfg2_shard8": (4096, 512, 4096, 16, 32, 32),
    "cfg3_75_shard8": (2048, 1376, 4096, 8, 32, 32),
    "cfg4_65b_shard8": (2048, 2752, 8192, 4, 32, 32),
}
SHARD_OF = {"cfg2_shard8": "cfg2", "cfg3_75_shard8": "cfg3_75", "cfg4_65b_shard8": "cfg4_65b"}
HEADLINE = "cfg2"
# one metric string for both arms (the driver pairs the lines by it)
METRIC = "effective TFLOPS (kept MACs) of C = A . B~, vector-wise N:M"
VARIANTS = ["cfg1:f32", "cfg2:bf16", "cfg3_62:f32", "cfg3_75:f32", "cfg4_13b:f32", "cfg4_13b_sq:f32",
            "cfg4_65b_sq:f32", "cfg4_65b:f32", "cfg4_65b_m256:f32", "cfg3_62:bf16", "cfg3_75:bf16",
            "cfg4_13b:bf16", "cfg4_13b_sq:bf16", "cfg4_65b_sq:bf16", "cfg4_65b:bf16", "cfg4_65b_m256:bf16",
            "cfg4_13b_m256:bf16", "cfg2:tf32", "cfg3_62:tf32", "cfg3_75:tf32",
            "cfg4_65b:tf32", "cfg2_shard8:f32", "cfg3_75_shard8:f32", "cfg4_65b_shard8:f32",
            "cfg2_shard8:bf16", "cfg3_75_shard8:bf16", "cfg4_65b_shard8:bf16", "cfg2:bf16at", "cfg2:f32at",
            "cfg4_65b:bf16at"]  # ...at: feature-major activations (A^T given, no per-call transpose)  # tf32 = fp32 operands on the tf32 sparse tensor cores (opt-in math)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "sm_max_mhz": 1965.0}, "fallback"


def fp32_alu_peak_tflops(sm_mhz: float, sms: int = 148) -> float:
    # FP32 FFMA: 128 lanes/SM x 2 FLOP x SMs x clock
    return sms * 128 * 2 * sm_mhz * 1e6 / 1e12


# ----------------------------------------------------------------------- clocks
class ClockSampler:
    """Samples SM clock and throttle reasons with NVML during the timed region."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x20: "sw_thermal_slowdown", 0x4: "sw_power_cap", 0x1: "gpu_idle", 0x2: "applications_clocks_setting"}

    def __init__(self, index: int):
        self.samples, self.reasons, self.ok = [], set(), False
        self.max_mhz = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.ok = False
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                try:
                    r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                except AttributeError:
                    r = self.nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.01)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ----------------------------------------------------------------------- inputs
def make_inputs(cfg, dtype, device, seed=0):
    import torch
    from paper_2503_01253_b200 import nmspmm, synth
    m, n, k, N, M, L = cfg
    gen = synth.uniform if dtype == torch.float32 else synth.bf16grid
    A = torch.from_numpy(gen((m, k), seed + 1, synth.TID_A)).to(device=device, dtype=dtype)
    Bd = torch.from_numpy(gen((k, n), seed + 2, synth.TID_B)).to(device=device, dtype=dtype)
    W = nmspmm.nm_compress(Bd, N, M, L)  # magnitude pruning on the device (offline, untimed)
    return A, Bd, W


def make_step(A, W, C, dtype, math=None, at=False):
    '''One hot-path step.  fp32: nm_spmm (CUDA-core path).  bf16 and tf32 (fp32 operands,
    math="tf32_tc"): the weight is prepacked once, outside the timed region (the paper's
    offline PreProcessing), and the step is nm_spmm_prepacked.  at=True (variants
    "f32at" / "bf16at"): the activations arrive feature-major (A^T, nm_spmm_at /
    nm_spmm_prepacked_at), so the step has no per-call transpose.'''
    import torch
    from paper_2503_01253_b200 import nmspmm
    if at:
        At = A.t().contiguous()  # the caller's layout (untimed)
        if dtype == torch.float32:
            return lambda: nmspmm.nm_spmm_at(At, W, out=C, math="f32_simt")
        PWa = nmspmm.nm_prepack(W, m_hint=A.shape[0])
        return lambda: nmspmm.nm_spmm_prepacked_at(At, PWa, out=C)
    if math == "tf32_tc":
        PWt = nmspmm.nm_prepack(W, math="tf32_tc", m_hint=A.shape[0])
        return lambda: nmspmm.nm_spmm_prepacked(A, PWt, out=C)
    if dtype == torch.float32:
        return lambda: nmspmm.nm_spmm(A, W, out=C, math="f32_simt")
    PW = nmspmm.nm_prepack(W, m_hint=A.shape[0])  # the serving batch is known when the layer is built
    return lambda: nmspmm.nm_spmm_prepacked(A, PW, out=C)


def time_steps(fn, steps, warmup, stream, flush=None):
    """W untimed warm-ups, then `steps` steps each bracketed by CUDA events on
    `stream` (L2 flush between steps, outside the events).  Returns per-step ms."""
    import torch
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    with torch.cuda.stream(stream):
        for s, e in ev:
            if flush is not None:
                flush()
            s.record(stream)
            fn()
            e.record(stream)
    torch.cuda.synchronize()
    return [s.elapsed_time(e) for s, e in ev]


def flop_count(cfg):
    m, n, k, N, M, L = cfg
    return 2.0 * m * n * (k // M * N)


def alg_bytes(cfg, e):
    m, n, k, N, M, L = cfg
    w, q = k // M * N, n // L
    return e * m * k + e * w * n + w * q + e * m * n


def measure_config(cfg, dtype, steps, warmup, flush, with_cublas=True, math=None, at=False):
    import torch
    from paper_2503_01253_b200 import nmspmm
    stream = torch.cuda.current_stream()
    A, Bd, W = make_inputs(cfg, dtype, "cuda")
    C = torch.empty(cfg[0], cfg[1], dtype=dtype, device="cuda")
    step = make_step(A, W, C, dtype, math, at)
    for _ in range(warmup):
        step()
    ms = time_steps(step, steps, 0, stream, flush)  # steps without the profiling events
    nmspmm.nm_profile_begin()
    time_steps(step, steps, 0, stream, flush)
    k_ms, k_cnt, launches = nmspmm.nm_profile_end()
    t = statistics.median(ms)
    kms = k_ms / max(1, k_cnt)
    res = {"ms": t, "tflops": flop_count(cfg) / (t * 1e-3) / 1e12, "kernel_ms": kms,
           "kernel_tflops": flop_count(cfg) / (kms * 1e-3) / 1e12, "launches_per_step": launches / steps,
           "plan": nmspmm.nm_plan_query(*cfg, dtype=dtype,
                                        math=math or ("f32_simt" if dtype == torch.float32 else "auto"))}
    if with_cublas:
        torch.backends.cuda.matmul.allow_tf32 = False
        Cd = torch.empty_like(C)
        msd = time_steps(lambda: torch.mm(A, Bd, out=Cd), steps, warmup, stream, flush)
        td = statistics.median(msd)
        m, n, k = cfg[:3]
        res.update({"cublas_ms": td, "cublas_dense_tflops": 2.0 * m * n * k / (td * 1e-3) / 1e12,
                    "speedup_vs_cublas": td / t, "target_speedup": 0.7 * cfg[4] / cfg[3]})
        if math == "tf32_tc":  # the like-for-like dense comparator: cuBLAS with TF32 tensor cores
            torch.backends.cuda.matmul.allow_tf32 = True
            mst = time_steps(lambda: torch.mm(A, Bd, out=Cd), steps, warmup, stream, flush)
            torch.backends.cuda.matmul.allow_tf32 = False
            tt = statistics.median(mst)
            res.update({"cublas_tf32_dense_tflops": 2.0 * m * n * k / (tt * 1e-3) / 1e12,
                        "speedup_vs_cublas_tf32": tt / t})
    del A, Bd, W, C
    return res, ms


def e2e_measure(cfg, dtype, steps, warmup):
    """Same metric through nm_spmm_host (host pinned buffers; H2D + kernel + D2H timed)."""
    import torch
    from paper_2503_01253_b200 import nmspmm
    m, n, k, N, M, L = cfg
    A, Bd, W = make_inputs(cfg, dtype, "cuda")
    Ah = A.cpu().pin_memory()
    Vh = W.values.cpu().pin_memory()
    Dh = W.idx.cpu().pin_memory()
    Ch = torch.empty(m, n, dtype=dtype).pin_memory()
    run = nmspmm.HostSpmm(m, n, k, N, M, L, ab_dtype=dtype, math="f32_simt" if dtype == torch.float32 else "auto")
    stream = torch.cuda.current_stream()
    ms = time_steps(lambda: run(Ah, Vh, Dh, Ch, stream=stream), steps, warmup, stream)
    t = statistics.median(ms)
    e = Ah.element_size()
    return {"value": round(flop_count(cfg) / (t * 1e-3) / 1e12, 4), "unit": "TFLOP/s (effective, kept MACs)",
            "ms_per_step": round(t, 4), "h2d_bytes_per_step": int(Ah.numel() * e + Vh.numel() * e + Dh.numel()),
            "d2h_bytes_per_step": int(Ch.numel() * Ch.element_size()),
            "path": "nm_spmm_host (C ABI, host pinned A/B'/D in, C out, synchronous)"}


def cpu_baseline(cfg, target_s=10.0):
    """The oracle as it stands (O2, fp64, OpenMP over rows) on a bounded row sample."""
    from oracle import oracle
    from paper_2503_01253_b200 import synth
    m, n, k, N, M, L = cfg
    A = synth.uniform((m, k), 1, synth.TID_A)
    B = synth.uniform((k, n), 2, synth.TID_B)
    vals, D = oracle.compress(B, N, M, L)
    threads = oracle.num_threads()
    probe = list(range(min(m, max(4, threads))))
    t0 = time.perf_counter()
    oracle.spmm_sparse_f64(A, vals, D, k, N, M, L, rows=probe)
    tp = time.perf_counter() - t0
    rows = int(min(m, max(len(probe), len(probe) * target_s / max(tp, 1e-6))))
    sample = np.linspace(0, m - 1, rows).astype(np.int64)
    t0 = time.perf_counter()
    oracle.spmm_sparse_f64(A, vals, D, k, N, M, L, rows=sample)
    t = time.perf_counter() - t0
    w = k // M * N
    return {"value": round(2.0 * rows * n * w / t / 1e12, 6), "unit": "TFLOP/s (effective, kept MACs)",
            "cores": threads, "kind": "oracle", "cpu_model": cpu_model(),
            "sample": f"{rows} of {m} rows (all {n} columns) of {cfg_name(cfg)}, O2 fp64 sparse loop, {t:.1f} s",
            "seconds": round(t, 3)}


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def cfg_name(cfg):
    for k, v in CONFIGS.items():
        if v == cfg:
            return k
    return str(cfg)


def config_dict(cfg, dtype_name, extra=None):
    m, n, k, N, M, L = cfg
    d = {"workload": f"{cfg_name(cfg)}: C[m,n] = A[m,k] . B~ (vector-wise {N}:{M}, L={L})", "m": m, "n": n,
         "k": k, "N": N, "M": M, "L": L, "sparsity": 1 - N / M, "operands": dtype_name,
         "l2": "flushed between timed steps (256 MiB write, outside the CUDA events)",
         "inputs": "synthetic U[-1,1) (splitmix64 counter PRNG), magnitude-pruned by nm_compress"}
    if extra:
        d.update(extra)
    return d


def traffic_for(kernel_key):
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f).get(kernel_key)
    return None


# ----------------------------------------------------------------------- arms
def run_reference(args):
    cfg = CONFIGS[args.config]
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    runs = []
    for _ in range(args.warmup + args.steps):
        runs.append(cpu_baseline(cfg, target_s=max(1.0, args.ref_seconds / max(1, args.steps))))
    timed = runs[args.warmup:]
    v = statistics.median(r["value"] for r in timed)
    w = cfg[2] // cfg[4] * cfg[3]
    line = {"impl": "reference", "metric": METRIC,
            "value": v, "unit": "TFLOP/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": None, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": config_dict(cfg, args.dtype, {"parallelism": "single GPU" if args.gpus == 1 else
                                                    f"col{args.gpus}"}),
            "cpu_baseline": {k: timed[-1][k] for k in ("kind", "cores", "sample", "cpu_model")} | {"value": v},
            "e2e": {"value": v, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "note": "CPU oracle (plain C, OpenMP over rows) on a bounded row sample per step; "
                    f"full step would be {2.0 * cfg[0] * cfg[1] * w / (v * 1e12):.1f} s"}
    print(json.dumps(line), flush=True)
    return 0


def bf16_kernel_name(cfg):
    """Name of the bf16 SpMM kernel the selector picks for cfg (nm_plan_query kernel id)."""
    from paper_2503_01253_b200 import nmspmm
    import torch
    m, n, k, N, M, L = cfg
    plan = nmspmm.nm_plan_query(m, n, k, N, M, L, torch.bfloat16, "bf16_tc")
    return {4: f"nm::tcs::spmm_tc_sp_kernel<{plan['bn'] // 128}> (sparse tensor cores, {plan['bn']} columns x "
               f"{plan['bm']} tokens per CTA)",
            2: "nm::spmm_tc_pair_kernel / nm::tc::spmm_tc_bf16_kernel"}.get(plan["kernel"], "spmm_generic_kernel")


def run_ours(args):
    import torch
    import torch.distributed as dist
    from paper_2503_01253_b200 import nmspmm

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    peaks, peaks_src = load_peaks()
    cfg = CONFIGS[args.config]
    dtype = torch.float32 if args.dtype == "f32" else torch.bfloat16
    flush_buf = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    flush = (lambda: flush_buf.fill_(1.0)) if not args.no_flush else None
    m, n, k, N, M, L = cfg

    if world == 1:
        stream = torch.cuda.current_stream()
        A, Bd, W = make_inputs(cfg, dtype, "cuda")
        C = torch.empty(m, n, dtype=dtype, device="cuda")
        step = make_step(A, W, C, dtype)
        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize()
        sampler = ClockSampler(local)
        with sampler:
            t0 = time.perf_counter()
            ms = time_steps(step, args.steps, 0, stream, flush)
            wall = time.perf_counter() - t0
        # the dominant kernel's time and the launch count from a second, profiled pass (the
        # library's profiling events around the kernel are kept out of the timed steps above)
        nmspmm.nm_profile_begin()
        time_steps(step, args.steps, 0, stream, flush)
        k_ms, k_cnt, launches = nmspmm.nm_profile_end()
        t_step = statistics.median(ms)
        value = flop_count(cfg) / (t_step * 1e-3) / 1e12
        kernel_ms = k_ms / max(1, k_cnt)  # dominant SpMM kernel, CUDA events on its stream
        del Bd
        if args.profile:
            print(json.dumps({"profile_run": True, "ms": t_step}), flush=True)
            return 0
        res = {}
        if not args.quick:
            torch.backends.cuda.matmul.allow_tf32 = False
            Ad = A
            Bdense = nmspmm.nm_decompress(W)  # same shape as the dense weight
            Cd = torch.empty_like(C)
            msd = time_steps(lambda: torch.mm(Ad, Bdense, out=Cd), args.steps, args.warmup, stream, flush)
            td = statistics.median(msd)
            res = {"cublas_ms": td, "cublas_dense_tflops": 2.0 * m * n * k / (td * 1e-3) / 1e12,
                   "speedup_vs_cublas": td / t_step, "target_speedup_0.7xM/N": 0.7 * M / N}
            del Bdense, Cd
        del A, W, C
        torch.cuda.empty_cache()
    else:
        raise SystemExit("multi-GPU path: see run_sharded")

    sm_mhz = peaks.get("sm_max_mhz", 1965.0)
    if dtype == torch.float32:
        peak = fp32_alu_peak_tflops(sm_mhz)
        roof = {"bound": "alu", "achieved": round(flop_count(cfg) / (kernel_ms * 1e-3) / 1e12, 3),
                "peak": round(peak, 2), "unit": "TFLOP/s", "frac": None,
                "peak_source": f"derived: 148 SMs x 128 FP32 lanes x 2 FLOP x {sm_mhz:.0f} MHz (sm_max_mhz, {peaks_src})",
                "kernel": "nm::simt::spmm_simt_f32_kernel",
                "kernel_ms_per_launch": round(kernel_ms, 4), "kernel_share_of_step": round(kernel_ms / t_step, 4),
                "algorithmic_flops_per_launch": flop_count(cfg),
                "algorithmic_bytes_per_launch": alg_bytes(cfg, 4)}
    else:
        peak = peaks.get("bf16_tflops", 1590.0)
        roof = {"bound": "tensor", "achieved": round(flop_count(cfg) / (kernel_ms * 1e-3) / 1e12, 3),
                "peak": peak, "unit": "TFLOP/s", "frac": None, "peak_source": f"bf16_tflops ({peaks_src})",
                "kernel": bf16_kernel_name(cfg), "kernel_ms_per_launch": round(kernel_ms, 4),
                "kernel_share_of_step": round(kernel_ms / t_step, 4), "algorithmic_flops_per_launch": flop_count(cfg),
                "algorithmic_bytes_per_launch": alg_bytes(cfg, 2)}
    roof["frac"] = round(roof["achieved"] / roof["peak"], 4)
    tr = traffic_for(f"{args.config}_{args.dtype}")
    roof["traffic"] = tr["dram_bytes_per_launch"] if tr else None
    roof["traffic_source"] = tr["source"] if tr else "no ncu capture for this config"

    line = {"metric": METRIC,
            "value": round(value, 4), "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(t_step, 4), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": args.dtype, "data": "synthetic",
            "config": config_dict(cfg, args.dtype, {"parallelism": "single GPU"}),
            "gpu_launches": launches, "roofline": roof, "clocks": sampler.summary(),
            "wall_s_timed_region": round(wall, 4)}
    line.update({k2: (round(v2, 4) if isinstance(v2, float) else v2) for k2, v2 in res.items()})
    if not args.quick:
        line["e2e"] = e2e_measure(cfg, dtype, max(3, args.steps // 4), args.warmup)
        line["cpu_baseline"] = cpu_baseline(cfg, target_s=args.ref_seconds)
        variants = []
        for item in args.variants.split(",") if args.variants else []:
            name, _, vdt_full = item.partition(":")
            vdt_full = vdt_full or args.dtype
            at = vdt_full.endswith("at")  # feature-major activations (A^T given): no per-call transpose
            vdt = vdt_full[:-2] if at else vdt_full
            vcfg = CONFIGS[name]
            tdt = torch.bfloat16 if vdt == "bf16" else torch.float32
            r, _ = measure_config(vcfg, tdt, max(5, args.steps // 2), args.warmup, flush,
                                  math="tf32_tc" if vdt == "tf32" else None, at=at)
            # tf32 dense peak = the measured bf16 peak x the nominal tf32/bf16 ratio 1/2
            peak_v = (fp32_alu_peak_tflops(sm_mhz) if vdt == "f32" else
                      peaks.get("bf16_tflops", 1590.0) / (2.0 if vdt == "tf32" else 1.0))
            # the relevant roofline: the slower of compute (FLOPs / peak) and HBM (algorithmic bytes /
            # measured copy bandwidth); frac = that time / the kernel's time
            e_v = 2 if vdt == "bf16" else 4
            t_c = flop_count(vcfg) / (peak_v * 1e12)
            t_m = alg_bytes(vcfg, e_v) / (peaks.get("hbm_gbs", 6650.0) * 1e9)
            t_k = r["kernel_ms"] * 1e-3
            variants.append({"config": name, "dtype": vdt, "m_n_k": vcfg[:3], "N:M": f"{vcfg[3]}:{vcfg[4]}",
                             "a_layout": "A^T given (nm_spmm_at)" if at else "A row-major",
                             "L": vcfg[5], "tflops": round(r["tflops"], 3), "ms": round(r["ms"], 4),
                             "kernel_tflops": round(r["kernel_tflops"], 3), "kernel_ms": round(r["kernel_ms"], 5),
                             "roofline_frac": round(max(t_c, t_m) / t_k, 4),
                             "roofline_bound": ("hbm" if t_m > t_c else "alu" if vdt == "f32" else "tensor"),
                             "hbm_gbs_achieved": round(alg_bytes(vcfg, e_v) / t_k / 1e9, 1),
                             "cublas_dense_tflops": round(r["cublas_dense_tflops"], 3),
                             "speedup_vs_cublas": round(r["speedup_vs_cublas"], 3),
                             "target_speedup": round(r["target_speedup"], 3)}
                            | ({"cublas_tf32_dense_tflops": round(r["cublas_tf32_dense_tflops"], 3),
                                "speedup_vs_cublas_tf32": round(r["speedup_vs_cublas_tf32"], 3)}
                               if "cublas_tf32_dense_tflops" in r else {}))
            torch.cuda.empty_cache()
        # kernel-only 8-GPU scaling of the column-sharded layer from one GPU: the full config's kernel
        # time over 8 x one shard's (the all-gather is not included; SURVEY 8(e) reporting (i))
        kms = {(u["config"], u["dtype"]): u["kernel_ms"] for u in variants if u["a_layout"] == "A row-major"}
        if roof.get("kernel_ms_per_launch"):
            kms.setdefault((args.config, args.dtype), roof["kernel_ms_per_launch"])
        for v in variants:
            full = kms.get((SHARD_OF.get(v["config"]), v["dtype"]))
            if full:
                v["kernel_only_scaling_8gpu"] = round(full / (8 * v["kernel_ms"]), 4)
        line["variants"] = variants
    print(json.dumps(line), flush=True)
    return 0


def run_sharded(args):
    """N > 1: column groups sharded over ranks, NCCL all-gather + unshard kernel."""
    import torch
    import torch.distributed as dist
    from paper_2503_01253_b200 import nmspmm, sharded

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29517")
    dist.init_process_group("nccl", device_id=torch.device("cuda", local), rank=rank, world_size=world)
    cfg = CONFIGS[args.config]
    dtype = torch.float32 if args.dtype == "f32" else torch.bfloat16
    m, n, k, N, M, L = cfg
    A, Bd, _ = make_inputs(cfg, dtype, "cuda")  # A replicated (column-parallel input), B generated identically
    # row slices for the NCCL overlap: measured per-rank compute (profiles/r02m_shard_chunks.txt)
    # grows with the slice count much faster than the all-gather it hides (cfg2 fp32 at G = 8:
    # 226 us in one slice, 306 / 609 us in 2 / 4, against a 76 us all-gather floor), so one slice
    # unless --chunks asks for more
    chunks = args.chunks if args.chunks > 0 else 1
    layer = sharded.ShardedNmLinear.from_dense(Bd, N, M, L, dist.group.WORLD, exchange=args.exchange, chunks=chunks,
                                               m_hint=m)
    del Bd
    flush_buf = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    flush = (lambda: flush_buf.fill_(1.0)) if not args.no_flush else None
    stream = torch.cuda.current_stream()
    step = lambda: layer(A)  # noqa: E731
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    sampler = ClockSampler(local)
    with sampler:
        ms = time_steps(step, args.steps, 0, stream, flush)
    dist.barrier()
    nmspmm.nm_profile_begin()  # kernel time and launches from a second, profiled pass
    time_steps(step, args.steps, 0, stream, flush)
    k_ms, k_cnt, launches = nmspmm.nm_profile_end()
    dist.barrier()
    t = torch.tensor([statistics.median(ms), k_ms / max(1, k_cnt)], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)  # max over ranks (step, dominant kernel)
    t_step, t_kernel = t[0].item(), t[1].item()
    # end to end: each rank copies A from pinned host memory, runs the layer, rank 0 reads C back
    Ah = A.cpu().pin_memory()
    Ch = torch.empty(m, n, dtype=dtype).pin_memory()
    Ad = torch.empty_like(A)

    def e2e_step():
        Ad.copy_(Ah, non_blocking=True)
        C = layer(Ad)
        if rank == 0:
            Ch.copy_(C, non_blocking=True)

    mse = time_steps(e2e_step, max(3, args.steps // 4), args.warmup, stream)
    te = torch.tensor([statistics.median(mse)], device="cuda")
    dist.all_reduce(te, op=dist.ReduceOp.MAX)
    if rank == 0:
        value = flop_count(cfg) / (t_step * 1e-3) / 1e12
        peaks, peaks_src = load_peaks()
        sm_mhz = peaks.get("sm_max_mhz", 1965.0)
        local_flops = flop_count(cfg) * layer.nr / n  # this rank's (padded) share
        peak = fp32_alu_peak_tflops(sm_mhz) if dtype == torch.float32 else peaks.get("bf16_tflops", 1590.0)
        ach = local_flops / (t_kernel * 1e-3) / 1e12
        line = {"metric": METRIC,
                "value": round(value, 4), "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": round(t_step, 4), "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": args.dtype, "data": "synthetic",
                "config": config_dict(cfg, args.dtype, {"parallelism": f"col{world} (column groups sharded, " + (
                    f"NCCL all-gather of C, {chunks} overlapped row slices)" if args.exchange == "nccl" else
                    "fused peer-store epilogue over CUDA IPC / NVLink + flag barrier)")}),
                "gpu_launches": int(launches), "clocks": sampler.summary(),
                "roofline": {"bound": "alu" if dtype == torch.float32 else "tensor", "achieved": round(ach, 3),
                             "peak": round(peak, 2), "unit": "TFLOP/s", "frac": round(ach / peak, 4),
                             "traffic": None, "kernel": "local nm_spmm (max over ranks)",
                             "kernel_ms_per_launch": round(t_kernel, 4)},
                "e2e": {"value": round(flop_count(cfg) / (te.item() * 1e-3) / 1e12, 4),
                        "unit": "TFLOP/s (effective, kept MACs)", "ms_per_step": round(te.item(), 4),
                        "h2d_bytes_per_step": int(Ah.numel() * Ah.element_size()),
                        "d2h_bytes_per_step": int(Ch.numel() * Ch.element_size()),
                        "path": f"pinned A -> each rank, sharded layer ({args.exchange} exchange), C -> host on rank 0"},
                "kernel_only_tflops_all_ranks": round(flop_count(cfg) / (t_kernel * 1e-3) / 1e12, 4),
                "allgather_floor_ms": round((world - 1) / world * m * n * A.element_size() / 770e9 * 1e3, 4)}
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()
    return 0


def launch_check() -> int:
    '''--launch-check: every rank joins a gloo group and contributes 1 to an all-reduce; rank 0
    prints how many ranks it saw (tests the --gpus N self-launch without a GPU).'''
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        dist.init_process_group("gloo")
    t = torch.ones(1)
    if world > 1:
        dist.all_reduce(t)
    if rank == 0:
        print(json.dumps({"launch_check": True, "world_size": world, "ranks_seen": int(t.item())}), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def self_launch(n: int) -> int:
    '''`python bench.py --gpus N` without torchrun: re-run this command as N ranks under
    torch.distributed.run (one process per GPU, rendezvous on 127.0.0.1); rank 0 prints the line.'''
    import socket
    import subprocess
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.run(cmd).returncode


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=HEADLINE, choices=sorted(CONFIGS))
    ap.add_argument("--dtype", default="f32", choices=["f32", "bf16"])
    ap.add_argument("--variants", default=",".join(VARIANTS))
    ap.add_argument("--quick", action="store_true", help="headline kernel only (no cuBLAS / e2e / oracle)")
    ap.add_argument("--profile", action="store_true", help="minimal run for ncu")
    ap.add_argument("--no-flush", action="store_true")
    ap.add_argument("--sharded", action="store_true", help="column-sharded path even at one rank (testing)")
    ap.add_argument("--ref-seconds", type=float, default=10.0)
    ap.add_argument("--chunks", type=int, default=0,
                    help="sharded NCCL path: row slices whose all-gather overlaps the next slice (0 = 1 slice)")
    ap.add_argument("--launch-check", action="store_true",
                    help="start the ranks, all-reduce a count over gloo, rank 0 prints it (no GPU needed)")
    ap.add_argument("--exchange", default="nccl", choices=["nccl", "p2p"],
                    help="sharded path: NCCL all-gather + unshard, or the fused peer-store epilogue (fp32)")
    args = ap.parse_args()
    if args.warmup < 3 and not args.profile:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return self_launch(args.gpus)
    if args.launch_check:
        return launch_check()
    if args.impl == "reference":
        return run_reference(args)
    if int(os.environ.get("WORLD_SIZE", "1")) > 1 or args.sharded:
        return run_sharded(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
