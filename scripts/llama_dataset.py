"""The paper's evaluation protocol on B200: a 100-point LLaMA-shape
dataset -- m in {256, 512, 1024, 2048, 4096} x 20 (n, k) tuples of LLaMA-7B/13B/30B/65B linear
layers (q/k/v/o, fused qkv, up/gate, fused gate+up, down) -- at 50 / 62.5 / 75 / 87.5 % (16:32,
12:32, 8:32, 4:32, L = 32), fp32 (SIMT kernel, vs cuBLAS SGEMM) and bf16 (sparse-TC kernel with prepacked
weights, vs cuBLAS bf16); LLAMA_DT=tf32 runs fp32 operands on the tf32 sparse-TC kernel against
cuBLAS with TF32 tensor cores.  Kernel-event times, synthetic weights, L2 not flushed (weights
and activations of the large shapes exceed L2).  Writes CSV rows to stdout."""
import sys, os, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2503_01253_b200 import nmspmm, synth

HID = {"7b": (4096, 11008), "13b": (5120, 13824), "30b": (6656, 17920), "65b": (8192, 22016)}
NK = []
for h, f in HID.values():
    NK += [(h, h), (3 * h, h), (f, h), (2 * f, h), (h, f)]  # o/q/k/v, fused qkv, up/gate, gate+up, down
MS = [256, 512, 1024, 2048, 4096]
NMS = [(16, 32), (12, 32), (8, 32), (4, 32)]  # 50 / 62.5 / 75 / 87.5 %


def timed(fn, reps=5):
    for _ in range(2):
        fn()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for s, e in ev:
        s.record(); fn(); e.record()
    torch.cuda.synchronize()
    return statistics.median(s.elapsed_time(e) for s, e in ev)


TF32 = os.environ.get("LLAMA_DT") == "tf32"
torch.backends.cuda.matmul.allow_tf32 = TF32
print("dtype,m,n,k,N,M,ms,tflops_eff,cublas_ms,speedup,target", flush=True)
for (n, k) in NK:
    for dt in ((torch.float32,) if TF32 else (torch.float32, torch.bfloat16)):
        gen = synth.uniform if dt == torch.float32 else synth.bf16grid
        Bd = torch.from_numpy(gen((k, n), 2, synth.TID_B)).cuda().to(dt)
        Ws = {nm_: nmspmm.nm_compress(Bd, nm_[0], nm_[1], 32) for nm_ in NMS}
        PWs = ({key: nmspmm.nm_prepack(W, math="tf32_tc" if TF32 else "auto") for key, W in Ws.items()}
               if (dt == torch.bfloat16 or TF32) else {})
        for m in MS:
            A = torch.from_numpy(gen((m, k), 1, synth.TID_A)).cuda().to(dt)
            C = torch.empty(m, n, device="cuda", dtype=dt)
            tdense = timed(lambda: torch.mm(A, Bd, out=C))
            for (N, M) in NMS:
                if dt == torch.float32 and not TF32:
                    W = Ws[(N, M)]
                    t = timed(lambda: nmspmm.nm_spmm(A, W, out=C, math="f32_simt"))
                else:
                    PW = PWs[(N, M)]
                    t = timed(lambda: nmspmm.nm_spmm_prepacked(A, PW, out=C))
                fl = 2.0 * m * n * (k // M * N)
                print(f"{'tf32' if TF32 else 'f32' if dt == torch.float32 else 'bf16'},{m},{n},{k},{N},{M},{t:.4f},{fl / t / 1e9:.2f},"
                      f"{tdense:.4f},{tdense / t:.3f},{0.7 * M / N:.2f}", flush=True)
            del A, C
        del Bd, Ws, PWs
        torch.cuda.empty_cache()
