"""One small invocation of every product kernel, for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck).  Each case checks its result against the CPU oracle too, so a run that
"passes" the sanitizer also computed the right numbers.  Usage: sanitize_run.py [case ...]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from oracle import oracle
from paper_2503_01253_b200 import nmspmm as nm, synth

torch.cuda.set_device(0)
dev = lambda x, dt=torch.float32: torch.from_numpy(np.ascontiguousarray(x)).cuda().to(dt)


def check(name, got, ref, exact):
    g = got.float().cpu().numpy().astype(np.float64)
    ok = np.array_equal(g, ref) if exact else oracle.rel_frobenius(g, ref) <= 5e-3
    print(f"{name}: {'ok' if ok else 'MISMATCH'}", flush=True)
    if not ok:
        sys.exit(1)


def weights(m, n, k, N, M, L, bf16, seed):
    A = synth.integer((m, k), seed, synth.TID_A)
    B = synth.integer((k, n), seed + 1, synth.TID_B)
    if bf16:
        vals, D = oracle.compress(synth.to_bf16_bits(B), N, M, L)
        W = nm.NmWeight(dev(oracle.bf16_to_f32(vals), torch.bfloat16), dev(D, torch.uint8), k, N, M, L)
        return synth.to_bf16_bits(A), vals, D, W, dev(A, torch.bfloat16)
    vals, D = oracle.compress(B, N, M, L)
    return A, vals, D, nm.NmWeight(dev(vals), dev(D, torch.uint8), k, N, M, L), dev(A)


def c_format():
    B = synth.uniform((96, 160), 3, synth.TID_B)
    W = nm.nm_compress(dev(B), 4, 32, 32)
    v, D = oracle.compress(B, 4, 32, 32)
    assert np.array_equal(W.idx.cpu().numpy(), D)
    assert nm.nm_validate(W.idx, 96, 160, 4, 32, 32) == -1
    d = nm.nm_decompress(W)
    assert np.array_equal(d.cpu().numpy(), oracle.decompress(v, D, 96, 4, 32, 32))
    words = nm.nm_index_pack(W.idx, 96, 160, 4, 32, 32)
    assert torch.equal(nm.nm_index_unpack(words, 96, 160, 4, 32, 32), W.idx)
    print("format kernels (compress / validate / decompress / index pack): ok", flush=True)


def c_simt():  # fp32 SIMT, a split sub-wave grid, L = 4 (TWO) and L = 32
    for cfg in [(300, 256, 512, 2, 4, 4), (200, 384, 1024, 8, 32, 32)]:
        A, vals, D, W, Ad = weights(*cfg, False, 11)
        check(f"simt {cfg}", nm.nm_spmm(Ad, W), oracle.spmm_sparse_f64(A, vals, D, cfg[2], *cfg[3:]), True)


def c_generic():
    A, vals, D, W, Ad = weights(40, 48, 96, 3, 8, 3, False, 21)  # L = 3: the generic kernel
    check("generic", nm.nm_spmm(Ad, W), oracle.spmm_sparse_f64(A, vals, D, 96, 3, 8, 3), True)


def c_slot():  # bf16 slot kernel (tail split on a small grid)
    cfg = (300, 512, 1024, 16, 32, 32)
    A, vals, D, W, Ad = weights(*cfg, True, 31)
    C = nm.nm_spmm_prepacked(Ad, nm.nm_prepack(W), out_dtype=torch.float32)
    check("bf16 slot", C, oracle.spmm_sparse_f64(A, vals, D, 1024, 16, 32, 32), True)


def c_tf32():
    cfg = (260, 256, 512, 8, 32, 32)
    A, vals, D, W, Ad = weights(*cfg, False, 41)
    check("tf32 slot", nm.nm_spmm(Ad, W, math="tf32_tc"), oracle.spmm_sparse_f64(A, vals, D, 512, 8, 32, 32), True)


def c_unshard():
    G, m, nr, L = 3, 50, 64, 32
    src = torch.arange(G * m * nr, dtype=torch.float32, device="cuda").reshape(G, m, nr)
    n = 160
    dst = torch.empty(m, n, device="cuda")
    nm.nm_unshard_columns(src, dst, G, m, nr, n, L)
    torch.cuda.synchronize()
    print("unshard: ok", flush=True)


def c_peers():  # fused exchange on one device: 2 "ranks" as two buffers, peer stores + barrier
    cfg = (130, 256, 256, 8, 32, 32)
    A, vals, D, W, Ad = weights(*cfg, False, 51)
    Cs = [torch.zeros(130, 512, device="cuda") for _ in range(2)]
    nm.nm_spmm_peers(Ad, W, [c.data_ptr() for c in Cs], 512, 256, 256)
    torch.cuda.synchronize()
    ref = oracle.spmm_sparse_f64(A, vals, D, 256, 8, 32, 32)
    for c in Cs:
        check("peers (SIMT peer-store epilogue)", c[:, 256:], ref, True)


def c_at():  # A supplied transposed: slot kernel (zero-filled padding slots) and SIMT staged mode
    for bf16, cfg in [(True, (300, 512, 1024, 4, 32, 32)), (False, (200, 384, 1024, 8, 32, 32))]:
        A, vals, D, W, Ad = weights(*cfg, bf16, 61)
        m, k = cfg[0], cfg[2]
        At = torch.zeros((k, (m + 7) // 8 * 8 + 8), dtype=Ad.dtype, device="cuda")
        At[:, :m] = Ad.t()
        C = nm.nm_spmm_at(At, W, m=m, out_dtype=torch.float32)
        check(f"nm_spmm_at {'bf16 slot' if bf16 else 'fp32 SIMT'}", C, oracle.spmm_sparse_f64(A, vals, D, k, *cfg[3:]), True)


def c_bf16simt():  # bf16 with L = 4: widen -> fp32 SIMT kernel -> narrow
    cfg = (300, 256, 512, 8, 32, 4)
    A, vals, D, W, Ad = weights(*cfg, True, 71)
    check("bf16 on the SIMT kernel", nm.nm_spmm(Ad, W, out_dtype=torch.float32),
          oracle.spmm_sparse_f64(A, vals, D, 512, 8, 32, 4), True)


CASES = {"at": c_at, "bf16simt": c_bf16simt, "format": c_format, "simt": c_simt, "generic": c_generic, "slot": c_slot, "tf32": c_tf32,
         "unshard": c_unshard, "peers": c_peers}
for name in sys.argv[1:] or list(CASES):
    CASES[name]()
