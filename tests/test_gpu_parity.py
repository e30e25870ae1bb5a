"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the
same seeded inputs.  Bars (BASELINE.json north star): compression and indices
bit-exact; fp32 CUDA-core C within 1e-5 relative Frobenius of the fp64 oracle
(O2); tf32/bf16 within 5e-3; integer-valued inputs bit-exact on every path."""
import os

import numpy as np
import pytest
import torch

from paper_2503_01253_b200 import synth

pytestmark = pytest.mark.gpu

TOL_F32 = 1e-5
TOL_BF16 = 5e-3


@pytest.fixture(scope="module")
def nm():
    from paper_2503_01253_b200 import nmspmm
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    nmspmm.lib()
    return nmspmm


def dev(x: np.ndarray, dtype=torch.float32):
    t = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    return t.to(dtype) if t.dtype != dtype else t


def bf16_bits(t: torch.Tensor) -> np.ndarray:
    return t.cpu().view(torch.int16).numpy().view(np.uint16)


# --------------------------------------------------------------- compression
COMPRESS_CASES = [(2, 4, 4), (3, 8, 1), (2, 8, 8), (1, 8, 4), (16, 32, 32), (12, 32, 32), (4, 32, 64),
                  (8, 32, 32), (5, 8, 3), (1, 2, 1), (64, 128, 16), (4, 4, 4)]


@pytest.mark.parametrize("N,M,L", COMPRESS_CASES)
@pytest.mark.parametrize("kind", ["uniform", "integer"])
def test_compress_bit_exact(nm, oracle, N, M, L, kind):
    k, n = 3 * M, 5 * L
    B = synth.make(kind, (k, n), 7 + N, synth.TID_B)
    vals_o, D_o = oracle.compress(B, N, M, L)
    W = nm.nm_compress(dev(B), N, M, L)
    assert np.array_equal(W.idx.cpu().numpy(), D_o)
    assert np.array_equal(W.values.cpu().numpy().view(np.uint32), vals_o.view(np.uint32))
    assert nm.nm_validate(W.idx, k, n, N, M, L) == -1
    dense = nm.nm_decompress(W)
    assert np.array_equal(dense.cpu().numpy(), oracle.decompress(vals_o, D_o, k, N, M, L))


@pytest.mark.parametrize("N,M,L", [(16, 32, 32), (2, 4, 4), (3, 8, 2)])
def test_compress_bf16_bit_exact(nm, oracle, N, M, L):
    k, n = 4 * M, 6 * L
    B = synth.uniform((k, n), 3, synth.TID_B)
    vals_o, D_o = oracle.compress(B, N, M, L, values_bf16=True)
    W = nm.nm_compress(dev(B), N, M, L, values_dtype=torch.bfloat16)
    assert np.array_equal(W.idx.cpu().numpy(), D_o)
    assert np.array_equal(bf16_bits(W.values), vals_o)
    Bh = synth.bf16grid((k, n), 4, synth.TID_B)
    vh_o, Dh_o = oracle.compress(synth.to_bf16_bits(Bh), N, M, L)
    Wh = nm.nm_compress(dev(Bh, torch.bfloat16), N, M, L)
    assert np.array_equal(Wh.idx.cpu().numpy(), Dh_o) and np.array_equal(bf16_bits(Wh.values), vh_o)


@pytest.mark.parametrize("k,n,N,M,L", [(4096, 4096, 16, 32, 32), (4096, 11008, 8, 32, 32), (8192, 22016, 4, 32, 32)])
def test_compress_bit_exact_full_size(nm, oracle, k, n, N, M, L):
    B = synth.uniform((k, n), 2, synth.TID_B)
    vals_o, D_o = oracle.compress(B, N, M, L)
    W = nm.nm_compress(dev(B), N, M, L)
    assert np.array_equal(W.idx.cpu().numpy(), D_o)
    assert np.array_equal(W.values.cpu().numpy().view(np.uint32), vals_o.view(np.uint32))


def test_compress_nan_and_inf(nm):
    B = synth.uniform((64, 64), 1, 2)
    B[5, 7] = np.nan
    with pytest.raises(nm.NmError) as e:
        nm.nm_compress(dev(B), 2, 4, 4)
    assert e.value.status == 4
    B[5, 7] = np.inf
    W = nm.nm_compress(dev(B), 1, 4, 4)
    assert W.idx[1, 1].item() == 1


def test_validate_matches_oracle(nm, oracle):
    k, n, N, M, L = 64, 32, 4, 16, 4
    D = synth.random_mask(k, n, N, M, L, seed=9)
    assert nm.nm_validate(dev(D, torch.uint8), k, n, N, M, L) == -1 == oracle.validate(D, k, n, N, M, L)
    bad = D.copy()
    bad[5, 3] = M
    bad[9, 1] = bad[8, 1]
    assert nm.nm_validate(dev(bad, torch.uint8), k, n, N, M, L) == oracle.validate(bad, k, n, N, M, L)


# --------------------------------------------------------------- fp32 SpMM
SPMM_CASES = [
    # (m, n, k, N, M, L): several tiles + ragged tails (m % 128, n % 128, partial last panel)
    (256, 256, 256, 2, 4, 4),      # cfg1
    (300, 288, 320, 16, 32, 32),
    (130, 136, 96, 12, 32, 8),
    (257, 384, 512, 8, 32, 32),
    (64, 520, 256, 4, 32, 8),
    (200, 192, 192, 1, 8, 4),
    (128, 256, 128, 3, 8, 16),
    (96, 128, 224, 32, 32, 32),    # N = M (dense)
    (129, 128, 256, 16, 32, 64),
    (33, 96, 96, 2, 8, 12),        # L not a divisor of the tile
    (70, 64, 64, 2, 4, 1),         # L = 1 -> generic kernel
    (70, 66, 64, 2, 8, 3),         # L = 3 -> generic kernel
    (40, 64, 256, 64, 128, 16),    # M > 64 -> generic kernel
    (1, 128, 64, 2, 4, 4),         # single row
]


def run_f32(nm, oracle, m, n, k, N, M, L, kind="uniform", seed=0):
    A = synth.make(kind, (m, k), 100 + seed, synth.TID_A)
    B = synth.make(kind, (k, n), 200 + seed, synth.TID_B)
    vals, D = oracle.compress(B, N, M, L)
    W = nm.NmWeight(dev(vals), dev(D, torch.uint8), k, N, M, L)
    C = nm.nm_spmm(dev(A), W).cpu().numpy()
    return A, vals, D, C


@pytest.mark.parametrize("m,n,k,N,M,L", SPMM_CASES)
def test_spmm_f32_vs_oracle(nm, oracle, m, n, k, N, M, L):
    A, vals, D, C = run_f32(nm, oracle, m, n, k, N, M, L)
    ref = oracle.spmm_sparse_f64(A, vals, D, k, N, M, L)
    err = oracle.rel_frobenius(C, ref)
    assert err <= TOL_F32, err


@pytest.mark.parametrize("m,n,k,N,M,L", SPMM_CASES)
def test_spmm_f32_integer_bit_exact(nm, oracle, m, n, k, N, M, L):
    A, vals, D, C = run_f32(nm, oracle, m, n, k, N, M, L, kind="integer", seed=1)
    ref = oracle.spmm_sparse_f64(A, vals, D, k, N, M, L)
    assert np.array_equal(C.astype(np.float64), ref)


def test_spmm_f32_identity_a(nm, oracle):
    k, n, N, M, L = 256, 256, 8, 32, 32
    B = synth.uniform((k, n), 5, synth.TID_B)
    vals, D = oracle.compress(B, N, M, L)
    W = nm.NmWeight(dev(vals), dev(D, torch.uint8), k, N, M, L)
    C = nm.nm_spmm(torch.eye(k, device="cuda"), W)
    assert torch.equal(C, nm.nm_decompress(W))


def test_spmm_f32_all_ones(nm):
    m, n, k, N, M, L = 130, 256, 192, 12, 32, 32
    w = k // M * N
    D = synth.random_mask(k, n, N, M, L, seed=4)
    W = nm.NmWeight(torch.ones(w, n, device="cuda"), dev(D, torch.uint8), k, N, M, L)
    C = nm.nm_spmm(torch.ones(m, k, device="cuda"), W)
    assert bool((C == w).all())


def test_spmm_f32_dense_matches_cublas(nm):
    """N = M: the method is a dense GEMM (pin i); compare with cuBLAS fp32 (TF32 off)."""
    m, n, k = 512, 384, 256
    torch.backends.cuda.matmul.allow_tf32 = False
    A = dev(synth.uniform((m, k), 1, 1))
    B = dev(synth.uniform((k, n), 2, 2))
    W = nm.nm_compress(B, 32, 32, 32)
    C = nm.nm_spmm(A, W)
    ref = A.double() @ B.double()
    assert ((C.double() - ref).norm() / ref.norm()).item() < TOL_F32
    assert ((torch.mm(A, B).double() - ref).norm() / ref.norm()).item() < TOL_F32


def test_spmm_f32_deterministic(nm, oracle):
    m, n, k, N, M, L = 512, 512, 1024, 8, 32, 32
    A = dev(synth.uniform((m, k), 3, 1))
    W = nm.nm_compress(dev(synth.uniform((k, n), 4, 2)), N, M, L)
    C1 = nm.nm_spmm(A, W)
    C2 = nm.nm_spmm(A, W)
    assert torch.equal(C1, C2)


def test_spmm_empty_and_errors(nm):
    W = nm.nm_compress(dev(synth.uniform((64, 64), 1, 2)), 2, 4, 4)
    C = nm.nm_spmm(torch.empty(0, 64, device="cuda"), W)
    assert C.shape == (0, 64)
    with pytest.raises(nm.NmError):
        nm.nm_spmm(torch.zeros(8, 64, device="cuda"), W, out_dtype=torch.bfloat16)


@pytest.mark.parametrize("cfg", ["cfg2", "cfg3_62", "cfg3_75", "cfg4_65b"])
def test_spmm_f32_full_size_sampled(nm, oracle, cfg):
    """BASELINE.json sizes, bench launch configuration; oracle on a row sample."""
    m, n, k, N, M, L = {"cfg2": (4096, 4096, 4096, 16, 32, 32), "cfg3_62": (2048, 11008, 4096, 12, 32, 32),
                        "cfg3_75": (2048, 11008, 4096, 8, 32, 32), "cfg4_65b": (2048, 22016, 8192, 4, 32, 32)}[cfg]
    A = synth.uniform((m, k), 11, synth.TID_A)
    B = synth.uniform((k, n), 12, synth.TID_B)
    W = nm.nm_compress(dev(B), N, M, L)
    C = nm.nm_spmm(dev(A), W)
    rows = np.array([0, 1, 127, 128, m // 2 + 3, m - 1])
    vals = W.values.cpu().numpy()
    D = W.idx.cpu().numpy()
    ref = oracle.spmm_sparse_f64(A, vals, D, k, N, M, L, rows=rows)
    err = oracle.rel_frobenius(C[torch.from_numpy(rows).cuda()].cpu().numpy(), ref)
    assert err <= TOL_F32, err


# --------------------------------------------------------------- bf16 SpMM
@pytest.mark.parametrize("m,n,k,N,M,L", [(256, 256, 256, 16, 32, 32), (130, 192, 96, 4, 32, 32),
                                         (64, 64, 64, 2, 4, 4)])
@pytest.mark.parametrize("cdt", [torch.bfloat16, torch.float32])
def test_spmm_bf16_vs_oracle(nm, oracle, m, n, k, N, M, L, cdt):
    A = synth.bf16grid((m, k), 21, synth.TID_A)
    B = synth.bf16grid((k, n), 22, synth.TID_B)
    vals, D = oracle.compress(synth.to_bf16_bits(B), N, M, L)
    W = nm.NmWeight(dev(oracle.bf16_to_f32(vals), torch.bfloat16), dev(D, torch.uint8), k, N, M, L)
    C = nm.nm_spmm(dev(A, torch.bfloat16), W, out_dtype=cdt).float().cpu().numpy()
    ref = oracle.spmm_sparse_f64(synth.to_bf16_bits(A), vals, D, k, N, M, L)
    assert oracle.rel_frobenius(C, ref) <= TOL_BF16


def test_spmm_bf16_integer_exact_fp32_out(nm, oracle):
    m, n, k, N, M, L = 200, 256, 256, 8, 32, 32
    A = synth.integer((m, k), 31, synth.TID_A)
    B = synth.integer((k, n), 32, synth.TID_B)
    vals, D = oracle.compress(synth.to_bf16_bits(B), N, M, L)
    W = nm.NmWeight(dev(oracle.bf16_to_f32(vals), torch.bfloat16), dev(D, torch.uint8), k, N, M, L)
    C = nm.nm_spmm(dev(A, torch.bfloat16), W, out_dtype=torch.float32).cpu().numpy()
    assert np.array_equal(C.astype(np.float64), oracle.spmm_sparse_f64(synth.to_bf16_bits(A), vals, D, k, N, M, L))


# --------------------------------------------------------------- host path / assembly
def test_spmm_host_path(nm, oracle):
    m, n, k, N, M, L = 257, 256, 512, 16, 32, 32
    A = synth.uniform((m, k), 41, 1)
    B = synth.uniform((k, n), 42, 2)
    vals, D = oracle.compress(B, N, M, L)
    run = nm.HostSpmm(m, n, k, N, M, L)
    C = torch.empty(m, n).pin_memory()
    run(torch.from_numpy(A).pin_memory(), torch.from_numpy(vals).pin_memory(), torch.from_numpy(D).pin_memory(), C)
    assert oracle.rel_frobenius(C.numpy(), oracle.spmm_sparse_f64(A, vals, D, k, N, M, L)) <= TOL_F32


@pytest.mark.parametrize("G", [1, 2, 3, 8])
def test_unshard_columns(nm, G):
    m, L, q = 37, 8, 43
    n = q * L
    full = torch.arange(m * n, dtype=torch.float32, device="cuda").reshape(m, n)
    nr = L * ((q + G - 1) // G)
    src = torch.full((G, m, nr), -1.0, device="cuda")
    for r in range(G):
        g0, g1 = r * q // G, (r + 1) * q // G
        src[r, :, :(g1 - g0) * L] = full[:, g0 * L:g1 * L]
    dst = torch.empty(m, n, device="cuda")
    nm.nm_unshard_columns(src, dst, G, m, nr, n, L)
    assert torch.equal(dst, full)


# --------------------------------------------------------------- tcgen05 bf16 path
TC_CASES = [
    # (m, n, k, N, M, L)
    (128, 128, 128, 16, 32, 32),
    (256, 256, 256, 16, 32, 32),
    (300, 384, 512, 16, 32, 32),    # ragged m, 3 column tiles, 4 panels
    (128, 192, 96, 4, 32, 32),      # ragged n tile, single partial panel
    (200, 256, 384, 12, 32, 32),    # BKW = 48
    (130, 256, 256, 8, 32, 16),     # L = 16 (N = 16 MMAs)
    (130, 256, 256, 8, 32, 64),     # L = 64 (128-byte swizzle)
    (64, 256, 256, 8, 32, 128),     # L = 128 (two 64-column atoms per group)
    (96, 128, 64, 8, 8, 32),        # M = 8 windows, dense N = M
    (257, 128, 640, 2, 16, 32),     # BKW padded 40 -> 48
]


# NM_TC_SP, NM_BF16_SIMT, kernel id (0: the generic correctness kernel, 5: bf16 on the fp32 SIMT kernel)
TC_PATHS = {"sp": ("1", "1", 4), "generic": ("0", "0", 0), "simt": ("0", "1", 5)}


def use_tc_path(monkeypatch, path):
    sp, simt, kid = TC_PATHS[path]
    monkeypatch.setenv("NM_TC_SP", sp)
    monkeypatch.setenv("NM_BF16_SIMT", simt)
    return kid


BF16_SIMT_CASES = [
    # (m, n, k, N, M, L): L outside {16, 32, 64, 128} -> bf16 on the fp32 SIMT kernel by default
    (256, 256, 256, 2, 4, 4),       # cfg1's pattern on bf16
    (300, 512, 1024, 8, 32, 4),     # cfg5's L = 4, ragged m
    (129, 264, 512, 4, 32, 8),      # L = 8, ragged m and n tile
    (64, 96, 192, 3, 8, 12),        # L = 12, odd N
]


@pytest.mark.parametrize("m,n,k,N,M,L", BF16_SIMT_CASES)
@pytest.mark.parametrize("cdt", [torch.bfloat16, torch.float32])
def test_spmm_bf16_simt_default_path(nm, oracle, monkeypatch, m, n, k, N, M, L, cdt):
    """bf16 operands whose L the slot kernel cannot take run the fp32 SIMT kernel on exact fp32
    copies (kernel id 5, AUTO and bf16_tc): uniform inputs within the bf16 bar, integer inputs
    bit-exact with fp32 C, and bf16 C = RNE of the exact result."""
    monkeypatch.delenv("NM_TC_SP", raising=False)
    monkeypatch.delenv("NM_BF16_SIMT", raising=False)
    for math in ("auto", "bf16_tc"):
        assert nm.nm_plan_query(m, n, k, N, M, L, torch.bfloat16, math)["kernel"] == 5
    A = synth.bf16grid((m, k), 61, synth.TID_A)
    B = synth.bf16grid((k, n), 62, synth.TID_B)
    vals, D = oracle.compress(synth.to_bf16_bits(B), N, M, L)
    W = nm.NmWeight(dev(oracle.bf16_to_f32(vals), torch.bfloat16), dev(D, torch.uint8), k, N, M, L)
    C = nm.nm_spmm(dev(A, torch.bfloat16), W, out_dtype=cdt).float().cpu().numpy()
    ref = oracle.spmm_sparse_f64(synth.to_bf16_bits(A), vals, D, k, N, M, L)
    assert oracle.rel_frobenius(C, ref) <= TOL_BF16
    Ai = synth.integer((m, k), 63, synth.TID_A)
    vi, Di = oracle.compress(synth.integer((k, n), 64, synth.TID_B), N, M, L)
    Wi = nm.NmWeight(dev(vi, torch.bfloat16), dev(Di, torch.uint8), k, N, M, L)
    Ci = nm.nm_spmm(dev(Ai, torch.bfloat16), Wi, out_dtype=cdt).float().cpu().numpy()
    refi = oracle.spmm_sparse_f64(Ai, vi, Di, k, N, M, L)
    if cdt == torch.float32:
        assert np.array_equal(Ci.astype(np.float64), refi)
    else:  # |C| <= 4 w < 2^24: exact in fp32, then one RNE to bf16 (torch's rounding of the exact value)
        assert np.array_equal(Ci, torch.from_numpy(refi).float().bfloat16().float().numpy())


@pytest.mark.parametrize("m,n,k,N,M,L", TC_CASES)
@pytest.mark.parametrize("cdt", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("path", ["sp", "generic", "simt"])
def test_spmm_tc_bf16_vs_oracle(nm, oracle, monkeypatch, m, n, k, N, M, L, cdt, path):
    kid = use_tc_path(monkeypatch, path)
    A = synth.bf16grid((m, k), 51, synth.TID_A)
    B = synth.bf16grid((k, n), 52, synth.TID_B)
    vals, D = oracle.compress(synth.to_bf16_bits(B), N, M, L)
    W = nm.NmWeight(dev(oracle.bf16_to_f32(vals), torch.bfloat16), dev(D, torch.uint8), k, N, M, L)
    plan = nm.nm_plan_query(m, n, k, N, M, L, torch.bfloat16, "bf16_tc")
    assert plan["kernel"] == kid, plan  # the tcgen05 kernel, not the generic fallback
    C = nm.nm_spmm(dev(A, torch.bfloat16), W, out_dtype=cdt, math="bf16_tc").float().cpu().numpy()
    ref = oracle.spmm_sparse_f64(synth.to_bf16_bits(A), vals, D, k, N, M, L)
    assert oracle.rel_frobenius(C, ref) <= TOL_BF16


@pytest.mark.parametrize("m,n,k,N,M,L", TC_CASES)
@pytest.mark.parametrize("path", ["sp", "generic"])
def test_spmm_tc_bf16_integer_exact(nm, oracle, monkeypatch, m, n, k, N, M, L, path):
    """Integer inputs: every partial sum is exact in fp32 -> bit-exact C (fp32 out)."""
    use_tc_path(monkeypatch, path)
    A = synth.integer((m, k), 61, synth.TID_A)
    B = synth.integer((k, n), 62, synth.TID_B)
    vals, D = oracle.compress(synth.to_bf16_bits(B), N, M, L)
    W = nm.NmWeight(dev(oracle.bf16_to_f32(vals), torch.bfloat16), dev(D, torch.uint8), k, N, M, L)
    C = nm.nm_spmm(dev(A, torch.bfloat16), W, out_dtype=torch.float32, math="bf16_tc").cpu().numpy()
    assert np.array_equal(C.astype(np.float64), oracle.spmm_sparse_f64(synth.to_bf16_bits(A), vals, D, k, N, M, L))


def test_spmm_tc_bf16_deterministic(nm):
    A = dev(synth.bf16grid((512, 1024), 1, 1), torch.bfloat16)
    W = nm.nm_compress(dev(synth.bf16grid((1024, 512), 2, 2), torch.bfloat16), 8, 32, 32)
    assert torch.equal(nm.nm_spmm(A, W), nm.nm_spmm(A, W))


@pytest.mark.parametrize("cfg", ["cfg2", "cfg3_62", "cfg3_75", "cfg4_65b"])
@pytest.mark.parametrize("path", ["sp"])
def test_spmm_tc_bf16_full_size_sampled(nm, oracle, monkeypatch, cfg, path):
    use_tc_path(monkeypatch, path)
    m, n, k, N, M, L = {"cfg2": (4096, 4096, 4096, 16, 32, 32), "cfg3_62": (2048, 11008, 4096, 12, 32, 32),
                        "cfg3_75": (2048, 11008, 4096, 8, 32, 32), "cfg4_65b": (2048, 22016, 8192, 4, 32, 32)}[cfg]
    A = synth.bf16grid((m, k), 71, synth.TID_A)
    B = synth.bf16grid((k, n), 72, synth.TID_B)
    W = nm.nm_compress(dev(B, torch.bfloat16), N, M, L)
    C = nm.nm_spmm(dev(A, torch.bfloat16), W)
    rows = np.array([0, 5, 127, 128, m // 2 + 7, m - 1])
    ref = oracle.spmm_sparse_f64(synth.to_bf16_bits(A), bf16_bits(W.values), W.idx.cpu().numpy(), k, N, M, L,
                                 rows=rows)
    got = C[torch.from_numpy(rows).cuda()].float().cpu().numpy()
    assert oracle.rel_frobenius(got, ref) <= TOL_BF16


# --------------------------------------------------------------- SIMT staging modes (selector ablation)
MODE_CASES = [(256, 256, 256, 2, 4, 4), (300, 288, 320, 16, 32, 32), (260, 384, 512, 8, 32, 32),
              (128, 520, 256, 4, 32, 8), (200, 192, 192, 1, 8, 4), (132, 128, 256, 16, 32, 64), (4, 256, 128, 4, 32, 32)]


@pytest.mark.parametrize("mode", ["0", "1", "2"])
@pytest.mark.parametrize("m,n,k,N,M,L", MODE_CASES)
def test_spmm_f32_staging_modes(nm, oracle, monkeypatch, mode, m, n, k, N, M, L):
    """mode 0: A panels straight from A; 1: A^T staged; 2: A^T + packed col_info loads
    (P:412-437).  All must give the same parity."""
    monkeypatch.setenv("NM_SIMT_MODE", mode)
    A, vals, D, C = run_f32(nm, oracle, m, n, k, N, M, L, kind="integer", seed=3)
    assert np.array_equal(C.astype(np.float64), oracle.spmm_sparse_f64(A, vals, D, k, N, M, L))
    A, vals, D, C = run_f32(nm, oracle, m, n, k, N, M, L)
    assert oracle.rel_frobenius(C, oracle.spmm_sparse_f64(A, vals, D, k, N, M, L)) <= TOL_F32


SK_CASES = [
    (4096, 1280, 1024, 16, 32, 32),   # 320 tiles > 296 resident: a 24-tile partial wave
    (1000, 640, 2048, 8, 32, 32),     # 40 tiles, ragged m: sub-wave grid
    (384, 384, 4096, 4, 32, 32),      # 9 tiles, long k, 87.5 %
    (256, 520, 1536, 3, 8, 8),        # odd N (odd row counts), n not a multiple of the tile
    (300, 256, 512, 2, 4, 4),         # L = 4: two column groups per thread chunk (TWO)
]


@pytest.mark.parametrize("split", ["auto", "1", "2", "3", "4"])
@pytest.mark.parametrize("m,n,k,N,M,L", SK_CASES)
def test_spmm_f32_split(nm, oracle, monkeypatch, split, m, n, k, N, M, L):
    """Split tiles (the partial last wave, or every tile of a sub-wave grid, as S k-range CTAs whose
    partials the last arriver adds in part order): integer inputs bit-exact for every S, uniform
    inputs within tolerance, and bit-reproducible run to run (fixed reduction order)."""
    if split != "auto":
        monkeypatch.setenv("NM_SIMT_SPLIT", split)
    A, vals, D, C = run_f32(nm, oracle, m, n, k, N, M, L, kind="integer", seed=5)
    rows = np.unique(np.concatenate([np.arange(0, m, 37), [m - 1]]))
    ref = oracle.spmm_sparse_f64(A, vals, D, k, N, M, L, rows=rows)
    assert np.array_equal(C[rows].astype(np.float64), ref)
    A, vals, D, C = run_f32(nm, oracle, m, n, k, N, M, L, seed=6)
    ref = oracle.spmm_sparse_f64(A, vals, D, k, N, M, L, rows=rows)
    assert oracle.rel_frobenius(C[rows], ref) <= TOL_F32
    W = nm.NmWeight(dev(vals), dev(D, torch.uint8), k, N, M, L)
    Ad = dev(A)
    assert torch.equal(nm.nm_spmm(Ad, W), nm.nm_spmm(Ad, W))


@pytest.mark.parametrize("bm", ["64", "128"])
@pytest.mark.parametrize("mode", ["0", "1"])
@pytest.mark.parametrize("m,n,k,N,M,L", [(300, 640, 512, 16, 32, 32), (97, 256, 384, 2, 4, 4),
                                         (513, 384, 1024, 3, 8, 8), (64, 128, 2048, 4, 32, 32)])
def test_spmm_f32_row_tiles(nm, oracle, monkeypatch, bm, mode, m, n, k, N, M, L):
    """Both SIMT row tiles (64: 4 warps, 3 CTAs/SM; 128: 8 warps) in both A stagings, integer inputs
    bit-exact (ragged m and n, the TWO path at L = 4, odd N)."""
    monkeypatch.setenv("NM_SIMT_BM", bm)
    monkeypatch.setenv("NM_SIMT_MODE", mode)
    A, vals, D, C = run_f32(nm, oracle, m, n, k, N, M, L, kind="integer", seed=7)
    assert np.array_equal(C.astype(np.float64), oracle.spmm_sparse_f64(A, vals, D, k, N, M, L))


# --------------------------------------------------------------- prepacked weights (P:470-475 offline step)
@pytest.mark.parametrize("m,n,k,N,M,L", TC_CASES)
@pytest.mark.parametrize("path", ["sp", "generic"])
def test_spmm_tc_prepacked_integer_exact(nm, oracle, monkeypatch, m, n, k, N, M, L, path):
    use_tc_path(monkeypatch, path)
    A = synth.integer((m, k), 81, synth.TID_A)
    B = synth.integer((k, n), 82, synth.TID_B)
    vals, D = oracle.compress(synth.to_bf16_bits(B), N, M, L)
    W = nm.NmWeight(dev(oracle.bf16_to_f32(vals), torch.bfloat16), dev(D, torch.uint8), k, N, M, L)
    PW = nm.nm_prepack(W)
    C = nm.nm_spmm_prepacked(dev(A, torch.bfloat16), PW, out_dtype=torch.float32).cpu().numpy()
    assert np.array_equal(C.astype(np.float64), oracle.spmm_sparse_f64(synth.to_bf16_bits(A), vals, D, k, N, M, L))
    assert PW.kind == {"sp": 2, "generic": 0}[path]
    C2 = nm.nm_spmm(dev(A, torch.bfloat16), W, out_dtype=torch.float32).cpu().numpy()
    assert np.array_equal(C, C2)


@pytest.mark.parametrize("L,kind", [(32, 4), (12, 0)])
def test_spmm_prepacked_fp32(nm, oracle, L, kind):
    """fp32 prepack: kind 4 (SIMT on bit-packed tile-major indices) when 128 % L == 0, else kind 0;
    the same bits as nm_spmm either way (the indices are the only difference)."""
    m, n, k, N, M = 200, 24 * L, 256, 8, 32
    A = synth.uniform((m, k), 91, 1)
    B = synth.uniform((k, n), 92, 2)
    vals, D = oracle.compress(B, N, M, L)
    W = nm.NmWeight(dev(vals), dev(D, torch.uint8), k, N, M, L)
    PW = nm.nm_prepack(W)
    assert PW.kind == kind
    C = nm.nm_spmm_prepacked(dev(A), PW)
    assert oracle.rel_frobenius(C.cpu().numpy(), oracle.spmm_sparse_f64(A, vals, D, k, N, M, L)) <= TOL_F32
    assert torch.equal(C, nm.nm_spmm(dev(A), W))


@pytest.mark.parametrize("N,M,L", [(2, 4, 4), (16, 32, 32), (4, 32, 8), (3, 8, 16), (1, 2, 64), (5, 64, 128),
                                   (12, 32, 32), (7, 100, 4), (60, 256, 32)])
def test_index_pack_bit_exact(nm, oracle, N, M, L):
    """nm_index_pack == the oracle's index_pack word for word (ragged last tile included);
    nm_index_unpack inverts it."""
    k, n = 8 * M, 128 * 3 + 2 * L
    _, D = oracle.compress(synth.uniform((k, n), 33, synth.TID_B), N, M, L)
    words = nm.nm_index_pack(dev(D, torch.uint8), k, n, N, M, L)
    torch.cuda.synchronize()
    assert np.array_equal(words.cpu().numpy().view(np.uint32), oracle.index_pack(D, k, n, N, M, L))
    assert np.array_equal(nm.nm_index_unpack(words, k, n, N, M, L).cpu().numpy(), D)


@pytest.mark.parametrize("m,n,k,N,M,L", [(300, 384, 512, 16, 32, 32), (257, 640, 1024, 4, 32, 32),
                                         (130, 256, 256, 2, 4, 4), (512, 1024, 2048, 8, 16, 16)])
def test_spmm_prepacked_packed_indices_integer_exact(nm, oracle, m, n, k, N, M, L):
    """kind 4: integer inputs, bit-exact vs the oracle through the packed-index loads."""
    A = synth.integer((m, k), 95, 1)
    vals, D = oracle.compress(synth.integer((k, n), 96, 2), N, M, L)
    W = nm.NmWeight(dev(vals), dev(D, torch.uint8), k, N, M, L)
    PW = nm.nm_prepack(W)
    assert PW.kind == 4
    C = nm.nm_spmm_prepacked(dev(A), PW).cpu().numpy()
    assert np.array_equal(C.astype(np.float64), oracle.spmm_sparse_f64(A, vals, D, k, N, M, L))


# --------------------------------------------------------------- sparse-tensor-core slot path edge cases
SP_EDGE = [
    (1, 128, 64, 16, 32, 32),        # single token (one partial token atom)
    (255, 160, 128, 16, 32, 16),     # n not a multiple of the 128-column tile; L = 16 (8 groups, 256 types)
    (513, 384, 1024, 1, 32, 32),     # very sparse (1:32): many padding slots
    (64, 256, 256, 32, 32, 32),      # N = M: dense windows (2 rows per group per quad exactly)
    (300, 256, 768, 3, 8, 64),       # odd N, M = 8
    (96, 128, 512, 5, 256, 128),     # M = 256 windows (uint8 offsets up to 255), L = 128 (one group per tile)
]


@pytest.mark.parametrize("m,n,k,N,M,L", SP_EDGE)
def test_spmm_tc_sp_edges_integer_exact(nm, oracle, monkeypatch, m, n, k, N, M, L):
    kid = use_tc_path(monkeypatch, "sp")
    assert nm.nm_plan_query(m, n, k, N, M, L, torch.bfloat16, "bf16_tc")["kernel"] == kid
    A = synth.integer((m, k), 101, synth.TID_A)
    B = synth.integer((k, n), 102, synth.TID_B)
    vals, D = oracle.compress(synth.to_bf16_bits(B), N, M, L)
    W = nm.NmWeight(dev(oracle.bf16_to_f32(vals), torch.bfloat16), dev(D, torch.uint8), k, N, M, L)
    ref = oracle.spmm_sparse_f64(synth.to_bf16_bits(A), vals, D, k, N, M, L)
    C = nm.nm_spmm(dev(A, torch.bfloat16), W, out_dtype=torch.float32).cpu().numpy()
    assert np.array_equal(C.astype(np.float64), ref)
    Cb = nm.nm_spmm(dev(A, torch.bfloat16), W, out_dtype=torch.bfloat16).float().cpu().numpy()
    assert oracle.rel_frobenius(Cb, ref) <= TOL_BF16


@pytest.mark.parametrize("nt", ["160", "176", "192", "208", "224"])
@pytest.mark.parametrize("cdt", [torch.bfloat16, torch.float32])
def test_spmm_tc_sp_token_tiles_all_rows(nm, oracle, monkeypatch, nt, cdt):
    """Every token-tile size the selector may pick, several token tiles deep, every row and column
    checked: integer inputs make fp32 C exact and bf16 C its RNE (catches epilogue chunks that
    spill into the next tile's rows)."""
    use_tc_path(monkeypatch, "sp")
    monkeypatch.setenv("NM_SP_H", "2")     # the H = 2 token tiles (a small grid would otherwise take H = 1)
    monkeypatch.setenv("NM_SP_NT", nt)
    m, n, k, N, M, L = 650, 512, 256, 16, 32, 32
    A = synth.integer((m, k), 111, synth.TID_A)
    B = synth.integer((k, n), 112, synth.TID_B)
    vals, D = oracle.compress(synth.to_bf16_bits(B), N, M, L)
    W = nm.NmWeight(dev(oracle.bf16_to_f32(vals), torch.bfloat16), dev(D, torch.uint8), k, N, M, L)
    ref = oracle.spmm_sparse_f64(synth.to_bf16_bits(A), vals, D, k, N, M, L)
    C = nm.nm_spmm(dev(A, torch.bfloat16), W, out_dtype=cdt).float().cpu().numpy()
    if cdt == torch.float32:
        assert np.array_equal(C.astype(np.float64), ref)
    else:
        want = torch.from_numpy(ref.astype(np.float32)).bfloat16().float().numpy()
        assert np.array_equal(C, want)


@pytest.mark.parametrize("tail", ["0", "1"])
@pytest.mark.parametrize("m,n,k,N,M,L", [(700, 768, 512, 16, 32, 32), (300, 640, 1024, 4, 32, 32)])
def test_spmm_tc_sp_tail_split_on_off(nm, oracle, monkeypatch, tail, m, n, k, N, M, L):
    """Small grids take the tail split (two half-range CTAs per tile, part 0 adds part 1's
    partial); NM_SP_TAIL=0 runs one CTA per tile.  Both bit-exact on integer inputs."""
    use_tc_path(monkeypatch, "sp")
    monkeypatch.setenv("NM_SP_TAIL", tail)
    monkeypatch.setenv("NM_SP_SPLIT", "2")  # these tiles are too short for the selector to split them
    A = synth.integer((m, k), 131, synth.TID_A)
    B = synth.integer((k, n), 132, synth.TID_B)
    vals, D = oracle.compress(synth.to_bf16_bits(B), N, M, L)
    W = nm.NmWeight(dev(oracle.bf16_to_f32(vals), torch.bfloat16), dev(D, torch.uint8), k, N, M, L)
    C = nm.nm_spmm(dev(A, torch.bfloat16), W, out_dtype=torch.float32).cpu().numpy()
    assert np.array_equal(C.astype(np.float64), oracle.spmm_sparse_f64(synth.to_bf16_bits(A), vals, D, k, N, M, L))


# --------------------------------------------------------------- tf32 sparse tensor cores (opt-in math)
# Tolerance: A is read by the tensor core at tf32 precision (10 explicit mantissa bits, relative
# error < 2^-10 per element), B' is rounded to tf32 offline (< 2^-11); the fp32 accumulation adds
# the fp32 path's error.  The north star's 5e-3 relative Frobenius bound for tf32
# holds with margin; integer inputs in {-2..2} are exact in tf32 and every partial sum is exact in
# fp32, so they must match the oracle bit for bit.
TF32_CASES = TC_CASES + SP_EDGE


def run_tf32(nm, oracle, m, n, k, N, M, L, kind, seed):
    A = synth.make(kind, (m, k), 141 + seed, synth.TID_A)
    B = synth.make(kind, (k, n), 142 + seed, synth.TID_B)
    vals, D = oracle.compress(B, N, M, L)
    W = nm.NmWeight(dev(vals), dev(D, torch.uint8), k, N, M, L)
    C = nm.nm_spmm(dev(A), W, math="tf32_tc").cpu().numpy()
    return C, oracle.spmm_sparse_f64(A, vals, D, k, N, M, L)


@pytest.mark.parametrize("m,n,k,N,M,L", TF32_CASES)
def test_spmm_tc_tf32_vs_oracle(nm, oracle, m, n, k, N, M, L):
    assert nm.nm_plan_query(m, n, k, N, M, L, torch.float32, "tf32_tc")["kernel"] == 3
    C, ref = run_tf32(nm, oracle, m, n, k, N, M, L, "uniform", 0)
    assert oracle.rel_frobenius(C, ref) <= TOL_BF16


@pytest.mark.parametrize("m,n,k,N,M,L", TF32_CASES)
def test_spmm_tc_tf32_integer_exact(nm, oracle, m, n, k, N, M, L):
    C, ref = run_tf32(nm, oracle, m, n, k, N, M, L, "integer", 1)
    assert np.array_equal(C.astype(np.float64), ref)


@pytest.mark.parametrize("nt", ["160", "176", "192", "208", "224"])
def test_spmm_tc_tf32_token_tiles_all_rows(nm, oracle, monkeypatch, nt):
    monkeypatch.setenv("NM_SP_H", "2")  # the H = 2 token tiles (a small grid would otherwise take H = 1)
    monkeypatch.setenv("NM_SP_NT", nt)
    C, ref = run_tf32(nm, oracle, 650, 512, 256, 16, 32, 32, "integer", 2)
    assert np.array_equal(C.astype(np.float64), ref)


@pytest.mark.parametrize("tail", ["0", "1"])
@pytest.mark.parametrize("m,n,k,N,M,L", [(700, 768, 512, 16, 32, 32), (300, 640, 1024, 4, 32, 32)])
def test_spmm_tc_tf32_tail_split_on_off(nm, oracle, monkeypatch, tail, m, n, k, N, M, L):
    monkeypatch.setenv("NM_SP_TAIL", tail)
    monkeypatch.setenv("NM_SP_SPLIT", "2")  # forced: these tiles are too short for the selector's split
    C, ref = run_tf32(nm, oracle, m, n, k, N, M, L, "integer", 3)
    assert np.array_equal(C.astype(np.float64), ref)


@pytest.mark.parametrize("cfg", ["cfg2", "cfg3_75", "cfg4_65b"])
def test_spmm_tc_tf32_full_size_sampled(nm, oracle, cfg):
    m, n, k, N, M, L = {"cfg2": (4096, 4096, 4096, 16, 32, 32), "cfg3_75": (2048, 11008, 4096, 8, 32, 32),
                        "cfg4_65b": (2048, 22016, 8192, 4, 32, 32)}[cfg]
    A = synth.uniform((m, k), 151, synth.TID_A)
    W = nm.nm_compress(dev(synth.uniform((k, n), 152, synth.TID_B)), N, M, L)
    C = nm.nm_spmm(dev(A), W, math="tf32_tc")
    rows = np.array([0, 3, 127, 128, m // 2 + 5, m - 1])
    ref = oracle.spmm_sparse_f64(A, W.values.cpu().numpy(), W.idx.cpu().numpy(), k, N, M, L, rows=rows)
    assert oracle.rel_frobenius(C[torch.from_numpy(rows).cuda()].cpu().numpy(), ref) <= TOL_BF16


def test_spmm_tc_tf32_deterministic_and_opt_in(nm):
    m, n, k, N, M, L = 512, 512, 1024, 8, 32, 32
    A = dev(synth.uniform((m, k), 5, 1))
    W = nm.nm_compress(dev(synth.uniform((k, n), 6, 2)), N, M, L)
    assert torch.equal(nm.nm_spmm(A, W, math="tf32_tc"), nm.nm_spmm(A, W, math="tf32_tc"))
    # AUTO keeps the paper's fp32 semantics (SIMT kernel); tf32 needs a slot-path geometry
    assert nm.nm_plan_query(m, n, k, N, M, L, torch.float32)["kernel"] == 1
    W8 = nm.nm_compress(dev(synth.uniform((64, 64), 7, 2)), 2, 4, 8)
    with pytest.raises(nm.NmError):
        nm.nm_spmm(dev(synth.uniform((16, 64), 8, 1)), W8, math="tf32_tc")


@pytest.mark.parametrize("m,n,k,N,M,L", [(300, 384, 512, 16, 32, 32), (513, 384, 1024, 1, 32, 32),
                                         (130, 256, 256, 8, 32, 16)])
def test_spmm_tc_tf32_prepacked(nm, oracle, monkeypatch, m, n, k, N, M, L):
    """nm_prepack_ex(math=tf32_tc): kind 3 images; same bits as nm_spmm(math=tf32_tc) at the same
    column-tile geometry (a per-call prepack may pick H = 1 for small grids: a different slot order,
    so only equal within tolerance -- the geometry is pinned here)."""
    monkeypatch.setenv("NM_SP_H", "2" if L >= 32 else "1")
    A = synth.uniform((m, k), 161, synth.TID_A)
    vals, D = oracle.compress(synth.uniform((k, n), 162, synth.TID_B), N, M, L)
    W = nm.NmWeight(dev(vals), dev(D, torch.uint8), k, N, M, L)
    PW = nm.nm_prepack(W, math="tf32_tc")
    assert PW.kind == 3
    C = nm.nm_spmm_prepacked(dev(A), PW)
    assert torch.equal(C, nm.nm_spmm(dev(A), W, math="tf32_tc"))
    ref = oracle.spmm_sparse_f64(A, vals, D, k, N, M, L)
    assert oracle.rel_frobenius(C.cpu().numpy(), ref) <= TOL_BF16
    assert nm.nm_prepack(W).kind == 4  # AUTO on fp32 keeps the SIMT path (with packed indices)


@pytest.mark.parametrize("dt", ["bf16", "tf32"])
@pytest.mark.parametrize("k,n,N,M,L", [(4096, 4096, 16, 32, 32), (4096, 1024, 8, 32, 32), (8192, 768, 4, 32, 32),
                                       (2048, 640, 12, 32, 16), (1536, 512, 3, 8, 64), (2048, 256, 5, 256, 128),
                                       (1024, 384, 1, 32, 32)])
def test_sp_pack_warp_matches_sequential(nm, monkeypatch, dt, k, n, N, M, L):
    """The warp-parallel slot packer reproduces the sequential reference packer exactly (slot
    lists, types, stage counts, weight and metadata images: the whole prepacked buffer)."""
    tdt = torch.bfloat16 if dt == "bf16" else torch.float32
    gen = synth.bf16grid if dt == "bf16" else synth.uniform
    W = nm.nm_compress(dev(gen((k, n), 171, synth.TID_B), tdt), N, M, L)
    math = "tf32_tc" if dt == "tf32" else "auto"
    fast = nm.nm_prepack(W, math=math)
    monkeypatch.setenv("NM_SP_PACK_SEQ", "1")
    ref = nm.nm_prepack(W, math=math)
    torch.cuda.synchronize()
    assert fast.kind == ref.kind == (3 if dt == "tf32" else 2)
    assert torch.equal(fast.buf, ref.buf)


@pytest.mark.parametrize("chunks,m", [("1", 700), ("2", 700), ("3", 700), ("4", 700), ("8", 700), ("0", 2100)])
def test_spmm_host_path_chunked(nm, oracle, monkeypatch, chunks, m):
    """nm_spmm_host's copy/compute overlap (row chunks 1 : 2 : .. : 2 : 1 on separate copy streams)
    gives the oracle's result for every chunk count, including a ragged last chunk, empty chunks
    (8 at m = 700) and the default (0: 9 chunks at m = 2100)."""
    monkeypatch.setenv("NM_HOST_CHUNKS", chunks)
    n, k, N, M, L = 512, 1024, 8, 32, 32
    A = synth.uniform((m, k), 43, 1)
    B = synth.uniform((k, n), 44, 2)
    vals, D = oracle.compress(B, N, M, L)
    run = nm.HostSpmm(m, n, k, N, M, L)
    C = torch.full((m, n), float("nan")).pin_memory()
    run(torch.from_numpy(A).pin_memory(), torch.from_numpy(vals).pin_memory(), torch.from_numpy(D).pin_memory(), C)
    assert oracle.rel_frobenius(C.numpy(), oracle.spmm_sparse_f64(A, vals, D, k, N, M, L)) <= TOL_F32
    Ai = synth.integer((m, k), 45, 1)
    vi, Di = oracle.compress(synth.integer((k, n), 46, 2), N, M, L)
    run(torch.from_numpy(Ai).pin_memory(), torch.from_numpy(vi).pin_memory(), torch.from_numpy(Di).pin_memory(), C)
    assert np.array_equal(C.numpy().astype(np.float64), oracle.spmm_sparse_f64(Ai, vi, Di, k, N, M, L))


# --------------------------------------------------------------- fused peer exchange (S10, p2p)
def _shards(nm, oracle, m, n, k, N, M, L, G, seed):
    from paper_2503_01253_b200 import sharded
    A = synth.uniform((m, k), seed, synth.TID_A)
    B = synth.uniform((k, n), seed + 1, synth.TID_B)
    vals, D = oracle.compress(B, N, M, L)
    q, out = n // L, []
    for r in range(G):
        v, d = sharded.shard_weight(torch.from_numpy(vals), torch.from_numpy(D), L, N, r, G)
        g0, g1 = sharded.shard_ranges(q, G)[r]
        out.append((nm.NmWeight(v.cuda(), d.cuda(), k, N, M, L), g0 * L, (g1 - g0) * L))
    return A, vals, D, out


@pytest.mark.parametrize("G,m,n,k,N,M,L", [(2, 300, 640, 512, 8, 32, 32), (3, 256, 768, 1024, 4, 32, 32),
                                           (2, 130, 520, 256, 4, 32, 8)])
def test_spmm_peers_two_streams(nm, oracle, G, m, n, k, N, M, L):
    """The fused exchange's device logic with G 'ranks' on G streams of one process: every rank's
    epilogue stores its shard into all G C buffers, the flag barrier orders them; after the
    barrier every buffer holds the whole C (oracle), for several epochs."""
    A, vals, D, shards = _shards(nm, oracle, m, n, k, N, M, L, G, 181)
    ref = oracle.spmm_sparse_f64(A, vals, D, k, N, M, L)
    Ad = dev(A)
    Cs = [torch.full((m, n), float("nan"), device="cuda") for _ in range(G)]
    flags = [torch.zeros(G, dtype=torch.int32, device="cuda") for _ in range(G)]
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream() for _ in range(G)]
    for epoch in (1, 2, 3):
        for r in range(G):
            W, col_off, n_valid = shards[r]
            with torch.cuda.stream(streams[r]):
                nm.nm_spmm_peers(Ad, W, [c.data_ptr() for c in Cs], n, col_off, n_valid, stream=streams[r])
                nm.nm_peer_barrier([f.data_ptr() for f in flags], r, epoch, stream=streams[r])
        torch.cuda.synchronize()
        for r in range(G):
            assert oracle.rel_frobenius(Cs[r].cpu().numpy(), ref) <= TOL_F32
            assert int(flags[r].min()) == epoch


def test_sharded_p2p_two_processes_one_gpu(nm, oracle):
    """The IPC plumbing of exchange='p2p': two processes (gloo for the handle exchange) on one
    GPU map each other's C buffers and flags; each call's C equals the oracle on both ranks."""
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29000 + os.getpid() % 1000
    import p2p_worker
    procs = [ctx.Process(target=p2p_worker.run, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for r in range(2):
        assert isinstance(res[r], float) and res[r] <= TOL_F32, res


@pytest.mark.parametrize("dt", ["bf16", "tf32"])
@pytest.mark.parametrize("cdt", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("G,m,n,k,N,M,L", [(2, 300, 1024, 512, 8, 32, 32), (3, 260, 768, 1024, 4, 32, 32)])
def test_spmm_prepacked_peers_two_streams(nm, oracle, dt, cdt, G, m, n, k, N, M, L):
    """Fused exchange on the sparse-tensor-core slot kernel (bf16 kind 2 / tf32 kind 3 shards):
    the direct-store epilogue writes each shard into all G buffers; integer inputs -> fp32 C
    bit-exact, bf16 C = its RNE."""
    if dt == "tf32" and cdt == torch.bfloat16:
        pytest.skip("fp32 operands need an fp32 C")
    from paper_2503_01253_b200 import sharded
    A = synth.integer((m, k), 201, synth.TID_A)
    B = synth.integer((k, n), 202, synth.TID_B)
    bits = synth.to_bf16_bits(B) if dt == "bf16" else B
    vals, D = oracle.compress(bits, N, M, L)
    vals_f = oracle.bf16_to_f32(vals) if dt == "bf16" else vals
    ref = oracle.spmm_sparse_f64(synth.to_bf16_bits(A) if dt == "bf16" else A, vals, D, k, N, M, L)
    tdt = torch.bfloat16 if dt == "bf16" else torch.float32
    Ad = dev(A, tdt)
    q = n // L
    Cs = [torch.full((m, n), float("nan"), device="cuda", dtype=cdt) for _ in range(G)]
    flags = [torch.zeros(G, dtype=torch.int32, device="cuda") for _ in range(G)]
    shards = []
    for r in range(G):
        v, d = sharded.shard_weight(torch.from_numpy(vals_f), torch.from_numpy(D), L, N, r, G)
        W = nm.NmWeight(v.cuda().to(tdt), d.cuda(), k, N, M, L)
        PW = nm.nm_prepack(W, math="tf32_tc" if dt == "tf32" else "auto")
        assert PW.kind == (3 if dt == "tf32" else 2)
        g0, g1 = sharded.shard_ranges(q, G)[r]
        shards.append((PW, g0 * L, (g1 - g0) * L))
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream() for _ in range(G)]
    want = ref if cdt == torch.float32 else torch.from_numpy(ref.astype(np.float32)).bfloat16().float().numpy()
    for epoch in (1, 2):
        for r in range(G):
            PW, col_off, n_valid = shards[r]
            with torch.cuda.stream(streams[r]):
                nm.nm_spmm_prepacked_peers(Ad, PW, [c.data_ptr() for c in Cs], n, col_off, n_valid, out_dtype=cdt,
                                           stream=streams[r])
                nm.nm_peer_barrier([f.data_ptr() for f in flags], r, epoch, stream=streams[r])
        torch.cuda.synchronize()
        for r in range(G):
            assert np.array_equal(Cs[r].float().cpu().numpy().astype(np.float64), want)


# --------------------------------------------------------------- Eq. 1 as printed: alpha = M/N
SCALED_PATHS = [  # (name, ab dtype, math, env, expected kernel id)
    ("simt", torch.float32, "f32_simt", {}, 1),
    ("generic", torch.float32, "f32_simt", {}, 0),          # L = 3 -> generic kernel + scaling pass
    ("sp_bf16", torch.bfloat16, "bf16_tc", {}, 4),
    ("generic_bf16", torch.bfloat16, "bf16_tc", {"NM_TC_SP": "0", "NM_BF16_SIMT": "0"}, 0),
    ("simt_bf16", torch.bfloat16, "bf16_tc", {"NM_TC_SP": "0"}, 5),   # alpha fused into the SIMT epilogue
    ("tf32", torch.float32, "tf32_tc", {}, 3),
]


@pytest.mark.parametrize("name,tdt,math,env,kid", SCALED_PATHS)
@pytest.mark.parametrize("cdt", [torch.float32, torch.bfloat16])
def test_spmm_scaled_eq1(nm, oracle, monkeypatch, name, tdt, math, env, kid, cdt):
    """nm_spmm_scaled with alpha = M/N against the oracle's Eq. 1 as printed (O2s): integer inputs
    and M/N a power of two, so fp32 C is exact and bf16 C is its RNE on every path."""
    if tdt == torch.float32 and cdt == torch.bfloat16:
        pytest.skip("fp32 operands need an fp32 C")
    for key, val in env.items():
        monkeypatch.setenv(key, val)
    m, n, k, N, M, L = (130, 258, 256, 2, 8, 3) if name == "generic" else (300, 512, 512, 8, 32, 32)
    assert nm.nm_plan_query(m, n, k, N, M, L, tdt, math)["kernel"] == kid
    A = synth.integer((m, k), 211, synth.TID_A)
    B = synth.integer((k, n), 212, synth.TID_B)
    bits = synth.to_bf16_bits(B) if tdt == torch.bfloat16 else B
    vals, D = oracle.compress(bits, N, M, L)
    vf = oracle.bf16_to_f32(vals) if tdt == torch.bfloat16 else vals
    W = nm.NmWeight(dev(vf, tdt), dev(D, torch.uint8), k, N, M, L)
    ref = oracle.spmm_eq1_scaled_f64(synth.to_bf16_bits(A) if tdt == torch.bfloat16 else A, vals, D, k, N, M, L)
    C = nm.nm_spmm(dev(A, tdt), W, out_dtype=cdt, math=math, alpha=M / N).float().cpu().numpy()
    want = ref if cdt == torch.float32 else torch.from_numpy(ref.astype(np.float32)).bfloat16().float().numpy()
    assert np.array_equal(C.astype(np.float64), want)


def test_spmm_scaled_uniform_and_unit_alpha(nm, oracle):
    """Uniform inputs within the fp32 bound; alpha = 1 gives nm_spmm's bits exactly."""
    m, n, k, N, M, L = 257, 384, 512, 12, 32, 32
    A = synth.uniform((m, k), 221, synth.TID_A)
    vals, D = oracle.compress(synth.uniform((k, n), 222, synth.TID_B), N, M, L)
    W = nm.NmWeight(dev(vals), dev(D, torch.uint8), k, N, M, L)
    C = nm.nm_spmm(dev(A), W, alpha=M / N).cpu().numpy()
    assert oracle.rel_frobenius(C, oracle.spmm_eq1_scaled_f64(A, vals, D, k, N, M, L)) <= TOL_F32
    assert torch.equal(nm.nm_spmm(dev(A), W, alpha=1.0), nm.nm_spmm(dev(A), W))


@pytest.mark.parametrize("dt", ["bf16", "tf32"])
@pytest.mark.parametrize("chunks", ["1", "3", "4"])
def test_spmm_host_path_chunked_slot_kernels(nm, oracle, monkeypatch, dt, chunks):
    """nm_spmm_host on the sparse-tensor-core slot kernels: one prepack per call, then the row
    chunks overlapped with the copies; integer inputs -> fp32 C bit-exact."""
    monkeypatch.setenv("NM_HOST_CHUNKS", chunks)
    m, n, k, N, M, L = 700, 512, 1024, 8, 32, 32
    A = synth.integer((m, k), 231, 1)
    B = synth.integer((k, n), 232, 2)
    tdt = torch.bfloat16 if dt == "bf16" else torch.float32
    bits = synth.to_bf16_bits(B) if dt == "bf16" else B
    vals, D = oracle.compress(bits, N, M, L)
    vf = oracle.bf16_to_f32(vals) if dt == "bf16" else vals
    run = nm.HostSpmm(m, n, k, N, M, L, ab_dtype=tdt, c_dtype=torch.float32,
                      math="tf32_tc" if dt == "tf32" else "bf16_tc")
    C = torch.full((m, n), float("nan")).pin_memory()
    run(torch.from_numpy(A).to(tdt).pin_memory(), torch.from_numpy(vf).to(tdt).pin_memory(),
        torch.from_numpy(D).pin_memory(), C)
    ref = oracle.spmm_sparse_f64(synth.to_bf16_bits(A) if dt == "bf16" else A, vals, D, k, N, M, L)
    assert np.array_equal(C.numpy().astype(np.float64), ref)


# --------------------------------------------------------------- A supplied transposed (nm_spmm_at)
AT_CASES = [  # (dtype, math, m, n, k, N, M, L, lda padding)
    (torch.float32, "auto", 300, 256, 512, 8, 32, 32, 4),      # SIMT staged-A^T mode, ragged m, lda > m
    (torch.float32, "auto", 1024, 512, 1024, 16, 32, 32, 0),   # full tiles
    (torch.bfloat16, "auto", 300, 384, 512, 16, 32, 32, 8),    # slot kernel, ragged m and n tile
    (torch.bfloat16, "auto", 129, 256, 1024, 4, 32, 32, 0),    # 87.5 %: many zero-filled padding slots
    (torch.bfloat16, "auto", 520, 256, 768, 3, 8, 64, 24),     # odd N, M = 8, L = 64
    (torch.float32, "tf32_tc", 200, 256, 512, 8, 32, 32, 4),   # tf32 slot kernel
]


@pytest.mark.parametrize("dt,math,m,n,k,N,M,L,pad", AT_CASES)
def test_spmm_at_matches_nm_spmm(nm, oracle, dt, math, m, n, k, N, M, L, pad):
    """nm_spmm_at (A given as A^T, k x lda, columns m .. lda-1 filled with NaN) computes the same C
    as nm_spmm bit for bit, and integer inputs match the oracle exactly; nm_spmm_prepacked_at the
    same on the prepacked weight (kind 2 bf16, 3 tf32, 4 fp32 bit-packed indices)."""
    tdt = dt
    for kind_inputs in ("uniform", "integer"):
        if kind_inputs == "uniform":
            A = synth.bf16grid((m, k), 71, synth.TID_A) if dt == torch.bfloat16 else synth.uniform((m, k), 71, synth.TID_A)
            B = synth.bf16grid((k, n), 72, synth.TID_B) if dt == torch.bfloat16 else synth.uniform((k, n), 72, synth.TID_B)
        else:
            A = synth.integer((m, k), 73, synth.TID_A)
            B = synth.integer((k, n), 74, synth.TID_B)
        bits = synth.to_bf16_bits(B) if dt == torch.bfloat16 else B
        vals, D = oracle.compress(bits, N, M, L)
        v = oracle.bf16_to_f32(vals) if dt == torch.bfloat16 else vals
        W = nm.NmWeight(dev(v, tdt), dev(D, torch.uint8), k, N, M, L)
        Ad = dev(A, tdt)
        lda = (m + 7) // 8 * 8 + pad  # rows 16-B aligned (bf16: 8 elements)
        At = torch.full((k, lda), float("nan"), dtype=tdt, device="cuda")
        At[:, :m] = Ad.t()
        C_ref = nm.nm_spmm(Ad, W, out_dtype=torch.float32, math=math)
        C_at = nm.nm_spmm_at(At, W, m=m, out_dtype=torch.float32, math=math)
        torch.cuda.synchronize()
        assert torch.equal(C_at, C_ref)
        PW = nm.nm_prepack(W, math=math)
        C_pat = nm.nm_spmm_prepacked_at(At, PW, m=m, out_dtype=torch.float32)
        C_pre = nm.nm_spmm_prepacked(Ad, PW, out_dtype=torch.float32)
        torch.cuda.synchronize()
        assert torch.equal(C_pat, C_pre)
        src = synth.to_bf16_bits(A) if dt == torch.bfloat16 else A
        ref = oracle.spmm_sparse_f64(src, vals, D, k, N, M, L)
        if kind_inputs == "integer":
            assert np.array_equal(C_at.cpu().numpy().astype(np.float64), ref)
        else:
            assert oracle.rel_frobenius(C_at.cpu().numpy(), ref) <= (TOL_F32 if math == "auto" and dt == torch.float32
                                                                     else TOL_BF16)


def test_spmm_at_rejects(nm):
    """lda < m -> NM_ERR_SHAPE; a shape that selects a kernel without an A^T input -> unsupported."""
    m, n, k, N, M, L = 64, 96, 96, 3, 8, 3   # L = 3: the generic kernel
    W = nm.nm_compress(torch.ones(k, n, device="cuda"), N, M, L)
    At = torch.zeros((k, m), device="cuda")
    with pytest.raises(nm.NmError, match="UNSUPPORTED"):
        nm.nm_spmm_at(At, W)
    W2 = nm.nm_compress(torch.ones(128, 128, device="cuda"), 16, 32, 32)
    At2 = torch.zeros((128, 64), device="cuda")
    with pytest.raises(nm.NmError):
        nm.nm_spmm_at(At2, W2, m=65)


@pytest.mark.parametrize("m,n,k,N,M,L,bn_hint", [(512, 1024, 1024, 16, 32, 32, 128),   # small grid: H = 1
                                                 (4096, 4096, 1024, 16, 32, 32, 256)])  # large grid: H = 2 stays
def test_prepack_m_hint(nm, oracle, m, n, k, N, M, L, bn_hint):
    """nm_prepack_m: with the token count known the slot prepack takes the tile nm_spmm would (H = 1
    when H = 2 leaves the grid under two waves); results are exact on integer inputs either way."""
    A = synth.integer((m, k), 81, synth.TID_A)
    B = synth.integer((k, n), 82, synth.TID_B)
    vals, D = oracle.compress(synth.to_bf16_bits(B), N, M, L)
    W = nm.NmWeight(dev(oracle.bf16_to_f32(vals), torch.bfloat16), dev(D, torch.uint8), k, N, M, L)
    ref = oracle.spmm_sparse_f64(synth.to_bf16_bits(A), vals, D, k, N, M, L)
    Ad = dev(A, torch.bfloat16)
    PW0, PWm = nm.nm_prepack(W), nm.nm_prepack(W, m_hint=m)
    assert PW0.kind == PWm.kind == 2 and PW0.desc.bn == 256 and PWm.desc.bn == bn_hint
    for PW in (PW0, PWm):
        C = nm.nm_spmm_prepacked(Ad, PW, out_dtype=torch.float32)
        torch.cuda.synchronize()
        assert np.array_equal(C.cpu().numpy().astype(np.float64), ref)


@pytest.mark.parametrize("m,n,k,N,M,L,split", [(512, 1024, 1024, 16, 32, 32, 2),   # 64-row tile, split 2
                                               (512, 512, 512, 16, 32, 32, 2),
                                               (200, 384, 768, 8, 32, 32, 0)])     # whatever the selector picks
def test_simt_small_grid_split_exact(nm, oracle, m, n, k, N, M, L, split):
    """The 64-row tile's k-split of small grids (fixed-order partial sums) on integer inputs: fp32 C
    equals the oracle exactly; the selector's split is the pinned one."""
    p = nm.nm_plan_query(m, n, k, N, M, L, torch.float32)
    if split:
        assert p["bm"] == 64 and p["split"] == split, p
    A = synth.integer((m, k), 91, synth.TID_A)
    vals, D = oracle.compress(synth.integer((k, n), 92, synth.TID_B), N, M, L)
    W = nm.NmWeight(dev(vals), dev(D, torch.uint8), k, N, M, L)
    C = nm.nm_spmm(dev(A), W, math="f32_simt")
    torch.cuda.synchronize()
    assert np.array_equal(C.cpu().numpy().astype(np.float64), oracle.spmm_sparse_f64(A, vals, D, k, N, M, L))


def test_host_path_bf16_simt_fallback(nm, oracle):
    """nm_spmm_host with bf16 operands at L = 4 (the SIMT fallback, kernel 5): integer inputs exact."""
    m, n, k, N, M, L = 300, 256, 512, 8, 32, 4
    A = synth.integer((m, k), 93, synth.TID_A)
    vals, D = oracle.compress(synth.integer((k, n), 94, synth.TID_B), N, M, L)
    run = nm.HostSpmm(m, n, k, N, M, L, ab_dtype=torch.bfloat16, c_dtype=torch.float32)
    C = torch.full((m, n), float("nan")).pin_memory()
    run(torch.from_numpy(A).to(torch.bfloat16).pin_memory(), torch.from_numpy(vals).to(torch.bfloat16).pin_memory(),
        torch.from_numpy(D).pin_memory(), C)
    assert np.array_equal(C.numpy().astype(np.float64), oracle.spmm_sparse_f64(A, vals, D, k, N, M, L))
