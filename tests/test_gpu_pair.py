"""GPU parity of the CTA-pair slot kernel (spmm_tc_sp2.cu: tcgen05.mma.sp.cta_group::2, persistent
clusters, 128-slot stages) against the CPU oracle.  It runs for bf16 operands on the H = 2 prepack
(L >= 32, N/M >= 1/4) when NM_SP_PAIR=1 (opt-in; the default is the one-CTA kernel).  Integer inputs in {-2..2}
make every partial sum exact, so fp32 C must equal the oracle bit for bit and bf16 C its RNE
(catches a wrong slot row, token, column half, stage or split part anywhere in the tile)."""
import numpy as np
import pytest
import torch

from paper_2503_01253_b200 import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def pair_on(monkeypatch):
    monkeypatch.setenv("NM_SP_PAIR", "1")
    monkeypatch.setenv("NM_SP_H", "2")  # the pair kernel runs on the H = 2 prepack (also at 75 %)


@pytest.fixture(scope="module")
def nm():
    from paper_2503_01253_b200 import nmspmm
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    nmspmm.lib()
    return nmspmm


def dev(x, dtype):
    t = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    return t.to(dtype) if t.dtype != dtype else t


def weight(nm, oracle, m, n, k, N, M, L, seed, kind="integer"):
    A = synth.make(kind, (m, k), seed, synth.TID_A)
    B = synth.make(kind, (k, n), seed + 1, synth.TID_B)
    Ab = synth.to_bf16_bits(A)
    vals, D = oracle.compress(synth.to_bf16_bits(B), N, M, L)
    W = nm.NmWeight(dev(oracle.bf16_to_f32(vals), torch.bfloat16), dev(D, torch.uint8), k, N, M, L)
    return Ab, vals, D, W


PAIR_CASES = [
    (256, 256, 256, 16, 32, 32),      # one tile, one pair, 4 prepack stages
    (300, 512, 1024, 16, 32, 32),     # ragged token tile, two column tiles
    (100, 256, 512, 8, 32, 32),       # m < 128: the peer CTA gathers only padding tokens
    (129, 768, 320, 12, 32, 32),      # peer CTA holds 1 token; k = 10 windows (odd prepack stage count)
    (520, 320, 96, 32, 32, 32),       # N = M, k = 3 windows; n not a multiple of the 256-column tile
    (2048, 4096, 512, 16, 32, 32),    # 128 tiles > 74 pairs: several units per persistent cluster
    (1000, 1536, 2048, 8, 32, 64),    # L = 64 (4 groups per tile), 75 %
    (64, 256, 4096, 16, 32, 32),      # one token tile, long k: the split of a sub-wave grid
]


@pytest.mark.parametrize("m,n,k,N,M,L", PAIR_CASES)
def test_pair_integer_exact(nm, oracle, monkeypatch, m, n, k, N, M, L):
    assert nm.nm_plan_query(m, n, k, N, M, L, torch.bfloat16, "bf16_tc")["kernel"] == 4
    Ab, vals, D, W = weight(nm, oracle, m, n, k, N, M, L, 201)
    ref = oracle.spmm_sparse_f64(Ab, vals, D, k, N, M, L)
    A = dev(oracle.bf16_to_f32(Ab), torch.bfloat16)
    PW = nm.nm_prepack(W)
    C = nm.nm_spmm_prepacked(A, PW, out_dtype=torch.float32).cpu().numpy()
    assert np.array_equal(C.astype(np.float64), ref)
    Cb = nm.nm_spmm_prepacked(A, PW, out_dtype=torch.bfloat16).float().cpu().numpy()
    assert np.array_equal(Cb, torch.from_numpy(ref.astype(np.float32)).bfloat16().float().numpy())
    # the per-call path (prepack into scratch) takes the same kernel
    C2 = nm.nm_spmm(A, W, out_dtype=torch.float32).cpu().numpy()
    assert np.array_equal(C2.astype(np.float64), ref)


@pytest.mark.parametrize("split", ["2", "3", "5"])
@pytest.mark.parametrize("m,n,k,N,M,L", [(700, 768, 2048, 16, 32, 32), (256, 512, 1024, 12, 32, 32)])
def test_pair_forced_split_integer_exact(nm, oracle, monkeypatch, split, m, n, k, N, M, L):
    """Split parts (pair-aligned stage ranges, last arriver adds the partials in part order),
    including parts whose range ends on an odd prepack stage and parts with no stage at all."""
    monkeypatch.setenv("NM_SP_SPLIT", split)
    Ab, vals, D, W = weight(nm, oracle, m, n, k, N, M, L, 211)
    ref = oracle.spmm_sparse_f64(Ab, vals, D, k, N, M, L)
    C = nm.nm_spmm(dev(oracle.bf16_to_f32(Ab), torch.bfloat16), W, out_dtype=torch.float32).cpu().numpy()
    assert np.array_equal(C.astype(np.float64), ref)


@pytest.mark.parametrize("tail", ["0", "1"])
def test_pair_tail_on_off(nm, oracle, monkeypatch, tail):
    monkeypatch.setenv("NM_SP_TAIL", tail)
    m, n, k, N, M, L = 1280, 2816, 512, 16, 32, 32   # 5 x 11 = 55 tiles < 74 pairs (sub-wave split)
    Ab, vals, D, W = weight(nm, oracle, m, n, k, N, M, L, 221)
    ref = oracle.spmm_sparse_f64(Ab, vals, D, k, N, M, L)
    C = nm.nm_spmm(dev(oracle.bf16_to_f32(Ab), torch.bfloat16), W, out_dtype=torch.float32).cpu().numpy()
    assert np.array_equal(C.astype(np.float64), ref)


@pytest.mark.parametrize("m,n,k,N,M,L", [(4096, 4096, 4096, 16, 32, 32), (2048, 11008, 4096, 12, 32, 32)])
def test_pair_uniform_tolerance_sampled(nm, oracle, monkeypatch, m, n, k, N, M, L):
    """BASELINE sizes (cfg2, cfg3 62.5 %) in the launch configuration bench.py times: bf16 C on
    uniform inputs within the 5e-3 bar on sampled rows (every column), and equal to the one-CTA
    kernel within the same bar."""
    Ab, vals, D, W = weight(nm, oracle, m, n, k, N, M, L, 231, kind="bf16grid")
    A = dev(oracle.bf16_to_f32(Ab), torch.bfloat16)
    PW = nm.nm_prepack(W)
    C = nm.nm_spmm_prepacked(A, PW).float().cpu().numpy()
    rows = np.unique(np.concatenate([np.arange(0, m, 97), [m - 1]]))
    ref = oracle.spmm_sparse_f64(Ab, vals, D, k, N, M, L, rows=rows)
    assert oracle.rel_frobenius(C[rows], ref) <= 5e-3
    monkeypatch.setenv("NM_SP_PAIR", "0")
    C1 = nm.nm_spmm_prepacked(A, PW).float().cpu().numpy()
    assert oracle.rel_frobenius(C, C1.astype(np.float64)) <= 5e-3


def test_pair_scaled_alpha(nm, oracle):
    """Eq. 1's M/N prefactor (nm_spmm_scaled) applied in the pair epilogue."""
    m, n, k, N, M, L = 384, 512, 512, 16, 32, 32
    Ab, vals, D, W = weight(nm, oracle, m, n, k, N, M, L, 241)
    ref = oracle.spmm_sparse_f64(Ab, vals, D, k, N, M, L) * (M / N)
    C = nm.nm_spmm(dev(oracle.bf16_to_f32(Ab), torch.bfloat16), W, out_dtype=torch.float32, alpha=M / N)
    assert np.array_equal(C.cpu().numpy().astype(np.float64), ref)
