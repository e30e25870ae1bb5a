"""Pins for the CPU oracle (oracle/nm_oracle.c) against what the paper and the
mathematics fix -- never against the oracle itself.  CPU only.

Pins used (SURVEY 8(c) "What pins each part"):
  * worked examples S:69
    (tests/golden/spec_examples.json);
  * an independent brute-force C(M,N) keep-set search for M <= 8 (pure Python);
  * integer-valued inputs: every partial sum is an exact integer, so the
    oracle must equal numpy's int64 matmul on the brute-force-pruned B;
  * N = M reduces to dense GEMM (numpy fp64 matmul, and bit-exact O1f==O2f);
  * A = I gives C = B~; all-ones A and B' give C == w;
  * invariants (N per window, strictly increasing, < M), round trip,
    idempotence, linearity, sharded concatenation.
"""
import itertools
import json
import os

import numpy as np
import pytest

from paper_2503_01253_b200 import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")


@pytest.fixture(scope="module")
def gold():
    with open(GOLDEN) as f:
        return json.load(f)


# --------------------------------------------------------------------------
# independent brute force (tests only; does not call the oracle)
# --------------------------------------------------------------------------
def brute_force_keep(window: np.ndarray, N: int):
    """window: M x L values of one (window, group).  Score of a vector = fp64 sum
    of squares in ascending c (R6 defines the score this way).  Among all C(M,N)
    subsets, pick the one whose descending-sorted score vector is
    lexicographically largest, then the lexicographically smallest offset tuple
    (SURVEY 8(c) item 4 / S:107)."""
    M = window.shape[0]
    scores = []
    for r in range(M):
        s = 0.0
        for x in window[r]:
            s = s + float(x) * float(x)
        scores.append(s)
    best = None
    for sub in itertools.combinations(range(M), N):
        key = (tuple(sorted((scores[r] for r in sub), reverse=True)), tuple(-r for r in sub))
        if best is None or key > best[0]:
            best = (key, sub)
    return list(best[1])


def sort_keep(window: np.ndarray, N: int):
    """Second, independent statement of the rule for large M, where C(M,N) is
    too big to enumerate: Python's stable sort on (-score, offset)."""
    scores = [sum((float(x) * float(x) for x in row), 0.0) for row in window]
    return sorted(sorted(range(window.shape[0]), key=lambda r: (-scores[r], r))[:N])


def brute_force_prune(B: np.ndarray, N: int, M: int, L: int) -> np.ndarray:
    k, n = B.shape
    out = np.zeros_like(B)
    keep = brute_force_keep if M <= 8 else sort_keep
    for t in range(k // M):
        for g in range(n // L):
            win = B[t * M:(t + 1) * M, g * L:(g + 1) * L]
            for r in keep(win, N):
                out[t * M + r, g * L:(g + 1) * L] = win[r]
    return out


# --------------------------------------------------------------------------
# worked examples
# --------------------------------------------------------------------------
def test_spec_prune_example(oracle, gold):
    ex = gold["prune_column"]
    B = np.array(ex["B"], dtype=np.float32)
    vals, D = oracle.compress(B, ex["N"], ex["M"], ex["L"])
    assert vals.tolist() == ex["values"]
    assert D.tolist() == ex["D"]
    dense = oracle.decompress(vals, D, 4, ex["N"], ex["M"], ex["L"])
    assert dense.tolist() == ex["pruned"]


def test_spec_compress_decompress_example(oracle, gold):
    ex = gold["compress_4x2"]
    B = np.array(ex["B"], dtype=np.float32)
    vals, D = oracle.compress(B, ex["N"], ex["M"], ex["L"])
    assert vals.tolist() == ex["values"]
    assert D.tolist() == ex["D"]
    back = oracle.decompress(np.array(ex["values"], np.float32), np.array(ex["D"], np.uint8), 4,
                             ex["N"], ex["M"], ex["L"])
    assert np.array_equal(back, B)


def test_spec_spmm_example(oracle, gold):
    ex, cx = gold["spmm_1x4"], gold["compress_4x2"]
    A = np.array(ex["A"], dtype=np.float32)
    vals = np.array(cx["values"], np.float32)
    D = np.array(cx["D"], np.uint8)
    C = oracle.spmm_sparse_f64(A, vals, D, 4, 2, 4, 1)
    assert C.tolist() == ex["C_unscaled"]
    # Eq. 1's M/N prefactor is the reading R4 "not applied"; scaled form:
    assert (C * (4 / 2)).tolist() == ex["C_scaled"]
    C32 = oracle.spmm_sparse_f32seq(A, vals, D, 4, 2, 4, 1)
    assert C32.tolist() == ex["C_unscaled"]


def test_spec_validate_examples(oracle, gold):
    ex = gold["validate"]
    a = np.array(ex["out_of_range"], np.uint8)
    b = np.array(ex["not_increasing"], np.uint8)
    assert oracle.validate(a, ex["k"], ex["n"], ex["N"], ex["M"], ex["L"]) == ex["out_of_range_first_bad"]
    assert oracle.validate(b, ex["k"], ex["n"], ex["N"], ex["M"], ex["L"]) == ex["not_increasing_first_bad"]
    ok = np.array([[0], [3]], np.uint8)
    assert oracle.validate(ok, 4, 1, 2, 4, 1) == -1


def test_spec_confusion_examples(oracle, gold):
    ex = gold["confusion"]
    W = oracle.confusion(np.array(ex["one_by_one"]["approx"]), np.array(ex["one_by_one"]["exact"]))
    assert W.tolist() == ex["one_by_one"]["W"]
    C = np.array(ex["two_by_two_plus_one"]["exact"])
    assert oracle.confusion(C + 1, C).tolist() == ex["two_by_two_plus_one"]["W"]
    assert not oracle.confusion(C, C).any()


# --------------------------------------------------------------------------
# compression: brute force, invariants, ties, underfull windows, errors
# --------------------------------------------------------------------------
CFGS_SMALL_M = [(1, 2), (2, 4), (1, 4), (3, 4), (2, 8), (3, 8), (1, 8), (5, 8), (4, 4)]


@pytest.mark.parametrize("N,M", CFGS_SMALL_M)
@pytest.mark.parametrize("L", [1, 2, 4])
@pytest.mark.parametrize("kind", ["uniform", "integer"])
def test_compress_matches_brute_force(oracle, N, M, L, kind):
    k, n = 4 * M, 6 * L
    B = synth.make(kind, (k, n), seed=11 + N * 7 + M, tid=synth.TID_B)
    vals, D = oracle.compress(B, N, M, L)
    pruned = brute_force_prune(B, N, M, L)
    assert np.array_equal(oracle.decompress(vals, D, k, N, M, L), pruned)
    # explicit index check per window
    for t in range(k // M):
        for g in range(n // L):
            exp = brute_force_keep(B[t * M:(t + 1) * M, g * L:(g + 1) * L], N)
            assert D[t * N:(t + 1) * N, g].tolist() == exp


@pytest.mark.parametrize("N,M", CFGS_SMALL_M)
def test_sort_keep_equals_brute_force(N, M):
    for seed in range(20):
        win = synth.integer((M, 3), seed, 77)
        assert sort_keep(win, N) == brute_force_keep(win, N)


def test_compress_tie_rule_smaller_offset(oracle):
    # all vectors of equal norm -> lowest N offsets
    B = np.ones((8, 4), np.float32)
    B[1::2] *= -1.0
    vals, D = oracle.compress(B, 3, 8, 2)
    assert D[:, 0].tolist() == [0, 1, 2] and D[:, 1].tolist() == [0, 1, 2]


def test_compress_all_zero_and_underfull(oracle):
    # all-zero B -> indices [0..N); underfull window keeps all nonzero vectors
    # and fills with the smallest unused offsets (R10)
    B = np.zeros((8, 1), np.float32)
    vals, D = oracle.compress(B, 3, 8, 1)
    assert D[:, 0].tolist() == [0, 1, 2] and not vals.any()
    B[6, 0] = -2.0
    vals, D = oracle.compress(B, 3, 8, 1)
    assert D[:, 0].tolist() == [0, 1, 6] and vals[:, 0].tolist() == [0.0, 0.0, -2.0]


def test_compress_nan_rejected_inf_allowed(oracle):
    B = synth.uniform((8, 4), 1, 2)
    B[3, 1] = np.nan
    with pytest.raises(oracle.OracleError) as e:
        oracle.compress(B, 2, 4, 2)
    assert e.value.status == oracle.ERR_NONFINITE
    B[3, 1] = np.inf
    vals, D = oracle.compress(B, 1, 4, 2)
    assert D[0, 0] == 3  # +Inf score wins its window
    assert np.isinf(vals[0, 1])


def test_compress_shape_and_config_errors(oracle):
    B = np.zeros((6, 4), np.float32)
    with pytest.raises(oracle.OracleError) as e:
        oracle.compress(B, 2, 4, 1)  # k % M != 0
    assert e.value.status == oracle.ERR_SHAPE
    with pytest.raises(oracle.OracleError) as e:
        oracle.compress(np.zeros((4, 3), np.float32), 2, 4, 2)  # n % L != 0
    assert e.value.status == oracle.ERR_SHAPE
    for N, M, L in [(0, 4, 1), (5, 4, 1), (1, 257, 1), (1, 4, 0)]:
        assert oracle.check_config(N, M, L) == oracle.ERR_INVALID_CONFIG
    assert oracle.check_config(256, 256, 1) == 0


@pytest.mark.parametrize("N,M,L", [(2, 4, 4), (16, 32, 32), (4, 32, 8), (3, 8, 1), (1, 8, 4)])
def test_compress_invariants_roundtrip_idempotence(oracle, N, M, L):
    k, n = 4 * M, 8 * L
    B = synth.uniform((k, n), 5, synth.TID_B)
    vals, D = oracle.compress(B, N, M, L)
    w, q = k // M * N, n // L
    assert vals.shape == (w, n) and D.shape == (w, q)
    Dw = D.reshape(k // M, N, q)
    assert (Dw < M).all()
    assert (np.diff(Dw.astype(int), axis=1) > 0).all()
    assert oracle.validate(D, k, n, N, M, L) == -1
    pruned = oracle.decompress(vals, D, k, N, M, L)
    # exactly the kept vectors survive, bit-exact copies of B
    kept = np.zeros((k, n), bool)
    for u in range(w):
        for g in range(q):
            kept[(u // N) * M + D[u, g], g * L:(g + 1) * L] = True
    assert np.array_equal(pruned[kept], B[kept]) and not pruned[~kept].any()
    assert kept.sum() == w * n
    # idempotence: compressing the pruned matrix gives the same result
    vals2, D2 = oracle.compress(pruned, N, M, L)
    assert np.array_equal(vals2, vals) and np.array_equal(D2, D)


def test_bf16_rne_matches_torch(oracle):
    torch = pytest.importorskip("torch")
    x = synth.uniform((4096,), 3, 9) * np.float32(3.7)
    edge = np.array([0.0, -0.0, 1.0, np.inf, -np.inf, 1e-40, -1e-40, 3.4e38,
                     np.float32(1.0) + np.float32(2 ** -8), np.float32(1.0) + np.float32(3 * 2 ** -8),
                     np.float32(1.0) + np.float32(2 ** -9)], np.float32)
    x = np.concatenate([x, edge])
    ours = oracle.f32_to_bf16(x)
    ref = torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(ours, ref)


def test_compress_bf16_values(oracle):
    B = synth.uniform((64, 64), 4, synth.TID_B)
    vals32, D32 = oracle.compress(B, 8, 32, 8)
    vals16, D16 = oracle.compress(B, 8, 32, 8, values_bf16=True)
    assert np.array_equal(D16, D32)  # selection on the input values (R11)
    assert np.array_equal(vals16, oracle.f32_to_bf16(vals32))
    # bf16 input -> bf16 copy
    Bh = synth.to_bf16_bits(synth.bf16grid((64, 64), 4, synth.TID_B))
    vh, Dh = oracle.compress(Bh, 8, 32, 8)
    assert vh.dtype == np.uint16
    vf, Df = oracle.compress(oracle.bf16_to_f32(Bh), 8, 32, 8)
    assert np.array_equal(Dh, Df) and np.array_equal(oracle.bf16_to_f32(vh), vf)


# --------------------------------------------------------------------------
# SpMM semantics
# --------------------------------------------------------------------------
@pytest.mark.parametrize("N,M", [(2, 4), (3, 8), (1, 4), (16, 32), (4, 32)])
@pytest.mark.parametrize("L", [1, 4, 8])
def test_integer_inputs_exact_vs_bruteforce(oracle, N, M, L):
    """pin (ii)+(vi): integer A, B -> every partial sum exact; compare with numpy
    int64 matmul of A and the independently brute-force-pruned B."""
    m, k, n = 24, 4 * M, 4 * L * 2
    A = synth.integer((m, k), 21, synth.TID_A)
    B = synth.integer((k, n), 22, synth.TID_B)
    vals, D = oracle.compress(B, N, M, L)
    exact = A.astype(np.int64) @ brute_force_prune(B, N, M, L).astype(np.int64)
    assert np.array_equal(oracle.spmm_sparse_f64(A, vals, D, k, N, M, L), exact)
    assert np.array_equal(oracle.spmm_sparse_f32seq(A, vals, D, k, N, M, L), exact)
    dense = oracle.decompress(vals, D, k, N, M, L)
    assert np.array_equal(oracle.gemm_dense_f64(A, dense), exact)


@pytest.mark.parametrize("N,M", [(2, 4), (3, 8), (2, 8), (1, 8), (16, 32)])
@pytest.mark.parametrize("L", [1, 4, 8])
@pytest.mark.parametrize("mkn", [(64, 64, 64), (128, 128, 256)])
def test_o1_equals_o2_bit_exact(oracle, N, M, L, mkn):
    """sparse loop == dense loop on the decompressed B, bit-exactly
    (same nonzero terms in the same order)."""
    m, k, n = mkn
    A = synth.uniform((m, k), 31, synth.TID_A)
    B = synth.uniform((k, n), 32, synth.TID_B)
    vals, D = oracle.compress(B, N, M, L)
    dense = oracle.decompress(vals, D, k, N, M, L)
    assert np.array_equal(oracle.spmm_sparse_f64(A, vals, D, k, N, M, L),
                          oracle.gemm_dense_f64(A, dense))
    assert np.array_equal(oracle.spmm_sparse_f32seq(A, vals, D, k, N, M, L),
                          oracle.gemm_dense_f32seq(A, dense))
    # and the fp64 result agrees with numpy's fp64 matmul (library routine)
    ref = A.astype(np.float64) @ dense.astype(np.float64)
    assert oracle.rel_frobenius(oracle.spmm_sparse_f64(A, vals, D, k, N, M, L), ref) < 1e-13


@pytest.mark.slow
def test_o1_equals_o2_512(oracle):
    m = k = n = 512
    for (N, M), L in [((2, 4), 4), ((16, 32), 8), ((1, 8), 1)]:
        A = synth.uniform((m, k), 41, synth.TID_A)
        B = synth.uniform((k, n), 42, synth.TID_B)
        vals, D = oracle.compress(B, N, M, L)
        dense = oracle.decompress(vals, D, k, N, M, L)
        assert np.array_equal(oracle.spmm_sparse_f64(A, vals, D, k, N, M, L),
                              oracle.gemm_dense_f64(A, dense))


def test_n_equals_m_is_dense_gemm(oracle):
    """pin (i): N = M keeps everything; D is the identity pattern."""
    m, k, n, M, L = 32, 64, 48, 8, 4
    A = synth.uniform((m, k), 51, synth.TID_A)
    B = synth.uniform((k, n), 52, synth.TID_B)
    vals, D = oracle.compress(B, M, M, L)
    assert np.array_equal(vals, B)
    assert (D == np.tile(np.arange(M, dtype=np.uint8), k // M)[:, None]).all()
    assert np.array_equal(oracle.spmm_sparse_f32seq(A, vals, D, k, M, M, L),
                          oracle.gemm_dense_f32seq(A, B))
    ref = A.astype(np.float64) @ B.astype(np.float64)
    assert oracle.rel_frobenius(oracle.spmm_sparse_f64(A, vals, D, k, M, M, L), ref) < 1e-14


def test_identity_a_gives_pruned_b(oracle):
    """pin (iii): A = I_k gives C = B~ exactly."""
    k, n, N, M, L = 64, 32, 3, 8, 4
    B = synth.uniform((k, n), 61, synth.TID_B)
    vals, D = oracle.compress(B, N, M, L)
    C = oracle.spmm_sparse_f64(np.eye(k, dtype=np.float32), vals, D, k, N, M, L)
    assert np.array_equal(C, brute_force_prune(B, N, M, L).astype(np.float64))


def test_all_ones_gives_w(oracle):
    """pin (iv): all-ones A and B' (any valid D) give C == w everywhere."""
    m, k, n, N, M, L = 8, 96, 64, 5, 32, 16
    w = k // M * N
    D = synth.random_mask(k, n, N, M, L, seed=3)
    C = oracle.spmm_sparse_f64(np.ones((m, k), np.float32), np.ones((w, n), np.float32), D, k, N, M, L)
    assert (C == w).all()


def test_linearity_in_a(oracle):
    m, k, n, N, M, L = 16, 64, 64, 4, 16, 8
    A1 = synth.uniform((m, k), 71, synth.TID_A)
    A2 = synth.uniform((m, k), 72, synth.TID_A)
    B = synth.uniform((k, n), 73, synth.TID_B)
    vals, D = oracle.compress(B, N, M, L)
    lhs = oracle.spmm_sparse_f64((np.float32(0.5) * A1 + A2).astype(np.float32), vals, D, k, N, M, L)
    rhs = 0.5 * oracle.spmm_sparse_f64(A1, vals, D, k, N, M, L) + oracle.spmm_sparse_f64(A2, vals, D, k, N, M, L)
    assert oracle.rel_frobenius(lhs, rhs) < 1e-6


def test_row_sample_equals_full(oracle):
    m, k, n, N, M, L = 40, 64, 64, 2, 8, 4
    A = synth.uniform((m, k), 81, synth.TID_A)
    B = synth.uniform((k, n), 82, synth.TID_B)
    vals, D = oracle.compress(B, N, M, L)
    full = oracle.spmm_sparse_f64(A, vals, D, k, N, M, L)
    rows = [0, 7, 39, 13]
    assert np.array_equal(oracle.spmm_sparse_f64(A, vals, D, k, N, M, L, rows=rows), full[rows])


@pytest.mark.parametrize("G", [2, 3, 8])
def test_sharded_concat_equals_full(oracle, G):
    """pin (viii): column j depends only on B'[:, j] and D[:, j//L]; the
    concatenation of per-shard results equals the full result bit-for-bit."""
    m, k, n, N, M, L = 16, 64, 11 * 8, 4, 16, 8
    A = synth.uniform((m, k), 91, synth.TID_A)
    B = synth.uniform((k, n), 92, synth.TID_B)
    vals, D = oracle.compress(B, N, M, L)
    q = n // L
    full = oracle.spmm_sparse_f64(A, vals, D, k, N, M, L)
    parts = []
    for r in range(G):
        g0, g1 = r * q // G, (r + 1) * q // G
        parts.append(oracle.spmm_sparse_f64(A, vals[:, g0 * L:g1 * L], D[:, g0:g1], k, N, M, L))
    assert np.array_equal(np.concatenate(parts, axis=1), full)


def test_bf16_operands_exact_products(oracle):
    """bf16 A and B' widen exactly; integer bf16 inputs reproduce the int64 matmul."""
    m, k, n, N, M, L = 16, 64, 64, 8, 32, 32
    A = synth.integer((m, k), 101, synth.TID_A)
    B = synth.integer((k, n), 102, synth.TID_B)
    vals, D = oracle.compress(synth.to_bf16_bits(B), N, M, L)
    C = oracle.spmm_sparse_f64(synth.to_bf16_bits(A), vals, D, k, N, M, L)
    exact = A.astype(np.int64) @ brute_force_prune(B, N, M, L).astype(np.int64)
    assert np.array_equal(C, exact)


def test_eq1_scaled_hand_example(oracle):
    """Eq. 1 as printed (with M/N) and Eq. 2 on a hand-worked case:
    A = [1 2 3 4], B = [1 5 2 3]^T, 2:4, L = 1 -> keep offsets 1 and 3 (|5|, |3|),
    sum = 2*5 + 4*3 = 22, C' = (4/2)*22 = 44; unpruned C = 1 + 10 + 6 + 12 = 29; W = |44-29|/1 = 15."""
    A = np.array([[1, 2, 3, 4]], dtype=np.float32)
    B = np.array([[1], [5], [2], [3]], dtype=np.float32)
    vals, D = oracle.compress(B, 2, 4, 1)
    assert D.ravel().tolist() == [1, 3] and vals.ravel().tolist() == [5.0, 3.0]
    Cs = oracle.spmm_eq1_scaled_f64(A, vals, D, 4, 2, 4, 1)
    assert Cs.tolist() == [[44.0]]
    assert oracle.spmm_sparse_f64(A, vals, D, 4, 2, 4, 1).tolist() == [[22.0]]
    C = oracle.gemm_dense_f64(A, B)
    assert C.tolist() == [[29.0]]
    assert oracle.confusion(Cs, C).tolist() == [[15.0]]


@pytest.mark.parametrize("L", [1, 4, 8])
def test_eq1_scaled_dense_window_is_gemm(oracle, L):
    """N = M: nothing is pruned and M/N = 1, so Eq. 1 as printed is the dense product (checked
    against the independent dense triple loop) and the confusion W of Eq. 2 is zero."""
    from paper_2503_01253_b200 import synth
    m, k, n = 9, 16, 4 * L
    A = synth.uniform((m, k), 61, synth.TID_A)
    B = synth.uniform((k, n), 62, synth.TID_B)
    vals, D = oracle.compress(B, 8, 8, L)
    Cs = oracle.spmm_eq1_scaled_f64(A, vals, D, k, 8, 8, L)
    C = oracle.gemm_dense_f64(A, B)
    assert np.allclose(Cs, C, rtol=1e-12, atol=1e-12)
    assert np.abs(oracle.confusion(Cs, C)).max() <= 1e-12


def test_rel_frobenius_hand_values(oracle):
    """SURVEY 8(c)5 tolerance metric ||C - C_ref||_F / ||C_ref||_F, pinned by hand-computed
    values (not by restating the formula): a dropped square root, a swapped numerator /
    denominator or a missing zero-reference branch each fails one of these."""
    # ||(0, -4)|| / ||(3, 4)|| = 4 / 5
    assert oracle.rel_frobenius(np.array([[3.0, 0.0]]), np.array([[3.0, 4.0]])) == 0.8
    # the reference is the denominator: ||(0, 4)|| / ||(3, 0)|| = 4 / 3
    assert abs(oracle.rel_frobenius(np.array([[3.0, 4.0]]), np.array([[3.0, 0.0]])) - 4.0 / 3.0) < 1e-15
    # Frobenius over all elements of a 2-D array: diff (1, 2; 2, 0) has norm 3, ref (2, 0; 0, 0) norm 2
    assert oracle.rel_frobenius(np.array([[3.0, 2.0], [2.0, 0.0]]), np.array([[2.0, 0.0], [0.0, 0.0]])) == 1.5
    # zero reference: the absolute norm of C (||(3, 4)|| = 5), and 0 for C = C_ref = 0
    assert oracle.rel_frobenius(np.array([[3.0, 4.0]]), np.zeros((1, 2))) == 5.0
    assert oracle.rel_frobenius(np.zeros((2, 2)), np.zeros((2, 2))) == 0.0
    # identical inputs give exactly 0; a uniform 1e-3 relative perturbation gives 1e-3
    R = np.arange(1.0, 13.0).reshape(3, 4)
    assert oracle.rel_frobenius(R, R) == 0.0
    assert abs(oracle.rel_frobenius(R * (1 + 1e-3), R) - 1e-3) < 1e-12
    # fp32 / bf16-widened inputs are compared in fp64 (no float32 cancellation): 1 + 2^-30 vs 1
    assert oracle.rel_frobenius(np.array([[1.0 + 2.0 ** -30]]), np.array([[1.0]], dtype=np.float32)) == 2.0 ** -30


# ----------------------------------------------------------------------------- bit-packed indices
def test_index_bits_closed_form(oracle):
    """an index needs only ceil(log2 M) bits: the largest offset M - 1 fits in b bits and
    not in b - 1 (b >= 1)."""
    for M in [1, 2, 3, 4, 5, 7, 8, 9, 16, 31, 32, 33, 64, 100, 128, 129, 255, 256]:
        b = oracle.index_bits(M)
        assert (M - 1) < (1 << b)
        assert b == 1 or (M - 1) >= (1 << (b - 1))


def test_index_pack_hand_example(oracle):
    """Hand-packed words (R28).  M = 4 -> 2-bit entries, 16 per word; L = 32 -> tiles of
    T = 4 groups, a tile's entries numbered x = u*T + t.  w = 4 rows -> 16 entries = 1 word per tile.
    Row 0 of groups 0..7 = [1, 3, 0, 2 | 2, 1, 3, 0], row 1 = [3, 0, 0, 0 | 0, 0, 0, 1]:
    tile 0 = 1 + 3*4 + 0*16 + 2*64 + 3*256 = 909, tile 1 = 2 + 1*4 + 3*16 + 0*64 + 1*2^14 = 16438."""
    k, n, N, M, L = 8, 256, 2, 4, 32
    D = np.zeros((4, 8), dtype=np.uint8)
    D[0] = [1, 3, 0, 2, 2, 1, 3, 0]
    D[1] = [3, 0, 0, 0, 0, 0, 0, 1]
    P = oracle.index_pack(D, k, n, N, M, L)
    assert list(P) == [909, 16438]
    # M = 32 -> 5-bit entries, 6 per word; L = 16 -> tiles of 8 groups; one row = 2 words:
    # [31, 0, 7, 16, 1, 2 | 30, 5] -> 31 + 7*2^10 + 16*2^15 + 2^20 + 2*2^25 = 68688927, 30 + 5*32 = 190
    D2 = np.array([[31, 0, 7, 16, 1, 2, 30, 5]], dtype=np.uint8)
    P2 = oracle.index_pack(D2, 32, 128, 1, 32, 16)
    assert list(P2) == [68688927, 190]


@pytest.mark.parametrize("N,M,L", [(2, 4, 4), (16, 32, 32), (4, 32, 8), (3, 8, 16), (1, 2, 64), (5, 256, 128),
                                   (12, 32, 32), (7, 100, 4)])
def test_index_pack_roundtrip_and_size(oracle, N, M, L):
    """Lossless (unpack . pack = identity on compressed indices, ragged last tile included) and the
    footprint of log2-M-bit entries: 32 / floor(32 / b) bits per entry + at most one partial word
    per tile (b = 5 at M = 32: 5.33 bits instead of the 8 of a byte)."""
    k, n = 8 * M, 128 * 3 + 2 * L
    B = synth.uniform((k, n), 31, synth.TID_B)
    _, D = oracle.compress(B, N, M, L)
    P = oracle.index_pack(D, k, n, N, M, L)
    assert np.array_equal(oracle.index_unpack(P, k, n, N, M, L), D)
    b, w, q, T = oracle.index_bits(M), k // M * N, n // L, 128 // L
    e = 32 // b
    ntiles = -(-q // T)
    assert P.size == ntiles * -(-(w * T) // e)
    assert P.nbytes * 8 * e <= ntiles * T * w * 32 + 32 * ntiles * e  # 32 / e bits per entry
