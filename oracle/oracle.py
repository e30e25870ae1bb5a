"""ctypes shim over ``oracle/libnmoracle.so`` (built from ``nm_oracle.c``).

TEST INFRASTRUCTURE ONLY: only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference``) may import
this module.  It shares no code with the CUDA path and never imports the
product package.  Every function cites the PAPER.md passage it follows in
``nm_oracle.c``; see that file's header for the notation.

bf16 arrays are passed as ``numpy.uint16`` bit patterns.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "nm_oracle.c")
_LIB = os.path.join(_HERE, "libnmoracle.so")

OK = 0
ERR_INVALID_CONFIG = 1
ERR_SHAPE = 2
ERR_NONFINITE = 4
ERR_INVALID_INDICES = 6


class OracleError(RuntimeError):
    def __init__(self, status: int, what: str):
        super().__init__(f"oracle {what} failed with status {status}")
        self.status = status


def build(force: bool = False) -> str:
    """Compile the oracle (gcc, -O2, OpenMP, no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=c11", "-fopenmp", "-ffp-contract=off", "-fno-fast-math",
               "-fPIC", "-shared", _SRC, "-o", _LIB + ".tmp", "-lm"]
        subprocess.run(cmd, check=True)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        P, I64, I = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
        L.nmo_check_config.argtypes = [I, I, I]
        L.nmo_compress.argtypes = [P, I, I64, I64, I, I, I, P, I, P]
        L.nmo_decompress.argtypes = [P, I, P, I64, I64, I, I, I, P]
        L.nmo_validate.argtypes = [P, I64, I64, I, I, I]
        L.nmo_validate.restype = I64
        L.nmo_spmm_sparse_f64.argtypes = [P, I, P, I, P, I64, I64, I64, I, I, I, P, I64, P, I]
        L.nmo_spmm_sparse_f32seq.argtypes = [P, I, P, I, P, I64, I64, I64, I, I, I, P, I]
        L.nmo_spmm_eq1_scaled_f64.argtypes = [P, I, P, I, P, I64, I64, I64, I, I, I, P, I]
        L.nmo_gemm_dense_f64.argtypes = [P, I, P, I, I64, I64, I64, P, I]
        L.nmo_gemm_dense_f32seq.argtypes = [P, I, P, I, I64, I64, I64, P, I]
        L.nmo_confusion.argtypes = [P, P, I64, I64, P]
        L.nmo_f32_to_bf16_rne.argtypes = [ctypes.c_float]
        L.nmo_f32_to_bf16_rne.restype = ctypes.c_uint16
        L.nmo_num_threads.argtypes = [I]
        L.nmo_index_bits.argtypes = [I]
        L.nmo_index_packed_words.argtypes = [I64, I64, I, I, I]
        L.nmo_index_packed_words.restype = I64
        L.nmo_index_pack.argtypes = [P, I64, I64, I, I, I, P]
        L.nmo_index_unpack.argtypes = [P, I64, I64, I, I, I, P]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _is_bf16(a: np.ndarray) -> int:
    if a.dtype == np.uint16:
        return 1
    if a.dtype == np.float32:
        return 0
    raise TypeError(f"oracle takes float32 or bf16-as-uint16 arrays, got {a.dtype}")


def _c(a: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(a)


def num_threads(nthreads: int = 0) -> int:
    return int(lib().nmo_num_threads(nthreads))


def check_config(N: int, M: int, L: int) -> int:
    return int(lib().nmo_check_config(N, M, L))


def compress(B: np.ndarray, N: int, M: int, L: int, values_bf16: bool | None = None):
    """P:93 compression; returns (B' (w x n), D (w x q) uint8).  See nm_oracle.c."""
    B = _c(B)
    k, n = B.shape
    b16 = _is_bf16(B)
    v16 = b16 if values_bf16 is None else int(values_bf16)
    s = check_config(N, M, L)
    if s:
        raise OracleError(s, "compress")
    if k % M or n % L:
        raise OracleError(ERR_SHAPE, "compress")
    w, q = k // M * N, n // L
    vals = np.empty((w, n), dtype=np.uint16 if v16 else np.float32)
    D = np.empty((w, q), dtype=np.uint8)
    s = lib().nmo_compress(_p(B), b16, k, n, N, M, L, _p(vals), v16, _p(D))
    if s:
        raise OracleError(s, "compress")
    return vals, D


def decompress(values: np.ndarray, D: np.ndarray, k: int, N: int, M: int, L: int) -> np.ndarray:
    """Inverse of P:93: dense k x n with +0.0 off the kept vectors."""
    values, D = _c(values), _c(D)
    v16 = _is_bf16(values)
    n = values.shape[1]
    out = np.empty((k, n), dtype=values.dtype)
    s = lib().nmo_decompress(_p(values), v16, _p(D), k, n, N, M, L, _p(out))
    if s:
        raise OracleError(s, "decompress")
    return out


def validate(D: np.ndarray, k: int, n: int, N: int, M: int, L: int) -> int:
    """-1 if valid, else the first bad flat index u*q+g (-2: bad config)."""
    D = _c(D.astype(np.uint8, copy=False))
    return int(lib().nmo_validate(_p(D), k, n, N, M, L))


def spmm_sparse_f64(A: np.ndarray, values: np.ndarray, D: np.ndarray, k: int, N: int, M: int,
                    L: int, rows=None, nthreads: int = 0) -> np.ndarray:
    """O2 (Eq. 1 corrected, unscaled): fp64 result, optional row sample."""
    A, values, D = _c(A), _c(values), _c(D)
    m = A.shape[0]
    n = values.shape[1]
    if A.shape[1] != k:
        raise OracleError(ERR_SHAPE, "spmm")
    if rows is not None:
        rows = np.ascontiguousarray(np.asarray(rows, dtype=np.int64))
        C = np.empty((rows.shape[0], n), dtype=np.float64)
        rp, nr = _p(rows), rows.shape[0]
    else:
        C = np.empty((m, n), dtype=np.float64)
        rp, nr = None, 0
    s = lib().nmo_spmm_sparse_f64(_p(A), _is_bf16(A), _p(values), _is_bf16(values), _p(D), m, n, k,
                                  N, M, L, rp, nr, _p(C), nthreads)
    if s:
        raise OracleError(s, "spmm_sparse_f64")
    return C


def spmm_eq1_scaled_f64(A, values, D, k, N, M, L, nthreads: int = 0) -> np.ndarray:
    """O2s: Eq. 1 as printed, with the M/N factor, fp64."""
    A, values, D = _c(A), _c(values), _c(D)
    m, n = A.shape[0], values.shape[1]
    C = np.empty((m, n), dtype=np.float64)
    s = lib().nmo_spmm_eq1_scaled_f64(_p(A), _is_bf16(A), _p(values), _is_bf16(values), _p(D), m, n, k, N, M,
                                      L, _p(C), nthreads)
    if s:
        raise OracleError(s, "spmm_eq1_scaled_f64")
    return C


def spmm_sparse_f32seq(A, values, D, k, N, M, L, nthreads: int = 0) -> np.ndarray:
    """O2f: Eq. 1 with a sequential fp32 accumulator."""
    A, values, D = _c(A), _c(values), _c(D)
    m, n = A.shape[0], values.shape[1]
    C = np.empty((m, n), dtype=np.float32)
    s = lib().nmo_spmm_sparse_f32seq(_p(A), _is_bf16(A), _p(values), _is_bf16(values), _p(D), m, n,
                                     k, N, M, L, _p(C), nthreads)
    if s:
        raise OracleError(s, "spmm_sparse_f32seq")
    return C


def gemm_dense_f64(A, B, nthreads: int = 0) -> np.ndarray:
    """Dense triple loop, fp64 accumulation; O1 = gemm_dense_f64(A, decompress(...))."""
    A, B = _c(A), _c(B)
    m, k = A.shape
    n = B.shape[1]
    C = np.empty((m, n), dtype=np.float64)
    lib().nmo_gemm_dense_f64(_p(A), _is_bf16(A), _p(B), _is_bf16(B), m, n, k, _p(C), nthreads)
    return C


def gemm_dense_f32seq(A, B, nthreads: int = 0) -> np.ndarray:
    """O1f: dense loop with a sequential fp32 accumulator."""
    A, B = _c(A), _c(B)
    m, k = A.shape
    n = B.shape[1]
    C = np.empty((m, n), dtype=np.float32)
    lib().nmo_gemm_dense_f32seq(_p(A), _is_bf16(A), _p(B), _is_bf16(B), m, n, k, _p(C), nthreads)
    return C


def confusion(C_approx: np.ndarray, C_exact: np.ndarray) -> np.ndarray:
    """Eq. 2 verbatim: |C' - C| / (m*n)."""
    a = _c(C_approx.astype(np.float64))
    b = _c(C_exact.astype(np.float64))
    W = np.empty_like(a)
    lib().nmo_confusion(_p(a), _p(b), a.shape[0], a.shape[1], _p(W))
    return W


def f32_to_bf16(x: np.ndarray) -> np.ndarray:
    """RNE fp32 -> bf16 bit patterns (R11), element by element."""
    f = lib().nmo_f32_to_bf16_rne
    flat = np.asarray(x, dtype=np.float32).ravel()
    return np.array([f(float(v)) for v in flat], dtype=np.uint16).reshape(np.shape(x))


def bf16_to_f32(h: np.ndarray) -> np.ndarray:
    """Exact widening of bf16 bit patterns."""
    return (np.asarray(h, dtype=np.uint32) << 16).view(np.float32)


def rel_frobenius(C: np.ndarray, C_ref: np.ndarray) -> float:
    """Tolerance metric: ||C - C_ref||_F / ||C_ref||_F in fp64."""
    d = np.asarray(C, dtype=np.float64) - np.asarray(C_ref, dtype=np.float64)
    den = np.linalg.norm(np.asarray(C_ref, dtype=np.float64))
    num = np.linalg.norm(d)
    return float(num / den) if den > 0 else float(num)


def index_bits(M: int) -> int:
    """bits per packed index entry, max(1, ceil(log2 M))."""
    return int(lib().nmo_index_bits(M))


def index_pack(D: np.ndarray, k: int, n: int, N: int, M: int, L: int) -> np.ndarray:
    """P:288 + P:419 (transformLayout): D (w x q uint8) -> the tile-major bit-packed words
    (R28; layout in nm_oracle.c).  Needs 128 % L == 0."""
    nw = int(lib().nmo_index_packed_words(k, n, N, M, L))
    if nw < 0:
        raise OracleError(ERR_SHAPE, "index_pack")
    out = np.empty(max(nw, 1), dtype=np.uint32)
    s = lib().nmo_index_pack(_p(_c(D.astype(np.uint8, copy=False))), k, n, N, M, L, _p(out))
    if s:
        raise OracleError(s, "index_pack")
    return out[:nw]


def index_unpack(P: np.ndarray, k: int, n: int, N: int, M: int, L: int) -> np.ndarray:
    w, q = k // M * N, n // L
    D = np.empty((w, q), dtype=np.uint8)
    s = lib().nmo_index_unpack(_p(_c(P.astype(np.uint32, copy=False))), k, n, N, M, L, _p(D))
    if s:
        raise OracleError(s, "index_unpack")
    return D
