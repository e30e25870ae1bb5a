"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This module holds NO arithmetic of the method (no compression, no product):
only a counter-based generator, so that the CPU oracle and the CUDA path can be
fed bit-identical inputs.  Recipe:

  h = splitmix64(seed ^ (tensor_id * 0x9E3779B97F4A7C15) ^ index)    (uint64)
  uniform : x = (h >> 40) * 2^-23 - 1   in [-1, 1), exact in fp32
  bf16grid: x = (h >> 56) * 2^-7  - 1   in [-1, 1), exact in bf16 and fp32
  integer : x = (h % 5) - 2             in {-2..2} (exact partial sums, pin ii)

Masks for benchmarks that bypass magnitude pruning:
  random: per (window t, group g) the N offsets with the smallest keys
          h(seed, tid, (t*q + g)*M + r), sorted ascending;
  shared: the same pattern for every group of a window (key index t*M + r).
"""
from __future__ import annotations

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)

# tensor ids (seed ^ tid*GOLDEN keeps streams independent)
TID_A = 1
TID_B = 2
TID_MASK = 3


def splitmix64(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = x + GOLDEN
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def _hash(count: int, seed: int, tid: int, start: int = 0) -> np.ndarray:
    idx = np.arange(start, start + count, dtype=np.uint64)
    with np.errstate(over="ignore"):
        key = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) ^ (np.uint64(tid) * GOLDEN)
    return splitmix64(idx ^ key)


def _gen(shape, seed, tid, fn, chunk=1 << 24):
    total = int(np.prod(shape))
    out = np.empty(total, dtype=np.float32)
    for s in range(0, total, chunk):
        e = min(total, s + chunk)
        out[s:e] = fn(_hash(e - s, seed, tid, s))
    return out.reshape(shape)


def uniform(shape, seed: int, tid: int) -> np.ndarray:
    """U[-1,1) on the 2^-23 grid (exact fp32)."""
    return _gen(shape, seed, tid,
                lambda h: ((h >> np.uint64(40)).astype(np.float64) * 2.0 ** -23 - 1.0))


def bf16grid(shape, seed: int, tid: int) -> np.ndarray:
    """U[-1,1) on the 2^-7 grid: exactly representable in bf16 (returned as fp32)."""
    return _gen(shape, seed, tid,
                lambda h: ((h >> np.uint64(56)).astype(np.float64) * 2.0 ** -7 - 1.0))


def integer(shape, seed: int, tid: int) -> np.ndarray:
    """Integers in {-2,...,2} (as fp32)."""
    return _gen(shape, seed, tid, lambda h: (h % np.uint64(5)).astype(np.float64) - 2.0)


def make(kind: str, shape, seed: int, tid: int) -> np.ndarray:
    return {"uniform": uniform, "bf16grid": bf16grid, "integer": integer}[kind](shape, seed, tid)


def to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Bit patterns of fp32 values that are exactly bf16 (bf16grid / integer):
    the upper 16 bits; raises if a value is not exactly representable."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    if np.any(u & np.uint32(0xFFFF)):
        raise ValueError("value not exactly representable in bf16")
    return (u >> np.uint32(16)).astype(np.uint16)


def random_mask(k: int, n: int, N: int, M: int, L: int, seed: int, shared: bool = False):
    """Index matrix D (w x q, uint8): a uniform N-subset per window (and group),
    sorted ascending.  shared=True gives every group of a window the same subset."""
    T, q = k // M, n // L
    if shared:
        keys = _hash(T * M, seed, TID_MASK).reshape(T, 1, M)
        keys = np.broadcast_to(keys, (T, q, M))
    else:
        keys = _hash(T * q * M, seed, TID_MASK).reshape(T, q, M)
    sel = np.sort(np.argsort(keys, axis=2, kind="stable")[:, :, :N], axis=2)  # T x q x N
    return np.ascontiguousarray(sel.transpose(0, 2, 1).reshape(T * N, q).astype(np.uint8))
