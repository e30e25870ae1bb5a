"""Column-sharded multi-GPU N:M SpMM, one process per GPU.

Column j of C depends only on A, B'[:, j] and D[:, j // L] (Eq. 1),
so the q = n/L column groups are split over the G ranks: rank r owns groups
[floor(r*q/G), floor((r+1)*q/G)).  Every rank's shard is padded to
ceil(q/G) groups (zero values, a valid index pattern) so that the NCCL
all-gather moves equal-size [m][nr] blocks; nm_unshard_columns (our kernel)
drops the padding and writes the m x n row-major C.  A is replicated (the
input of a column-parallel layer).  No reduction is needed.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_ranges(q: int, G: int):
    """[(g0, g1)] per rank: rank r owns groups [floor(r*q/G), floor((r+1)*q/G))."""
    return [(r * q // G, (r + 1) * q // G) for r in range(G)]


def groups_per_shard(q: int, G: int) -> int:
    return -(-q // G)


def shard_weight(values: torch.Tensor, idx: torch.Tensor, L: int, N: int, rank: int, G: int):
    """This rank's slice of (B', D), padded to ceil(q/G) groups: padded values are
    +0.0 and padded index columns hold the valid pattern 0..N-1 per window."""
    w, n = values.shape
    q = n // L
    g0, g1 = shard_ranges(q, G)[rank]
    gp = groups_per_shard(q, G)
    v = torch.zeros((w, gp * L), dtype=values.dtype, device=values.device)
    d = torch.arange(N, dtype=torch.uint8, device=idx.device).repeat(w // N).reshape(w, 1).repeat(1, gp)
    v[:, :(g1 - g0) * L] = values[:, g0 * L:g1 * L]
    d[:, :g1 - g0] = idx[:, g0:g1]
    return v.contiguous(), d.contiguous()


class ShardedNmLinear:
    """y = x . B~ with B~'s column groups sharded over a process group (NCCL)."""

    def __init__(self, local_weight, n: int, group=None):
        from . import nmspmm
        self.W = local_weight  # nmspmm.NmWeight of this rank's padded shard
        # the offline weight prepack once per layer: the bf16 sparse-tensor-core
        # kernel's slot packing and images; plain values/idx for the fp32 path
        self.PW = nmspmm.nm_prepack(local_weight) if local_weight.values.is_cuda else None
        self.group = group
        self.G = dist.get_world_size(group)
        self.n = n
        self.nr = local_weight.n

    @classmethod
    def from_dense(cls, B: torch.Tensor, N: int, M: int, L: int, group=None):
        """Compress only this rank's columns (compression is per column group, so
        the shard of compress(B) equals compress of the shard)."""
        from . import nmspmm
        G, r = dist.get_world_size(group), dist.get_rank(group)
        k, n = B.shape
        q = n // L
        g0, g1 = shard_ranges(q, G)[r]
        gp = groups_per_shard(q, G)
        Bs = torch.zeros((k, gp * L), dtype=B.dtype, device=B.device)
        Bs[:, :(g1 - g0) * L] = B[:, g0 * L:g1 * L]
        # padding groups are all-zero: compress gives zero values and the pattern 0..N-1
        W = nmspmm.nm_compress(Bs.contiguous(), N, M, L)
        return cls(W, n, group)

    def local(self, A: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        from . import nmspmm
        if self.PW is not None:
            return nmspmm.nm_spmm_prepacked(A, self.PW, out=out)
        return nmspmm.nm_spmm(A, self.W, out=out)

    def __call__(self, A: torch.Tensor) -> torch.Tensor:
        from . import nmspmm
        m = A.shape[0]
        c_local = self.local(A)
        if self.G == 1 and self.nr == self.n:  # a single shard is already C (no exchange step)
            return c_local
        gathered = torch.empty((self.G, m, self.nr), dtype=c_local.dtype, device=A.device)
        dist.all_gather_into_tensor(gathered, c_local, group=self.group)
        C = torch.empty((m, self.n), dtype=c_local.dtype, device=A.device)
        nmspmm.nm_unshard_columns(gathered, C, self.G, m, self.nr, self.n, self.W.L)
        return C
