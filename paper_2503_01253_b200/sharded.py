"""Column-sharded multi-GPU N:M SpMM, one process per GPU.

Column j of C depends only on A, B'[:, j] and D[:, j // L] (Eq. 1),
so the q = n/L column groups are split over the G ranks: rank r owns groups
[floor(r*q/G), floor((r+1)*q/G)).  Every rank's shard is padded to
ceil(q/G) groups (zero values, a valid index pattern) so that the NCCL
all-gather moves equal-size [m][nr] blocks; nm_unshard_columns (our kernel)
drops the padding and writes the m x n row-major C.  A is replicated (the
input of a column-parallel layer).  No reduction is needed.

exchange="p2p" fuses the exchange into the SpMM (fp32 SIMT or bf16 slot kernel): the ranks' C buffers are
mapped into every process by CUDA IPC, each rank's SpMM epilogue stores its
columns into all of them over NVLink (nm_spmm_peers), and a flag barrier in
peer memory (nm_peer_barrier) orders the ranks -- stream-ordered, no all-gather
pass, no unshard pass.  The C buffers are double-buffered: the tensor returned
by call i stays valid for work this rank enqueues on its stream before its call
i + 1 (the peers overwrite it in call i + 2, which they start only after call
i + 1's barrier has seen this rank's stream reach call i + 1).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def host_staged_all_gather(out: torch.Tensor, inp: torch.Tensor, group=None, async_op=False):
    """all_gather_into_tensor through host memory (for backends without device collectives, e.g.
    gloo): out[r] = rank r's inp.  Synchronous (returns no work handle)."""
    parts = [torch.empty(inp.shape, dtype=inp.dtype) for _ in range(dist.get_world_size(group))]
    dist.all_gather(parts, inp.cpu(), group=group)
    out.copy_(torch.stack(parts))
    return None


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


class PeerExchange:
    """Per-layer peer mappings for exchange="p2p": two C buffers (m x n) and one int[G] flag
    array per rank, allocated by torch, exported by CUDA IPC, exchanged with
    all_gather_object over the group and opened in every other process."""

    def __init__(self, group, m: int, n: int, dtype, device):
        from . import nmspmm
        self.G, self.rank = dist.get_world_size(group), dist.get_rank(group)
        self.m, self.n = m, n
        self.C = [torch.empty((m, n), dtype=dtype, device=device) for _ in range(2)]
        self.flags = torch.zeros(self.G, dtype=torch.int32, device=device)
        torch.cuda.synchronize(device)  # zeroed flags before any peer can write them
        mine = [nmspmm.nm_ipc_get_handle(t) for t in (self.C[0], self.C[1], self.flags)]
        allh = [None] * self.G
        dist.all_gather_object(allh, mine, group=group)
        self.opened = []  # (ptr, offset) to close
        self.ptrs = [[0] * self.G for _ in range(3)]  # [buffer][rank]
        for r in range(self.G):
            for b in range(3):
                if r == self.rank:
                    self.ptrs[b][r] = (self.C[0], self.C[1], self.flags)[b].data_ptr()
                else:
                    h, off = allh[r][b]
                    ptr = nmspmm.nm_ipc_open_handle(h, off)
                    self.opened.append((ptr, off))
                    self.ptrs[b][r] = ptr
        self.epoch = 0
        dist.barrier(group=group)  # every rank mapped before anyone stores

    def close(self):
        from . import nmspmm
        torch.cuda.synchronize()  # no kernel of ours may still be storing through a mapping
        for ptr, off in self.opened:
            nmspmm.nm_ipc_close(ptr, off)
        self.opened = []


class ShardedNmLinear:
    """y = x . B~ with B~'s column groups sharded over a process group: exchange="nccl"
    (all-gather + unshard kernel) or "p2p" (fused peer-store epilogue: fp32 SIMT kernel, or the bf16
    sparse-tensor-core kernel's direct-store epilogue)."""

    def __init__(self, local_weight, n: int, group=None, exchange: str = "nccl", all_gather=None, chunks: int = 1,
                 m_hint: int | None = None):
        from . import nmspmm
        if exchange not in ("nccl", "p2p"):
            raise ValueError("exchange must be 'nccl' or 'p2p'")
        self.W = local_weight  # nmspmm.NmWeight of this rank's padded shard
        # the offline weight prepack once per layer: the bf16 sparse-tensor-core
        # kernel's slot packing and images; plain values/idx for the fp32 path
        # m_hint: the expected token count, so the slot prepack picks the tile nm_spmm would (nm_prepack_m)
        self.PW = nmspmm.nm_prepack(local_weight, m_hint=m_hint) if local_weight.values.is_cuda else None
        self.group = group
        self.G = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.n = n
        self.nr = local_weight.n
        self.exchange = exchange
        # exchange="nccl": the collective that fills [G][m][nr] from every rank's [m][nr] block
        # (default torch.distributed.all_gather_into_tensor over the group, i.e. NCCL on GPUs;
        # injectable so the same branch runs with other backends, e.g. gloo with host staging)
        self.all_gather = all_gather or (lambda out, inp, group, async_op=False: dist.all_gather_into_tensor(
            out, inp, group=group, async_op=async_op))
        # exchange="nccl" with chunks > 1: the rows of A go in `chunks` slices; the
        # all-gather of slice c runs asynchronously (NCCL's stream) while slice c + 1 is computed
        self.chunks = max(1, int(chunks))
        self.peers = None
        q = n // local_weight.L
        g0, g1 = shard_ranges(q, self.G)[self.rank]
        self.col_off, self.n_valid = g0 * local_weight.L, (g1 - g0) * local_weight.L
        # the fused exchange has two epilogues: the bf16 / tf32 slot kernels (prepack kind 2 / 3) and
        # the fp32 SIMT kernel; any other weight (e.g. bf16 with L outside {16, 32, 64, 128}) has none
        if exchange == "p2p" and local_weight.values.dtype != torch.float32 and (
                self.PW is None or self.PW.kind not in (2, 3)):
            raise ValueError("exchange='p2p' needs an fp32 weight or a bf16 weight the slot kernel takes "
                             "(L in {16, 32, 64, 128}); use exchange='nccl'")

    @classmethod
    def from_dense(cls, B: torch.Tensor, N: int, M: int, L: int, group=None, exchange: str = "nccl", all_gather=None,
                   chunks: int = 1, m_hint: int | None = None):
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
        return cls(W, n, group, exchange, all_gather, chunks, m_hint)

    def local(self, A: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        from . import nmspmm
        if self.PW is not None:
            return nmspmm.nm_spmm_prepacked(A, self.PW, out=out)
        return nmspmm.nm_spmm(A, self.W, out=out)

    def _call_p2p(self, A: torch.Tensor) -> torch.Tensor:
        from . import nmspmm
        m = A.shape[0]
        if self.peers is None or self.peers.m != m:  # collective: every rank calls with the same m
            if self.peers is not None:
                self.peers.close()
            self.peers = PeerExchange(self.group, m, self.n, A.dtype, A.device)
        ex = self.peers
        ex.epoch += 1
        b = ex.epoch & 1
        if self.PW is not None and self.PW.kind in (2, 3):  # bf16 / tf32 slot kernel, direct-store epilogue
            nmspmm.nm_spmm_prepacked_peers(A, self.PW, ex.ptrs[b], self.n, self.col_off, self.n_valid)
        else:  # fp32 SIMT kernel's peer epilogue
            nmspmm.nm_spmm_peers(A, self.W, ex.ptrs[b], self.n, self.col_off, self.n_valid)
        nmspmm.nm_peer_barrier(ex.ptrs[2], self.rank, ex.epoch, device=A.device)
        return ex.C[b]

    def __call__(self, A: torch.Tensor) -> torch.Tensor:
        from . import nmspmm
        if self.exchange == "p2p":
            return self._call_p2p(A)
        m = A.shape[0]
        if self.G == 1 and self.nr == self.n:  # a single shard is already C (no exchange step)
            return self.local(A)
        # row slices of 128-multiples; slice c's all-gather overlaps slice c+1's SpMM
        nch = min(self.chunks, max(1, m // 128))
        rc = -(-m // nch)
        rc = -(-rc // 128) * 128 if nch > 1 else m
        pending = []
        for r0 in range(0, m, rc):
            r1 = min(m, r0 + rc)
            c_local = self.local(A[r0:r1])
            gathered = torch.empty((self.G, r1 - r0, self.nr), dtype=c_local.dtype, device=A.device)
            pending.append((self.all_gather(gathered, c_local, self.group, async_op=nch > 1), gathered, r0, r1))
        C = torch.empty((m, self.n), dtype=pending[0][1].dtype, device=A.device)
        for work, gathered, r0, r1 in pending:
            if work is not None:
                work.wait()  # the current stream waits for this slice's collective
            nmspmm.nm_unshard_columns(gathered, C[r0:r1], self.G, r1 - r0, self.nr, self.n, self.W.L)
        return C
