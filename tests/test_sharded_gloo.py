"""Multi-process (world_size 2 and 3, gloo, CPU) checks of the column-sharded
host logic (paper_2503_01253_b200/sharded.py): partition, padding and the
assembly mapping that nm_unshard_columns implements on the GPU.  The local
product on each rank is the CPU oracle (test infrastructure); the check is
that the assembled result equals the unsharded oracle bit-for-bit (column j
depends only on B'[:, j] and D[:, j//L])."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def assemble_reference(gathered: np.ndarray, q: int, L: int) -> np.ndarray:
    """Host statement of the nm_unshard_columns mapping: dst[:, L*g0(r) + j] = src[r][:, j]."""
    from paper_2503_01253_b200.sharded import shard_ranges
    G, m, nr = gathered.shape
    out = np.empty((m, q * L), dtype=gathered.dtype)
    for r, (g0, g1) in enumerate(shard_ranges(q, G)):
        out[:, g0 * L:g1 * L] = gathered[r][:, :(g1 - g0) * L]
    return out


def _worker(rank, world, port, case, errs):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from oracle import oracle
        from paper_2503_01253_b200 import synth
        from paper_2503_01253_b200.sharded import groups_per_shard, shard_weight
        m, n, k, N, M, L = case
        q = n // L
        A = synth.uniform((m, k), 5, synth.TID_A)
        B = synth.uniform((k, n), 6, synth.TID_B)
        vals, D = oracle.compress(B, N, M, L)
        v_r, d_r = shard_weight(torch.from_numpy(vals), torch.from_numpy(D), L, N, rank, world)
        assert v_r.shape[1] == groups_per_shard(q, world) * L
        assert oracle.validate(d_r.numpy(), k, v_r.shape[1], N, M, L) == -1  # padding keeps D valid
        c_r = torch.from_numpy(oracle.spmm_sparse_f64(A, v_r.numpy(), d_r.numpy(), k, N, M, L))
        parts = [torch.empty_like(c_r) for _ in range(world)]
        dist.all_gather(parts, c_r)
        C = assemble_reference(torch.stack(parts).numpy(), q, L)
        full = oracle.spmm_sparse_f64(A, vals, D, k, N, M, L)
        if not np.array_equal(C, full):
            errs.put(f"rank {rank}: assembled result differs")
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # surface the failure in the parent
        errs.put(f"rank {rank}: {e!r}")


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("case", [(16, 11 * 8, 64, 4, 16, 8), (8, 64, 32, 2, 4, 4), (4, 5 * 32, 64, 16, 32, 32)])
def test_sharded_assembly_gloo(world, case):
    ctx = mp.get_context("spawn")
    errs = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, errs)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    msgs = []
    while not errs.empty():
        msgs.append(errs.get())
    assert all(p.exitcode == 0 for p in procs), msgs
    assert not msgs, msgs


def test_shard_ranges_cover_and_balance():
    from paper_2503_01253_b200.sharded import groups_per_shard, shard_ranges
    for q in [1, 7, 128, 172, 344, 688]:
        for G in [1, 2, 3, 4, 8]:
            rs = shard_ranges(q, G)
            assert rs[0][0] == 0 and rs[-1][1] == q
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            assert max(g1 - g0 for g0, g1 in rs) <= groups_per_shard(q, G)


def _p2p_worker(rank, world, port, case, errs):
    """Host statement of the fused exchange (exchange='p2p'): every rank stores its shard's
    n_valid real columns at [row][col_off + j] of EVERY rank's C (nm_spmm_peers' epilogue), with
    col_off / n_valid as ShardedNmLinear computes them; after the barrier each rank's C must be
    the unsharded oracle, bit for bit, and the ranks' column ranges must tile [0, n) exactly."""
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from oracle import oracle
        from paper_2503_01253_b200 import nmspmm, synth
        from paper_2503_01253_b200.sharded import ShardedNmLinear, shard_weight
        m, n, k, N, M, L = case
        A = synth.uniform((m, k), 7, synth.TID_A)
        B = synth.uniform((k, n), 8, synth.TID_B)
        vals, D = oracle.compress(B, N, M, L)
        v_r, d_r = shard_weight(torch.from_numpy(vals), torch.from_numpy(D), L, N, rank, world)
        layer = ShardedNmLinear(nmspmm.NmWeight(v_r, d_r, k, N, M, L), n, exchange="p2p")  # CPU: no prepack
        c_r = oracle.spmm_sparse_f64(A, v_r.numpy(), d_r.numpy(), k, N, M, L)
        stores = [None] * world
        dist.all_gather_object(stores, (layer.col_off, layer.n_valid, c_r[:, :layer.n_valid]))
        C = np.full((m, n), np.nan)
        covered = np.zeros(n, dtype=np.int64)
        for col_off, n_valid, block in stores:  # every rank's epilogue stores into this rank's C
            C[:, col_off:col_off + n_valid] = block
            covered[col_off:col_off + n_valid] += 1
        if not (covered == 1).all():
            errs.put(f"rank {rank}: column ranges do not tile [0, n)")
        if not np.array_equal(C, oracle.spmm_sparse_f64(A, vals, D, k, N, M, L)):
            errs.put(f"rank {rank}: p2p-assembled result differs")
        try:
            ShardedNmLinear(nmspmm.NmWeight(v_r, d_r, k, N, M, L), n, exchange="allreduce")
            errs.put(f"rank {rank}: unknown exchange accepted")
        except ValueError:
            pass
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:
        errs.put(f"rank {rank}: {e!r}")


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("case", [(16, 11 * 8, 64, 4, 16, 8), (4, 5 * 32, 64, 16, 32, 32)])
def test_sharded_p2p_store_mapping_gloo(world, case):
    ctx = mp.get_context("spawn")
    errs = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_p2p_worker, args=(r, world, port, case, errs)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    msgs = []
    while not errs.empty():
        msgs.append(errs.get())
    assert all(p.exitcode == 0 for p in procs), msgs
    assert not msgs, msgs
