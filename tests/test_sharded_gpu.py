"""The column-sharded layer's exchange="nccl" branch end to end on the GPU with G = 2 and 3
ranks (processes sharing cuda:0): each rank compresses its column groups (nm_compress), runs its
local SpMM (nm_spmm / nm_spmm_prepacked), the [G][m][nr] blocks are all-gathered (gloo with host
staging, injected in place of NCCL -- the box has one GPU) and nm_unshard_columns assembles C.
Every rank's C is compared element by element with the CPU oracle on the unsharded weight."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, case, errs):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        from oracle import oracle
        from paper_2503_01253_b200 import synth
        from paper_2503_01253_b200.sharded import ShardedNmLinear, host_staged_all_gather
        m, n, k, N, M, L, dt, kind, chunks = case
        gen = synth.integer if kind == "integer" else (synth.uniform if dt == "f32" else synth.bf16grid)
        A = gen((m, k), 11, synth.TID_A)
        B = gen((k, n), 12, synth.TID_B)
        tdt = torch.float32 if dt == "f32" else torch.bfloat16
        layer = ShardedNmLinear.from_dense(torch.from_numpy(B).cuda().to(tdt), N, M, L,
                                           all_gather=host_staged_all_gather, chunks=chunks)
        C = layer(torch.from_numpy(A).cuda().to(tdt)).float().cpu().numpy().astype(np.float64)
        Bo = B if dt == "f32" else synth.to_bf16_bits(B)
        Ao = A if dt == "f32" else synth.to_bf16_bits(A)
        vals, D = oracle.compress(Bo, N, M, L)
        ref = oracle.spmm_sparse_f64(Ao, vals, D, k, N, M, L)
        if kind == "integer" and dt == "f32":
            ok = np.array_equal(C, ref)  # every partial sum is an exact integer
        else:
            tol = 1e-5 if dt == "f32" else 5e-3
            ok = oracle.rel_frobenius(C, ref) <= tol
        if not ok:
            errs.put(f"rank {rank}: C differs (rel {oracle.rel_frobenius(C, ref):.3e})")
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:
        errs.put(f"rank {rank}: {e!r}")


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("case", [
    (256, 11 * 32, 512, 16, 32, 32, "f32", "uniform", 1),   # 11 groups: uneven shards, padding
    (200, 8 * 32, 256, 8, 32, 32, "f32", "integer", 1),     # bit-exact through the exchange
    (300, 12 * 32, 512, 12, 32, 32, "bf16", "uniform", 1),  # slot kernel (prepacked) shards
    (128, 9 * 16, 256, 4, 16, 16, "bf16", "uniform", 1),
    (700, 10 * 32, 512, 8, 32, 32, "f32", "integer", 3),    # row slices (overlapped exchange), ragged
    (520, 12 * 32, 512, 12, 32, 32, "bf16", "uniform", 4),
])
def test_sharded_nccl_branch_multi_rank_one_gpu(world, case):
    ctx = mp.get_context("spawn")
    errs = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, errs)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
    msgs = []
    while not errs.empty():
        msgs.append(errs.get())
    assert all(p.exitcode == 0 for p in procs), msgs
    assert not msgs, msgs
