"""Worker process of tests/test_gpu_parity.py::test_sharded_p2p_two_processes_one_gpu (a
module of its own so that multiprocessing's spawn can import it)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2503_01253_b200 import synth  # noqa: E402


def run(rank, G, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    from oracle import oracle
    from paper_2503_01253_b200 import nmspmm as nm, sharded
    try:
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=G)
        m, n, k, N, M, L = 260, 640, 512, 8, 32, 32
        A = synth.uniform((m, k), 191, synth.TID_A)
        B = synth.uniform((k, n), 192, synth.TID_B)
        layer = sharded.ShardedNmLinear.from_dense(torch.from_numpy(B).cuda(), N, M, L, exchange="p2p")
        vals, D = oracle.compress(B, N, M, L)
        ref = oracle.spmm_sparse_f64(A, vals, D, k, N, M, L)
        errs = []
        for _ in range(3):
            C = layer(torch.from_numpy(A).cuda())
            torch.cuda.synchronize()
            errs.append(oracle.rel_frobenius(C.cpu().numpy(), ref))
        dist.barrier()
        layer.peers.close()
        dist.destroy_process_group()
        q.put((rank, max(errs)))
    except Exception as e:  # report, do not hang the parent
        q.put((rank, repr(e)))
