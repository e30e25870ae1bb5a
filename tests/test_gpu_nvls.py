"""NVLS multicast C (nm_mc_*, nm_spmm_mc) on the one GPU of the box: a multicast
object over this device, its buffer bound and mapped (unicast replica + multicast view), the SIMT
kernel's multimem.st epilogue writing two column shards of one layer through the multicast view.
The replica must equal the oracle bit for bit on integer inputs (the multi-rank replication itself
needs >= 2 GPUs on an NVSwitch and is not exercised here)."""
import ctypes

import numpy as np
import pytest
import torch

from paper_2503_01253_b200 import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nm():
    from paper_2503_01253_b200 import nmspmm
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    nmspmm.lib()
    if not nmspmm.nm_mc_supported():
        # the round-2 box: multicast attribute 1, but cuMulticastCreate -> CUDA_ERROR_INVALID_VALUE with
        # one visible GPU (profiles/r02i_nvls_probe.txt)
        pytest.skip("multicast objects unavailable to this process (one visible GPU)")
    return nmspmm


def dev(x, dtype=torch.float32):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda().to(dtype)


def copy_from(ptr, nbytes, shape):
    """Device-to-device copy of the unicast replica into a torch tensor (test plumbing)."""
    out = torch.empty(shape, dtype=torch.float32, device="cuda")
    torch.cuda.synchronize()
    rt = ctypes.CDLL("libcudart.so.12")
    rt.cudaMemcpy.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
    assert rt.cudaMemcpy(ctypes.c_void_p(out.data_ptr()), ptr, nbytes, 3) == 0
    return out


@pytest.mark.parametrize("m,n,k,N,M,L", [(260, 512, 512, 8, 32, 32), (128, 256, 1024, 16, 32, 32),
                                         (97, 384, 256, 2, 4, 4)])
def test_spmm_mc_two_shards_integer_exact(nm, oracle, m, n, k, N, M, L):
    A = synth.integer((m, k), 301, synth.TID_A)
    B = synth.integer((k, n), 302, synth.TID_B)
    vals, D = oracle.compress(B, N, M, L)
    ref = oracle.spmm_sparse_f64(A, vals, D, k, N, M, L)
    buf = nm.McBuffer(m * n * 4, num_devices=1)
    try:
        buf.add_device()
        buf.bind_map()
        q = n // L
        g_half = q // 2
        for g0, g1 in ((0, g_half), (g_half, q)):  # two column shards, each written through the multicast view
            c0, c1 = g0 * L, g1 * L
            Ws = nm.NmWeight(dev(vals[:, c0:c1]), dev(D[:, g0:g1], torch.uint8), k, N, M, L)
            nm.nm_spmm_mc(dev(A), Ws, buf.mc_ptr.value, n, c0, c1 - c0)
        C = copy_from(buf.uc_ptr, m * n * 4, (m, n)).cpu().numpy()
    finally:
        buf.free()
    assert np.array_equal(C.astype(np.float64), ref)


def test_spmm_mc_rejects_bad_geometry(nm):
    A = torch.zeros((64, 96), device="cuda")
    W = nm.NmWeight(torch.zeros((48, 64), device="cuda"), torch.zeros((48, 2), dtype=torch.uint8, device="cuda"),
                    96, 16, 32, 32)
    with pytest.raises(nm.NmError):
        nm.nm_spmm_mc(A, W, 0x1000, 64, 2, 62)  # n_valid % 4 != 0
