"""Thin Python binding of libnmspmm.so (include/nmspmm.h): argument
marshalling only -- every step of the path runs in the library's sm_100a
kernels.  torch supplies device memory and streams.  There is no CPU
fallback: if the library or a CUDA device is missing, calls raise.

Names follow the C ABI: nm_compress, nm_decompress, nm_validate, nm_spmm,
nm_spmm_host, nm_plan_query, nm_unshard_columns.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
# NM_LIB_PATH: an alternative build of the same library (A/B timing studies in scripts/ only)
LIB_PATH = os.environ.get("NM_LIB_PATH") or os.path.join(_PKG, "libnmspmm.so")

NM_OK = 0
STATUS = {0: "NM_OK", 1: "NM_ERR_INVALID_CONFIG", 2: "NM_ERR_SHAPE", 3: "NM_ERR_ALIGNMENT",
          4: "NM_ERR_NONFINITE", 5: "NM_ERR_UNSUPPORTED", 6: "NM_ERR_INVALID_INDICES", 7: "NM_ERR_CUDA",
          8: "NM_ERR_NULL"}
NM_F32, NM_BF16 = 0, 1
MATH = {"auto": 0, "f32_simt": 1, "tf32_tc": 2, "bf16_tc": 3}

EXPORTS = ["nm_version", "nm_last_error", "nm_check_config", "nm_compress", "nm_decompress", "nm_validate",
           "nm_spmm", "nm_spmm_host_ws_bytes", "nm_spmm_host", "nm_plan_query", "nm_unshard_columns",
           "nm_profile_begin", "nm_profile_end", "nm_prepack_bytes", "nm_prepack", "nm_spmm_prepacked",
           "nm_prepack_bytes_ex", "nm_prepack_ex", "nm_ipc_get_handle", "nm_ipc_open_handle", "nm_ipc_close",
           "nm_spmm_peers", "nm_peer_barrier", "nm_spmm_prepacked_peers", "nm_spmm_scaled", "nm_prepack_size",
           "nm_index_packed_words", "nm_index_pack", "nm_index_unpack", "nm_mc_supported", "nm_mc_create",
           "nm_mc_export", "nm_mc_import", "nm_mc_add_device", "nm_mc_bind_map", "nm_mc_free", "nm_spmm_mc",
           "nm_spmm_at", "nm_spmm_prepacked_at", "nm_prepack_size_m", "nm_prepack_m"]


class NmError(RuntimeError):
    def __init__(self, status: int, fn: str, msg: str):
        super().__init__(f"{fn}: {STATUS.get(status, status)}: {msg}")
        self.status = status


class Prepacked(ctypes.Structure):
    _fields_ = [("magic", ctypes.c_int32), ("kind", ctypes.c_int32), ("dtype", ctypes.c_int32), ("N", ctypes.c_int32),
                ("M", ctypes.c_int32), ("L", ctypes.c_int32), ("n", ctypes.c_int64), ("k", ctypes.c_int64),
                ("bn", ctypes.c_int32), ("wp", ctypes.c_int32), ("bk", ctypes.c_int32), ("bkw", ctypes.c_int32),
                ("bkw_pad", ctypes.c_int32), ("npanels", ctypes.c_int32), ("values", ctypes.c_void_p),
                ("idx", ctypes.c_void_p), ("perm", ctypes.c_void_p), ("tbl", ctypes.c_void_p),
                ("bperm", ctypes.c_void_p)]


class Plan(ctypes.Structure):
    _fields_ = [("math", ctypes.c_int32), ("kernel", ctypes.c_int32), ("bm", ctypes.c_int32),
                ("bn", ctypes.c_int32), ("bk", ctypes.c_int32), ("bkw", ctypes.c_int32),
                ("stages", ctypes.c_int32), ("grid", ctypes.c_int32), ("threads", ctypes.c_int32),
                ("smem_bytes", ctypes.c_int32), ("flops", ctypes.c_double), ("bytes", ctypes.c_double),
                ("t_compute_us", ctypes.c_double), ("t_memory_us", ctypes.c_double), ("bound", ctypes.c_int32),
                ("split", ctypes.c_int32), ("split_tiles", ctypes.c_int32), ("waves", ctypes.c_double)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


_lib = None


def lib():
    """Load libnmspmm.so (built in-tree by __graft_entry__.build()); raise if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} missing: run __graft_entry__.build() (no CPU fallback exists)")
        L = ctypes.CDLL(LIB_PATH)
        P, I64, I = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
        L.nm_version.restype = ctypes.c_char_p
        L.nm_last_error.restype = ctypes.c_char_p
        L.nm_check_config.argtypes = [I, I, I]
        L.nm_compress.argtypes = [P, I, I64, I64, I, I, I, P, I, P, P]
        L.nm_decompress.argtypes = [P, I, P, I64, I64, I, I, I, P, P]
        L.nm_validate.argtypes = [P, I64, I64, I, I, I, ctypes.POINTER(ctypes.c_int64), P]
        L.nm_spmm.argtypes = [P, P, P, P, I64, I64, I64, I, I, I, I, I, I, P]
        L.nm_spmm_scaled.argtypes = [P, P, P, P, I64, I64, I64, I, I, I, I, I, I, ctypes.c_float, P]
        L.nm_spmm_host_ws_bytes.argtypes = [I64, I64, I64, I, I, I, I, I]
        L.nm_spmm_host_ws_bytes.restype = I64
        L.nm_spmm_host.argtypes = [P, P, P, P, I64, I64, I64, I, I, I, I, I, I, P, P]
        L.nm_plan_query.argtypes = [I64, I64, I64, I, I, I, I, I, ctypes.c_double, ctypes.c_double,
                                    ctypes.POINTER(Plan)]
        L.nm_unshard_columns.argtypes = [P, P, I64, I64, I64, I64, I, I, P]
        L.nm_profile_begin.argtypes = []
        L.nm_prepack_bytes.argtypes = [I64, I64, I, I, I, I]
        L.nm_prepack_bytes.restype = I64
        L.nm_prepack.argtypes = [P, P, I64, I64, I, I, I, I, P, I64, ctypes.POINTER(Prepacked), P]
        L.nm_spmm_prepacked.argtypes = [P, ctypes.POINTER(Prepacked), P, I64, I, P]
        L.nm_spmm_at.argtypes = [P, I64, P, P, P, I64, I64, I64, I, I, I, I, I, I, P]
        L.nm_spmm_prepacked_at.argtypes = [P, I64, ctypes.POINTER(Prepacked), P, I64, I, P]
        L.nm_prepack_bytes_ex.argtypes = [I64, I64, I, I, I, I, I]
        L.nm_prepack_bytes_ex.restype = I64
        L.nm_prepack_ex.argtypes = [P, P, I64, I64, I, I, I, I, I, P, I64, ctypes.POINTER(Prepacked), P]
        L.nm_prepack_size.argtypes = [P, P, I64, I64, I, I, I, I, I, ctypes.POINTER(I64), P]
        L.nm_prepack_size_m.argtypes = [P, P, I64, I64, I, I, I, I, I, I64, ctypes.POINTER(I64), P]
        L.nm_prepack_m.argtypes = [P, P, I64, I64, I, I, I, I, I, I64, P, I64, ctypes.POINTER(Prepacked), P]
        L.nm_index_packed_words.argtypes = [I64, I64, I, I, I]
        L.nm_index_packed_words.restype = I64
        L.nm_index_pack.argtypes = [P, I64, I64, I, I, I, P, P]
        L.nm_index_unpack.argtypes = [P, I64, I64, I, I, I, P, P]
        L.nm_profile_end.argtypes = [ctypes.POINTER(ctypes.c_double), ctypes.POINTER(I64), ctypes.POINTER(I64)]
        L.nm_ipc_get_handle.argtypes = [P, P, ctypes.POINTER(I64)]
        L.nm_ipc_open_handle.argtypes = [P, I64, ctypes.POINTER(P)]
        L.nm_ipc_close.argtypes = [P, I64]
        L.nm_spmm_peers.argtypes = [P, P, P, ctypes.POINTER(P), I, I64, I64, I64, I64, I64, I64, I, I, I, P]
        L.nm_peer_barrier.argtypes = [ctypes.POINTER(P), I, I, I, P]
        L.nm_spmm_prepacked_peers.argtypes = [P, ctypes.POINTER(Prepacked), ctypes.POINTER(P), I, I64, I64, I64, I64, I,
                                              P]
        U64 = ctypes.c_uint64
        L.nm_mc_supported.argtypes = [ctypes.POINTER(I)]
        L.nm_mc_create.argtypes = [I64, I, ctypes.POINTER(U64), ctypes.POINTER(I64)]
        L.nm_mc_export.argtypes = [U64, P]
        L.nm_mc_import.argtypes = [P, ctypes.POINTER(U64)]
        L.nm_mc_add_device.argtypes = [U64]
        L.nm_mc_bind_map.argtypes = [U64, I64, ctypes.POINTER(U64), ctypes.POINTER(P), ctypes.POINTER(P)]
        L.nm_mc_free.argtypes = [U64, U64, P, P, I64]
        L.nm_spmm_mc.argtypes = [P, P, P, P, I64, I64, I64, I64, I64, I64, I, I, I, P]
        for name in EXPORTS[2:]:
            if name not in ("nm_spmm_host_ws_bytes", "nm_prepack_bytes", "nm_prepack_bytes_ex", "nm_index_packed_words"):
                getattr(L, name).restype = I
        _lib = L
    return _lib


def _check(status: int, fn: str):
    if status != NM_OK:
        raise NmError(status, fn, lib().nm_last_error().decode())


def _dt(t: torch.Tensor) -> int:
    if t.dtype == torch.float32:
        return NM_F32
    if t.dtype == torch.bfloat16:
        return NM_BF16
    raise TypeError(f"unsupported dtype {t.dtype}")


def _stream(t: torch.Tensor, stream=None):
    if stream is not None:
        return ctypes.c_void_p(stream.cuda_stream)
    return ctypes.c_void_p(torch.cuda.current_stream(t.device).cuda_stream)


def _dev(t: torch.Tensor, name: str):
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous (row-major)")


def _check_out(out: torch.Tensor, A: torch.Tensor, m: int, n: int):
    '''A caller-supplied C: a contiguous CUDA tensor on A's device with shape (m, n) (the kernels
    write m x n elements of out's dtype at its data pointer).'''
    _dev(out, "out")
    if out.device != A.device:
        raise ValueError(f"out is on {out.device}, A on {A.device}")
    if tuple(out.shape) != (m, n):
        raise ValueError(f"out has shape {tuple(out.shape)}, expected {(m, n)}")
    _dt(out)


def version() -> str:
    return lib().nm_version().decode()


@dataclass
class NmWeight:
    """Compressed weight: values B' (w x n) + index matrix D (w x q, uint8)."""
    values: torch.Tensor
    idx: torch.Tensor
    k: int
    N: int
    M: int
    L: int

    @property
    def n(self) -> int:
        return self.values.shape[1]

    @property
    def w(self) -> int:
        return self.values.shape[0]


def nm_compress(B: torch.Tensor, N: int, M: int, L: int, values_dtype=None, stream=None) -> NmWeight:
    """nm_compress: magnitude-prune B (k x n) to vector-wise N:M and compress."""
    _dev(B, "B")
    k, n = B.shape
    vdt = values_dtype or B.dtype
    _check(lib().nm_check_config(N, M, L), "nm_check_config")
    if k % M or n % L:
        raise NmError(2, "nm_compress", "k % M and n % L must be 0 (caller pads, P:94)")
    w, q = k // M * N, n // L
    values = torch.empty((w, n), dtype=vdt, device=B.device)
    idx = torch.empty((w, q), dtype=torch.uint8, device=B.device)
    _check(lib().nm_compress(B.data_ptr(), _dt(B), k, n, N, M, L, values.data_ptr(), _dt(values), idx.data_ptr(),
                             _stream(B, stream)), "nm_compress")
    return NmWeight(values, idx, k, N, M, L)


def nm_decompress(W: NmWeight, stream=None) -> torch.Tensor:
    _dev(W.values, "values")
    out = torch.empty((W.k, W.n), dtype=W.values.dtype, device=W.values.device)
    _check(lib().nm_decompress(W.values.data_ptr(), _dt(W.values), W.idx.data_ptr(), W.k, W.n, W.N, W.M, W.L,
                               out.data_ptr(), _stream(out, stream)), "nm_decompress")
    return out


def nm_validate(idx: torch.Tensor, k: int, n: int, N: int, M: int, L: int, stream=None) -> int:
    """-1 if valid, else the first bad flat index."""
    _dev(idx, "idx")
    bad = ctypes.c_int64(0)
    st = lib().nm_validate(idx.data_ptr(), k, n, N, M, L, ctypes.byref(bad), _stream(idx, stream))
    if st not in (NM_OK, 6):
        _check(st, "nm_validate")
    return int(bad.value)


def nm_spmm(A: torch.Tensor, W: NmWeight, out: torch.Tensor | None = None, out_dtype=None, math: str = "auto",
            stream=None, alpha: float = 1.0) -> torch.Tensor:
    """C = alpha . A . decompress(W) on the device (Eq. 1: alpha = 1 is the product,
    alpha = M/N the paper's scaled approximation C'; nm_spmm_scaled)."""
    _dev(A, "A")
    _dev(W.values, "values")
    _dev(W.idx, "idx")
    m, k = A.shape
    if k != W.k:
        raise NmError(2, "nm_spmm", f"A has k={k}, weight has k={W.k}")
    if A.dtype != W.values.dtype:
        raise TypeError("A and values must share a dtype")
    cdt = out_dtype or A.dtype
    if out is None:
        out = torch.empty((m, W.n), dtype=cdt, device=A.device)
    else:
        _check_out(out, A, m, W.n)
    if alpha == 1.0:
        _check(lib().nm_spmm(A.data_ptr(), W.values.data_ptr(), W.idx.data_ptr(), out.data_ptr(), m, W.n, k, W.N,
                             W.M, W.L, _dt(A), _dt(out), MATH[math], _stream(A, stream)), "nm_spmm")
    else:
        _check(lib().nm_spmm_scaled(A.data_ptr(), W.values.data_ptr(), W.idx.data_ptr(), out.data_ptr(), m, W.n, k,
                                    W.N, W.M, W.L, _dt(A), _dt(out), MATH[math], float(alpha), _stream(A, stream)),
               "nm_spmm_scaled")
    return out


def _at_args(At: torch.Tensor, k: int, m: int | None):
    """A^T operand checks (nm_spmm_at): k x lda contiguous rows, lda >= m."""
    _dev(At, "At")
    if At.dim() != 2 or At.stride(1) != 1:
        raise ValueError("At must be a 2-D tensor with unit column stride (k x lda)")
    if At.shape[0] != k:
        raise NmError(2, "nm_spmm_at", f"At has {At.shape[0]} rows, weight has k={k}")
    lda = At.stride(0)
    m = At.shape[1] if m is None else m
    if m > At.shape[1]:
        raise NmError(2, "nm_spmm_at", f"m={m} exceeds At's {At.shape[1]} columns")
    return lda, m


def nm_spmm_at(At: torch.Tensor, W: NmWeight, m: int | None = None, out: torch.Tensor | None = None, out_dtype=None,
               math: str = "auto", stream=None) -> torch.Tensor:
    """C = A . decompress(W) with A supplied transposed (At: k x lda, feature-major activations):
    the per-call transpose of nm_spmm is skipped; same kernels, same results."""
    _dev(W.values, "values")
    _dev(W.idx, "idx")
    lda, m = _at_args(At, W.k, m)
    if At.dtype != W.values.dtype:
        raise TypeError("At and values must share a dtype")
    cdt = out_dtype or At.dtype
    if out is None:
        out = torch.empty((m, W.n), dtype=cdt, device=At.device)
    else:
        _check_out(out, At, m, W.n)
    _check(lib().nm_spmm_at(At.data_ptr(), lda, W.values.data_ptr(), W.idx.data_ptr(), out.data_ptr(), m, W.n, W.k,
                            W.N, W.M, W.L, _dt(At), _dt(out), MATH[math], _stream(At, stream)), "nm_spmm_at")
    return out


class PrepackedWeight:
    '''A weight after nm_prepack (the paper's offline PreProcessing): keeps the
    original NmWeight (referenced by the descriptor), the device buffer and the descriptor.'''

    def __init__(self, W: NmWeight, stream=None, math: str = "auto", m_hint: int | None = None):
        self.W = W
        mh = int(m_hint or 0)
        dt = _dt(W.values)
        if lib().nm_prepack_bytes_ex(W.n, W.k, W.N, W.M, W.L, dt, MATH[math]) < 0:
            raise NmError(2, "nm_prepack_bytes", "bad shape")
        # the exact size of the compact slot images (one packing pass; synchronizes the stream)
        nb = ctypes.c_int64(0)
        _check(lib().nm_prepack_size_m(W.values.data_ptr(), W.idx.data_ptr(), W.n, W.k, W.N, W.M, W.L, dt, MATH[math],
                                       mh, ctypes.byref(nb), _stream(W.values, stream)), "nm_prepack_size")
        nbytes = int(nb.value)
        self.buf = torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device=W.values.device)
        self.desc = Prepacked()
        _check(lib().nm_prepack_m(W.values.data_ptr(), W.idx.data_ptr(), W.n, W.k, W.N, W.M, W.L, dt, MATH[math], mh,
                                  self.buf.data_ptr(), int(nbytes), ctypes.byref(self.desc), _stream(W.values, stream)),
               "nm_prepack")

    @property
    def kind(self) -> int:
        return int(self.desc.kind)

    def __getattr__(self, name):  # n, k, N, M, L, values, idx ... of the underlying weight
        return getattr(self.W, name)


def nm_prepack(W: NmWeight, stream=None, math: str = "auto", m_hint: int | None = None) -> PrepackedWeight:
    """math="tf32_tc" on an fp32 weight prepares the tf32 sparse-tensor-core path (kind 3); m_hint =
    the expected token count lets the slot prepack pick its tile for that m (nm_prepack_m)."""
    return PrepackedWeight(W, stream, math, m_hint)


def nm_spmm_prepacked(A: torch.Tensor, PW: PrepackedWeight, out: torch.Tensor | None = None, out_dtype=None,
                      stream=None) -> torch.Tensor:
    _dev(A, "A")
    m, k = A.shape
    if k != PW.W.k:
        raise NmError(2, "nm_spmm_prepacked", f"A has k={k}, weight has k={PW.W.k}")
    if A.dtype != PW.W.values.dtype:  # the kernels read A's bytes as the weight's element type
        raise TypeError(f"A is {A.dtype}, the prepacked weight is {PW.W.values.dtype}")
    cdt = out_dtype or A.dtype
    if out is None:
        out = torch.empty((m, PW.W.n), dtype=cdt, device=A.device)
    else:
        _check_out(out, A, m, PW.W.n)
    _check(lib().nm_spmm_prepacked(A.data_ptr(), ctypes.byref(PW.desc), out.data_ptr(), m, _dt(out),
                                   _stream(A, stream)), "nm_spmm_prepacked")
    return out


def nm_spmm_prepacked_at(At: torch.Tensor, PW: "PrepackedWeight", m: int | None = None, out: torch.Tensor | None = None,
                         out_dtype=None, stream=None) -> torch.Tensor:
    """nm_spmm_prepacked with A supplied transposed (At: k x lda); no per-call transpose."""
    lda, m = _at_args(At, PW.W.k, m)
    if At.dtype != PW.W.values.dtype:
        raise TypeError(f"At is {At.dtype}, the prepacked weight is {PW.W.values.dtype}")
    cdt = out_dtype or At.dtype
    if out is None:
        out = torch.empty((m, PW.W.n), dtype=cdt, device=At.device)
    else:
        _check_out(out, At, m, PW.W.n)
    _check(lib().nm_spmm_prepacked_at(At.data_ptr(), lda, ctypes.byref(PW.desc), out.data_ptr(), m, _dt(out),
                                      _stream(At, stream)), "nm_spmm_prepacked_at")
    return out


class HostSpmm:
    """End-to-end path through nm_spmm_host: host (pinned) operands in, host C out;
    the device workspace is allocated once by torch."""

    def __init__(self, m, n, k, N, M, L, ab_dtype=torch.float32, c_dtype=None, math="auto", device="cuda"):
        self.m, self.n, self.k, self.N, self.M, self.L = m, n, k, N, M, L
        self.ab = NM_F32 if ab_dtype == torch.float32 else NM_BF16
        cd = c_dtype or ab_dtype
        self.cd = NM_F32 if cd == torch.float32 else NM_BF16
        self.math = MATH[math]
        ws = lib().nm_spmm_host_ws_bytes(m, n, k, N, M, L, self.ab, self.cd)
        if ws < 0:
            raise NmError(2, "nm_spmm_host_ws_bytes", "bad shape")
        self.ws = torch.empty(ws, dtype=torch.uint8, device=device)

    def __call__(self, A_host, values_host, idx_host, C_host, stream=None):
        _check(lib().nm_spmm_host(A_host.data_ptr(), values_host.data_ptr(), idx_host.data_ptr(), C_host.data_ptr(),
                                  self.m, self.n, self.k, self.N, self.M, self.L, self.ab, self.cd, self.math,
                                  self.ws.data_ptr(), _stream(self.ws, stream)), "nm_spmm_host")
        return C_host


def nm_plan_query(m, n, k, N, M, L, dtype=torch.float32, math="auto", peak_flops=0.0, peak_hbm=0.0) -> dict:
    p = Plan()
    _check(lib().nm_plan_query(m, n, k, N, M, L, NM_F32 if dtype == torch.float32 else NM_BF16, MATH[math],
                               float(peak_flops), float(peak_hbm), ctypes.byref(p)), "nm_plan_query")
    return p.as_dict()


def nm_profile_begin():
    _check(lib().nm_profile_begin(), "nm_profile_begin")


def nm_profile_end():
    '''(summed ms of the dominant SpMM kernels, their number, total kernel launches).'''
    ms, cnt, nl = ctypes.c_double(0), ctypes.c_int64(0), ctypes.c_int64(0)
    _check(lib().nm_profile_end(ctypes.byref(ms), ctypes.byref(cnt), ctypes.byref(nl)), "nm_profile_end")
    return ms.value, cnt.value, nl.value


def nm_unshard_columns(src: torch.Tensor, dst: torch.Tensor, G: int, m: int, nr: int, n: int, L: int, stream=None):
    _dev(src, "src")
    _dev(dst, "dst")
    _check(lib().nm_unshard_columns(src.data_ptr(), dst.data_ptr(), G, m, nr, n, L, src.element_size(),
                                    _stream(src, stream)), "nm_unshard_columns")
    return dst


# ----------------------------------------------------------------------------- bit-packed indices
def nm_index_pack(idx: torch.Tensor, k: int, n: int, N: int, M: int, L: int, stream=None) -> torch.Tensor:
    """D (w x q uint8) -> ceil(log2 M)-bit tile-major words (P:288, P:419 transformLayout)."""
    _dev(idx, "idx")
    nw = lib().nm_index_packed_words(k, n, N, M, L)
    if nw < 0:
        raise NmError(5, "nm_index_pack", "needs 128 % L == 0 and a valid shape")
    out = torch.empty(max(int(nw), 1), dtype=torch.int32, device=idx.device)
    _check(lib().nm_index_pack(idx.data_ptr(), k, n, N, M, L, out.data_ptr(), _stream(idx, stream)), "nm_index_pack")
    return out[:int(nw)]


def nm_index_unpack(words: torch.Tensor, k: int, n: int, N: int, M: int, L: int, stream=None) -> torch.Tensor:
    _dev(words, "words")
    out = torch.empty((k // M * N, n // L), dtype=torch.uint8, device=words.device)
    _check(lib().nm_index_unpack(words.data_ptr(), k, n, N, M, L, out.data_ptr(), _stream(words, stream)),
           "nm_index_unpack")
    return out


# ----------------------------------------------------------------------------- fused peer exchange
def nm_ipc_get_handle(t: torch.Tensor) -> tuple[bytes, int]:
    """(64-byte CUDA IPC handle of t's allocation, byte offset of t in it)."""
    h = ctypes.create_string_buffer(64)
    off = ctypes.c_int64()
    _check(lib().nm_ipc_get_handle(t.data_ptr(), h, ctypes.byref(off)), "nm_ipc_get_handle")
    return h.raw, int(off.value)


def nm_ipc_open_handle(handle: bytes, offset: int) -> int:
    """Map another process's allocation; returns the device address of (its base + offset)."""
    p = ctypes.c_void_p()
    _check(lib().nm_ipc_open_handle(ctypes.create_string_buffer(handle, 64), offset, ctypes.byref(p)),
           "nm_ipc_open_handle")
    return int(p.value)


def nm_ipc_close(ptr: int, offset: int) -> None:
    _check(lib().nm_ipc_close(ctypes.c_void_p(ptr), offset), "nm_ipc_close")


def _ptr_array(ptrs):
    arr = (ctypes.c_void_p * len(ptrs))()
    for i, v in enumerate(ptrs):
        arr[i] = v
    return arr


def nm_spmm_peers(A: torch.Tensor, W: NmWeight, c_ptrs, ldc: int, col_off: int, n_valid: int, stream=None) -> None:
    """Fused sharded product: this shard's C columns [0, n_valid) stored at [row][col_off + j] of
    every buffer in c_ptrs (own or IPC-mapped device addresses, row pitch ldc)."""
    _dev(A, "A")
    m, k = A.shape
    if A.dtype != torch.float32 or W.values.dtype != torch.float32:
        raise TypeError("nm_spmm_peers is the fp32 SIMT peer path: A and values must be float32")
    _check(lib().nm_spmm_peers(A.data_ptr(), W.values.data_ptr(), W.idx.data_ptr(), _ptr_array(c_ptrs), len(c_ptrs),
                               ldc, col_off, n_valid, m, W.n, k, W.N, W.M, W.L, _stream(A, stream)), "nm_spmm_peers")


def nm_peer_barrier(flag_ptrs, rank: int, epoch: int, device=None, stream=None) -> None:
    s = ctypes.c_void_p(stream.cuda_stream) if stream is not None else \
        ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)
    _check(lib().nm_peer_barrier(_ptr_array(flag_ptrs), len(flag_ptrs), rank, epoch, s), "nm_peer_barrier")


def nm_spmm_prepacked_peers(A: torch.Tensor, PW: "PrepackedWeight", c_ptrs, ldc: int, col_off: int, n_valid: int,
                            out_dtype=None, stream=None) -> None:
    """nm_spmm_peers for a prepacked shard (bf16 / tf32 slot kernels, or kind 0 -> the SIMT path)."""
    _dev(A, "A")
    if A.dtype != PW.W.values.dtype:
        raise TypeError(f"A is {A.dtype}, the prepacked weight is {PW.W.values.dtype}")
    cdt = _dt_of(out_dtype or A.dtype)
    _check(lib().nm_spmm_prepacked_peers(A.data_ptr(), ctypes.byref(PW.desc), _ptr_array(c_ptrs), len(c_ptrs), ldc,
                                         col_off, n_valid, A.shape[0], cdt, _stream(A, stream)),
           "nm_spmm_prepacked_peers")


def _dt_of(dtype) -> int:
    if dtype == torch.float32:
        return NM_F32
    if dtype == torch.bfloat16:
        return NM_BF16
    raise TypeError(f"unsupported dtype {dtype}")


# ----------------------------------------------------------------------------- NVLS multicast C
class McBuffer:
    """A multicast (NVLS) buffer of this process's device (nm_mc_*): `mc_ptr` is the multicast
    view (stores through it reach every bound rank's replica), `uc_ptr` this device's replica.
    Single-process form (num_devices = 1); the collective multi-rank setup is the same calls with
    the fabric handle exchanged (MulticastExchange in sharded.py)."""

    def __init__(self, nbytes: int, num_devices: int = 1, fabric_handle: bytes | None = None):
        L = lib()
        self.mc, self.mem = ctypes.c_uint64(), ctypes.c_uint64()
        self.bytes = ctypes.c_int64()
        self.uc_ptr, self.mc_ptr = ctypes.c_void_p(), ctypes.c_void_p()
        if fabric_handle is None:
            _check(L.nm_mc_create(int(nbytes), num_devices, ctypes.byref(self.mc), ctypes.byref(self.bytes)),
                   "nm_mc_create")
        else:
            buf = ctypes.create_string_buffer(bytes(fabric_handle), 64)
            _check(L.nm_mc_import(buf, ctypes.byref(self.mc)), "nm_mc_import")
            self.bytes.value = int(nbytes)

    def export(self) -> bytes:
        buf = ctypes.create_string_buffer(64)
        _check(lib().nm_mc_export(self.mc, buf), "nm_mc_export")
        return buf.raw

    def add_device(self):
        _check(lib().nm_mc_add_device(self.mc), "nm_mc_add_device")

    def bind_map(self):
        _check(lib().nm_mc_bind_map(self.mc, self.bytes, ctypes.byref(self.mem), ctypes.byref(self.uc_ptr),
                                    ctypes.byref(self.mc_ptr)), "nm_mc_bind_map")

    def free(self):
        if self.mc.value:
            _check(lib().nm_mc_free(self.mc, self.mem, self.uc_ptr, self.mc_ptr, self.bytes), "nm_mc_free")
            self.mc.value = 0


def nm_mc_supported() -> bool:
    v = ctypes.c_int(0)
    _check(lib().nm_mc_supported(ctypes.byref(v)), "nm_mc_supported")
    return bool(v.value)


def nm_spmm_mc(A: torch.Tensor, W: "NmWeight", c_mc: int, ldc: int, col_off: int, n_valid: int, stream=None) -> None:
    """C_mc[i][col_off + j] = (A . B~)[i][j] through a multicast address (nm_spmm_mc, fp32 SIMT)."""
    _dev(A, "A")
    if A.dtype != torch.float32 or W.values.dtype != torch.float32:
        raise TypeError("nm_spmm_mc: fp32 A and values (the SIMT kernel's multicast epilogue)")
    m, k = A.shape
    _check(lib().nm_spmm_mc(A.data_ptr(), W.values.data_ptr(), W.idx.data_ptr(), ctypes.c_void_p(c_mc), ldc, col_off,
                            n_valid, m, W.n, k, W.N, W.M, W.L, _stream(A, stream)), "nm_spmm_mc")
