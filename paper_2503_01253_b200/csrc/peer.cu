// peer.cu -- the multi-GPU exchange of the column-sharded layer fused into
// the SpMM: every rank's SpMM epilogue stores its C columns straight into every rank's C buffer
// over NVLink peer memory (CUDA IPC mappings), then a flag barrier in peer memory orders the
// ranks -- no separate all-gather pass and no unshard pass.  Column j of C depends only on A,
// B'[:, j] and D[:, j / L] (Eq. 1), so the ranks' stores never overlap.
#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "common.cuh"

namespace nm {

nm_status simt_f32_launch(const float* A, const float* Bv, const uint8_t* D, float* C, int64_t m, int64_t n, int64_t k,
                          int N, int M, int L, int mode, cudaStream_t s, const PeerOut* po, float alpha, const uint32_t* Dw,
                          const float* At_in = nullptr, int64_t lda = 0);
bool simt_f32_applicable(const void* A, const void* Bv, const void* C, int64_t m, int64_t n, int64_t k, int N, int M,
                         int L);
nm_status require_device();
nm_status tc_sp_run(const void* A, const void* buf, int H, void* C, bool c_bf16, int64_t m, int64_t n, int64_t k, int N,
                    int M, int L, bool tf, cudaStream_t s, const PeerOut* po, float alpha, const void* At_in,
                    int64_t lda);
bool tc_sp_applicable(int64_t m, int64_t n, int64_t k, int N, int M, int L);

struct PeerFlags {
    int* f[8];  // f[p] = rank p's flag array (int[G]) as mapped in this process
};

// One warp.  Lane p < G: publish "rank `rank` reached `epoch`" in rank p's flags (system-scope
// release after a system fence, so this rank's earlier peer stores -- the SpMM kernel before
// this one on the stream -- are visible to whoever acquires the flag), then wait until rank p
// has published the same epoch in ours.  Bounded spin: a missing rank is a bug, trap, do not hang.
__global__ void peer_barrier_kernel(PeerFlags pf, int G, int rank, int epoch, unsigned long long timeout_ns) {
    const int t = threadIdx.x;
    if (t < G) {
        __threadfence_system();
        asm volatile("st.release.sys.global.b32 [%0], %1;" ::"l"(pf.f[t] + rank), "r"(epoch) : "memory");
    }
    __syncwarp();
    if (t < G) {
        const int* mine = pf.f[rank] + t;
        unsigned long long t0, now;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        for (;;) {
            int v;
            asm volatile("ld.acquire.sys.global.b32 %0, [%1];" : "=r"(v) : "l"(mine) : "memory");
            if (v - epoch >= 0) break;  // epochs increase by one per call (wrap-safe compare)
            __nanosleep(128);
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
            // a peer that never arrives is a bug (a crashed rank): fail loudly after the timeout
            // (NM_PEER_TIMEOUT_MS, default 120 s, wall time) instead of hanging the stream forever
            if (now - t0 > timeout_ns) __trap();
        }
    }
}

typedef CUresult (*AddrRangeFn)(CUdeviceptr*, size_t*, CUdeviceptr);

static AddrRangeFn get_addr_range() {
    static AddrRangeFn fn = nullptr;
    static bool done = false;
    if (!done) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<AddrRangeFn>(p);
        cudaGetLastError();
        done = true;
    }
    return fn;
}

}  // namespace nm

using namespace nm;

extern "C" {

nm_status nm_ipc_get_handle(const void* dptr, void* handle, int64_t* offset) {
    if (!dptr || !handle || !offset) return fail(NM_ERR_NULL, "nm_ipc_get_handle: NULL pointer");
    nm_status st = require_device();
    if (st) return st;
    AddrRangeFn fn = get_addr_range();
    if (!fn) return fail(NM_ERR_CUDA, "cuMemGetAddressRange unavailable");
    CUdeviceptr base = 0;
    size_t size = 0;
    if (fn(&base, &size, reinterpret_cast<CUdeviceptr>(dptr)) != CUDA_SUCCESS)
        return fail(NM_ERR_CUDA, "cuMemGetAddressRange failed (not a device allocation?)");
    NM_CUDA_TRY(cudaIpcGetMemHandle(static_cast<cudaIpcMemHandle_t*>(handle), reinterpret_cast<void*>(base)));
    *offset = static_cast<int64_t>(reinterpret_cast<CUdeviceptr>(dptr) - base);
    return NM_OK;
}

nm_status nm_ipc_open_handle(const void* handle, int64_t offset, void** dptr) {
    if (!handle || !dptr) return fail(NM_ERR_NULL, "nm_ipc_open_handle: NULL pointer");
    nm_status st = require_device();
    if (st) return st;
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    void* base = nullptr;
    NM_CUDA_TRY(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
    *dptr = static_cast<uint8_t*>(base) + offset;
    return NM_OK;
}

nm_status nm_ipc_close(void* dptr, int64_t offset) {
    if (!dptr) return fail(NM_ERR_NULL, "nm_ipc_close: NULL pointer");
    NM_CUDA_TRY(cudaIpcCloseMemHandle(static_cast<uint8_t*>(dptr) - offset));
    return NM_OK;
}

nm_status nm_peer_barrier(void* const* flag_peers, int G, int rank, int epoch, void* stream) {
    if (G < 1 || G > 8 || rank < 0 || rank >= G) return fail(NM_ERR_SHAPE, "nm_peer_barrier: 1 <= G <= 8, 0 <= rank < G");
    if (!flag_peers) return fail(NM_ERR_NULL, "nm_peer_barrier: NULL pointer");
    PeerFlags pf{};
    for (int i = 0; i < G; ++i) {
        if (!flag_peers[i]) return fail(NM_ERR_NULL, "nm_peer_barrier: NULL flag pointer");
        pf.f[i] = static_cast<int*>(flag_peers[i]);
    }
    nm_status st = require_device();
    if (st) return st;
    const char* te = std::getenv("NM_PEER_TIMEOUT_MS");
    const long long ms = te ? std::atoll(te) : 120000;
    const unsigned long long timeout_ns = static_cast<unsigned long long>(ms > 0 ? ms : 120000) * 1000000ull;
    peer_barrier_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(pf, G, rank, epoch, timeout_ns);
    note_launch();
    NM_LAUNCH_CHECK("peer_barrier_kernel");
    return NM_OK;
}

nm_status nm_spmm_peers(const void* A, const void* values, const uint8_t* idx, void* const* C_peers, int G, int64_t ldc,
                        int64_t col_off, int64_t n_valid, int64_t m, int64_t nr, int64_t k, int N, int M, int L,
                        void* stream) {
    if (N < 1 || M < N || M > 256 || L < 1) return fail(NM_ERR_INVALID_CONFIG, "invalid N:M/L");
    if (m < 0 || nr < 0 || k < 0 || k % M || nr % L) return fail(NM_ERR_SHAPE, "nm_spmm_peers: shape");
    if (G < 1 || G > 8) return fail(NM_ERR_SHAPE, "nm_spmm_peers: 1 <= G <= 8");
    if (col_off < 0 || n_valid < 0 || n_valid > nr || col_off + n_valid > ldc)
        return fail(NM_ERR_SHAPE, "nm_spmm_peers: columns [col_off, col_off + n_valid) outside ldc, or n_valid > nr");
    // the SIMT peer epilogue stores float4s guarded by col < n_valid: a ragged n_valid would write
    // up to 3 columns of another rank's range
    if (n_valid % 4) return fail(NM_ERR_SHAPE, "nm_spmm_peers: n_valid must be a multiple of 4");
    if (m == 0 || nr == 0 || n_valid == 0) return NM_OK;
    if (!A || !C_peers || (k > 0 && (!values || !idx))) return fail(NM_ERR_NULL, "nm_spmm_peers: NULL pointer");
    PeerOut po{};
    po.np = G;
    po.ldc = ldc;
    po.col_off = col_off;
    po.n_valid = n_valid;
    uintptr_t al = static_cast<uintptr_t>(ldc | col_off) * 4u;
    for (int i = 0; i < G; ++i) {
        if (!C_peers[i]) return fail(NM_ERR_NULL, "nm_spmm_peers: NULL C pointer");
        po.c[i] = C_peers[i];
        al |= reinterpret_cast<uintptr_t>(C_peers[i]);
    }
    // the fused path is the fp32 SIMT kernel's epilogue: 16-B stores at [row][col_off + col]
    if (k == 0 || (al & 15) || !simt_f32_applicable(A, values, po.c[0], m, nr, k, N, M, L))
        return fail(NM_ERR_UNSUPPORTED, "nm_spmm_peers: needs the fp32 SIMT kernel's geometry (L % 4 == 0, M <= 64, "
                                        "N <= 32, k > 0, 16-B aligned operands, ldc and col_off multiples of 4)");
    nm_status st = require_device();
    if (st) return st;
    const int mode = m % 4 == 0 ? 1 : 0;  // A^T staging needs m % 4 == 0 (as in the selector)
    return simt_f32_launch(static_cast<const float*>(A), static_cast<const float*>(values), idx,
                           static_cast<float*>(po.c[0]), m, nr, k, N, M, L, mode, static_cast<cudaStream_t>(stream), &po,
                           1.f, nullptr);
}

nm_status nm_spmm_mc(const void* A, const void* values, const uint8_t* idx, void* C_mc, int64_t ldc, int64_t col_off,
                     int64_t n_valid, int64_t m, int64_t nr, int64_t k, int N, int M, int L, void* stream) {
    if (N < 1 || M < N || M > 256 || L < 1) return fail(NM_ERR_INVALID_CONFIG, "invalid N:M/L");
    if (m < 0 || nr < 0 || k < 0 || k % M || nr % L) return fail(NM_ERR_SHAPE, "nm_spmm_mc: shape");
    if (col_off < 0 || n_valid < 0 || n_valid > nr || col_off + n_valid > ldc || n_valid % 4)
        return fail(NM_ERR_SHAPE, "nm_spmm_mc: columns [col_off, col_off + n_valid) outside ldc, n_valid > nr or "
                                  "n_valid % 4 != 0");
    if (m == 0 || nr == 0 || n_valid == 0) return NM_OK;
    if (!A || !C_mc || (k > 0 && (!values || !idx))) return fail(NM_ERR_NULL, "nm_spmm_mc: NULL pointer");
    PeerOut po{};
    po.np = 1;
    po.mc = 1;
    po.ldc = ldc;
    po.col_off = col_off;
    po.n_valid = n_valid;
    po.c[0] = C_mc;
    const uintptr_t al = static_cast<uintptr_t>(ldc | col_off) * 4u | reinterpret_cast<uintptr_t>(C_mc);
    if (k == 0 || (al & 15) || !simt_f32_applicable(A, values, C_mc, m, nr, k, N, M, L))
        return fail(NM_ERR_UNSUPPORTED, "nm_spmm_mc: needs the fp32 SIMT kernel's geometry (L % 4 == 0, M <= 64, "
                                        "N <= 32, k > 0, 16-B aligned operands, ldc and col_off multiples of 4)");
    nm_status st = require_device();
    if (st) return st;
    const int mode = m % 4 == 0 ? 1 : 0;
    return simt_f32_launch(static_cast<const float*>(A), static_cast<const float*>(values), idx,
                           static_cast<float*>(C_mc), m, nr, k, N, M, L, mode, static_cast<cudaStream_t>(stream), &po,
                           1.f, nullptr);
}

nm_status nm_spmm_prepacked_peers(const void* A, const nm_prepacked* w, void* const* C_peers, int G, int64_t ldc,
                                  int64_t col_off, int64_t n_valid, int64_t m, nm_dtype c_dt, void* stream) {
    if (!w || w->magic != 0x4B504D4E) return fail(NM_ERR_NULL, "nm_spmm_prepacked_peers: descriptor not filled by nm_prepack");
    if (w->kind == 0 || w->kind == 4) {  // fp32 weights: the SIMT kernel's peer epilogue (fp32 A, B', C)
        if (w->dtype != NM_F32 || c_dt != NM_F32)
            return fail(NM_ERR_UNSUPPORTED, "nm_spmm_prepacked_peers: a weight without slot images (prepack kind 0) "
                                            "takes the fp32 SIMT peer path, which needs fp32 values and an fp32 C");
        return nm_spmm_peers(A, w->values, w->idx, C_peers, G, ldc, col_off, n_valid, m, w->n, w->k, w->N, w->M, w->L,
                             stream);
    }
    if (w->kind != 2 && w->kind != 3)
        return fail(NM_ERR_UNSUPPORTED, "nm_spmm_prepacked_peers: prepack kind 0, 2 or 3 (slot kernels) only");
    if (G < 1 || G > 8) return fail(NM_ERR_SHAPE, "nm_spmm_prepacked_peers: 1 <= G <= 8");
    if (m < 0 || col_off < 0 || n_valid < 0 || n_valid > w->n || col_off + n_valid > ldc)
        return fail(NM_ERR_SHAPE, "nm_spmm_prepacked_peers: columns [col_off, col_off + n_valid) outside ldc");
    const bool tf = w->kind == 3;
    if (tf && c_dt != NM_F32) return fail(NM_ERR_UNSUPPORTED, "fp32 operands need an fp32 C");
    // the direct-store epilogue writes bf16 C as column pairs guarded by pair < n_valid
    if (c_dt == NM_BF16 && (n_valid % 2))
        return fail(NM_ERR_SHAPE, "nm_spmm_prepacked_peers: bf16 C needs an even n_valid");
    if (m == 0 || w->n == 0 || n_valid == 0) return NM_OK;
    if (!A || !C_peers) return fail(NM_ERR_NULL, "nm_spmm_prepacked_peers: NULL pointer");
    PeerOut po{};
    po.np = G;
    po.ldc = ldc;
    po.col_off = col_off;
    po.n_valid = n_valid;
    const int eb = c_dt == NM_BF16 ? 2 : 4;
    uintptr_t al = reinterpret_cast<uintptr_t>(A) & 15;
    for (int i = 0; i < G; ++i) {
        if (!C_peers[i]) return fail(NM_ERR_NULL, "nm_spmm_prepacked_peers: NULL C pointer");
        po.c[i] = C_peers[i];
        al |= (reinterpret_cast<uintptr_t>(C_peers[i]) | static_cast<uintptr_t>((ldc | col_off) * eb)) & 3;
    }
    if (al || w->k % 8 || !tc_sp_applicable(m, w->n, w->k, w->N, w->M, w->L))
        return fail(NM_ERR_UNSUPPORTED, "nm_spmm_prepacked_peers: A 16-B aligned, C pointers / ldc / col_off 4-B aligned, "
                                        "k % 8 == 0");
    nm_status st = require_device();
    if (st) return st;
    return tc_sp_run(A, w->bperm, w->bn / 128, po.c[0], c_dt == NM_BF16, m, w->n, w->k, w->N, w->M, w->L, tf,
                     static_cast<cudaStream_t>(stream), &po, 1.f, nullptr, 0);
}

}  // extern "C"
