// format.cu -- N:M compression, decompression, validation and multi-GPU
// column assembly kernels (sm_100a).  Offline / plumbing kernels: memory-bound,
// one pass, coalesced along n.
//
// Compression follows P:93 (Sec. II-A, "select N vectors from every M vector
// along the k dimension of matrix B") with DESIGN.md readings R6 (L2 score in
// fp64, ties -> smaller offset, NaN rejected), R7 (offsets ascending), R10
// (underfull windows keep zero vectors at the smallest unused offsets, which
// the tie rule produces) and R11 (bf16 values by RNE).
#include <cuda_bf16.h>

#include "common.cuh"

namespace nm {

template <typename T>
__device__ __forceinline__ double to_f64(T x);
template <>
__device__ __forceinline__ double to_f64<float>(float x) { return static_cast<double>(x); }
template <>
__device__ __forceinline__ double to_f64<__nv_bfloat16>(__nv_bfloat16 x) {
    return static_cast<double>(__bfloat162float(x));
}

template <typename TI, typename TO>
__device__ __forceinline__ TO convert_value(TI x);
template <>
__device__ __forceinline__ float convert_value<float, float>(float x) { return x; }
template <>
__device__ __forceinline__ __nv_bfloat16 convert_value<float, __nv_bfloat16>(float x) {
    return __float2bfloat16_rn(x);  // RNE (R11)
}
template <>
__device__ __forceinline__ __nv_bfloat16 convert_value<__nv_bfloat16, __nv_bfloat16>(__nv_bfloat16 x) {
    return x;
}
template <>
__device__ __forceinline__ float convert_value<__nv_bfloat16, float>(__nv_bfloat16 x) {
    return __bfloat162float(x);
}

// One thread per (window t, column group g); threads of a warp take
// consecutive g so the L-wide row segments they read are adjacent in memory.
// scores[] lives in local memory (M <= 256 doubles).
template <typename TI, typename TO>
__global__ void __launch_bounds__(128) compress_kernel(const TI* __restrict__ B, int64_t k, int64_t n, int N,
                                                       int M, int L, TO* __restrict__ values,
                                                       uint8_t* __restrict__ idx, int* __restrict__ nan_flag) {
    const int64_t q = n / L, windows = k / M;
    const int64_t tg = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (tg >= windows * q) return;
    const int64_t t = tg / q, g = tg % q;
    double score[256];
    bool has_nan = false;
    for (int r = 0; r < M; ++r) {
        const TI* row = B + (t * M + r) * n + g * L;
        double acc = 0.0;
        for (int c = 0; c < L; ++c) {
            const double x = to_f64<TI>(row[c]);
            has_nan |= (x != x);
            acc = __dadd_rn(acc, __dmul_rn(x, x));  // fixed order, no FMA (R6)
        }
        score[r] = acc;
    }
    if (has_nan) atomicExch(nan_flag, 1);
    // rank_r = #{r' : s_r' > s_r or (s_r' == s_r and r' < r)}; keep iff rank_r < N.
    int pos = 0;
    for (int r = 0; r < M && pos < N; ++r) {
        const double s = score[r];
        int rank = 0;
        for (int r2 = 0; r2 < M; ++r2) {
            const double s2 = score[r2];
            rank += (s2 > s) || (s2 == s && r2 < r);
        }
        if (rank < N) {
            const int64_t u = t * N + pos;
            idx[u * q + g] = static_cast<uint8_t>(r);
            const TI* src = B + (t * M + r) * n + g * L;
            TO* dst = values + u * n + g * L;
            for (int c = 0; c < L; ++c) dst[c] = convert_value<TI, TO>(src[c]);
            ++pos;
        }
    }
}

// B_out[t*M + idx[u][j/L]][j] = values[u][j]; B_out zeroed beforehand.
template <typename T>
__global__ void decompress_kernel(const T* __restrict__ values, const uint8_t* __restrict__ idx, int64_t k,
                                  int64_t n, int N, int M, int L, T* __restrict__ out) {
    const int64_t w = k / M * N, q = n / L;
    const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= w * n) return;
    const int64_t u = e / n, j = e % n;
    const int d = idx[u * q + j / L];
    if (d >= M) return;
    out[((u / N) * M + d) * n + j] = values[e];
}

__global__ void validate_kernel(const uint8_t* __restrict__ idx, int64_t w, int64_t q, int N, int M,
                                unsigned long long* __restrict__ first_bad) {
    const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= w * q) return;
    const int64_t u = e / q;
    const int d = idx[e];
    bool bad = d >= M;
    if (!bad && (u % N) != 0) bad = idx[e - q] >= d;
    if (bad) atomicMin(first_bad, static_cast<unsigned long long>(e));
}

// dst[i][L*g0(r) + j] = src[r][i][j] for j < L*cnt(r), g0(r) = floor(r*q/G).
template <typename T>
__global__ void unshard_kernel(const T* __restrict__ src, T* __restrict__ dst, int64_t G, int64_t m,
                               int64_t nr, int64_t q, int L) {
    const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= G * m * nr) return;
    const int64_t r = e / (m * nr), rem = e % (m * nr), i = rem / nr, j = rem % nr;
    const int64_t g0 = r * q / G, g1 = (r + 1) * q / G;
    if (j >= (g1 - g0) * L) return;
    dst[i * (q * L) + g0 * L + j] = src[e];
}

// ------------------------------------------------------------------ launchers
template <typename TI, typename TO>
static void launch_compress(const void* B, int64_t k, int64_t n, int N, int M, int L, void* values, uint8_t* idx,
                            int* flag, cudaStream_t s) {
    const int64_t total = (k / M) * (n / L);
    const int threads = 128;
    const int64_t blocks = ceil_div(total, threads);
    compress_kernel<TI, TO><<<static_cast<unsigned>(blocks), threads, 0, s>>>(
        static_cast<const TI*>(B), k, n, N, M, L, static_cast<TO*>(values), idx, flag);
}

nm_status compress_launch(const void* B, nm_dtype b_dt, int64_t k, int64_t n, int N, int M, int L, void* values,
                          nm_dtype v_dt, uint8_t* idx, cudaStream_t s) {
    if (k == 0 || n == 0) return NM_OK;
    int* flag = nullptr;
    NM_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&flag), sizeof(int), s));
    NM_CUDA_TRY(cudaMemsetAsync(flag, 0, sizeof(int), s));
    if (b_dt == NM_F32 && v_dt == NM_F32)
        launch_compress<float, float>(B, k, n, N, M, L, values, idx, flag, s);
    else if (b_dt == NM_F32 && v_dt == NM_BF16)
        launch_compress<float, __nv_bfloat16>(B, k, n, N, M, L, values, idx, flag, s);
    else if (b_dt == NM_BF16 && v_dt == NM_BF16)
        launch_compress<__nv_bfloat16, __nv_bfloat16>(B, k, n, N, M, L, values, idx, flag, s);
    else
        launch_compress<__nv_bfloat16, float>(B, k, n, N, M, L, values, idx, flag, s);
    NM_LAUNCH_CHECK("compress_kernel");
    int h = 0;
    NM_CUDA_TRY(cudaMemcpyAsync(&h, flag, sizeof(int), cudaMemcpyDeviceToHost, s));
    NM_CUDA_TRY(cudaFreeAsync(flag, s));
    NM_CUDA_TRY(cudaStreamSynchronize(s));
    if (h) return fail(NM_ERR_NONFINITE, "nm_compress: NaN in B (score undefined, reading R6)");
    return NM_OK;
}

nm_status decompress_launch(const void* values, nm_dtype v_dt, const uint8_t* idx, int64_t k, int64_t n, int N,
                            int M, int L, void* out, cudaStream_t s) {
    const size_t esz = v_dt == NM_BF16 ? 2 : 4;
    if (k == 0 || n == 0) return NM_OK;
    NM_CUDA_TRY(cudaMemsetAsync(out, 0, static_cast<size_t>(k * n) * esz, s));
    const int64_t total = (k / M * N) * n;
    const int threads = 256;
    const unsigned blocks = static_cast<unsigned>(ceil_div(total, threads));
    if (v_dt == NM_BF16)
        decompress_kernel<__nv_bfloat16><<<blocks, threads, 0, s>>>(
            static_cast<const __nv_bfloat16*>(values), idx, k, n, N, M, L, static_cast<__nv_bfloat16*>(out));
    else
        decompress_kernel<float><<<blocks, threads, 0, s>>>(static_cast<const float*>(values), idx, k, n, N, M,
                                                            L, static_cast<float*>(out));
    NM_LAUNCH_CHECK("decompress_kernel");
    return NM_OK;
}

nm_status validate_launch(const uint8_t* idx, int64_t k, int64_t n, int N, int M, int L, int64_t* first_bad_host,
                          cudaStream_t s) {
    const int64_t w = k / M * N, q = n / L;
    *first_bad_host = -1;
    if (w * q == 0) return NM_OK;
    unsigned long long* d = nullptr;
    NM_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&d), sizeof(unsigned long long), s));
    NM_CUDA_TRY(cudaMemsetAsync(d, 0xFF, sizeof(unsigned long long), s));
    const int threads = 256;
    validate_kernel<<<static_cast<unsigned>(ceil_div(w * q, threads)), threads, 0, s>>>(idx, w, q, N, M, d);
    NM_LAUNCH_CHECK("validate_kernel");
    unsigned long long h = 0;
    NM_CUDA_TRY(cudaMemcpyAsync(&h, d, sizeof(h), cudaMemcpyDeviceToHost, s));
    NM_CUDA_TRY(cudaFreeAsync(d, s));
    NM_CUDA_TRY(cudaStreamSynchronize(s));
    if (h != ~0ull) {
        *first_bad_host = static_cast<int64_t>(h);
        return fail(NM_ERR_INVALID_INDICES, "nm_validate: index entry out of range or not strictly increasing");
    }
    return NM_OK;
}

nm_status unshard_launch(const void* src, void* dst, int64_t G, int64_t m, int64_t nr, int64_t q, int L,
                         int elem_bytes, cudaStream_t s) {
    const int64_t total = G * m * nr;
    if (total == 0) return NM_OK;
    const int threads = 256;
    const unsigned blocks = static_cast<unsigned>(ceil_div(total, threads));
    if (elem_bytes == 2)
        unshard_kernel<uint16_t><<<blocks, threads, 0, s>>>(static_cast<const uint16_t*>(src),
                                                            static_cast<uint16_t*>(dst), G, m, nr, q, L);
    else
        unshard_kernel<uint32_t><<<blocks, threads, 0, s>>>(static_cast<const uint32_t*>(src),
                                                            static_cast<uint32_t*>(dst), G, m, nr, q, L);
    note_launch();
    NM_LAUNCH_CHECK("unshard_kernel");
    return NM_OK;
}

// ------------------------------------------------------------ bit-packed indices
// The index matrix D with ceil(log2 M) bits per entry in a tile-major layout
// (transformLayout, P:419 / Listing 3): per column tile of T = 128 / L groups (one SIMT CTA tile of
// 128 output columns) its entries x = u * T + t (row u, group t of the tile) are a contiguous
// stream of 32-bit words, floor(32 / b) entries per word, entry x at word x / e, bit (x % e) * b.
// A CTA's whole index stream is one coalesced run (R28).
struct IdxPack {
    int b, e, T;
    int64_t w, q, Wt, ntiles;
};
static IdxPack idx_pack_geom(int64_t k, int64_t n, int N, int M, int L) {
    IdxPack g{};
    g.b = 1;
    while ((1 << g.b) < M) ++g.b;
    g.e = 32 / g.b;
    g.T = 128 / L;
    g.w = k / M * N;
    g.q = n / L;
    g.ntiles = (g.q + g.T - 1) / g.T;
    g.Wt = (g.w * g.T + g.e - 1) / g.e;
    return g;
}

__global__ void index_pack_kernel(const uint8_t* __restrict__ D, uint32_t* __restrict__ P, IdxPack g) {
    const int64_t wi = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;  // one word
    if (wi >= g.ntiles * g.Wt) return;
    const int64_t tile = wi / g.Wt, x0 = (wi % g.Wt) * g.e;
    uint32_t word = 0;
    for (int i = 0; i < g.e; ++i) {
        const int64_t x = x0 + i, u = x / g.T, gg = tile * g.T + x % g.T;
        if (u < g.w && gg < g.q) word |= static_cast<uint32_t>(D[u * g.q + gg]) << (i * g.b);
    }
    P[wi] = word;
}

__global__ void index_unpack_kernel(const uint32_t* __restrict__ P, uint8_t* __restrict__ D, IdxPack g) {
    const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;  // one entry of D
    if (e >= g.w * g.q) return;
    const int64_t u = e / g.q, gg = e % g.q, x = u * g.T + gg % g.T;
    const uint32_t word = P[(gg / g.T) * g.Wt + x / g.e];
    D[e] = static_cast<uint8_t>((word >> ((x % g.e) * g.b)) & ((1u << g.b) - 1u));
}

int64_t index_packed_words(int64_t k, int64_t n, int N, int M, int L) {
    if (L < 1 || 128 % L || M < 1 || k % M || n % L) return -1;
    const IdxPack g = idx_pack_geom(k, n, N, M, L);
    return g.ntiles * g.Wt;
}

nm_status index_pack_launch(const uint8_t* D, uint32_t* P, int64_t k, int64_t n, int N, int M, int L, bool unpack,
                            cudaStream_t s) {
    const IdxPack g = idx_pack_geom(k, n, N, M, L);
    const int64_t total = unpack ? g.w * g.q : g.ntiles * g.Wt;
    if (total == 0) return NM_OK;
    const unsigned blocks = static_cast<unsigned>(ceil_div(total, 256));
    if (unpack)
        index_unpack_kernel<<<blocks, 256, 0, s>>>(P, const_cast<uint8_t*>(D), g);
    else
        index_pack_kernel<<<blocks, 256, 0, s>>>(D, P, g);
    note_launch();
    NM_LAUNCH_CHECK("index_pack_kernel");
    return NM_OK;
}

}  // namespace nm
