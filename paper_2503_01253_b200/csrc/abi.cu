// abi.cu -- the extern "C" boundary of libnmspmm.so (declared in include/nmspmm.h):
// argument validation, the selector, dispatch to the sm_100a kernels, status /
// thread-local error reporting.  No CPU fallback: every compute entry point
// needs a CUDA device and returns NM_ERR_CUDA without one.
#include <cuda_bf16.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <atomic>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace nm {

// ------------------------------------------------------------ error plumbing
static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

nm_status fail(nm_status s, const std::string& msg) {
    g_last_error = msg;
    return s;
}

nm_status cuda_fail(cudaError_t e, const char* what) {
    g_last_error = std::string("CUDA error in ") + what + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")";
    return NM_ERR_CUDA;
}

// Device properties, cached per device ordinal (a process may drive several GPUs): SM count and
// compute capability of the CURRENT device.  Benign races: every thread computes the same values.
constexpr int kMaxDev = 64;
static std::atomic<int> g_sms[kMaxDev];
static std::atomic<int> g_ccs[kMaxDev];

int current_device() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) {
        cudaGetLastError();
        return -1;
    }
    return dev;
}

static void read_props(int dev) {
    if (dev < 0 || dev >= kMaxDev || g_ccs[dev].load(std::memory_order_acquire) != 0) return;
    int sms = 0, major = 0, minor = 0;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess) g_sms[dev].store(sms);
    if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) == cudaSuccess &&
        cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev) == cudaSuccess)
        g_ccs[dev].store(major * 10 + minor, std::memory_order_release);
    cudaGetLastError();
}

int num_sms() {
    const int dev = current_device();
    read_props(dev);
    const int v = (dev >= 0 && dev < kMaxDev) ? g_sms[dev].load() : 0;
    return v > 0 ? v : 148;
}

nm_status require_device() {  // also used by peer.cu
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0) {
        cudaGetLastError();
        return fail(NM_ERR_CUDA, "no CUDA device: libnmspmm has no CPU fallback");
    }
    const int dev = current_device();
    read_props(dev);
    const int cc = (dev >= 0 && dev < kMaxDev) ? g_ccs[dev].load() : 0;
    if (cc != 100)
        return fail(NM_ERR_UNSUPPORTED, "libnmspmm is built for sm_100a (B200); device compute capability is " +
                                            std::to_string(cc));
    return NM_OK;
}

bool attr_once(std::atomic<uint64_t>& mask) {
    const int dev = current_device();
    if (dev < 0 || dev >= 64) return true;
    return (mask.load(std::memory_order_acquire) >> dev) & 1u;
}
void attr_done(std::atomic<uint64_t>& mask) {
    const int dev = current_device();
    if (dev >= 0 && dev < 64) mask.fetch_or(1ull << dev, std::memory_order_acq_rel);
}

// ------------------------------------------------------------ profiling
struct ProfState {
    bool on = false;
    int64_t launches = 0;
    std::vector<cudaEvent_t> ev;  // begin/end pairs
    size_t used = 0;
};
static std::mutex g_prof_mu;
static ProfState g_prof;

void note_launch() {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    if (g_prof.on) ++g_prof.launches;
}
static void prof_record(cudaStream_t s) {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    if (!g_prof.on) return;
    if (g_prof.used == g_prof.ev.size()) {
        cudaEvent_t e;
        if (cudaEventCreate(&e) != cudaSuccess) return;
        g_prof.ev.push_back(e);
    }
    cudaEventRecord(g_prof.ev[g_prof.used++], s);
}
void prof_begin(cudaStream_t s) { prof_record(s); }
void prof_end(cudaStream_t s) { prof_record(s); }

// --------------------------------------------------------- scratch memory pool
// Per-call scratch (the tcgen05 path's cell tables) comes from a library-owned
// stream-ordered pool whose release threshold keeps freed blocks cached, so a
// steady stream of nm_spmm calls allocates nothing after the first one.
// One pool per device (the pool of the current device, which owns the caller's stream).
static std::mutex g_pool_mu;
static cudaMemPool_t g_pool[kMaxDev] = {};
static bool g_pool_tried[kMaxDev] = {};

nm_status scratch_alloc(void** p, size_t bytes, cudaStream_t s) {
    const int dev = current_device();
    cudaMemPool_t pool = nullptr;
    if (dev >= 0 && dev < kMaxDev) {
        std::lock_guard<std::mutex> lk(g_pool_mu);
        if (!g_pool_tried[dev]) {
            g_pool_tried[dev] = true;
            cudaMemPoolProps props{};
            props.allocType = cudaMemAllocationTypePinned;
            props.location.type = cudaMemLocationTypeDevice;
            props.location.id = dev;
            if (cudaMemPoolCreate(&g_pool[dev], &props) == cudaSuccess) {
                uint64_t thr = ~0ull;
                cudaMemPoolSetAttribute(g_pool[dev], cudaMemPoolAttrReleaseThreshold, &thr);
            } else {
                g_pool[dev] = nullptr;
            }
            cudaGetLastError();
        }
        pool = g_pool[dev];
    }
    cudaError_t e = pool ? cudaMallocFromPoolAsync(p, bytes, pool, s) : cudaMallocAsync(p, bytes, s);
    if (e != cudaSuccess) return cuda_fail(e, "scratch allocation");
    return NM_OK;
}

// ------------------------------------------------------------------ TMA
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encode() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
        cudaGetLastError();
    });
    return fn;
}

nm_status make_tma_2d(CUtensorMap* map, const void* base, CUtensorMapDataType dt, int elem_bytes, int64_t rows,
                      int64_t cols, int box_rows, int box_cols, int swizzle) {
    EncodeTiledFn enc = get_encode();
    if (!enc) return fail(NM_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    cuuint64_t gdim[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
    cuuint64_t gstride[1] = {static_cast<cuuint64_t>(cols) * elem_bytes};
    cuuint32_t box[2] = {static_cast<cuuint32_t>(box_cols), static_cast<cuuint32_t>(box_rows)};
    cuuint32_t estr[2] = {1, 1};
    CUtensorMapSwizzle sw = swizzle == 128  ? CU_TENSOR_MAP_SWIZZLE_128B
                            : swizzle == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                            : swizzle == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                            : CU_TENSOR_MAP_SWIZZLE_NONE;
    CUresult r = enc(map, dt, 2, const_cast<void*>(base), gdim, gstride, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        char buf[256];
        snprintf(buf, sizeof(buf), "cuTensorMapEncodeTiled failed (%d): rows=%lld cols=%lld box=%dx%d swizzle=%d",
                 static_cast<int>(r), static_cast<long long>(rows), static_cast<long long>(cols), box_rows, box_cols,
                 swizzle);
        return fail(NM_ERR_ALIGNMENT, buf);
    }
    return NM_OK;
}

nm_status make_tma_2d_pitched(CUtensorMap* map, const void* base, CUtensorMapDataType dt, int elem_bytes, int64_t rows,
                              int64_t cols, int64_t pitch_elems, int box_rows, int box_cols, int swizzle) {
    EncodeTiledFn enc = get_encode();
    if (!enc) return fail(NM_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    cuuint64_t gdim[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
    cuuint64_t gstride[1] = {static_cast<cuuint64_t>(pitch_elems) * elem_bytes};
    cuuint32_t box[2] = {static_cast<cuuint32_t>(box_cols), static_cast<cuuint32_t>(box_rows)};
    cuuint32_t estr[2] = {1, 1};
    CUtensorMapSwizzle sw = swizzle == 128  ? CU_TENSOR_MAP_SWIZZLE_128B
                            : swizzle == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                            : swizzle == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                            : CU_TENSOR_MAP_SWIZZLE_NONE;
    CUresult r = enc(map, dt, 2, const_cast<void*>(base), gdim, gstride, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        char buf[256];
        snprintf(buf, sizeof(buf), "cuTensorMapEncodeTiled failed (%d): rows=%lld cols=%lld pitch=%lld box=%dx%d",
                 static_cast<int>(r), static_cast<long long>(rows), static_cast<long long>(cols),
                 static_cast<long long>(pitch_elems), box_rows, box_cols);
        return fail(NM_ERR_ALIGNMENT, buf);
    }
    return NM_OK;
}

// ---------------------------------------------------------- kernels (extern)
nm_status compress_launch(const void* B, nm_dtype b_dt, int64_t k, int64_t n, int N, int M, int L, void* values,
                          nm_dtype v_dt, uint8_t* idx, cudaStream_t s);
nm_status decompress_launch(const void* values, nm_dtype v_dt, const uint8_t* idx, int64_t k, int64_t n, int N,
                            int M, int L, void* out, cudaStream_t s);
nm_status validate_launch(const uint8_t* idx, int64_t k, int64_t n, int N, int M, int L, int64_t* first_bad_host,
                          cudaStream_t s);
nm_status unshard_launch(const void* src, void* dst, int64_t G, int64_t m, int64_t nr, int64_t q, int L,
                         int elem_bytes, cudaStream_t s);
int64_t index_packed_words(int64_t k, int64_t n, int N, int M, int L);
nm_status index_pack_launch(const uint8_t* D, uint32_t* P, int64_t k, int64_t n, int N, int M, int L, bool unpack,
                            cudaStream_t s);
bool simt_f32_applicable(const void* A, const void* Bv, const void* C, int64_t m, int64_t n, int64_t k, int N, int M,
                         int L);
void simt_f32_geometry(int N, int M, int* wp, int* bk, int* bkw);
int simt_split_factor(int ntiles, int64_t w, int npanels, int bm);
int simt_row_tile(int64_t m, int64_t n, int64_t w);
nm_status simt_f32_launch(const float* A, const float* Bv, const uint8_t* D, float* C, int64_t m, int64_t n, int64_t k,
                          int N, int M, int L, int mode, cudaStream_t s, const PeerOut* po = nullptr,
                          float alpha = 1.f, const uint32_t* Dw = nullptr, const float* At_in = nullptr,
                          int64_t lda = 0);
bool tc_sp_applicable(int64_t m, int64_t n, int64_t k, int N, int M, int L);
// tf: fp32 operands on the tf32 sparse tensor cores (1:2 slot pairs), else bf16 (2:4 slot quads)
size_t tc_sp_prepack_bytes(int64_t n, int64_t k, int N, int M, int L, bool tf);  // bound (no data)
int tc_sp_halves(int N, int M, int L);
int tc_sp_halves_m(int N, int M, int L, int64_t m, int64_t n, int64_t k);  // per-call prepack (m known)
void tc_sp_geometry(int64_t m, int64_t n, int64_t k, int N, int M, int L, int* halves, int* tokens);
nm_status tc_sp_prepack(const void* Bv, const uint8_t* D, int64_t n, int64_t k, int N, int M, int L, bool tf, int H,
                        void* buf, int64_t buf_bytes, int64_t* exact, bool query_only, cudaStream_t s);
nm_status tc_sp_run(const void* A, const void* buf, int H, void* C, bool c_bf16, int64_t m, int64_t n, int64_t k, int N,
                    int M, int L, bool tf, cudaStream_t s, const PeerOut* po = nullptr, float alpha = 1.f,
                    const void* At_in = nullptr, int64_t lda = 0);
nm_status tc_sp_launch(const void* A, const void* Bv, const uint8_t* D, void* C, bool c_bf16, int64_t m, int64_t n,
                       int64_t k, int N, int M, int L, bool tf, cudaStream_t s, float alpha = 1.f,
                       const void* At_in = nullptr, int64_t lda = 0);

// Sparse-tensor-core slot path (spmm_tc_sp.cu): bf16, L in {16, 32, 64, 128}, A 16-B aligned with
// k % 8 == 0 (the per-call transpose reads 16-B chunks), C 4-B aligned.  NM_TC_SP=0 disables it.
static bool tc_sp_ok(const void* A, const void* C, int64_t m, int64_t n, int64_t k, int N, int M, int L) {
    const char* e = getenv("NM_TC_SP");
    if (e && e[0] == '0') return false;
    return tc_sp_applicable(m, n, k, N, M, L) && k % 8 == 0 && (reinterpret_cast<uintptr_t>(A) & 15) == 0 &&
           (reinterpret_cast<uintptr_t>(C) & 3) == 0;
}

// ---------------------------------------------------------- generic kernel
// One thread per C element; correct for every valid (N, M, L) and alignment.
// Used when no tiled kernel applies (L % 4 != 0, M > 64, N > 32, misaligned).
template <typename T>
__device__ __forceinline__ float ld_f(const T* p, int64_t i);
template <>
__device__ __forceinline__ float ld_f<float>(const float* p, int64_t i) { return p[i]; }
template <>
__device__ __forceinline__ float ld_f<__nv_bfloat16>(const __nv_bfloat16* p, int64_t i) {
    return __bfloat162float(p[i]);
}
template <typename T>
__device__ __forceinline__ void st_f(T* p, int64_t i, float v);
template <>
__device__ __forceinline__ void st_f<float>(float* p, int64_t i, float v) { p[i] = v; }
template <>
__device__ __forceinline__ void st_f<__nv_bfloat16>(__nv_bfloat16* p, int64_t i, float v) {
    p[i] = __float2bfloat16_rn(v);
}

template <typename TA, typename TC>
__global__ void spmm_generic_kernel(const TA* __restrict__ A, const TA* __restrict__ Bv, const uint8_t* __restrict__ D,
                                    TC* __restrict__ C, int64_t m, int64_t n, int64_t k, int N, int M, int L) {
    const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t i = static_cast<int64_t>(blockIdx.y) * blockDim.y + threadIdx.y;
    if (i >= m || j >= n) return;
    const int64_t q = n / L, w = k / M * N, g = j / L;
    const TA* arow = A + i * k;
    float acc = 0.f;
    for (int64_t u = 0; u < w; ++u) {
        const int64_t kabs = (u / N) * M + D[u * q + g];  // Eq. 1 with R1-R3
        acc = fmaf(ld_f<TA>(arow, kabs), ld_f<TA>(Bv, u * n + j), acc);
    }
    st_f<TC>(C, i * n + j, acc);
}

template <typename TA, typename TC>
static nm_status generic_launch(const void* A, const void* Bv, const uint8_t* D, void* C, int64_t m, int64_t n,
                                int64_t k, int N, int M, int L, cudaStream_t s) {
    const dim3 block(32, 8);
    const int64_t gy = ceil_div(m, 8);
    if (gy > 65535) return fail(NM_ERR_UNSUPPORTED, "generic kernel: m too large");
    const dim3 grid(static_cast<unsigned>(ceil_div(n, 32)), static_cast<unsigned>(gy));
    prof_begin(s);
    spmm_generic_kernel<TA, TC><<<grid, block, 0, s>>>(static_cast<const TA*>(A), static_cast<const TA*>(Bv), D,
                                                       static_cast<TC*>(C), m, n, k, N, M, L);
    prof_end(s);
    note_launch();
    NM_LAUNCH_CHECK("spmm_generic_kernel");
    return NM_OK;
}

// ------------------------------------------------------------------ selector
// A^T staging for the SIMT kernel costs one read + one write of A (8*m*k bytes,
// measured ~2.9 TB/s) and saves ~15 % of the SpMM time (2 LDS.128 instead of 8 LDS.32
// per gathered fragment; r01 profiles).  Break-even: 0.15 * 2*m*n*w / 48 TF/s >
// 8*m*k / 2.9 TB/s  <=>  n*N/M > ~440.  NM_SIMT_AT=0/1 overrides (ablation).
static bool simt_use_at(int64_t m, int64_t n, int64_t k, int N, int M) {
    const char* e = getenv("NM_SIMT_AT");
    if (e && (e[0] == '0' || e[0] == '1')) return e[0] == '1';
    (void)k;
    return m % 4 == 0 && n * N >= 512 * static_cast<int64_t>(M);
}

// Packing (the paper's high-sparsity mode, Listing 3): fetch only the
// union of the columns the G = 128/L groups of a column tile select.  For masks that
// are independent across groups the expected union is 1 - (1 - N/M)^G of the panel
// (16:32 -> 0.94, 12:32 -> 0.85, 8:32 -> 0.68, 4:32 -> 0.41 at L = 32); packing pays
// when it removes at least a fifth of the A-panel bytes (the paper's fixed 70 %
// sparsity threshold, re-derived here from the traffic it saves).
// NM_SIMT_MODE=0/1/2 overrides (ablation).
static int simt_mode(int64_t m, int64_t n, int64_t k, int N, int M, int L) {
    const char* e = getenv("NM_SIMT_MODE");
    if (e && e[0] >= '0' && e[0] <= '2') {
        int mode = e[0] - '0';
        if (mode >= 1 && m % 4 != 0) mode = 0;
        return mode;
    }
    if (!simt_use_at(m, n, k, N, M)) return 0;
    const int G = (128 + L - 1) / L;
    const double keep = 1.0 - std::pow(1.0 - static_cast<double>(N) / M, G);
    // Measured on B200 (profiles/r01_summary.md): the per-row bulk copies of the packed
    // mode cost more than the L2->SM bytes they save -- L2 serves the re-streamed A^T
    // panels of the other column tiles -- so packing is off by default.
    (void)keep;
    return 1;
}

enum KernelId { K_GENERIC = 0, K_SIMT_F32 = 1, K_TC_BF16 = 2, K_TC_TF32 = 3, K_TC_SP = 4, K_SIMT_BF16 = 5 };

// bf16 operands the slot kernel cannot take (L not in {16, 32, 64, 128}, k % 8 != 0, e.g. cfg5's
// L = 4): the fp32 SIMT kernel on exact fp32 copies of A and B' (bf16 -> fp32 is exact, and so is
// every product), C rounded to bf16 (RNE) after the fp32 accumulation when c_dt is bf16 -- instead
// of the one-thread-per-element generic kernel.  NM_BF16_SIMT=0 disables (tests of the generic
// kernel).  The shape conditions are the SIMT kernel's on 16-B-aligned scratch copies.
static bool simt_bf16_ok(int64_t m, int64_t n, int64_t k, int N, int M, int L) {
    const char* e = getenv("NM_BF16_SIMT");
    if (e && e[0] == '0') return false;
    alignas(16) static const float dummy[4] = {0, 0, 0, 0};
    return simt_f32_applicable(dummy, dummy, dummy, m, n, k, N, M, L);
}

__global__ void widen_bf16_kernel(const __nv_bfloat16* __restrict__ in, float* __restrict__ out, int64_t count) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    const int64_t nv = count / 8;  // 8 elements (16 B in, 32 B out) per step; the scratch / caller
                                   // buffers are 16-B aligned (checked by the caller)
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < nv; i += stride) {
        const uint4 v = reinterpret_cast<const uint4*>(in)[i];
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
        float4 a, b;
        a.x = __uint_as_float(w[0] << 16), a.y = __uint_as_float(w[0] & 0xffff0000u);
        a.z = __uint_as_float(w[1] << 16), a.w = __uint_as_float(w[1] & 0xffff0000u);
        b.x = __uint_as_float(w[2] << 16), b.y = __uint_as_float(w[2] & 0xffff0000u);
        b.z = __uint_as_float(w[3] << 16), b.w = __uint_as_float(w[3] & 0xffff0000u);
        reinterpret_cast<float4*>(out)[2 * i] = a;
        reinterpret_cast<float4*>(out)[2 * i + 1] = b;
    }
    for (int64_t i = nv * 8 + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += stride)
        out[i] = __bfloat162float(in[i]);
}
__global__ void narrow_f32_kernel(const float* __restrict__ in, __nv_bfloat16* __restrict__ out, int64_t count) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += stride)
        out[i] = __float2bfloat16_rn(in[i]);
}

static nm_status simt_bf16_launch(const void* A, const void* Bv, const uint8_t* D, void* C, bool c_bf16, int64_t m,
                                  int64_t n, int64_t k, int N, int M, int L, int mode, float alpha, cudaStream_t s) {
    const int64_t w = k / M * N;
    if ((reinterpret_cast<uintptr_t>(A) & 15) || (reinterpret_cast<uintptr_t>(Bv) & 15))
        return fail(NM_ERR_ALIGNMENT, "bf16 SIMT path: A and values must be 16-B aligned");
    float *fa = nullptr, *fb = nullptr, *fc = nullptr;
    auto release = [&]() {
        if (fa) cudaFreeAsync(fa, s);
        if (fb) cudaFreeAsync(fb, s);
        if (fc) cudaFreeAsync(fc, s);
    };
    nm_status st = scratch_alloc(reinterpret_cast<void**>(&fa), static_cast<size_t>(m * k) * 4, s);
    if (!st) st = scratch_alloc(reinterpret_cast<void**>(&fb), static_cast<size_t>(w * n) * 4, s);
    if (!st && c_bf16) st = scratch_alloc(reinterpret_cast<void**>(&fc), static_cast<size_t>(m * n) * 4, s);
    if (st) {
        release();
        return st;
    }
    const unsigned blocks = static_cast<unsigned>(4 * num_sms());
    widen_bf16_kernel<<<blocks, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(A), fa, m * k);
    note_launch();
    widen_bf16_kernel<<<blocks, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(Bv), fb, w * n);
    note_launch();
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) st = cuda_fail(e, "widen_bf16_kernel");
    if (!st) st = simt_f32_launch(fa, fb, D, c_bf16 ? fc : static_cast<float*>(C), m, n, k, N, M, L, mode, s, nullptr, alpha);
    if (!st && c_bf16) {
        narrow_f32_kernel<<<blocks, 256, 0, s>>>(fc, static_cast<__nv_bfloat16*>(C), m * n);
        note_launch();
        if ((e = cudaGetLastError()) != cudaSuccess) st = cuda_fail(e, "narrow_f32_kernel");
    }
    release();
    return st;
}

static nm_status select(const void* A, const void* Bv, const void* C, int64_t m, int64_t n, int64_t k, int N, int M,
                        int L, nm_dtype ab, nm_dtype cd, nm_math math, int* kernel, nm_math* used) {
    if (ab == NM_F32) {
        if (cd != NM_F32) return fail(NM_ERR_UNSUPPORTED, "fp32 operands need an fp32 C");
        if (math == NM_MATH_AUTO || math == NM_MATH_F32_SIMT) {
            *used = NM_MATH_F32_SIMT;
            *kernel = simt_f32_applicable(A, Bv, C, m, n, k, N, M, L) ? K_SIMT_F32 : K_GENERIC;
            return NM_OK;
        }
        if (math == NM_MATH_TF32_TC) {
            // explicit opt-in only (tf32 rounds the operands; AUTO keeps the paper's fp32 semantics)
            if (!tc_sp_ok(A, C, m, n, k, N, M, L))
                return fail(NM_ERR_UNSUPPORTED, "tf32 sparse-tensor-core path needs L in {16,32,64,128}, k % 8 == 0, "
                                                "A 16-B and C 4-B aligned");
            *used = NM_MATH_TF32_TC;
            *kernel = K_TC_TF32;
            return NM_OK;
        }
        return fail(NM_ERR_UNSUPPORTED, "bf16 math requested on fp32 operands");
    }
    if (math == NM_MATH_AUTO || math == NM_MATH_BF16_TC) {
        *used = NM_MATH_BF16_TC;
        *kernel = tc_sp_ok(A, C, m, n, k, N, M, L) ? K_TC_SP : simt_bf16_ok(m, n, k, N, M, L) ? K_SIMT_BF16 : K_GENERIC;
        return NM_OK;
    }
    return fail(NM_ERR_UNSUPPORTED, "math mode not available for bf16 operands");
}

// C *= alpha (nm_spmm_scaled after a kernel without a fused alpha); grid-stride, 4 elements per
// iteration where aligned, rounding bf16 to nearest even as the fused epilogues do.
__global__ void scale_kernel(void* C, int c_bf16, int64_t count, float alpha) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += stride) {
        if (c_bf16) {
            __nv_bfloat16* c = static_cast<__nv_bfloat16*>(C) + i;
            *c = __float2bfloat16_rn(__bfloat162float(*c) * alpha);
        } else {
            static_cast<float*>(C)[i] *= alpha;
        }
    }
}

static nm_status scale_launch(void* C, bool c_bf16, int64_t count, float alpha, cudaStream_t s) {
    const int64_t blocks = std::min<int64_t>(ceil_div(count, 256), 8 * static_cast<int64_t>(num_sms()));
    scale_kernel<<<static_cast<unsigned>(blocks), 256, 0, s>>>(C, c_bf16 ? 1 : 0, count, alpha);
    note_launch();
    NM_LAUNCH_CHECK("scale_kernel");
    return NM_OK;
}

static nm_status check_common(int64_t m, int64_t n, int64_t k, int N, int M, int L) {
    if (N < 1 || M < N || M > 256 || L < 1)
        return fail(NM_ERR_INVALID_CONFIG, "invalid N:M/L: need 1 <= N <= M <= 256 and L >= 1");
    if (m < 0 || n < 0 || k < 0) return fail(NM_ERR_SHAPE, "negative dimension");
    if (k % M != 0) return fail(NM_ERR_SHAPE, "k must be a multiple of M (caller pads, P:94)");
    if (n % L != 0) return fail(NM_ERR_SHAPE, "n must be a multiple of L (caller pads, P:94)");
    return NM_OK;
}

}  // namespace nm

using namespace nm;

extern "C" {

const char* nm_version(void) { return "nmspmm 0.1 sm_100a"; }

const char* nm_last_error(void) { return g_last_error.c_str(); }

nm_status nm_check_config(int N, int M, int L) {
    if (N < 1 || M < N || M > 256 || L < 1)
        return fail(NM_ERR_INVALID_CONFIG, "invalid N:M/L: need 1 <= N <= M <= 256 and L >= 1");
    return NM_OK;
}

nm_status nm_compress(const void* B, nm_dtype b_dt, int64_t k, int64_t n, int N, int M, int L, void* values,
                      nm_dtype v_dt, uint8_t* idx, void* stream) {
    nm_status st = check_common(0, n, k, N, M, L);
    if (st) return st;
    if (b_dt > NM_BF16 || v_dt > NM_BF16) return fail(NM_ERR_UNSUPPORTED, "dtype");
    if (k * n > 0 && (!B || !values || !idx)) return fail(NM_ERR_NULL, "nm_compress: NULL pointer");
    if ((st = require_device())) return st;
    return compress_launch(B, b_dt, k, n, N, M, L, values, v_dt, idx, static_cast<cudaStream_t>(stream));
}

nm_status nm_decompress(const void* values, nm_dtype v_dt, const uint8_t* idx, int64_t k, int64_t n, int N, int M,
                        int L, void* B_out, void* stream) {
    nm_status st = check_common(0, n, k, N, M, L);
    if (st) return st;
    if (v_dt > NM_BF16) return fail(NM_ERR_UNSUPPORTED, "dtype");
    if (k * n > 0 && (!values || !idx || !B_out)) return fail(NM_ERR_NULL, "nm_decompress: NULL pointer");
    if ((st = require_device())) return st;
    return decompress_launch(values, v_dt, idx, k, n, N, M, L, B_out, static_cast<cudaStream_t>(stream));
}

nm_status nm_validate(const uint8_t* idx, int64_t k, int64_t n, int N, int M, int L, int64_t* first_bad_host,
                      void* stream) {
    nm_status st = check_common(0, n, k, N, M, L);
    if (st) return st;
    if (!first_bad_host || (k * n > 0 && !idx)) return fail(NM_ERR_NULL, "nm_validate: NULL pointer");
    if ((st = require_device())) return st;
    return validate_launch(idx, k, n, N, M, L, first_bad_host, static_cast<cudaStream_t>(stream));
}

nm_status nm_spmm_scaled(const void* A, const void* values, const uint8_t* idx, void* C, int64_t m, int64_t n,
                         int64_t k, int N, int M, int L, nm_dtype ab_dt, nm_dtype c_dt, nm_math math, float alpha,
                         void* stream) {
    nm_status st = check_common(m, n, k, N, M, L);
    if (st) return st;
    if (ab_dt > NM_BF16 || c_dt > NM_BF16 || math > NM_MATH_BF16_TC) return fail(NM_ERR_UNSUPPORTED, "dtype/math");
    if (m == 0 || n == 0) return NM_OK;
    if (!A || !C || (k > 0 && (!values || !idx))) return fail(NM_ERR_NULL, "nm_spmm: NULL pointer");
    if ((st = require_device())) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (k == 0) {
        NM_CUDA_TRY(cudaMemsetAsync(C, 0, static_cast<size_t>(m * n) * (c_dt == NM_BF16 ? 2 : 4), s));
        return NM_OK;
    }
    int kernel = K_GENERIC;
    nm_math used = NM_MATH_AUTO;
    if ((st = select(A, values, C, m, n, k, N, M, L, ab_dt, c_dt, math, &kernel, &used))) return st;
    // alpha is fused into the epilogues of the SIMT and sparse-tensor-core kernels; the
    // others are followed by one scaling pass over C when alpha != 1
    bool fused = false;
    if (kernel == K_SIMT_F32) {
        const int mode = simt_mode(m, n, k, N, M, L);
        st = simt_f32_launch(static_cast<const float*>(A), static_cast<const float*>(values), idx,
                             static_cast<float*>(C), m, n, k, N, M, L, mode, s, nullptr, alpha);
        fused = true;
    } else if (kernel == K_TC_SP || kernel == K_TC_TF32) {
        st = tc_sp_launch(A, values, idx, C, c_dt == NM_BF16, m, n, k, N, M, L, kernel == K_TC_TF32, s, alpha);
        fused = true;
    } else if (kernel == K_SIMT_BF16) {
        st = simt_bf16_launch(A, values, idx, C, c_dt == NM_BF16, m, n, k, N, M, L, simt_mode(m, n, k, N, M, L), alpha, s);
        fused = true;
    } else if (ab_dt == NM_F32) {
        st = generic_launch<float, float>(A, values, idx, C, m, n, k, N, M, L, s);
    } else if (c_dt == NM_BF16) {
        st = generic_launch<__nv_bfloat16, __nv_bfloat16>(A, values, idx, C, m, n, k, N, M, L, s);
    } else {
        st = generic_launch<__nv_bfloat16, float>(A, values, idx, C, m, n, k, N, M, L, s);
    }
    if (st || fused || alpha == 1.f) return st;
    return scale_launch(C, c_dt == NM_BF16, m * n, alpha, s);
}

nm_status nm_spmm(const void* A, const void* values, const uint8_t* idx, void* C, int64_t m, int64_t n, int64_t k,
                  int N, int M, int L, nm_dtype ab_dt, nm_dtype c_dt, nm_math math, void* stream) {
    return nm_spmm_scaled(A, values, idx, C, m, n, k, N, M, L, ab_dt, c_dt, math, 1.f, stream);
}

int64_t nm_spmm_host_ws_bytes(int64_t m, int64_t n, int64_t k, int N, int M, int L, nm_dtype ab_dt, nm_dtype c_dt) {
    if (N < 1 || M < N || L < 1 || k % M || n % L) return -1;
    const int64_t e = ab_dt == NM_BF16 ? 2 : 4, ec = c_dt == NM_BF16 ? 2 : 4;
    const int64_t w = k / M * N, q = n / L;
    auto al = [](int64_t b) { return (b + 255) / 256 * 256; };
    return al(m * k * e) + al(w * n * e) + al(w * q) + al(m * n * ec);
}

}  // extern "C"
namespace nm {
// Row chunks for the host path's copy/compute overlap (nch + 1 chunks sized 1 : 2 : .. : 2 : 1, see
// nm_spmm_host): nch = 4 once m >= 1024, 8 for the fp32 SIMT kernel once m >= 2048.  Measured on
// B200 (profiles/r01p_host_e2e_chunks.txt with equal chunks: 4 beat 2 and 3 at cfg2 and cfg4-65B
// even where a chunk's grid ends in a partial wave; profiles/r02l_host_e2e.txt with the 1:2:..:1
// sizes: cfg2 3.04 -> 2.88 ms (4) / 2.79 ms (8), cfg4-65B 6.0 -> 5.73 / 5.58 ms).  NM_HOST_CHUNKS=1..8
// overrides (ablation).
// kernel: the selector's choice; the slot kernels (bf16 / tf32 sparse TC) chunk too, with the
// weight prepacked once per call ahead of the chunks.
static int host_chunks(int64_t m, int kernel, nm_math math) {
    const char* e = getenv("NM_HOST_CHUNKS");
    int force = e ? atoi(e) : 0;
    if (force < 0 || force > 8) force = 0;
    const bool simt = kernel == K_SIMT_F32 && (math == NM_MATH_AUTO || math == NM_MATH_F32_SIMT);
    if (!simt && kernel != K_TC_SP && kernel != K_TC_TF32) return 1;
    if (force) return force;
    if (simt && m >= 2048) return 8;  // 1:2:..:2:1 sizing, fp32: 8 beats 4 by 3 % at cfg2 / cfg4-65B (r02l)
    return m >= 1024 ? 4 : 1;
}
}  // namespace nm
extern "C" {

nm_status nm_spmm_host(const void* A_host, const void* values_host, const uint8_t* idx_host, void* C_host, int64_t m,
                       int64_t n, int64_t k, int N, int M, int L, nm_dtype ab_dt, nm_dtype c_dt, nm_math math,
                       void* dev_ws, void* stream) {
    nm_status st = check_common(m, n, k, N, M, L);
    if (st) return st;
    if (m == 0 || n == 0) return NM_OK;
    if (!A_host || !C_host || !dev_ws || (k > 0 && (!values_host || !idx_host)))
        return fail(NM_ERR_NULL, "nm_spmm_host: NULL pointer");
    if ((st = require_device())) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int64_t e = ab_dt == NM_BF16 ? 2 : 4, ec = c_dt == NM_BF16 ? 2 : 4;
    const int64_t w = k / M * N, q = n / L;
    auto al = [](int64_t b) { return (b + 255) / 256 * 256; };
    uint8_t* base = static_cast<uint8_t*>(dev_ws);
    uint8_t* dA = base;
    uint8_t* dV = dA + al(m * k * e);
    uint8_t* dD = dV + al(w * n * e);
    uint8_t* dC = dD + al(w * q);
    NM_CUDA_TRY(cudaMemcpyAsync(dV, values_host, static_cast<size_t>(w * n * e), cudaMemcpyHostToDevice, s));
    NM_CUDA_TRY(cudaMemcpyAsync(dD, idx_host, static_cast<size_t>(w * q), cudaMemcpyHostToDevice, s));
    int kernel = K_GENERIC;
    nm_math used = NM_MATH_AUTO;
    if ((st = select(dA, dV, dC, m, n, k, N, M, L, ab_dt, c_dt, math, &kernel, &used))) return st;
    const int nch = k > 0 ? host_chunks(m, kernel, math) : 1;
    if (nch == 1) {
        NM_CUDA_TRY(cudaMemcpyAsync(dA, A_host, static_cast<size_t>(m * k * e), cudaMemcpyHostToDevice, s));
        if ((st = nm_spmm(dA, dV, dD, dC, m, n, k, N, M, L, ab_dt, c_dt, math, stream))) return st;
        NM_CUDA_TRY(cudaMemcpyAsync(C_host, dC, static_cast<size_t>(m * n * ec), cudaMemcpyDeviceToHost, s));
        NM_CUDA_TRY(cudaStreamSynchronize(s));
        return NM_OK;
    }
    // Row chunks of A / C, three-stage pipeline: H2D of chunk i+1 (copy stream) and D2H of chunk
    // i-1 (second copy stream) overlap the SpMM of chunk i (the caller's stream).  Every chunk
    // is the same product on a row range, so C is unchanged up to the k-split of sub-wave grids
    // (fixed order).  Chunk sizes 1 : 2 : ... : 2 : 1 (nch + 1 chunks, whole 128-row
    // tiles): the first chunk is on the critical path behind the weight upload and the last
    // chunk's D2H after the last SpMM, so both are half-size (CUPTI timeline at cfg2,
    // profiles/r02l_host_timeline.txt: equal chunks leave ~0.3 ms of D2H and the first chunk's
    // H2D exposed).
    const int nck = nch + 1;
    int64_t rb[10];
    rb[0] = 0;
    for (int i = 1; i < nck; ++i) rb[i] = std::min(m, ceil_div(m * (2 * i - 1), 2 * static_cast<int64_t>(nch) * 128) * 128);
    rb[nck] = m;
    int64_t rc = 0;  // the largest chunk (the slot kernels' H is chosen for it)
    for (int i = 0; i < nck; ++i) rc = std::max(rc, rb[i + 1] - rb[i]);
    // slot kernels: prepack the weight once (the paper's offline step, here per call) on s
    const bool slot = kernel == K_TC_SP || kernel == K_TC_TF32, tf = kernel == K_TC_TF32;
    const int hsp = tc_sp_halves_m(N, M, L, rc, n, k);  // the chunk's token count
    void* pbuf = nullptr;
    if (slot) {
        const size_t pb = tc_sp_prepack_bytes(n, k, N, M, L, tf);
        if ((st = scratch_alloc(&pbuf, pb, s))) return st;
        if ((st = tc_sp_prepack(dV, dD, n, k, N, M, L, tf, hsp, pbuf, static_cast<int64_t>(pb), nullptr, false, s))) {
            cudaFreeAsync(pbuf, s);
            return st;
        }
    }
    // Two compute streams (the caller's s and cs2) alternate over the chunks: a chunk's SpMM may
    // start while the previous one still runs, so the sub-wave grids of consecutive chunks share
    // the SMs instead of each leaving some idle (CUPTI timeline: the chunked SpMMs, not the copies,
    // are the critical path once the weights are up, profiles/r02l_host_timeline.txt).
    cudaStream_t hs = nullptr, ds = nullptr, cs2 = nullptr;
    cudaEvent_t ev[2 * 9 + 3] = {};
    auto cleanup = [&]() {
        for (cudaEvent_t x : ev)
            if (x) cudaEventDestroy(x);
        if (hs) cudaStreamDestroy(hs);
        if (ds) cudaStreamDestroy(ds);
        if (cs2) cudaStreamDestroy(cs2);
        if (pbuf) cudaFreeAsync(pbuf, s);
    };
    cudaError_t ce = cudaStreamCreateWithFlags(&hs, cudaStreamNonBlocking);
    if (ce == cudaSuccess) ce = cudaStreamCreateWithFlags(&ds, cudaStreamNonBlocking);
    if (ce == cudaSuccess) ce = cudaStreamCreateWithFlags(&cs2, cudaStreamNonBlocking);
    for (int i = 0; ce == cudaSuccess && i < 2 * nck + 3; ++i) ce = cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming);
    cudaEvent_t ev_w = ev[2 * nck + 1], ev_c2 = ev[2 * nck + 2];
    if (ce == cudaSuccess) ce = cudaEventRecord(ev_w, s);  // the weights (and the slot prepack) are ready
    if (ce == cudaSuccess) ce = cudaStreamWaitEvent(cs2, ev_w, 0);
    for (int i = 0; ce == cudaSuccess && i < nck; ++i) {
        const int64_t r0 = rb[i], r1 = rb[i + 1];
        if (r0 >= r1) continue;
        cudaStream_t cs = (i & 1) ? cs2 : s;
        ce = cudaMemcpyAsync(dA + r0 * k * e, static_cast<const uint8_t*>(A_host) + r0 * k * e,
                             static_cast<size_t>((r1 - r0) * k * e), cudaMemcpyHostToDevice, hs);
        if (ce == cudaSuccess) ce = cudaEventRecord(ev[2 * i], hs);
        if (ce == cudaSuccess) ce = cudaStreamWaitEvent(cs, ev[2 * i], 0);
        if (ce != cudaSuccess) break;
        st = slot ? tc_sp_run(dA + r0 * k * e, pbuf, hsp, dC + r0 * n * ec, c_dt == NM_BF16, r1 - r0, n, k, N, M, L, tf, cs)
                  : nm_spmm(dA + r0 * k * e, dV, dD, dC + r0 * n * ec, r1 - r0, n, k, N, M, L, ab_dt, c_dt, math, cs);
        if (st) {
            cudaStreamSynchronize(s);
            cudaStreamSynchronize(cs2);
            cudaStreamSynchronize(hs);
            cleanup();
            return st;
        }
        ce = cudaEventRecord(ev[2 * i + 1], cs);
        if (ce == cudaSuccess) ce = cudaStreamWaitEvent(ds, ev[2 * i + 1], 0);
        if (ce == cudaSuccess)
            ce = cudaMemcpyAsync(static_cast<uint8_t*>(C_host) + r0 * n * ec, dC + r0 * n * ec,
                                 static_cast<size_t>((r1 - r0) * n * ec), cudaMemcpyDeviceToHost, ds);
    }
    if (ce == cudaSuccess) ce = cudaEventRecord(ev_c2, cs2);
    if (ce == cudaSuccess) ce = cudaStreamWaitEvent(s, ev_c2, 0);  // before pbuf is released on s
    if (ce == cudaSuccess) ce = cudaEventRecord(ev[2 * nck], ds);
    if (ce == cudaSuccess) ce = cudaStreamWaitEvent(s, ev[2 * nck], 0);  // the caller's stream sees C_host
    const cudaError_t se = cudaStreamSynchronize(s);
    cudaStreamSynchronize(cs2);
    cudaStreamSynchronize(hs);
    cudaStreamSynchronize(ds);
    cleanup();
    if (ce != cudaSuccess) return cuda_fail(ce, "nm_spmm_host pipeline");
    if (se != cudaSuccess) return cuda_fail(se, "nm_spmm_host");
    return NM_OK;
}

nm_status nm_plan_query(int64_t m, int64_t n, int64_t k, int N, int M, int L, nm_dtype ab_dt, nm_math math,
                        double peak_flops, double peak_hbm, nm_plan* out) {
    nm_status st = check_common(m, n, k, N, M, L);
    if (st) return st;
    if (!out) return fail(NM_ERR_NULL, "nm_plan_query: NULL out");
    *out = nm_plan{};
    const int64_t w = k / M * N, q = n / L;
    const double e = ab_dt == NM_BF16 ? 2.0 : 4.0;
    out->flops = 2.0 * double(m) * double(n) * double(w);
    out->bytes = e * double(m) * double(k) + e * double(w) * double(n) + double(w) * double(q) + e * double(m) * double(n);
    int kernel = K_GENERIC;
    nm_math used = NM_MATH_AUTO;
    alignas(16) static const float dummy[4] = {0, 0, 0, 0};  // 16-B aligned stand-in pointers for the alignment test
    if ((st = select(dummy, dummy, dummy, m, n, k, N, M, L, ab_dt, ab_dt, math, &kernel, &used))) return st;
    out->math = used;
    out->kernel = kernel;
    const int sms = num_sms();
    if (kernel == K_SIMT_F32 || kernel == K_SIMT_BF16) {
        int wp, bk, bkw;
        simt_f32_geometry(N, M, &wp, &bk, &bkw);
        const int bm = simt_row_tile(m, n, w);
        out->bm = bm;
        out->bn = 128;
        out->bk = bk;
        out->bkw = bkw;
        out->stages = 2;
        out->threads = 2 * bm;
        const int64_t tiles = ceil_div(m, bm) * ceil_div(n, 128);
        const int npanels = static_cast<int>(ceil_div(k / M, wp));
        const int sp = simt_split_factor(static_cast<int>(tiles), w, npanels, bm);
        const int64_t resident = (bm == 128 ? 2 : 3) * static_cast<int64_t>(sms);
        out->split = sp;
        out->split_tiles = sp > 1 ? static_cast<int32_t>(tiles % resident) : 0;
        out->grid = static_cast<int32_t>(tiles - out->split_tiles + out->split_tiles * static_cast<int64_t>(sp));
        out->waves = double(out->grid) / double(resident);
        out->smem_bytes = 2 * (bm * 64 * 4 + 32 * 128 * 4) + 2 * 32 * 33 * 4 + 64 + 1024;
    } else if (kernel == K_TC_SP || kernel == K_TC_TF32) {
        // tokens x output columns per CTA (MMA N x M per column half), 64 (bf16) / 32 (tf32) slots
        // per stage, the same bytes per stage
        int hh = 1, nt = 256;
        tc_sp_geometry(m, n, k, N, M, L, &hh, &nt);
        out->bm = nt;
        out->bn = 128 * hh;
        out->bk = kernel == K_TC_SP ? 64 : 32;
        out->bkw = out->bk / 2;
        out->threads = 288;
        out->grid = static_cast<int32_t>(ceil_div(m, out->bm) * ceil_div(n, out->bn));
        {
            const int per = 64 * ((nt + 63) / 64) * 128 + hh * (128 * 64 + 128 * 16);
            const int st = std::min(8, (232448 - 1280) / per);
            out->stages = st;
            out->smem_bytes = st * per + 1280;
        }
    } else {
        out->bm = 8;
        out->bn = 32;
        out->threads = 256;
        out->grid = static_cast<int32_t>(ceil_div(m, 8) * ceil_div(n, 32));
    }
    // nominal peaks when none are given: FP32 FFMA = SMs * 128 lanes * 2 * 1.965 GHz; bf16 TC 2.25 PF, tf32 half
    // of it; HBM 7.7 TB/s
    if (peak_flops <= 0)
        peak_flops = used == NM_MATH_F32_SIMT ? double(sms) * 128 * 2 * 1.965e9 : used == NM_MATH_TF32_TC ? 1.125e15 : 2.25e15;
    if (peak_hbm <= 0) peak_hbm = 7.7e12;
    out->t_compute_us = out->flops / peak_flops * 1e6;
    out->t_memory_us = out->bytes / peak_hbm * 1e6;
    out->bound = out->t_memory_us > out->t_compute_us ? 1 : 0;
    return NM_OK;
}

// ------------------------------------------------------------------ prepack
}  // extern "C"
namespace nm {
static const int32_t kPrepackMagic = 0x4B504D4E;

// kind 3 iff the tf32 slot kernel is asked for and applies (aligned operands assumed)
static bool prepack_kind3(int64_t n, int64_t k, int N, int M, int L, nm_dtype dt, nm_math math) {
    static const float dummy[4] = {0, 0, 0, 0};
    return dt == NM_F32 && math == NM_MATH_TF32_TC && k > 0 && tc_sp_ok(dummy, dummy, 1, n, k, N, M, L);
}
// kind 2 iff the sparse-tensor-core slot kernel would run (aligned operands assumed)
static bool prepack_kind2(int64_t n, int64_t k, int N, int M, int L, nm_dtype dt) {
    static const float dummy[4] = {0, 0, 0, 0};
    return dt == NM_BF16 && k > 0 && tc_sp_ok(dummy, dummy, 1, n, k, N, M, L);
}
// kind 4 iff the fp32 SIMT kernel runs the weight and its tiles hold whole groups (128 % L == 0):
// the bit-packed tile-major index words replace D on the hot path
static bool prepack_kind4(int64_t n, int64_t k, int N, int M, int L, nm_dtype dt, nm_math math) {
    static const float dummy[4] = {0, 0, 0, 0};
    return dt == NM_F32 && (math == NM_MATH_AUTO || math == NM_MATH_F32_SIMT) && k > 0 && 128 % L == 0 &&
           simt_f32_applicable(dummy, dummy, dummy, 1, n, k, N, M, L);
}
// 2 / 3 = slot images (bf16 / tf32), 4 = packed indices (fp32 SIMT), 0 = none (values / idx directly)
static int prepack_kind(int64_t n, int64_t k, int N, int M, int L, nm_dtype dt, nm_math math) {
    if (prepack_kind3(n, k, N, M, L, dt, math)) return 3;
    if (prepack_kind2(n, k, N, M, L, dt)) return 2;
    if (prepack_kind4(n, k, N, M, L, dt, math)) return 4;
    return 0;
}
}  // namespace nm
extern "C" {

int64_t nm_prepack_bytes_ex(int64_t n, int64_t k, int N, int M, int L, nm_dtype dt, nm_math math) {
    if (check_common(0, n, k, N, M, L) != NM_OK || dt > NM_BF16 || math > NM_MATH_BF16_TC) return -1;
    const int kind = prepack_kind(n, k, N, M, L, dt, math);
    if (kind == 4) return 4 * index_packed_words(k, n, N, M, L);
    return kind ? static_cast<int64_t>(tc_sp_prepack_bytes(n, k, N, M, L, kind == 3)) : 0;
}

int64_t nm_prepack_bytes(int64_t n, int64_t k, int N, int M, int L, nm_dtype dt) {
    return nm_prepack_bytes_ex(n, k, N, M, L, dt, NM_MATH_AUTO);
}

// H of a slot prepack: without a token count the sparsity rule (tc_sp_halves); with the expected m
// (nm_prepack_m) also the small-grid rule of the per-call path (tc_sp_halves_m: H = 1 when H = 2
// would leave the grid under two waves; the A-F study)
static int prepack_halves(int64_t m_hint, int64_t n, int64_t k, int N, int M, int L) {
    return m_hint > 0 ? tc_sp_halves_m(N, M, L, m_hint, n, k) : tc_sp_halves(N, M, L);
}

nm_status nm_prepack_size(const void* values, const uint8_t* idx, int64_t n, int64_t k, int N, int M, int L, nm_dtype dt,
                          nm_math math, int64_t* bytes, void* stream) {
    return nm_prepack_size_m(values, idx, n, k, N, M, L, dt, math, 0, bytes, stream);
}

nm_status nm_prepack_size_m(const void* values, const uint8_t* idx, int64_t n, int64_t k, int N, int M, int L,
                            nm_dtype dt, nm_math math, int64_t m_hint, int64_t* bytes, void* stream) {
    nm_status st = check_common(0, n, k, N, M, L);
    if (st) return st;
    if (!bytes || (n * k > 0 && (!values || !idx))) return fail(NM_ERR_NULL, "nm_prepack_size: NULL pointer");
    if (dt > NM_BF16 || math > NM_MATH_BF16_TC) return fail(NM_ERR_UNSUPPORTED, "dtype/math");
    const int kind = prepack_kind(n, k, N, M, L, dt, math);
    *bytes = 0;
    if (kind == 4) *bytes = 4 * index_packed_words(k, n, N, M, L);
    if (kind == 0 || kind == 4) return NM_OK;
    if ((st = require_device())) return st;
    return tc_sp_prepack(values, idx, n, k, N, M, L, kind == 3, prepack_halves(m_hint, n, k, N, M, L), nullptr, 0, bytes,
                         true, static_cast<cudaStream_t>(stream));
}

nm_status nm_prepack_ex(const void* values, const uint8_t* idx, int64_t n, int64_t k, int N, int M, int L, nm_dtype dt,
                        nm_math math, void* buf, int64_t buf_bytes, nm_prepacked* out, void* stream) {
    return nm_prepack_m(values, idx, n, k, N, M, L, dt, math, 0, buf, buf_bytes, out, stream);
}

nm_status nm_prepack_m(const void* values, const uint8_t* idx, int64_t n, int64_t k, int N, int M, int L, nm_dtype dt,
                       nm_math math, int64_t m_hint, void* buf, int64_t buf_bytes, nm_prepacked* out, void* stream) {
    nm_status st = check_common(0, n, k, N, M, L);
    if (st) return st;
    if (!out || (n * k > 0 && (!values || !idx))) return fail(NM_ERR_NULL, "nm_prepack: NULL pointer");
    if (dt > NM_BF16 || math > NM_MATH_BF16_TC) return fail(NM_ERR_UNSUPPORTED, "dtype/math");
    *out = nm_prepacked{};
    out->dtype = dt;
    out->N = N;
    out->M = M;
    out->L = L;
    out->n = n;
    out->k = k;
    out->values = values;
    out->idx = idx;
    const int kind = prepack_kind(n, k, N, M, L, dt, math);
    if (kind == 4) {
        const int64_t need = 4 * index_packed_words(k, n, N, M, L);
        if (!buf || buf_bytes < need) return fail(NM_ERR_NULL, "nm_prepack: buffer missing or below nm_prepack_size");
        if ((st = require_device())) return st;
        if ((st = index_pack_launch(idx, static_cast<uint32_t*>(buf), k, n, N, M, L, false,
                                    static_cast<cudaStream_t>(stream))))
            return st;
        out->kind = 4;
        out->tbl = buf;  // the packed index words
    } else if (kind) {
        if (!buf) return fail(NM_ERR_NULL, "nm_prepack: buffer missing (size: nm_prepack_size)");
        if ((st = require_device())) return st;
        const int H = prepack_halves(m_hint, n, k, N, M, L);
        // exact size check when the buffer is below the data-independent bound (synchronizes)
        const bool check = buf_bytes < static_cast<int64_t>(tc_sp_prepack_bytes(n, k, N, M, L, kind == 3));
        int64_t need = 0;
        st = tc_sp_prepack(values, idx, n, k, N, M, L, kind == 3, H, buf, buf_bytes, check ? &need : nullptr, false,
                           static_cast<cudaStream_t>(stream));
        if (st) return st;
        out->kind = kind;
        out->bperm = buf;
        out->bn = 128 * H;                                                    // output columns per tile
        out->npanels = static_cast<int32_t>((n + 128 * H - 1) / (128 * H));  // column tiles
    }
    out->magic = kPrepackMagic;
    return NM_OK;
}

nm_status nm_prepack(const void* values, const uint8_t* idx, int64_t n, int64_t k, int N, int M, int L, nm_dtype dt,
                     void* buf, int64_t buf_bytes, nm_prepacked* out, void* stream) {
    return nm_prepack_ex(values, idx, n, k, N, M, L, dt, NM_MATH_AUTO, buf, buf_bytes, out, stream);
}

nm_status nm_spmm_prepacked(const void* A, const nm_prepacked* w, void* C, int64_t m, nm_dtype c_dt, void* stream) {
    if (!w || w->magic != kPrepackMagic) return fail(NM_ERR_NULL, "nm_spmm_prepacked: descriptor not filled by nm_prepack");
    if (w->kind == 2 || w->kind == 3) {
        const bool tf = w->kind == 3;
        nm_status st = check_common(m, w->n, w->k, w->N, w->M, w->L);
        if (st) return st;
        if (tf && c_dt != NM_F32) return fail(NM_ERR_UNSUPPORTED, "fp32 operands need an fp32 C");
        if (m == 0 || w->n == 0) return NM_OK;
        if (!A || !C) return fail(NM_ERR_NULL, "nm_spmm_prepacked: NULL pointer");
        if ((st = require_device())) return st;
        if (tc_sp_ok(A, C, m, w->n, w->k, w->N, w->M, w->L))
            return tc_sp_run(A, w->bperm, w->bn / 128, C, c_dt == NM_BF16, m, w->n, w->k, w->N, w->M, w->L, tf,
                             static_cast<cudaStream_t>(stream));
        if (tf) return fail(NM_ERR_UNSUPPORTED, "tf32 sparse-tensor-core path needs A 16-B and C 4-B aligned");
    }
    if (w->kind == 4) {  // fp32 SIMT kernel on the bit-packed tile-major indices
        nm_status st = check_common(m, w->n, w->k, w->N, w->M, w->L);
        if (st) return st;
        if (c_dt != NM_F32) return fail(NM_ERR_UNSUPPORTED, "fp32 operands need an fp32 C");
        if (m == 0 || w->n == 0) return NM_OK;
        if (!A || !C) return fail(NM_ERR_NULL, "nm_spmm_prepacked: NULL pointer");
        if ((st = require_device())) return st;
        const int mode = simt_mode(m, w->n, w->k, w->N, w->M, w->L);
        if (mode != 3 && simt_f32_applicable(A, w->values, C, m, w->n, w->k, w->N, w->M, w->L))
            return simt_f32_launch(static_cast<const float*>(A), static_cast<const float*>(w->values), w->idx,
                                   static_cast<float*>(C), m, w->n, w->k, w->N, w->M, w->L, mode,
                                   static_cast<cudaStream_t>(stream), nullptr, 1.f,
                                   static_cast<const uint32_t*>(w->tbl));
    }
    return nm_spmm(A, w->values, w->idx, C, m, w->n, w->k, w->N, w->M, w->L, static_cast<nm_dtype>(w->dtype), c_dt,
                   NM_MATH_AUTO, stream);
}

static nm_status at_check(const void* At, int64_t lda, int64_t m, int64_t e) {
    if (lda < m) return fail(NM_ERR_SHAPE, "nm_spmm_at: lda < m");
    if ((reinterpret_cast<uintptr_t>(At) & 15) || (lda * e) % 16)
        return fail(NM_ERR_ALIGNMENT, "nm_spmm_at: At must be 16-B aligned with lda * element size % 16 == 0");
    return NM_OK;
}

nm_status nm_spmm_at(const void* At, int64_t lda, const void* values, const uint8_t* idx, void* C, int64_t m, int64_t n,
                     int64_t k, int N, int M, int L, nm_dtype ab_dt, nm_dtype c_dt, nm_math math, void* stream) {
    nm_status st = check_common(m, n, k, N, M, L);
    if (st) return st;
    if (ab_dt > NM_BF16 || c_dt > NM_BF16 || math > NM_MATH_BF16_TC) return fail(NM_ERR_UNSUPPORTED, "dtype/math");
    if (m == 0 || n == 0) return NM_OK;
    if (!At || !C || (k > 0 && (!values || !idx))) return fail(NM_ERR_NULL, "nm_spmm_at: NULL pointer");
    if ((st = at_check(At, lda, m, ab_dt == NM_BF16 ? 2 : 4))) return st;
    if ((st = require_device())) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (k == 0) {
        NM_CUDA_TRY(cudaMemsetAsync(C, 0, static_cast<size_t>(m * n) * (c_dt == NM_BF16 ? 2 : 4), s));
        return NM_OK;
    }
    int kernel = K_GENERIC;
    nm_math used = NM_MATH_AUTO;
    if ((st = select(At, values, C, m, n, k, N, M, L, ab_dt, c_dt, math, &kernel, &used))) return st;
    if (kernel == K_SIMT_F32)
        return simt_f32_launch(nullptr, static_cast<const float*>(values), idx, static_cast<float*>(C), m, n, k, N, M, L,
                               1, s, nullptr, 1.f, nullptr, static_cast<const float*>(At), lda);
    if (kernel == K_TC_SP || kernel == K_TC_TF32)
        return tc_sp_launch(nullptr, values, idx, C, c_dt == NM_BF16, m, n, k, N, M, L, kernel == K_TC_TF32, s, 1.f, At,
                            lda);
    return fail(NM_ERR_UNSUPPORTED, "nm_spmm_at: this shape selects a kernel without an A^T input (generic / bf16 SIMT)");
}

nm_status nm_spmm_prepacked_at(const void* At, int64_t lda, const nm_prepacked* w, void* C, int64_t m, nm_dtype c_dt,
                               void* stream) {
    if (!w || w->magic != kPrepackMagic) return fail(NM_ERR_NULL, "nm_spmm_prepacked_at: descriptor not filled by nm_prepack");
    if (w->kind != 2 && w->kind != 3 && w->kind != 4)
        return nm_spmm_at(At, lda, w->values, w->idx, C, m, w->n, w->k, w->N, w->M, w->L, static_cast<nm_dtype>(w->dtype),
                          c_dt, NM_MATH_AUTO, stream);
    nm_status st = check_common(m, w->n, w->k, w->N, w->M, w->L);
    if (st) return st;
    const bool tf = w->kind == 3, simt = w->kind == 4;
    if ((tf || simt) && c_dt != NM_F32) return fail(NM_ERR_UNSUPPORTED, "fp32 operands need an fp32 C");
    if (m == 0 || w->n == 0) return NM_OK;
    if (!At || !C) return fail(NM_ERR_NULL, "nm_spmm_prepacked_at: NULL pointer");
    if ((st = at_check(At, lda, m, w->kind == 2 ? 2 : 4))) return st;
    if ((st = require_device())) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (simt) {
        if (!simt_f32_applicable(At, w->values, C, m, w->n, w->k, w->N, w->M, w->L))
            return fail(NM_ERR_UNSUPPORTED, "nm_spmm_prepacked_at: the SIMT kernel's shape / alignment rules");
        return simt_f32_launch(nullptr, static_cast<const float*>(w->values), w->idx, static_cast<float*>(C), m, w->n,
                               w->k, w->N, w->M, w->L, 1, s, nullptr, 1.f, static_cast<const uint32_t*>(w->tbl),
                               static_cast<const float*>(At), lda);
    }
    if (!tc_sp_ok(At, C, m, w->n, w->k, w->N, w->M, w->L))
        return fail(NM_ERR_UNSUPPORTED, "nm_spmm_prepacked_at: slot kernel needs C 4-B aligned, k % 8 == 0");
    return tc_sp_run(nullptr, w->bperm, w->bn / 128, C, c_dt == NM_BF16, m, w->n, w->k, w->N, w->M, w->L, tf, s, nullptr,
                     1.f, At, lda);
}

nm_status nm_profile_begin(void) {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    g_prof.on = true;
    g_prof.launches = 0;
    g_prof.used = 0;
    return NM_OK;
}

nm_status nm_profile_end(double* kernel_ms, int64_t* kernel_count, int64_t* launches) {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    g_prof.on = false;
    double tot = 0.0;
    int64_t cnt = 0;
    for (size_t i = 0; i + 1 < g_prof.used; i += 2) {
        cudaError_t e = cudaEventSynchronize(g_prof.ev[i + 1]);
        if (e != cudaSuccess) return cuda_fail(e, "nm_profile_end");
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, g_prof.ev[i], g_prof.ev[i + 1]) == cudaSuccess) {
            tot += ms;
            ++cnt;
        }
    }
    if (kernel_ms) *kernel_ms = tot;
    if (kernel_count) *kernel_count = cnt;
    if (launches) *launches = g_prof.launches;
    return NM_OK;
}

int64_t nm_index_packed_words(int64_t k, int64_t n, int N, int M, int L) {
    if (check_common(0, n, k, N, M, L) != NM_OK) return -1;
    return index_packed_words(k, n, N, M, L);
}

nm_status nm_index_pack(const uint8_t* idx, int64_t k, int64_t n, int N, int M, int L, uint32_t* words, void* stream) {
    nm_status st = check_common(0, n, k, N, M, L);
    if (st) return st;
    if (128 % L) return fail(NM_ERR_UNSUPPORTED, "nm_index_pack: tiles of 128 columns need 128 % L == 0");
    if (k * n > 0 && (!idx || !words)) return fail(NM_ERR_NULL, "nm_index_pack: NULL pointer");
    if ((st = require_device())) return st;
    return index_pack_launch(idx, words, k, n, N, M, L, false, static_cast<cudaStream_t>(stream));
}

nm_status nm_index_unpack(const uint32_t* words, int64_t k, int64_t n, int N, int M, int L, uint8_t* idx, void* stream) {
    nm_status st = check_common(0, n, k, N, M, L);
    if (st) return st;
    if (128 % L) return fail(NM_ERR_UNSUPPORTED, "nm_index_unpack: tiles of 128 columns need 128 % L == 0");
    if (k * n > 0 && (!idx || !words)) return fail(NM_ERR_NULL, "nm_index_unpack: NULL pointer");
    if ((st = require_device())) return st;
    return index_pack_launch(idx, const_cast<uint32_t*>(words), k, n, N, M, L, true, static_cast<cudaStream_t>(stream));
}

nm_status nm_unshard_columns(const void* src, void* dst, int64_t G, int64_t m, int64_t nr, int64_t n, int L,
                             int elem_bytes, void* stream) {
    if (G < 1 || m < 0 || nr < 0 || n < 0 || L < 1 || n % L) return fail(NM_ERR_SHAPE, "nm_unshard_columns: shape");
    if (elem_bytes != 2 && elem_bytes != 4) return fail(NM_ERR_UNSUPPORTED, "elem_bytes must be 2 or 4");
    const int64_t q = n / L;
    if (L * ceil_div(q, G) > nr) return fail(NM_ERR_SHAPE, "nm_unshard_columns: nr < L*ceil(q/G)");
    if (m * n > 0 && (!src || !dst)) return fail(NM_ERR_NULL, "nm_unshard_columns: NULL pointer");
    nm_status st = require_device();
    if (st) return st;
    return unshard_launch(src, dst, G, m, nr, q, L, elem_bytes, static_cast<cudaStream_t>(stream));
}

}  // extern "C"
