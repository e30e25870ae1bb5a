// Probe of tcgen05.mma.sp kind::tf32 (1:2-sparse A, fp32 accumulate) semantics on sm_100a:
// compressed-A smem layout (K-major, 128-B swizzle), metadata TMEM layout and nibble encoding,
// metadata delivery (tcgen05.st vs tcgen05.cp), and TMA tile::gather4 for the B operand (MN-major).
// M = 128 rows, K = 128 logical (4 MMAs of K = 32), N tokens.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o ubench_sp ubench_sp.cu
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <random>
#include <vector>

#define CK(x)                                                                       \
    do {                                                                            \
        cudaError_t e = (x);                                                        \
        if (e != cudaSuccess) {                                                     \
            printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
            exit(1);                                                                \
        }                                                                           \
    } while (0)

constexpr int M = 128, K = 64, KP = K / 2;  // tf32: 4 MMAs of K = 16 logical (8 physical)

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
    uint32_t ok = 0;
    long long spins = 0;
    while (!ok) {
        if (++spins > (1ll << 26)) __trap();
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}"
                     : "=r"(ok)
                     : "r"(su32(b)), "r"(ph)
                     : "memory");
    }
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(dst)),
                 "l"(src), "r"(bytes), "r"(su32(bar))
                 : "memory");
}
__device__ __forceinline__ void gather4(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int r0, int r1, int r2,
                                        int r3) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(su32(dst)),
        "l"(map), "r"(su32(bar)), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3)
        : "memory");
}
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
    d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
    d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
    d |= static_cast<uint64_t>(1) << 46;
    d |= static_cast<uint64_t>(layout & 7) << 61;
    return d;
}

struct Args {
    const uint8_t* aimg;   // M x KP bf16, K-major SW128 image (16 KB)
    const uint8_t* bimg;   // K x N bf16 MN-major SW128 image
    const uint32_t* meta;  // [4 mma][128 lanes]
    float* D;              // M x N
    int N;
    int mode;  // 1: metadata via tcgen05.cp; 2: B via gather4 (rows perm[k])
    const int* perm;
};

__global__ void __launch_bounds__(128, 1) sp_kernel(const __grid_constant__ CUtensorMap tm, Args a) {
    extern __shared__ __align__(1024) uint8_t sm_raw[];
    uint8_t* sm = sm_raw + ((1024u - (su32(sm_raw) & 1023u)) & 1023u);
    uint8_t* sA = sm;                    // 16 KB
    uint8_t* sE = sm + 16384;            // 2 KB
    uint8_t* sB = sm + 16384 + 2048;     // K * N * 4
    __shared__ __align__(8) uint64_t bar[2];
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int N = a.N;
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&slot)) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = slot;
    const uint32_t tE = tmem + 256;
    if (threadIdx.x == 0) {
        const uint32_t bbytes = K * N * 4;
        mbar_expect(&bar[0], 16384 + 2048 + bbytes);
        bulk(sA, a.aimg, 16384, &bar[0]);
        bulk(sE, a.meta, 2048, &bar[0]);  // only used in cp mode (layout: lane-major 16 B rows, see host)
        if (a.mode & 2) {
            for (int at = 0; at < N / 64; ++at)
                for (int r = 0; r < K; r += 4)
                    gather4(sB + at * (K * 128) + r * 128, &tm, &bar[0], at * 64, a.perm[r], a.perm[r + 1], a.perm[r + 2],
                            a.perm[r + 3]);
        } else {
            bulk(sB, a.bimg, bbytes, &bar[0]);
        }
    }
    mbar_wait(&bar[0], 0);
    if (!(a.mode & 1)) {
        // metadata via tcgen05.st: global meta is [mma j][lane]
        const uint32_t l = warp * 32 + lane;
        uint32_t v0 = a.meta[0 * 128 + l], v1 = a.meta[1 * 128 + l], v2 = a.meta[2 * 128 + l], v3 = a.meta[3 * 128 + l];
        asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(tE + ((warp * 32) << 16)), "r"(v0),
                     "r"(v1), "r"(v2), "r"(v3));
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (threadIdx.x == 0) {
        if (a.mode & 1) {
            // smem sE: 128 rows (lanes) x 16 B; K-major no-swizzle: core matrix 8 rows x 16 B, SBO = 128
            const uint64_t ed = sdesc(su32(sE), 2048, 128, 0);
            asm volatile("tcgen05.cp.cta_group::1.128x128b [%0], %1;" ::"r"(tE), "l"(ed) : "memory");
        }
        const uint32_t sp = (a.mode & 4) ? 0u : (1u << 2);
        const uint32_t idesc = sp | (1u << 4) | (2u << 7) | (2u << 10) | (1u << 16) |
                               (static_cast<uint32_t>(N >> 3) << 17) | (static_cast<uint32_t>(M >> 4) << 24);
        for (int j = 0; j < 4; ++j) {
            const uint64_t ad = sdesc(su32(sA) + 32 * j, 16, 1024, 2);
            const uint64_t bd = sdesc(su32(sB) + 2048 * j, K * 128, 512, 1);
            const uint32_t acc = j ? 1u : 0u;
            if (a.mode & 4) {
                // dense: A = first 8 physical columns (32 B) of each row = logical K 0..7 only; B rows 0..7
                asm volatile(
                    "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                    "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                    "l"(sdesc(su32(sA), 16, 1024, 2)), "l"(sdesc(su32(sB), K * 128, 512, 1)), "r"(idesc), "r"(0u)
                    : "memory");
                break;
            }
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.sp.cta_group::1.kind::tf32 [%0], %1, %2, [%5], %3, p;\n\t}" ::"r"(tmem),
                "l"(ad), "l"(bd), "r"(idesc | static_cast<uint32_t>(j & 1)), "r"(acc), "r"(tE + (j & ~1))
                : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar[1]))
                     : "memory");
    }
    __syncwarp();
    mbar_wait(&bar[1], 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int row = warp * 32 + lane;
    for (int c = 0; c < N; c += 8) {
        uint32_t v[8];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                     : "r"(tmem + ((warp * 32) << 16) + c));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        for (int i = 0; i < 8; ++i) a.D[row * N + c + i] = __uint_as_float(v[i]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
}

static uint16_t f2bf(float f) {
    uint32_t u;
    memcpy(&u, &f, 4);
    return static_cast<uint16_t>(u >> 16);  // exact for small integers
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// metadata position of (row m, chunk c of MMA j): lane, bit (hypothesis from the CUTLASS TMEM atom)
static void meta_pos(int m, int c, int* lane, int* bit) {
    const int k1 = c / 4;
    *lane = (m % 8) + 8 * k1 + 16 * (m / 16);
    *bit = 16 * ((m / 8) % 2) + 4 * (c % 4);
}

int run(int N, int mode, int probe, int box_rows, unsigned seed) {
    std::mt19937 rng(seed);
    std::vector<float> W(M * K, 0.f), X(K * N);
    std::vector<uint32_t> cval(M * KP, 0);
    std::vector<uint32_t> meta(4 * 128, 0);
    for (int m = 0; m < M; ++m)
        for (int ch = 0; ch < K / 2; ++ch) {  // chunk = pair of logical elements, one kept
            const int i0 = rng() % 2;
            float v0 = static_cast<float>(static_cast<int>(rng() % 7) - 3);
            if (probe) v0 = (m % KP == ch) ? 1.f : 0.f;
            W[m * K + ch * 2 + i0] = v0;
            memcpy(&cval[m * KP + ch], &v0, 4);
            const int j = ch / 8, c = ch % 8;
            int ln, bt;
            meta_pos(m, c, &ln, &bt);
            meta[j * 128 + ln] |= static_cast<uint32_t>(i0 ? 0xEu : 0x4u) << bt;
        }
    for (int k = 0; k < K; ++k)
        for (int t = 0; t < N; ++t) X[k * N + t] = probe ? (t == 0 ? static_cast<float>(k + 1) : 1.f) : static_cast<float>(static_cast<int>(rng() % 5) - 2);
    std::vector<int> perm(K);
    for (int k = 0; k < K; ++k) perm[k] = k;
    if (mode & 2) std::shuffle(perm.begin(), perm.end(), rng);
    // B operand row k = X row perm[k]; X stored in global as Xg[K][N] (bf16) for the gather
    std::vector<float> Xg(K * N);
    for (int k = 0; k < K; ++k)
        for (int t = 0; t < N; ++t) Xg[k * N + t] = X[k * N + t];
    // A image: K-major SW128: row m at (m/8)*1024 + (m%8)*128, 16-B chunk ^= m%8
    std::vector<uint8_t> aimg(16384, 0);
    for (int m = 0; m < M; ++m)
        for (int p = 0; p < KP; ++p) {
            const int b = 4 * p;
            const int off = (m / 8) * 1024 + (m % 8) * 128 + ((((b >> 4) ^ (m % 8))) << 4) + (b & 15);
            memcpy(&aimg[off], &cval[m * KP + p], 4);
        }
    // B image (non-gather mode): MN-major SW128: token atom at * (K*128), k row at k*128, chunk ^= k%8
    std::vector<uint8_t> bimg(K * N * 4, 0);
    for (int k = 0; k < K; ++k)
        for (int t = 0; t < N; ++t) {
            // 32-bit MN-major operands take SWIZZLE_128B_BASE32B (descriptor layout 1): 32-B
            // chunks of a 128-B row XOR (k % 4), 4-row groups (SBO 512), token atoms LBO apart
            const int b = (t % 32) * 4;
            const int off = (t / 32) * (K * 128) + k * 128 + (((b >> 5) ^ (k % 4)) << 5) + (b & 31);
            memcpy(&bimg[off], &Xg[perm[k] * N + t], 4);
        }
    // metadata smem image for tcgen05.cp: lane-major rows of 16 B: word j of lane l = meta[j][l]
    std::vector<uint32_t> emeta(4 * 128);
    for (int l = 0; l < 128; ++l)
        for (int j = 0; j < 4; ++j) emeta[l * 4 + j] = meta[j * 128 + l];
    std::vector<double> ref(M * N, 0.0);
    if (mode & 4) {
        for (int m = 0; m < M; ++m)
            for (int p = 0; p < 8; ++p) {
                float av;
                memcpy(&av, &cval[m * KP + p], 4);
                for (int t = 0; t < N; ++t) ref[m * N + t] += static_cast<double>(av) * X[p * N + t];
            }
    } else
    for (int m = 0; m < M; ++m)
        for (int k = 0; k < K; ++k)
            if (!(mode & 4) && W[m * K + k] != 0.f)
                for (int t = 0; t < N; ++t) ref[m * N + t] += W[m * K + k] * X[perm[k] * N + t];
    uint8_t *dA, *dB;
    uint32_t* dM;
    float* dX;
    float* dD;
    int* dP;
    CK(cudaMalloc(&dA, 16384));
    CK(cudaMalloc(&dB, K * N * 4));
    CK(cudaMalloc(&dM, 2048));
    CK(cudaMalloc(&dX, K * N * 4));
    CK(cudaMalloc(&dD, M * N * 4));
    CK(cudaMalloc(&dP, K * 4));
    CK(cudaMemcpy(dA, aimg.data(), 16384, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, bimg.data(), K * N * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dM, (mode & 1) ? emeta.data() : meta.data(), 2048, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dX, Xg.data(), K * N * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dP, perm.data(), K * 4, cudaMemcpyHostToDevice));
    CK(cudaMemset(dD, 0xFF, M * N * 4));
    CUtensorMap tm;
    memset(&tm, 0, sizeof(tm));
    if (mode & 2) {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
        cuuint64_t gdim[2] = {static_cast<cuuint64_t>(N), static_cast<cuuint64_t>(K)};
        cuuint64_t gstr[1] = {static_cast<cuuint64_t>(N) * 2};
        cuuint32_t box[2] = {64, static_cast<cuuint32_t>(box_rows)};
        cuuint32_t es[2] = {1, 1};
        CUresult r = reinterpret_cast<EncFn>(fn)(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dX, gdim, gstr, box, es,
                                                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                                 CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) {
            printf("  encode failed %d (box rows %d)\n", static_cast<int>(r), box_rows);
            return 1;
        }
    }
    Args a{dA, dB, dM, dD, N, mode, dP};
    const int smem = 1024 + 16384 + 2048 + K * N * 4;
    CK(cudaFuncSetAttribute(sp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    sp_kernel<<<1, 128, smem>>>(tm, a);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        printf("  kernel error: %s\n", cudaGetErrorString(e));
        exit(2);
    }
    std::vector<float> D(M * N);
    CK(cudaMemcpy(D.data(), dD, M * N * 4, cudaMemcpyDeviceToHost));
    int bad = 0;
    for (int m = 0; m < M; ++m)
        for (int t = 0; t < N; ++t)
            if (static_cast<double>(D[m * N + t]) != ref[m * N + t]) {
                if (bad < 8) {
                    if (probe && t == 0) {
                        const int p = m % KP, ch = p;
                        int want = -1;
                        for (int kk = 0; kk < 2; ++kk)
                            if (W[m * K + ch * 2 + kk] != 0.f) want = ch * 2 + kk;
                        printf("  probe m=%d p=%d: got k=%g want k=%d\n", m, p, D[m * N] - 1.0, want);
                    } else {
                        printf("  m=%d t=%d got %g want %g\n", m, t, D[m * N + t], ref[m * N + t]);
                    }
                }
                ++bad;
            }
    printf("N=%d mode=%d probe=%d box_rows=%d: %s (%d bad of %d)\n", N, mode, probe, box_rows, bad ? "FAIL" : "PASS", bad,
           M * N);
    cudaFree(dA);
    cudaFree(dB);
    cudaFree(dM);
    cudaFree(dX);
    cudaFree(dD);
    cudaFree(dP);
    return bad != 0;
}

int main() {
    int fails = 0;
    fails += run(64, 4, 0, 1, 5);
    fails += run(64, 0, 1, 1, 1);
    fails += run(64, 0, 0, 1, 2);
    printf("total fails %d\n", fails);
    return 0;
}
