// Probe: tcgen05.mma.sp.kind::f16 with the sparse A operand (the compressed weights) in TMEM
// instead of shared memory -- does it run, and which TMEM layout does it read?  Hypothesis
// (as for the dense .ts form): lane = row m, column c = compressed elements (2c, 2c+1) as a packed
// bf16 pair.  One MMA M=128 x N=64 x K=32 (logical), metadata nibble 0x4 (slots 0,1 of every quad)
// or per-quad varied, B MN-major 128-B swizzled in smem, integer values (exact in fp32).
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o ubench_sp_ts ubench_sp_ts.cu
#include <cuda_bf16.h>
#include <cstdint>
#include <cstdio>
#include <cstring>

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
    d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
    d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
    d |= static_cast<uint64_t>(1) << 46;
    d |= static_cast<uint64_t>(layout & 7) << 61;
    return d;
}

// A: 128 x 16 compressed bf16 (row-major), meta: per row 8 nibbles, B: 32 x 64 bf16 (k-major rows)
__global__ void probe(const __nv_bfloat16* A, const uint32_t* Erow /* [128 lanes][4 words] image */,
                      const __nv_bfloat16* B, float* D, int variant) {
    __shared__ __align__(1024) uint8_t sB[32 * 128];
    __shared__ __align__(16) uint32_t sE[128 * 4];
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t slot;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // B (k, n) -> MN-major SW128: byte (k/8)*1024 + (k%8)*128 + (((n/8) ^ (k%8)) * 16) + (n%8)*2
    for (int e = tid; e < 32 * 64; e += blockDim.x) {
        const int k = e / 64, n = e % 64;
        *reinterpret_cast<__nv_bfloat16*>(sB + (k / 8) * 1024 + (k % 8) * 128 + (((n / 8) ^ (k % 8)) * 16) + (n % 8) * 2) = B[e];
    }
    for (int e = tid; e < 128 * 4; e += blockDim.x) sE[e] = Erow[e];
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su32(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = slot;
    const uint32_t dcol = 0, acol = 64, mcol = 96;  // D: 64 columns, A: 8 (or 16) columns, metadata 4
    // A -> TMEM by the 4 warps (warp q writes lanes 32q .. 32q+31): 8 words per lane
    {
        const int r = 32 * warp + lane;
        uint32_t v[8];
        for (int c = 0; c < 8; ++c) {
            __nv_bfloat16 lo, hi;
            if (variant == 0) { lo = A[r * 16 + 2 * c]; hi = A[r * 16 + 2 * c + 1]; }     // col c = (2c, 2c+1)
            else { lo = A[r * 16 + c]; hi = A[r * 16 + c + 8]; }                          // col c = (c, c+8)
            v[c] = static_cast<uint32_t>(__bfloat16_as_ushort(lo)) | (static_cast<uint32_t>(__bfloat16_as_ushort(hi)) << 16);
        }
        const uint32_t ta = tmem + (static_cast<uint32_t>(32 * warp) << 16) + acol;
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(ta), "r"(v[0]),
                     "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]));
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (tid == 0) {
        asm volatile("tcgen05.cp.cta_group::1.128x128b [%0], %1;" ::"r"(tmem + mcol), "l"(sdesc(su32(sE), 2048, 128, 0)));
        const uint32_t idesc = (1u << 2) | (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) | ((64u >> 3) << 17) |
                               ((128u >> 4) << 24);
        const uint64_t bdesc = sdesc(su32(sB), 4096, 1024, 2);
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.sp.cta_group::1.kind::f16 [%0], [%1], %2, [%5], %3, p;\n\t}" ::"r"(tmem + dcol),
                     "r"(tmem + acol), "l"(bdesc), "r"(idesc), "r"(0), "r"(tmem + mcol)
                     : "memory");
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
    }
    {
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0,1,0,p;\n\t}"
                         : "=r"(ok) : "r"(su32(&bar)) : "memory");
    }
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    for (int c0 = 0; c0 < 64; c0 += 8) {
        uint32_t v[8];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                     : "r"(tmem + (static_cast<uint32_t>(32 * warp) << 16) + dcol + c0));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        for (int i = 0; i < 8; ++i) D[(32 * warp + lane) * 64 + c0 + i] = __uint_as_float(v[i]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

int main() {
    const int M = 128, KC = 16, K = 32, N = 64;
    static __nv_bfloat16 hA[M * KC], hB[K * N];
    static uint32_t hE[128 * 4];
    static int pos[M][8][2];
    static float hD[M * N];
    for (int r = 0; r < M; ++r)
        for (int j = 0; j < KC; ++j) hA[r * KC + j] = __float2bfloat16(float((r * 3 + j * 7) % 5 - 2));
    for (int k = 0; k < K; ++k)
        for (int n = 0; n < N; ++n) hB[k * N + n] = __float2bfloat16(float((k * 5 + n * 3) % 7 - 3));
    // metadata: per (row, quad) two distinct sorted slots, varied
    memset(hE, 0, sizeof(hE));
    const int pairs[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
    for (int r = 0; r < M; ++r)
        for (int c = 0; c < 8; ++c) {
            const int* pp = pairs[(r + 3 * c) % 6];
            pos[r][c][0] = pp[0], pos[r][c][1] = pp[1];
            const int ln = (r % 8) + 8 * (c / 4) + 16 * (r / 16);
            const int bit = 16 * ((r / 8) % 2) + 4 * (c % 4);
            hE[ln * 4 + 0] |= static_cast<uint32_t>(pp[0] | (pp[1] << 2)) << bit;
        }
    __nv_bfloat16 *dA, *dB;
    uint32_t* dE;
    float* dD;
    cudaMalloc(&dA, sizeof(hA)), cudaMalloc(&dB, sizeof(hB)), cudaMalloc(&dE, sizeof(hE)), cudaMalloc(&dD, sizeof(hD));
    cudaMemcpy(dA, hA, sizeof(hA), cudaMemcpyHostToDevice);
    cudaMemcpy(dB, hB, sizeof(hB), cudaMemcpyHostToDevice);
    cudaMemcpy(dE, hE, sizeof(hE), cudaMemcpyHostToDevice);
    for (int variant = 0; variant < 2; ++variant) {
        cudaMemset(dD, 0, sizeof(hD));
        probe<<<1, 128>>>(dA, dE, dB, dD, variant);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(hD, dD, sizeof(hD), cudaMemcpyDeviceToHost);
        int bad = 0;
        double maxerr = 0;
        for (int r = 0; r < M; ++r)
            for (int n = 0; n < N; ++n) {
                float ref = 0.f;
                for (int j = 0; j < KC; ++j) {
                    const int c = j / 2, k = 4 * c + pos[r][c][j % 2];
                    ref += __bfloat162float(hA[r * KC + j]) * __bfloat162float(hB[k * N + n]);
                }
                const double d = hD[r * N + n] - ref;
                if (d != 0) ++bad;
                if (d * d > maxerr) maxerr = d * d;
            }
        printf("variant %d (%s): %s, mismatches %d / %d%s\n", variant,
               variant == 0 ? "column c = compressed (2c, 2c+1)" : "column c = compressed (c, c+8)",
               cudaGetErrorString(e), bad, M * N, bad == 0 ? "  <-- layout confirmed" : "");
    }
    return 0;
}
