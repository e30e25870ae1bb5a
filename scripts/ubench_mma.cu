// Micro-benchmark: tcgen05.mma kind::f16 M=128, K=16, A from TMEM, B MN-major in smem,
// issue/execute rate vs N, with and without concurrent tcgen05.st traffic from 12 warps.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_mma ubench_mma.cu
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ bool try_wait(uint64_t* b, uint32_t ph) {
    uint32_t ok;
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}"
                 : "=r"(ok) : "r"(su32(b)), "r"(ph) : "memory");
    return ok;
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
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d), "r"(a), "l"(bdesc), "r"(idesc), "r"(acc)
                 : "memory");
}
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc)
                 : "memory");
}

// per "panel": G = 128/N groups x 4 k-steps of M128 x N x K16 (same MAC count per panel for every N)
__global__ void kern(int N, int panels, int stores, int ss, long long* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ __align__(8) uint64_t bars[2];
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bars[0])) : "memory");
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bars[1])) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int G = 128 / N;
    const int rb = (N >= 64 ? 64 : N) * 2;
    const uint32_t layout = rb == 128 ? 2u : rb == 64 ? 4u : 6u;
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) | (static_cast<uint32_t>(N >> 3) << 17) |
                           (static_cast<uint32_t>(128 >> 4) << 24);
    const uint32_t base = su32(sm);
    const uint32_t abase = base + 64 * 1024;  // SS: A K-major SW128 atoms (128 rows x 64 B)
    long long t0 = clock64();
    if (warp == 0) {
        for (int pnl = 0; pnl < panels; ++pnl) {
            if (threadIdx.x == 0) {
                for (int g = 0; g < G; ++g)
                    for (int kk = 0; kk < 4; ++kk) {
                        const uint64_t bd = sdesc(base + g * 16384 % 65536 + kk * 16 * rb, 64 * 128, 8 * rb, layout);
                        if (ss)
                            mma_ss(g * N, sdesc(abase + kk * 32, 16, 1024, 2), bd, idesc, 1);
                        else
                            mma_ts(g * N, 128 + (pnl % 3) * 128 + kk * 8, bd, idesc, 1);
                    }
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bars[pnl & 1])) : "memory");
            }
            __syncwarp();
            if (pnl >= 1) while (!try_wait(&bars[(pnl - 1) & 1], ((pnl - 1) >> 1) & 1)) {}
        }
        while (!try_wait(&bars[(panels - 1) & 1], ((panels - 1) >> 1) & 1)) {}
        if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
    } else if (stores && warp >= 4) {
        // 12 warps hammer tcgen05.st.16x128b.x4 into columns 128..511 (A buffers)
        const int q = warp & 3;
        uint32_t v[8] = {1, 2, 3, 4, 5, 6, 7, 8};
        for (int i = 0; i < panels * 6; ++i) {
            const uint32_t ta = (static_cast<uint32_t>(q * 32 + (i & 1) * 16) << 16) + 128 + ((i * 16 + warp * 48) % 384);
            asm volatile("tcgen05.st.sync.aligned.16x128b.x4.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(ta), "r"(v[0]),
                         "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]));
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
}

__device__ __forceinline__ bool elect1() {
    uint32_t pred;
    asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(pred));
    return pred != 0;
}
// compile-time N, descriptors from uniform values, whole warp runs the loop, elected lane issues
template <int N, int KK = 4>
__global__ void kern2(int panels, int load, long long* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ __align__(8) uint64_t bars[3];
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bars[0])) : "memory");
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bars[1])) : "memory");
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bars[2])) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    constexpr int G = 128 / N;
    constexpr int rb = (N >= 64 ? 64 : N) * 2;
    constexpr uint32_t layout = rb == 128 ? 2u : rb == 64 ? 4u : 6u;
    constexpr uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) | (static_cast<uint32_t>(N >> 3) << 17) |
                               (static_cast<uint32_t>(128 >> 4) << 24);
    const uint64_t d0 = sdesc(su32(sm), 64 * 128, 8 * rb, layout);
    long long t0 = clock64();
    if (warp == 0) {
        for (int pnl = 0; pnl < panels; ++pnl) {
            const uint32_t abuf = 128 + (pnl % 3) * 128;
            if (elect1()) {
#pragma unroll
                for (int g = 0; g < G; ++g)
#pragma unroll
                    for (int kk = 0; kk < KK; ++kk)
                        mma_ts(g * N, abuf + (kk % 4) * 8, d0 + (((g * 16384) % 65536 + (kk % 4) * 16 * rb) >> 4), idesc, 1);
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bars[pnl & 1])) : "memory");
            }
            __syncwarp();
            if (pnl >= 1) while (!try_wait(&bars[(pnl - 1) & 1], ((pnl - 1) >> 1) & 1)) {}
        }
        while (!try_wait(&bars[(panels - 1) & 1], ((panels - 1) >> 1) & 1)) {}
        if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
        if (threadIdx.x == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&bars[2])) : "memory");
    } else if (load == 4) {
        while (!try_wait(&bars[2], 0)) {}  // completes only when the MMA warp finishes -> spins
    } else if (warp >= 4 && load) {
        const int q = warp & 3;
        uint32_t v[8] = {1, 2, 3, 4, 5, 6, 7, 8};
        uint32_t acc = 0;
        for (int i = 0; i < panels * 8; ++i) {
            if (load & 1) {
                const uint32_t ta = (static_cast<uint32_t>(q * 32 + (i & 1) * 16) << 16) + 128 + ((i * 16 + warp * 48) % 384);
                asm volatile("tcgen05.st.sync.aligned.16x128b.x4.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(ta), "r"(v[0]),
                             "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]));
            }
            if (load & 2) {
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const uint32_t a = su32(sm) + 70000 + ((threadIdx.x * 4 + j * 256 + i * 64) & 16383);
                    uint32_t x;
                    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(x) : "r"(a));
                    acc += x;
                }
                v[i & 7] += acc;
            }
        }
        if (load & 1) asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        if (acc == 12345) out[1] = acc;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
}

template <int N, int KK = 4>
void run2(long long* d, int panels, int grid, int load = 0) {
    cudaFuncSetAttribute(kern2<N, KK>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    kern2<N, KK><<<grid, 512, 100 * 1024>>>(10, load, d);
    kern2<N, KK><<<grid, 512, 100 * 1024>>>(panels, load, d);
    long long c;
    cudaError_t e = cudaMemcpy(&c, d, sizeof(c), cudaMemcpyDeviceToHost);
    const int mmas = panels * (128 / N) * KK;
    printf("KK=%2d TS-unrolled grid=%d load=%d N=%3d: %7.1f clk/MMA  %6.0f MAC/clk  %s\n", KK, grid, load, N, double(c) / mmas,
           128.0 * N * 16 * mmas / double(c), cudaGetErrorString(e));
}

int main() {
    long long* d;
    cudaMalloc(&d, 148 * sizeof(long long));
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    const int panels = 2000;
    for (int load : {0, 4}) {
        run2<32, 16>(d, 500, 1, load);
        run2<32, 4>(d, 2000, 1, load);
    }
    return 0;
}
