// Micro-benchmark of the slot kernel's stage ring (sm_100a): 8 producer warps + 1 consumer warp,
// a 5-stage full/empty mbarrier ring, one CTA per SM, clk per stage for protocol variants.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_ring ubench_ring.cu
// mode bits: 1 plain per-thread arrive (else cp.async.mbarrier.arrive.noinc), 2 one arrive per warp,
//            4 consumer releases with a plain arrive (else tcgen05.commit), 8 empty wait by lane 0 only,
//            16 each producer thread issues 8 x 16-B cp.async per stage (L2-resident source)
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void init(uint64_t* b, int c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ bool try_wait(uint64_t* b, uint32_t ph) {
    uint32_t ok;
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}"
                 : "=r"(ok) : "r"(su32(b)), "r"(ph) : "memory");
    return ok;
}
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) { while (!try_wait(b, ph)) {} }

constexpr int ST = 5, PW = 8;
__global__ void __launch_bounds__(288, 1) kern(int mode, int iters, long long* out, const uint8_t* src) {
    __shared__ __align__(8) uint64_t full[ST], empty[ST];
    __shared__ uint32_t slot;
    extern __shared__ __align__(1024) uint8_t buf[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < ST; ++s) {
            init(&full[s], 1 + ((mode & 2) ? PW : 32 * PW));
            init(&empty[s], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == PW) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(su32(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    __syncthreads();
    long long t0 = clock64();
    if (warp < PW) {
        for (int st = 0; st < iters; ++st) {
            const int s = st % ST;
            if (st >= ST) {
                if (mode & 8) {
                    if (lane == 0) wait(&empty[s], ((st / ST) - 1) & 1);
                    __syncwarp();
                } else {
                    wait(&empty[s], ((st / ST) - 1) & 1);
                }
            }
            if (warp == 0 && lane == 0) arrive(&full[s]);  // the weight copy's expect_tx arrival
            if (mode & 16) {
                const uint32_t d = su32(buf + s * 32768 + warp * 4096 + lane * 16);
                const uint8_t* g = src + ((st * 977 + warp * 131) % 4096) * 4096 + lane * 16;
#pragma unroll
                for (int i = 0; i < 8; ++i)
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d + i * 512), "l"(g + i * 512) : "memory");
            }
            if (mode & 2) {
                if (mode & 16) {
                    asm volatile("cp.async.wait_all;" ::: "memory");
                }
                __syncwarp();
                if (lane == 0) arrive(&full[s]);
            } else if (mode & 1) {
                if (mode & 16) asm volatile("cp.async.wait_all;" ::: "memory");
                arrive(&full[s]);
            } else {
                asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(su32(&full[s])) : "memory");
            }
        }
    } else if (warp == PW) {
        for (int st = 0; st < iters; ++st) {
            const int s = st % ST;
            wait(&full[s], (st / ST) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            if (lane == 0) {
                if (mode & 4) arrive(&empty[s]);
                else asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&empty[s])) : "memory");
            }
            __syncwarp();
        }
        if (lane == 0) out[blockIdx.x] = clock64() - t0;
    }
    __syncthreads();
    if (warp == PW) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(slot));
}

int main() {
    long long* d;
    uint8_t* src;
    cudaMalloc(&d, 148 * sizeof(long long));
    cudaMalloc(&src, 4096 * 4096 + 8192);
    cudaMemset(src, 1, 4096 * 4096 + 8192);
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, ST * 32768);
    const int modes[] = {0, 1, 2, 4, 5, 6, 8, 9, 12, 14, 16, 17, 18, 20, 22, 24, 30};
    for (int mode : modes) {
        const int iters = 4000;
        for (int rep = 0; rep < 2; ++rep) kern<<<148, 288, ST * 32768>>>(mode, iters, d, src);
        long long h[148];
        cudaError_t e = cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        double mx = 0, mean = 0;
        for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx, mean += h[i] / 148.0;
        printf("mode %2d [%s%s%s%s%s] %7.1f clk/stage mean, %7.1f max  (%s)\n", mode,
               (mode & 2) ? "warp-arrive " : (mode & 1) ? "plain-arrive " : "noinc ",
               (mode & 4) ? "plain-release " : "commit ", (mode & 8) ? "lane0-wait " : "all-wait ",
               (mode & 16) ? "+8cp.async/thr" : "", "", mean / iters, mx / iters, cudaGetErrorString(e));
    }
    return 0;
}
