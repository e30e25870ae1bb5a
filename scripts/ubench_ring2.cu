// Stage-ring protocol floor vs producer layout (sm_100a), one CTA per SM (148 CTAs).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_ring2 ubench_ring2.cu
// layout 0: 8 producer warps share every stage (each lane: 8 x 16-B cp.async, noinc arrive)
// layout 1: one producer warp does every stage (each lane: 64 cp.async, noinc arrive)
// layout 2: 8 producer warps own stages round-robin (warp st % 8; each lane 64 cp.async, noinc)
// layout 3: 4 producer warps share every stage (16 cp.async per lane)
// cp: 0 = protocol only (plain per-thread arrive), 1 = with the copies (64 x 512 B = 32 KB per stage)
#include <cstdint>
#include <cstdio>
#include <cstdlib>

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

constexpr int MAXST = 8;
__global__ void __launch_bounds__(288, 1) kern(int layout, int ST, int cp, int iters, long long* out, const uint8_t* src) {
    __shared__ __align__(8) uint64_t full[MAXST], empty[MAXST];
    __shared__ uint32_t slot;
    extern __shared__ __align__(1024) uint8_t buf[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int NPW = layout == 0 ? 8 : layout == 3 ? 4 : 1;  // warps sharing one stage
    const int OWN = layout == 2 ? 8 : layout == 4 ? 4 : layout == 5 ? 2 : 1;  // stage-owning warps (round robin)
    const int CPL = 64 / NPW;                                  // 512-B rows per warp and stage
    if (threadIdx.x == 0) {
        for (int s = 0; s < ST; ++s) {
            init(&full[s], 32 * NPW);
            init(&empty[s], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 8) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(su32(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    __syncthreads();
    long long t0 = clock64();
    const bool producer = layout == 0 ? warp < 8 : layout == 1 ? warp == 0 : layout == 3 ? warp < 4 : warp < OWN;
    if (producer) {
        const int first = OWN > 1 ? warp : 0, step = OWN;
        const int part = (layout == 0 || layout == 3) ? warp : 0;
        for (int st = first; st < iters; st += step) {
            const int s = st % ST;
            if (st >= ST) wait(&empty[s], ((st / ST) - 1) & 1);
            if (cp) {
                const uint8_t* g = src + ((st * 977 + part * 131) % 4096) * 4096 + lane * 16;
                const uint32_t d = su32(buf + s * 32768 + part * CPL * 512 + lane * 16);
                for (int i = 0; i < CPL; ++i)
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d + i * 512), "l"(g + i * 4096 * 3) : "memory");
                asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(su32(&full[s])) : "memory");
            } else {
                arrive(&full[s]);
            }
        }
    } else if (warp == 8) {
        for (int st = 0; st < iters; ++st) {
            const int s = st % ST;
            wait(&full[s], (st / ST) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            if (lane == 0)
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&empty[s])) : "memory");
            __syncwarp();
        }
        if (lane == 0) out[blockIdx.x] = clock64() - t0;
    }
    __syncthreads();
    if (warp == 8) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(slot));
}

int main(int argc, char** argv) {
    const int layout = atoi(argv[1]), ST = atoi(argv[2]), cp = atoi(argv[3]);
    long long* d;
    uint8_t* src;
    cudaMalloc(&d, 148 * sizeof(long long));
    const size_t sb = 4096ull * 4096 * 4;
    cudaMalloc(&src, sb);
    cudaMemset(src, 1, sb);
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 6 * 32768);
    const int iters = 4096;
    for (int rep = 0; rep < 2; ++rep) kern<<<148, 288, 6 * 32768>>>(layout, ST, cp, iters, d, src);
    long long h[148];
    cudaError_t e = cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double mx = 0, mean = 0;
    for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx, mean += h[i] / 148.0;
    printf("cp=%d layout %d ST=%d: %7.1f clk/stage mean, %7.1f max  (%s)\n", cp, layout, ST, mean / iters, mx / iters,
           cudaGetErrorString(e));
    return 0;
}
