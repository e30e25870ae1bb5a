// Micro-benchmark of the synchronisation primitives the tcgen05 pipeline uses (sm_100a).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_sync ubench_sync.cu -lcuda
// Prints clocks per operation for: tcgen05.commit -> mbarrier round trip, warp-to-warp
// mbarrier ping-pong (1 elected arrival vs 32-thread arrivals), and the same ping-pong
// while other warps poll a barrier (try_wait vs test_wait).
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
__device__ __forceinline__ bool test_wait(uint64_t* b, uint32_t ph) {
    uint32_t ok;
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}"
                 : "=r"(ok) : "r"(su32(b)), "r"(ph) : "memory");
    return ok;
}
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) { while (!try_wait(b, ph)) {} }
__device__ __forceinline__ void wait_test(uint64_t* b, uint32_t ph) { while (!test_wait(b, ph)) {} }

struct Res { long long c[8]; };

// mode 0: commit round trip (1 thread)
// mode 1: ping-pong warp0 <-> warp1, 1 arrival each (lane 0)
// mode 2: ping-pong warp0 <-> warps1..12, 384 arrivals (all threads) -> warp0, warp0 lane0 -> all
// mode 3: mode 1 + warps 2..16 spinning try_wait on a never-completing barrier
// mode 4: mode 1 + warps 2..16 spinning test_wait on a never-completing barrier
__global__ void kern(int mode, int iters, Res* out) {
    __shared__ __align__(8) uint64_t bars[4];
    __shared__ uint32_t slot;
    __shared__ volatile int stop;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        init(&bars[0], 1);
        init(&bars[1], mode == 2 ? 384 : 1);
        init(&bars[2], 1);
        init(&bars[3], 1);
        stop = 0;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(su32(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    __syncthreads();
    long long t0 = clock64();
    if (mode == 0) {
        if (threadIdx.x == 0) {
            for (int i = 0; i < iters; ++i) {
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bars[0])) : "memory");
                wait(&bars[0], i & 1);
            }
            out->c[0] = (clock64() - t0);
        }
    } else if (mode == 2) {
        if (warp == 0) {
            for (int i = 0; i < iters; ++i) {
                if (lane == 0) arrive(&bars[0]);
                wait(&bars[1], i & 1);
            }
            if (lane == 0) out->c[0] = clock64() - t0;
        } else if (warp <= 12) {
            for (int i = 0; i < iters; ++i) {
                wait(&bars[0], i & 1);
                arrive(&bars[1]);
            }
        }
    } else {
        if (warp == 0) {
            for (int i = 0; i < iters; ++i) {
                if (lane == 0) arrive(&bars[0]);
                wait(&bars[1], i & 1);
            }
            if (lane == 0) out->c[0] = clock64() - t0;
            __syncwarp();
            if (lane == 0) { stop = 1; arrive(&bars[2]); }
        } else if (warp == 1) {
            for (int i = 0; i < iters; ++i) {
                wait(&bars[0], i & 1);
                if (lane == 0) arrive(&bars[1]);
            }
        } else if (mode == 3) {
            wait(&bars[2], 0);
        } else if (mode == 4) {
            wait_test(&bars[2], 0);
        }
    }
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(slot));
}

int main() {
    Res* d;
    cudaMalloc(&d, sizeof(Res));
    const char* names[] = {"commit round trip", "ping-pong 1 arrival", "ping-pong 384 arrivals",
                           "ping-pong + 15 warps try_wait", "ping-pong + 15 warps test_wait"};
    for (int mode = 0; mode < 5; ++mode) {
        const int iters = 2000;
        kern<<<1, 544>>>(mode, iters, d);
        kern<<<1, 544>>>(mode, iters, d);
        Res r;
        cudaError_t e = cudaMemcpy(&r, d, sizeof(Res), cudaMemcpyDeviceToHost);
        printf("%-34s %8.1f clk/iter  (%s)\n", names[mode], double(r.c[0]) / iters, cudaGetErrorString(e));
    }
    // many CTAs at once (one per SM) for the commit round trip and the ping-pong
    for (int mode = 0; mode < 3; ++mode) {
        kern<<<148, 544>>>(mode, 2000, d);
        Res r;
        cudaMemcpy(&r, d, sizeof(Res), cudaMemcpyDeviceToHost);
        printf("148 CTAs: %-24s %8.1f clk/iter\n", names[mode], double(r.c[0]) / 2000);
    }
    return 0;
}
