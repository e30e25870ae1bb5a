// Per-iteration cost of the consumer-side barrier operations (sm_100a), one warp per CTA,
// 148 CTAs.  Each iteration: the barrier gets its one arrival and the warp waits on it.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_loop ubench_loop.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
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
// mode: 0 arrive+try_wait, 1 arrive+test_wait, 2 arrive+try_wait+fence, 3 commit+try_wait,
//       4 commit+try_wait+fence, 5 pre-completed barrier: try_wait only (already complete),
//       6 fence only, 7 empty loop
__global__ void kern(int mode, int iters, long long* out) {
    __shared__ __align__(8) uint64_t bar[2];
    __shared__ uint32_t slot;
    const int lane = threadIdx.x;
    if (lane == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[0])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[1])));
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&bar[1])));  // phase 0 complete
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(su32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    __syncwarp();
    long long t0 = clock64();
    int acc = 0;
    for (int i = 0; i < iters; ++i) {
        if (mode <= 4) {
            if (lane == 0) {
                if (mode >= 3)
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar[0])) : "memory");
                else
                    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&bar[0])) : "memory");
            }
            if (mode == 1) while (!test_wait(&bar[0], i & 1)) {}
            else while (!try_wait(&bar[0], i & 1)) {}
            if (mode == 2 || mode == 4) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            __syncwarp();
        } else if (mode == 5) {
            acc += try_wait(&bar[1], 0);
        } else if (mode == 6) {
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        } else {
            __syncwarp();
        }
    }
    if (lane == 0) out[blockIdx.x] = (clock64() - t0) + (acc == -1);
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(slot));
}
int main() {
    long long* d;
    cudaMalloc(&d, 148 * 8);
    const char* nm[] = {"arrive + try_wait", "arrive + test_wait", "arrive + try_wait + tc fence", "commit + try_wait",
                        "commit + try_wait + tc fence", "try_wait on complete barrier", "tc fence only", "syncwarp only"};
    for (int mode = 0; mode < 8; ++mode) {
        const int iters = 20000;
        kern<<<148, 32>>>(mode, iters, d);
        kern<<<148, 32>>>(mode, iters, d);
        long long h[148];
        cudaError_t e = cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        double mean = 0;
        for (int i = 0; i < 148; ++i) mean += h[i] / 148.0;
        printf("%-34s %7.1f clk/iter (%s)\n", nm[mode], mean / iters, cudaGetErrorString(e));
        fflush(stdout);
    }
    return 0;
}
