// Who waits in the slot kernel's stage ring?  (sm_100a; 148 CTAs, 8 producer warps + 1 consumer
// warp, 5-stage full/empty ring, no data.)  Reports clk/stage and the share of time the consumer
// spends blocked in wait(full) and producer warp 0 in wait(empty).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_ring3 ubench_ring3.cu
// argv[1] = variant bits: 1 consumer plain arrive (else tcgen05.commit), 2 producers plain arrive
// (else cp.async.mbarrier.arrive.noinc), 4 no tcgen05.fence, 8 producer lane 0 waits + syncwarp,
// 16 consumer lane 0 only (other lanes exit), 32 test_wait spin instead of try_wait
#include <cstdint>
#include <cstdio>
#include <cstdlib>
__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
template <bool TEST>
__device__ __forceinline__ bool poll(uint64_t* b, uint32_t ph) {
    uint32_t ok;
    if (TEST)
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}"
                     : "=r"(ok) : "r"(su32(b)), "r"(ph) : "memory");
    else
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}"
                     : "=r"(ok) : "r"(su32(b)), "r"(ph) : "memory");
    return ok;
}
template <int V>
__global__ void __launch_bounds__(288, 1) kern(int iters, long long* out) {
    constexpr int ST = 5;
    constexpr bool TEST = V & 32;
    __shared__ __align__(8) uint64_t full[ST], empty[ST];
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < ST; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&full[s])), "r"(1 + 256));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&empty[s])), "r"(1));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 8) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(su32(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    __syncthreads();
    const long long t0 = clock64();
    long long blocked = 0;
    if (warp < 8) {
        int s = 0;
        uint32_t ph = 0;
        for (int st = 0; st < iters; ++st) {
            if (st >= ST) {
                const long long a = clock64();
                if (V & 8) {
                    if (lane == 0) while (!poll<TEST>(&empty[s], ph ^ 1)) {}
                    __syncwarp();
                } else {
                    while (!poll<TEST>(&empty[s], ph ^ 1)) {}
                }
                blocked += clock64() - a;
            }
            if (warp == 0 && lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&full[s])) : "memory");
            if (V & 2) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&full[s])) : "memory");
            else asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(su32(&full[s])) : "memory");
            if (++s == ST) s = 0, ph ^= 1;
        }
        if (warp == 0 && lane == 0) out[2 * blockIdx.x + 1] = blocked;
    } else if (warp == 8 && (!(V & 16) || lane == 0)) {
        int s = 0;
        uint32_t ph = 0;
        for (int st = 0; st < iters; ++st) {
            const long long a = clock64();
            while (!poll<TEST>(&full[s], ph)) {}
            blocked += clock64() - a;
            if (!(V & 4)) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            if (lane == 0) {
                if (V & 1) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[s])) : "memory");
                else asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&empty[s])) : "memory");
            }
            if (!(V & 16)) __syncwarp();
            if (++s == ST) s = 0, ph ^= 1;
        }
        if (lane == 0) out[2 * blockIdx.x] = (clock64() - t0) * 1000000 + blocked;
    }
    __syncthreads();
    if (warp == 8) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(slot));
}
template <int V>
void run(long long* d) {
    const int iters = 4000;
    kern<V><<<148, 288>>>(iters, d);
    kern<V><<<148, 288>>>(iters, d);
    long long h[296];
    cudaError_t e = cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double tot = 0, cb = 0, pb = 0;
    for (int i = 0; i < 148; ++i) tot += (h[2 * i] / 1000000) / 148.0, cb += (h[2 * i] % 1000000) / 148.0, pb += h[2 * i + 1] / 148.0;
    printf("V=%2d: %6.1f clk/stage, consumer blocked %5.1f%%, producer warp0 blocked %5.1f%% (%s)\n", V, tot / iters,
           100 * cb / tot, 100 * pb / tot, cudaGetErrorString(e));
    fflush(stdout);
}
int main() {
    long long* d;
    cudaMalloc(&d, 296 * 8);
    run<0>(d); run<1>(d); run<2>(d); run<3>(d); run<4>(d); run<8>(d); run<16>(d); run<17>(d); run<21>(d);
    run<32>(d); run<33>(d); run<2 + 8>(d); run<1 + 2 + 4 + 8 + 16>(d); run<1 + 2 + 4 + 8 + 16 + 32>(d);
    return 0;
}
