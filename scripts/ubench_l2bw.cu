// Micro-benchmark: L2 -> SM feed bandwidth on B200 with every SM loading an L2-resident buffer
// (the slot kernel's token gather and weight stream both come from L2).  One CTA per SM
// (clusters of CS CTAs for the multicast case), a ring of 8 x 16 KB shared-memory slots.
//   kind 0: cp.async.bulk (1-D bulk copy) of 16 KB per slot, one issuing thread
//   kind 1: 16-B cp.async by 8 warps (the gather's instruction), completion by
//           cp.async.mbarrier.arrive.noinc (as in the slot kernel), 32 KB per slot round
//   kind 2: bulk copy, CTAs of a group of G read the SAME addresses at the same time (L2 dedup?)
//   kind 3: bulk copy .multicast::cluster, each CTA of a cluster of CS loads 1/CS of the slot
//           into every CTA of the cluster
// Bytes delivered to shared memory per SM clock are reported (chip total and per SM).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_l2bw ubench_l2bw.cu
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ bool try_wait(uint64_t* b, uint32_t ph) {
    uint32_t ok;
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}"
                 : "=r"(ok) : "r"(su32(b)), "r"(ph) : "memory");
    return ok;
}
__device__ __forceinline__ void expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ uint32_t cta_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

constexpr int SLOT = 16384, NSLOT = 8;

__global__ void __launch_bounds__(256, 1) l2bw(const uint8_t* __restrict__ src, int64_t src_bytes, int kind, int group,
                                               int cs, int rounds, long long* out) {
    extern __shared__ __align__(1024) uint8_t sm_raw[];
    uint8_t* sm = sm_raw + ((1024u - (su32(sm_raw) & 1023u)) & 1023u);
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + NSLOT * SLOT);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t crank = cs > 1 ? cta_rank() : 0u;
    if (tid == 0) {
        for (int s = 0; s < NSLOT; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&full[s])), "r"(kind == 1 ? 256 : 1));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (cs > 1) cluster_sync(); else __syncthreads();
    const int64_t nchunks = src_bytes / SLOT;
    // which chunk sequence this CTA walks: kind 2 -> all CTAs of a group share one sequence
    const int64_t seq = kind == 2 ? blockIdx.x / group : (kind == 3 ? blockIdx.x / cs : blockIdx.x);
    long long t0 = clock64();
    if (kind == 1) {
        // 8 warps x 32 lanes x 4 x 16 B = 32 KB per round: two slots
        for (int r = 0; r < rounds; ++r) {
            const int s = (2 * r) % NSLOT;
            if (r >= NSLOT / 2) {
                while (!try_wait(&full[s], ((2 * r / NSLOT) - 1) & 1)) {
                }
            }
            const int64_t ch = (seq * 7919 + r * 2) % (nchunks - 1);
            const uint8_t* g = src + ch * SLOT;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const uint32_t off = (i * 256 + tid) * 16;  // 0 .. 32 KB
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su32(sm + s * SLOT) + off), "l"(g + off) : "memory");
            }
            asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(su32(&full[s])) : "memory");
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncthreads();
    } else if (kind == 3) {
        // double-buffered halves of the ring; a cluster barrier after each half completes keeps every
        // CTA's barrier phases aligned with its peers' multicast writes
        const uint32_t part = SLOT / cs;
        auto issue = [&](int r) {
            const int s = r % NSLOT;
            const int64_t ch = (seq * 7919 + r) % nchunks;
            expect_tx(&full[s], SLOT);
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], %4;" ::"r"(
                    su32(sm + s * SLOT + crank * part)),
                "l"(src + ch * SLOT + crank * part), "r"(part), "r"(su32(&full[s])), "h"(static_cast<uint16_t>((1u << cs) - 1))
                : "memory");
        };
        if (tid == 0)
            for (int r = 0; r < NSLOT / 2; ++r) issue(r);
        for (int r0 = 0; r0 < rounds; r0 += NSLOT / 2) {
            if (tid == 0) {
                if (r0 + NSLOT / 2 < rounds)
                    for (int r = r0 + NSLOT / 2; r < r0 + NSLOT; ++r) issue(r);
                for (int r = r0; r < r0 + NSLOT / 2; ++r)
                    while (!try_wait(&full[r % NSLOT], (r / NSLOT) & 1)) {
                    }
            }
            cluster_sync();
        }
    } else if (tid == 0) {
        for (int r = 0; r < rounds; ++r) {
            const int s = r % NSLOT;
            if (r >= NSLOT) {
                while (!try_wait(&full[s], ((r / NSLOT) - 1) & 1)) {
                }
            }
            const int64_t ch = (seq * 7919 + r) % nchunks;
            const uint8_t* g = src + ch * SLOT;
            expect_tx(&full[s], SLOT);
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                             su32(sm + s * SLOT)),
                         "l"(g), "r"(SLOT), "r"(su32(&full[s]))
                         : "memory");
        }
        for (int s = 0; s < NSLOT; ++s) {
            const int r = rounds - NSLOT + s;
            const int ss = r % NSLOT;
            while (!try_wait(&full[ss], (r / NSLOT) & 1)) {
            }
        }
    }
    long long t1 = clock64();
    if (cs > 1) cluster_sync(); else __syncthreads();
    if (tid == 0) {
        out[2 * blockIdx.x] = t1 - t0;
        out[2 * blockIdx.x + 1] = static_cast<long long>(rounds) * (kind == 1 ? 2 * SLOT : SLOT);
    }
    (void)warp; (void)lane;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int64_t bytes = 32ll << 20;  // 32 MB: L2 resident
    uint8_t* src;
    cudaMalloc(&src, bytes);
    cudaMemset(src, 1, bytes);
    long long* out;
    cudaMalloc(&out, sizeof(long long) * 2 * 160);
    const int smem = NSLOT * SLOT + 1024 + 128;
    cudaFuncSetAttribute(l2bw, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(l2bw, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    struct C { int kind, group, cs; const char* name; };
    const C cases[] = {{0, 1, 1, "bulk, distinct"}, {1, 1, 1, "cp.async16 8 warps"}, {2, 2, 1, "bulk, 2 CTAs same addr"},
                       {2, 4, 1, "bulk, 4 CTAs same addr"}, {2, 8, 1, "bulk, 8 CTAs same addr"},
                       {3, 1, 2, "bulk multicast cs 2"}, {3, 1, 4, "bulk multicast cs 4"}, {3, 1, 8, "bulk multicast cs 8"},
                       {0, 1, 1, "bulk, distinct (again)"}};
    printf("# ubench_l2bw: %d CTAs (1/SM), 32 MB L2-resident source, 8 x 16 KB ring\n", sms);
    for (const C& c : cases) {
        const int grid = (sms / c.cs) * c.cs;
        const int rounds = 4096;
        cudaMemset(out, 0, sizeof(long long) * 2 * 160);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(256);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = c.cs;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cudaError_t e = cudaLaunchKernelEx(&cfg, l2bw, (const uint8_t*)src, bytes, c.kind, c.group, c.cs, rounds, out);
        if (e == cudaSuccess) e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("%-28s error %s\n", c.name, cudaGetErrorString(e)); cudaGetLastError(); continue; }
        long long h[2 * 160];
        cudaMemcpy(h, out, sizeof(long long) * 2 * grid, cudaMemcpyDeviceToHost);
        double clk = 0, by = 0, mx = 0;
        for (int i = 0; i < grid; ++i) { clk += h[2 * i]; by += h[2 * i + 1]; if (h[2 * i] > mx) mx = h[2 * i]; }
        // delivered bytes per SM clock: total bytes into shared memory over the slowest CTA's clocks
        printf("%-28s grid %3d: %6.1f B/clk per SM (mean CTA), chip %7.0f B/clk delivered\n", c.name, grid,
               by / clk, by / mx);
    }
    return 0;
}
