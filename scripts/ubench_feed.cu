// Micro-benchmark: concurrent L2 -> SM feed paths on B200, one CTA per SM, from an L2-resident
// 32 MB buffer: which ones share a bandwidth limit?  Roles run concurrently in one CTA:
//   cp warps  : 16-B cp.async (LDGSTS) into a per-warp ring of 4 x 2 KB, cp.async.mbarrier.arrive.noinc
//   bulk thr  : 1-D cp.async.bulk of BS bytes into a per-thread ring of 4 slots (complete_tx)
//   tma thr   : 2-D TMA tile loads (64 rows x 128 B, 128-B swizzle) into a ring of 4 x 8 KB
//   ldg warps : LDG.128 into registers (8 independent loads per lane in flight), summed
// Each role reports its bytes and clocks; the line gives per-role B/clk per SM and the total.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_feed ubench_feed.cu -lcuda
#include <cuda.h>
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

struct Cfg {
    int cp_warps, bulk_thr, bulk_bytes, tma_thr, ldg_warps, rounds;
    int seq;  // 1: rows sequential per warp instead of pseudo-random
};
constexpr int CP_SLOT = 2048, CP_RING = 4, BK_RING = 4, TMA_SLOT = 8192, TMA_RING = 4;
// shared layout: cp rings 8 x 8 KB = 64 KB | bulk rings 2 x 4 x 16 KB = 128 KB max | tma ring 32 KB (bulk <= 1 then)
__global__ void __launch_bounds__(1024, 1) feed(const uint8_t* __restrict__ src, int64_t nbytes, const __grid_constant__ CUtensorMap tm,
                                               Cfg c, long long* out, float* sink) {
    extern __shared__ __align__(1024) uint8_t sm_raw[];
    uint8_t* sm = sm_raw + ((1024u - (su32(sm_raw) & 1023u)) & 1023u);
    uint8_t* cp_base = sm;
    uint8_t* bk_base = sm + 65536;  // may alias cp rings of warps >= 8 (contents are never read)
    uint8_t* tma_base = sm + 196608;
    uint64_t* bars = reinterpret_cast<uint64_t*>(tma_base + TMA_RING * TMA_SLOT);
    uint64_t* cp_bar = bars;              // 16 warps x 4
    uint64_t* bk_bar = bars + 64;         // 2 threads x 4
    uint64_t* tma_bar = bars + 72;        // 4
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int i = 0; i < 64; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 32;" ::"r"(su32(&cp_bar[i])));
        for (int i = 0; i < 12; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bk_bar[i])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int64_t nchunk = nbytes / 16384;
    long long t0 = clock64(), bytes = 0;
    int role = -1;
    if (warp < c.cp_warps) {
        role = 0;
        uint64_t* b = cp_bar + 4 * warp;
        uint8_t* ring = cp_base + warp * CP_RING * CP_SLOT;
        for (int r = 0; r < c.rounds; ++r) {
            const int s = r % CP_RING;
            if (r >= CP_RING)
                while (!try_wait(&b[s], ((r / CP_RING) - 1) & 1)) {
                }
            // 4 rows of 512 B at pseudo-random 512-B-aligned offsets (the gather's access shape)
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int64_t row = c.seq ? (static_cast<int64_t>(blockIdx.x) * 409 + warp * 8191 + r * 4 + i) & (nbytes / 512 - 1)
                                          : ((static_cast<int64_t>(blockIdx.x) * 7919 + warp * 131 + r * 4 + i) * 2654435761ull) & (nbytes / 512 - 1);
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su32(ring + s * CP_SLOT) + i * 512 + lane * 16),
                             "l"(src + row * 512 + lane * 16) : "memory");
            }
            asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(su32(&b[s])) : "memory");
            bytes += 4 * 16;
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
        bytes *= 32;  // per warp (lane 0 reports)
    } else if (warp == 31 && lane < c.bulk_thr) {
        role = 1;
        uint64_t* b = bk_bar + 4 * lane;
        uint8_t* ring = bk_base + lane * BK_RING * 16384;
        const int rounds = static_cast<int>(static_cast<int64_t>(c.rounds) * 2048 * c.cp_warps / c.bulk_bytes / (c.bulk_thr ? c.bulk_thr : 1)) + 64;
        for (int r = 0; r < rounds; ++r) {
            const int s = r % BK_RING;
            if (r >= BK_RING)
                while (!try_wait(&b[s], ((r / BK_RING) - 1) & 1)) {
                }
            const int64_t ch = (static_cast<int64_t>(blockIdx.x) * 7919 + lane * 31 + r) & (nchunk - 1);
            expect_tx(&b[s], c.bulk_bytes);
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                             su32(ring + s * 16384)), "l"(src + ch * 16384), "r"(c.bulk_bytes), "r"(su32(&b[s])) : "memory");
            bytes += c.bulk_bytes;
        }
        for (int r = rounds - BK_RING; r < rounds; ++r)
            while (!try_wait(&b[r % BK_RING], (r / BK_RING) & 1)) {
            }
    } else if (warp == 30 && lane == 0 && c.tma_thr) {
        role = 2;
        const int rounds = c.rounds * 2;
        for (int r = 0; r < rounds; ++r) {
            const int s = r % TMA_RING;
            if (r >= TMA_RING)
                while (!try_wait(&tma_bar[s], ((r / TMA_RING) - 1) & 1)) {
                }
            const int row = static_cast<int>(((static_cast<int64_t>(blockIdx.x) * 7919 + r) * 64) & (nbytes / 128 - 1)) & ~63;
            expect_tx(&tma_bar[s], TMA_SLOT);
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
                             su32(tma_base + s * TMA_SLOT)), "l"(&tm), "r"(su32(&tma_bar[s])), "r"(0), "r"(row) : "memory");
            bytes += TMA_SLOT;
        }
        for (int r = rounds - TMA_RING; r < rounds; ++r)
            while (!try_wait(&tma_bar[r % TMA_RING], (r / TMA_RING) & 1)) {
            }
    } else if (warp >= 16 && warp < 16 + c.ldg_warps) {
        role = 3;
        float acc = 0.f;
        const int w = warp - 16;
        for (int r = 0; r < c.rounds / 2; ++r) {
            float4 v[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int64_t row = c.seq ? (static_cast<int64_t>(blockIdx.x) * 409 + w * 8191 + r * 8 + i) & (nbytes / 512 - 1)
                                          : ((static_cast<int64_t>(blockIdx.x) * 7919 + w * 131 + r * 8 + i) * 2654435761ull) & (nbytes / 512 - 1);
                v[i] = __ldcg(reinterpret_cast<const float4*>(src + row * 512) + lane);
            }
#pragma unroll
            for (int i = 0; i < 8; ++i) acc += v[i].x + v[i].y + v[i].z + v[i].w;
            bytes += 8 * 16;
        }
        bytes *= 32;
        if (acc == 12345.f) sink[0] = acc;
    }
    long long t1 = clock64();
    if (role >= 0 && (role == 1 || role == 2 || lane == 0)) {
        atomicAdd(reinterpret_cast<unsigned long long*>(&out[(blockIdx.x * 4 + role) * 2]), static_cast<unsigned long long>(bytes));
        atomicMax(reinterpret_cast<unsigned long long*>(&out[(blockIdx.x * 4 + role) * 2 + 1]), static_cast<unsigned long long>(t1 - t0));
    }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int64_t nbytes = 32ll << 20;
    uint8_t* src;
    cudaMalloc(&src, nbytes);
    cudaMemset(src, 0, nbytes);
    float* sink;
    cudaMalloc(&sink, 4);
    long long* out;
    cudaMalloc(&out, sizeof(long long) * 8 * 160);
    EncodeFn enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &q);
    CUtensorMap tm;
    cuuint64_t dims[2] = {64, static_cast<cuuint64_t>(nbytes / 128)};  // [rows][64 bf16]
    cuuint64_t strides[1] = {128};
    cuuint32_t box[2] = {64, 64}, es[2] = {1, 1};
    enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, src, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int smem = 196608 + TMA_RING * TMA_SLOT + 1024 + 1024;
    cudaFuncSetAttribute(feed, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    struct C { Cfg c; int grid_div; const char* name; };
    const C cases[] = {
        {{8, 0, 16384, 0, 0, 8192, 0}, 1, "cp 8w"},
        {{4, 0, 16384, 0, 0, 8192, 0}, 1, "cp 4w"},
        {{8, 0, 16384, 0, 0, 8192, 0}, 2, "cp 8w, half the SMs"},
        {{0, 1, 16384, 0, 0, 8192, 0}, 1, "bulk 1 thr 16K"},
        {{0, 2, 16384, 0, 0, 8192, 0}, 1, "bulk 2 thr 16K"},
        {{0, 2, 4096, 0, 0, 8192, 0}, 1, "bulk 2 thr 4K"},
        {{0, 1, 16384, 0, 0, 8192, 0}, 2, "bulk 1 thr 16K, half the SMs"},
        {{0, 0, 16384, 1, 0, 8192, 0}, 1, "tma 2d 8K"},
        {{0, 0, 16384, 0, 8, 8192, 0}, 1, "ldg 8w"},
        {{0, 0, 16384, 0, 12, 8192, 0}, 1, "ldg 12w"},
        {{8, 1, 16384, 0, 0, 8192, 0}, 1, "cp 8w + bulk 1"},
        {{8, 2, 16384, 0, 0, 8192, 0}, 1, "cp 8w + bulk 2"},
        {{8, 0, 16384, 1, 0, 8192, 0}, 1, "cp 8w + tma"},
        {{8, 0, 16384, 0, 8, 8192, 0}, 1, "cp 8w + ldg 8w"},
        {{0, 1, 16384, 0, 8, 8192, 0}, 1, "bulk 1 + ldg 8w"},
        {{8, 0, 16384, 0, 0, 8192, 1}, 1, "cp 8w seq rows"},
        {{0, 0, 16384, 0, 8, 8192, 1}, 1, "ldg 8w seq rows"},
        {{8, 1, 16384, 0, 0, 8192, 1}, 1, "cp 8w seq + bulk 1"},
        {{16, 0, 16384, 0, 0, 8192, 0}, 1, "cp 16w"},
        {{16, 1, 16384, 0, 0, 8192, 0}, 1, "cp 16w + bulk 1"},
        {{16, 2, 16384, 0, 0, 8192, 0}, 1, "cp 16w + bulk 2"},
        {{8, 2, 8192, 0, 0, 8192, 0}, 1, "cp 8w + bulk 2 x 8K"},
    };
    const char* rn[4] = {"cp", "bulk", "tma", "ldg"};
    printf("# ubench_feed: 1 CTA/SM, 32 MB L2-resident source; B/clk per SM per role (bytes / role clocks), mean over CTAs\n");
    for (const C& cc : cases) {
        const int grid = sms / cc.grid_div;
        cudaMemset(out, 0, sizeof(long long) * 8 * 160);
        feed<<<grid, 1024, smem>>>(src, nbytes, tm, cc.c, out, sink);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("%s: error %s\n", cc.name, cudaGetErrorString(e)); return 1; }
        long long h[8 * 160];
        cudaMemcpy(h, out, sizeof(long long) * 8 * grid, cudaMemcpyDeviceToHost);
        printf("%-30s grid %3d:", cc.name, grid);
        double tot = 0, tmax = 0;
        for (int r = 0; r < 4; ++r) {
            double by = 0, ck = 0;
            for (int i = 0; i < grid; ++i) by += h[(i * 4 + r) * 2], ck += h[(i * 4 + r) * 2 + 1];
            if (by == 0) continue;
            printf("  %s %6.1f", rn[r], by / ck);
            tot += by / grid;
            if (ck / grid > tmax) tmax = ck / grid;
        }
        printf("  | total %6.1f B/clk per SM, chip %6.0f B/clk\n", tot / tmax, tot / tmax * grid);
    }
    return 0;
}
