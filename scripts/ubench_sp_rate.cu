// Micro-benchmark: throughput of tcgen05.mma.sp kind::f16 (the slot kernel's contraction) on
// B200, and how concurrent shared-memory writes (the token gather) slow it.  One CTA per SM,
// one elected thread issues R "stages" back to back (per stage and half: two MMAs M = 128,
// K = 32 slots, N = NT tokens; the B operand ring of 4 stages is the slot kernel's MN-major
// 128-B-swizzled layout, the A images its 64-B-swizzled K-major layout), one commit at the
// end.  Writers (warps 0-7) meanwhile store to shared memory: 0 none, 1 st.shared.v4 from
// registers, 2 16-B cp.async from an L2-resident buffer (the gather's instruction), 3 tcgen05.st
// into spare TMEM columns (4 warps, one per lane quarter), counting
// bytes until the MMA thread raises a flag.
//   mode 0: sparse SS, H halves (A images differ, B shared)   mode 1: dense SS K = 16 (same bytes)
//   mode 2: sparse, A operand from TMEM (TS)
//   mode 3 / 4: mode 0 + a metadata tcgen05.cp per half every second stage, read by the next MMAs / unread
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_sp_rate ubench_sp_rate.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>

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
__device__ __forceinline__ bool elect() {
    uint32_t p;
    asm volatile("{\n\t.reg .pred q;\n\telect.sync _|q, 0xffffffff;\n\tselp.u32 %0,1,0,q;\n\t}" : "=r"(p));
    return p;
}
__device__ __forceinline__ bool try_wait(uint64_t* b, uint32_t ph) {
    uint32_t ok;
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}"
                 : "=r"(ok) : "r"(su32(b)), "r"(ph) : "memory");
    return ok;
}

constexpr int SLOTS = 64, A_BYTES = 8192, E_BYTES = 2048, RING = 4, WR_BYTES = 16384;

struct Args {
    int mode, nt, h, reps, writer;
    const uint8_t* gsrc;  // writer 2 source (L2 resident), 1 MB
    long long* out;       // per CTA: [mma clk, writer bytes, ns]
};

__global__ void __launch_bounds__(288, 1) bench(Args a) {
    extern __shared__ __align__(1024) uint8_t sm_raw[];
    uint8_t* sm = sm_raw + ((1024u - (su32(sm_raw) & 1023u)) & 1023u);
    const int NT = a.nt, H = a.h;
    const int B_BYTES = SLOTS * ((NT + 63) / 64) * 128;
    uint8_t* sB = sm;
    uint8_t* sA = sB + RING * B_BYTES;                 // RING x H x A
    uint8_t* sE = sA + RING * H * A_BYTES;             // H x E (metadata source)
    uint8_t* sWr = sE + H * E_BYTES;                   // writers' region
    uint64_t* bar = reinterpret_cast<uint64_t*>(sWr + WR_BYTES);
    volatile int* done = reinterpret_cast<volatile int*>(bar + 1);
    uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 2);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // operands: arbitrary finite bf16 (0x3c00 pattern), metadata 0x44 (elements 0, 1 of every quad)
    for (int i = tid; i < (RING * B_BYTES + RING * H * A_BYTES) / 4; i += blockDim.x)
        reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
    for (int i = tid; i < H * E_BYTES / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sE)[i] = 0x44444444u;
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
        *done = 0;
    }
    if (warp == 8) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *slot;
    // TMEM: D at h * NT (H x NT <= 448), metadata at 448 + 4 h, TS A operand at 456 + 8 h
    const uint32_t MCOL = 448, ACOL = 464;
    if (warp == 8) {
        long long t0 = 0, t1 = 0;
        unsigned long long g0 = 0, g1 = 0;
        if (elect()) {
            for (int h = 0; h < H; ++h)
                asm volatile("tcgen05.cp.cta_group::1.128x128b [%0], %1;" ::"r"(tmem + MCOL + 4 * h),
                             "l"(sdesc(su32(sE + h * E_BYTES), 2048, 128, 0)) : "memory");
            const uint32_t sp = a.mode == 1 ? 0u : 1u;
            const uint32_t idesc = (sp << 2) | (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) |
                                   (static_cast<uint32_t>(NT >> 3) << 17) | (static_cast<uint32_t>(128 >> 4) << 24);
            const uint64_t b0 = sdesc(su32(sB), SLOTS * 128, 1024, 2);
            const uint64_t a0 = sdesc(su32(sA), 16, 512, 4);
            asm volatile("mov.u64 %0, %%clock64;" : "=l"(t0));
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
            for (int it = 0; it < a.reps; ++it) {
                const int s = it & (RING - 1);
                const uint64_t bo = static_cast<uint64_t>(s * (B_BYTES >> 4));
                // modes 3 / 4: the slot kernel's metadata delivery -- one tcgen05.cp 128x128b per half on
                // every even stage (a stage pair's metadata)
                if ((a.mode == 3 || a.mode == 4) && !(it & 1))
                    for (int h = 0; h < H; ++h) {
                        // mode 3: into the columns the next MMAs read; mode 4: into columns no MMA reads
                        asm volatile("tcgen05.cp.cta_group::1.128x128b [%0], %1;" ::"r"(tmem + MCOL + (a.mode == 4 ? 8 : 0) + 4 * h),
                                     "l"(sdesc(su32(sE + h * E_BYTES), 2048, 128, 0)) : "memory");
                    }
                for (int h = 0; h < H; ++h) {
                    const uint64_t ao = static_cast<uint64_t>((s * H + h) * (A_BYTES >> 4));
                    for (int j = 0; j < 2; ++j) {
                        const uint32_t acc = (it | j) ? 1u : 0u;
                        const uint64_t bd = b0 + bo + ((4096u * j) >> 4);
                        if (a.mode == 0 || a.mode == 3 || a.mode == 4) {
                            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                         "tcgen05.mma.sp.cta_group::1.kind::f16 [%0], %1, %2, [%5], %3, p;\n\t}" ::"r"(tmem + h * NT),
                                         "l"(a0 + ao + ((32u * j) >> 4)), "l"(bd), "r"(idesc | j), "r"(acc), "r"(tmem + MCOL + 4 * h)
                                         : "memory");
                        } else if (a.mode == 2) {
                            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                         "tcgen05.mma.sp.cta_group::1.kind::f16 [%0], [%1], %2, [%5], %3, p;\n\t}" ::"r"(tmem + h * NT),
                                         "r"(tmem + ACOL + 8 * h), "l"(bd), "r"(idesc | j), "r"(acc), "r"(tmem + MCOL + 4 * h)
                                         : "memory");
                        } else {  // dense K = 16: two MMAs per K = 32 half-step (same B bytes per clk as sparse K = 32)
                            for (int q = 0; q < 2; ++q)
                                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                             "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem + h * NT),
                                             "l"(a0 + ao + ((32u * j) >> 4)), "l"(bd + ((2048u * q) >> 4)), "r"(idesc), "r"((acc | q) ? 1u : 0u)
                                             : "memory");
                        }
                    }
                }
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar)) : "memory");
            while (!try_wait(bar, 0)) {
            }
            asm volatile("mov.u64 %0, %%clock64;" : "=l"(t1));
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
            *done = 1;
            a.out[3 * blockIdx.x + 0] = t1 - t0;
            a.out[3 * blockIdx.x + 2] = static_cast<long long>(g1 - g0);
        }
        __syncwarp();
    } else if (a.writer) {
        long long bytes = 0;
        const uint32_t dst = su32(sWr) + (warp * 32 + lane) * 16;  // 8 warps x 512 B = 4 KB per round
        if (a.writer == 1) {
            uint4 v = make_uint4(tid, tid + 1, tid + 2, tid + 3);
            while (!*done) {
#pragma unroll
                for (int r = 0; r < 4; ++r)
                    asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(dst + r * 4096), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                                 : "memory");
                bytes += 4 * 16;
            }
        } else if (a.writer == 3) {  // tcgen05.st into spare TMEM columns 480..495 (warps 0-3: lane quarters)
            if (warp < 4) {
                uint4 v[4];
                for (int i = 0; i < 4; ++i) v[i] = make_uint4(tid, tid + i, 0x3c003c00u, i);
                const uint32_t ta = tmem + (static_cast<uint32_t>(warp * 32) << 16) + 480;
                while (!*done) {
                    asm volatile(
                        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(ta),
                        "r"(v[0].x), "r"(v[0].y), "r"(v[0].z), "r"(v[0].w), "r"(v[1].x), "r"(v[1].y), "r"(v[1].z), "r"(v[1].w),
                        "r"(v[2].x), "r"(v[2].y), "r"(v[2].z), "r"(v[2].w), "r"(v[3].x), "r"(v[3].y), "r"(v[3].z), "r"(v[3].w)
                        : "memory");
                    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                    bytes += 64;  // per lane
                }
            }
        } else {
            int r0 = 0;
            while (!*done) {
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    const uint8_t* src = a.gsrc + ((((r0 + r) * 37 + blockIdx.x * 11) & 255) * 4096) + (warp * 32 + lane) * 16;
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + r * 4096), "l"(src) : "memory");
                }
                asm volatile("cp.async.wait_all;" ::: "memory");
                r0 += 4;
                bytes += 4 * 16;
            }
        }
        atomicAdd(reinterpret_cast<unsigned long long*>(&a.out[3 * blockIdx.x + 1]), static_cast<unsigned long long>(bytes));
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 8) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    }
}

int main(int argc, char** argv) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint8_t* g;
    cudaMalloc(&g, 1 << 20);
    cudaMemset(g, 0x11, 1 << 20);
    long long* out;
    cudaMalloc(&out, sizeof(long long) * 3 * sms);
    const int reps = 2048;
    struct Case { int mode, nt, h, writer; const char* name; };
    const Case cases[] = {
        {0, 64, 1, 0, "sparse SS"},  {0, 128, 1, 0, "sparse SS"}, {0, 192, 1, 0, "sparse SS"}, {0, 256, 1, 0, "sparse SS"},
        {0, 192, 2, 0, "sparse SS"}, {0, 224, 2, 0, "sparse SS"},
        {1, 128, 1, 0, "dense SS "}, {1, 256, 1, 0, "dense SS "}, {1, 192, 2, 0, "dense SS "},
        {2, 128, 1, 0, "sparse TS"}, {2, 256, 1, 0, "sparse TS"}, {2, 192, 2, 0, "sparse TS"},
        {0, 192, 2, 1, "sparse SS"}, {0, 192, 2, 2, "sparse SS"}, {0, 256, 1, 1, "sparse SS"}, {0, 256, 1, 2, "sparse SS"},
        {2, 192, 2, 1, "sparse TS"}, {2, 192, 2, 2, "sparse TS"}, {2, 256, 1, 2, "sparse TS"},
        {1, 256, 1, 1, "dense SS "}, {1, 256, 1, 2, "dense SS "},
        {3, 192, 2, 0, "sp SS+cp "}, {4, 192, 2, 0, "sp SS+cp4"}, {3, 256, 1, 0, "sp SS+cp "}, {4, 256, 1, 0, "sp SS+cp4"},
        {3, 160, 2, 0, "sp SS+cp "},
        {2, 192, 2, 3, "sparse TS"}, {0, 192, 2, 3, "sparse SS"}, {2, 256, 1, 3, "sparse TS"},
    };
    printf("# ubench_sp_rate: %d CTAs x %d stages (per stage and half: 2 x M128 K32 sparse MMAs or 4 x K16 dense)\n", sms, reps);
    printf("# clk/stage-half = MMA clk per (half, 64 slots); ideal sparse = NT/2 clk... (2:4 at 2x dense: 128x NT x 64 / 8192 x 2 / 2)\n");
    for (const Case& c : cases) {
        const int B_BYTES = SLOTS * ((c.nt + 63) / 64) * 128;
        const int smem = RING * B_BYTES + RING * c.h * A_BYTES + c.h * E_BYTES + WR_BYTES + 64 + 1024;
        if (smem > 232448) { printf("skip %s nt %d h %d (smem %d)\n", c.name, c.nt, c.h, smem); continue; }
        cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaMemset(out, 0, sizeof(long long) * 3 * sms);
        Args a{c.mode, c.nt, c.h, reps, c.writer, g, out};
        bench<<<sms, 288, smem>>>(a);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("%s nt %d: error %s\n", c.name, c.nt, cudaGetErrorString(e)); return 1; }
        long long* h = (long long*)malloc(sizeof(long long) * 3 * sms);
        cudaMemcpy(h, out, sizeof(long long) * 3 * sms, cudaMemcpyDeviceToHost);
        double clk = 0, wb = 0, ns = 0;
        for (int i = 0; i < sms; ++i) clk += h[3 * i], wb += h[3 * i + 1], ns += h[3 * i + 2];
        clk /= sms; wb /= sms; ns /= sms;
        const double per = clk / (reps * c.h);
        // bytes the MMA reads per (half, stage): B tile + A image (sparse: 8 KB of values; dense mode reads it too)
        const double rd = B_BYTES + (c.mode == 2 ? 0 : A_BYTES);
        const double ideal = c.nt * 64.0 * 128 * 2 / (c.mode == 1 ? 8192.0 : 16384.0);
        printf("%s NT %3d H %d writer %d: %7.1f clk per half-stage (ideal %5.1f, %4.0f%%), MMA smem read %5.1f B/clk, writer %6.1f B/clk, %.2f GHz\n",
               c.name, c.nt, c.h, c.writer, per, ideal, 100 * ideal / per, rd / per, wb / clk, clk / ns);
        free(h);
    }
    return 0;
}
