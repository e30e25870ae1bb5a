// spmm_tc.cu -- bf16 N:M SpMM on the 5th-generation tensor cores (tcgen05 + TMEM), sm_100a.
//
// The method (Eq. 1 with readings R1-R4): for column group g (L output
// columns) C[:, gL:(g+1)L] = A_g . B'_g, where A_g = A[:, kabs(u, g)] gathers the
// selected k of every window.  Each group has its own selected-k set, so one MMA
// can only span the L columns of one group (SURVEY 7 "hard parts"): the kernel
// compacts A_g per group and issues one tcgen05.mma (M=128, N=L, K=16) per group
// and k-step, with the compacted operand in TMEM (A-from-TMEM "TS" form) so that
// the gathered bytes cross the shared-memory port once (read), never twice.
//
// Roles (288 threads, 1 CTA per SM, persistent over nothing -- one 128 x 128
// output tile per CTA):
//   warps 0-7  "gather": load the dense A panel (128 rows x BK) global -> regs ->
//              padded smem (row pitch BK*2+4 B: the 32 rows a warp touches at one
//              column hit 32 distinct banks), then per group build A_g rows
//              (thread = TMEM lane = token row) with LDS.32 + PRMT, store them with
//              tcgen05.st.32x32b into a double-buffered TMEM A region; after the
//              k loop they are the epilogue (tcgen05.ld -> cvt -> st.global).
//   warp 8     "control": TMEM alloc/dealloc; lane 0 issues the TMA loads of the
//              B' panel (one box per group, MN-major, swizzle = L*2 bytes, which is
//              the canonical UMMA MN-major layout) and the MMAs, and signals
//              completion with tcgen05.commit -> mbarrier.
// Paper structure kept: CTA tile over C with the k loop inside (Listing 1,
// P:241-268), double buffering (Listing 4), per-panel index table
// prefetch.  Everything else is B200-specific.
#include <cuda_bf16.h>

#include "common.cuh"

namespace nm {
namespace tc {

constexpr int BM = 128, BN = 128;
constexpr int GATHER_WARPS = 8, GATHER_THREADS = GATHER_WARPS * 32;
constexpr int THREADS = GATHER_THREADS + 32;
constexpr int B_STAGES = 3;
constexpr int BK_MAX = 128;     // dense k per panel
constexpr int BKW_MAX = 64;     // compressed rows per panel (padded to a multiple of 16)
constexpr int G_MAX = BN / 16;  // groups per tile (L >= 16)
constexpr int A_PITCH_MAX = BK_MAX * 2 + 4;
constexpr int A_STAGE_BYTES = BM * A_PITCH_MAX;            // 33,280
constexpr int B_STAGE_BYTES = BKW_MAX * BN * 2;            // 16 KB
constexpr int TBL_BYTES = G_MAX * BKW_MAX * 2;             // uint16 kloc table per panel
constexpr int LDG_PER_THREAD = BM * BK_MAX / 8 / GATHER_THREADS;  // 16-byte chunks: 8

struct Smem {
    // offsets (bytes) from the 1024-aligned base
    static constexpr int B = 0;                                   // B_STAGES x 16 KB (1024-aligned)
    static constexpr int A = B + B_STAGES * B_STAGE_BYTES;        // 2 x padded A panel
    static constexpr int T = A + 2 * A_STAGE_BYTES;               // 2 x kloc table
    static constexpr int BAR = (T + 2 * TBL_BYTES + 7) / 8 * 8;   // mbarriers
    static constexpr int NBAR = 2 * B_STAGES + 2 + 2 + 1;
    static constexpr int TMEM_SLOT = BAR + NBAR * 8;
    static constexpr int END = TMEM_SLOT + 16;
};
constexpr int SMEM_BYTES = Smem::END + 1024;

struct Params {
    const __nv_bfloat16* A;
    const uint8_t* D;
    void* C;
    int m, n, k, N, M, L;
    int q, wp, bk, bkw, bkw_pad, npanels;
    int c_bf16;
};

// ------------------------------------------------------------------ PTX
__device__ __forceinline__ void tmem_alloc(uint32_t* slot, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)), "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
// D[tmem] (+)= A[tmem] . B[smem]  (kind::f16, bf16 inputs, fp32 accumulate)
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
        "r"(a), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&v)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(v[0]),
                 "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr)
        : "memory");
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void bar_gather() { asm volatile("bar.sync 1, %0;" ::"n"(GATHER_THREADS) : "memory"); }

// UMMA shared-memory descriptor (SM100 version 1): start, LBO, SBO (>>4), layout type.
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
    d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
    d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
    d |= static_cast<uint64_t>(1) << 46;  // version
    d |= static_cast<uint64_t>(layout & 7) << 61;
    return d;
}

// ------------------------------------------------------------------ kernel
__global__ void __launch_bounds__(THREADS, 1)
    spmm_tc_bf16_kernel(const __grid_constant__ CUtensorMap tmB, const Params p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* sB = smem + Smem::B;
    uint8_t* sA = smem + Smem::A;
    uint16_t* sT = reinterpret_cast<uint16_t*>(smem + Smem::T);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Smem::BAR);
    uint64_t* b_full = bars;                   // [B_STAGES] TMA -> MMA
    uint64_t* b_free = bars + B_STAGES;        // [B_STAGES] MMA -> TMA
    uint64_t* a_full = bars + 2 * B_STAGES;    // [2] gather -> MMA (GATHER_THREADS arrivals)
    uint64_t* a_free = a_full + 2;             // [2] MMA -> gather
    uint64_t* acc_full = a_free + 2;           // MMA -> epilogue
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + Smem::TMEM_SLOT);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
    const int L = p.L, G = BN / L;
    const int bk = p.bk, bkw = p.bkw, bkwp = p.bkw_pad;
    const int a_pitch = bk * 2 + 4;
    const int a_cols = G * (bkwp / 2);  // TMEM columns of one A buffer

    if (warp == GATHER_WARPS) {
        if (lane == 0) {
            tma_prefetch_desc(&tmB);
            for (int s = 0; s < B_STAGES; ++s) {
                mbar_init(&b_full[s], 1);
                mbar_init(&b_free[s], 1);
            }
            for (int b = 0; b < 2; ++b) {
                mbar_init(&a_full[b], GATHER_THREADS);
                mbar_init(&a_free[b], 1);
            }
            mbar_init(acc_full, 1);
            fence_mbar_init();
        }
        __syncwarp();
        tmem_alloc(tmem_slot, 512);
    } else {
        // zero the B stages once: rows past the panel's bkw (k padding to 16) stay +0.0
        for (int i = tid; i < B_STAGES * B_STAGE_BYTES / 16; i += GATHER_THREADS)
            reinterpret_cast<uint4*>(sB)[i] = make_uint4(0, 0, 0, 0);
        fence_proxy_async_smem();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == GATHER_WARPS) {
        // ===================== control warp: TMA (B') + MMA issue =====================
        if (lane == 0) {
            const int rb = (L >= 64 ? 64 : L) * 2;            // bytes per B row inside one atom
            const int atoms = (L * 2 + 127) / 128;           // 64-column atoms per group (L > 64)
            const int gbytes = bkwp * L * 2;                  // one group's B_g region
            const uint32_t layout = rb == 128 ? 2u : rb == 64 ? 4u : 6u;  // SW128 / SW64 / SW32
            const uint32_t sbo = 8u * rb, lbo = static_cast<uint32_t>(bkwp * 128);
            const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) |
                                   (static_cast<uint32_t>(L >> 3) << 17) | (static_cast<uint32_t>(BM >> 4) << 24);
            const uint32_t stage_tx = static_cast<uint32_t>(G * atoms * bkw * rb);
            auto issue_b = [&](int panel) {
                const int s = panel % B_STAGES;
                mbar_arrive_expect_tx(&b_full[s], stage_tx);
                uint8_t* dst = sB + s * B_STAGE_BYTES;
                for (int g = 0; g < G; ++g)
                    for (int a = 0; a < atoms; ++a)
                        tma_load_2d(dst + g * gbytes + a * bkwp * 128, &tmB, &b_full[s], n0 + g * L + a * 64,
                                    panel * bkw);
            };
            for (int i = 0; i < B_STAGES - 1 && i < p.npanels; ++i) issue_b(i);
            for (int panel = 0; panel < p.npanels; ++panel) {
                const int nxt = panel + B_STAGES - 1;
                if (nxt < p.npanels) {
                    if (nxt >= B_STAGES) mbar_wait(&b_free[nxt % B_STAGES], ((nxt / B_STAGES) - 1) & 1);
                    issue_b(nxt);
                }
                const int s = panel % B_STAGES, ab = panel & 1;
                mbar_wait(&b_full[s], (panel / B_STAGES) & 1);
                mbar_wait(&a_full[ab], (panel >> 1) & 1);
                tc_fence_after();
                const uint32_t sb = smem_u32(sB + s * B_STAGE_BYTES);
                const uint32_t abase = tmem + BN + ab * a_cols;
                for (int g = 0; g < G; ++g) {
                    for (int kk = 0; kk < bkwp / 16; ++kk) {
                        const uint64_t bd = smem_desc(sb + g * gbytes + kk * 16 * rb, lbo, sbo, layout);
                        mma_ts(tmem + g * L, abase + g * (bkwp / 2) + kk * 8, bd, idesc, (panel | kk) ? 1u : 0u);
                    }
                }
                tc_commit(&a_free[ab]);
                tc_commit(&b_free[s]);
            }
            tc_commit(acc_full);
        }
        __syncwarp();
    } else {
        // ===================== gather warps (then epilogue) =====================
        const int quarter = warp & 3;            // TMEM lane quarter = rows quarter*32 .. +31
        const int ghalf = warp >> 2;             // groups ghalf, ghalf+2, ...
        const int row = quarter * 32 + lane;     // tile row = TMEM lane
        const uint32_t lane_addr = static_cast<uint32_t>(quarter * 32) << 16;
        const int chunks_per_row = bk / 8;       // 16-byte chunks per A panel row
        const int windows = p.k / p.M;

        uint4 ldg[LDG_PER_THREAD];
        uint16_t dreg[(G_MAX * BKW_MAX + GATHER_THREADS - 1) / GATHER_THREADS];
        constexpr int DPT = (G_MAX * BKW_MAX + GATHER_THREADS - 1) / GATHER_THREADS;

        // A panel tile, row-major units of 16 bytes: unit -> (row = unit / cpr, chunk = unit % cpr)
        auto load_a = [&](int panel) {
            const int k0 = panel * bk;
            const int kv = min(bk, p.k - k0);
#pragma unroll
            for (int i = 0; i < LDG_PER_THREAD; ++i) {
                const int unit = i * GATHER_THREADS + tid;
                const int r = unit / chunks_per_row, c = unit - r * chunks_per_row;
                uint4 v = make_uint4(0, 0, 0, 0);
                if (r < BM && m0 + r < p.m && c * 8 < kv)
                    v = __ldg(reinterpret_cast<const uint4*>(p.A + static_cast<int64_t>(m0 + r) * p.k + k0 + c * 8));
                ldg[i] = v;
            }
        };
        auto store_a = [&](int panel) {
            uint8_t* dst = sA + (panel & 1) * A_STAGE_BYTES;
#pragma unroll
            for (int i = 0; i < LDG_PER_THREAD; ++i) {
                const int unit = i * GATHER_THREADS + tid;
                const int r = unit / chunks_per_row, c = unit - r * chunks_per_row;
                if (r < BM) {
                    uint32_t* d = reinterpret_cast<uint32_t*>(dst + r * a_pitch + c * 16);
                    d[0] = ldg[i].x;
                    d[1] = ldg[i].y;
                    d[2] = ldg[i].z;
                    d[3] = ldg[i].w;
                }
            }
            // the pad word of each row is the zero source for k padding (sentinel kloc = bk)
            if (tid < BM) *reinterpret_cast<uint32_t*>(dst + tid * a_pitch + bk * 2) = 0u;
        };
        // per-panel kloc table: T[g][u] = dense column of compressed row u of group g inside the panel
        auto load_d = [&](int panel) {
            const int u0 = panel * bkw;
            const int wtot = windows * p.N;
#pragma unroll
            for (int r = 0; r < DPT; ++r) {
                const int e = r * GATHER_THREADS + tid;
                const int g = e / BKW_MAX, u = e % BKW_MAX;
                uint16_t v = static_cast<uint16_t>(bk);  // sentinel -> zero word
                if (g < G && u < bkw && u0 + u < wtot) {
                    const int gg = (n0 / L) + g;
                    if (gg < p.q) {
                        const int d = p.D[static_cast<int64_t>(u0 + u) * p.q + gg];
                        v = static_cast<uint16_t>((u / p.N) * p.M + d);
                    }
                }
                dreg[r] = v;
            }
        };
        auto store_d = [&](int panel) {
            uint16_t* t = sT + (panel & 1) * (G_MAX * BKW_MAX);
#pragma unroll
            for (int r = 0; r < DPT; ++r) t[r * GATHER_THREADS + tid] = dreg[r];
        };

        load_a(0);
        load_d(0);
        store_a(0);
        store_d(0);

        for (int panel = 0; panel < p.npanels; ++panel) {
            bar_gather();  // panel's A tile + table visible; previous gathers done
            const bool more = panel + 1 < p.npanels;
            if (more) {
                load_a(panel + 1);
                load_d(panel + 1);
            }
            const int ab = panel & 1;
            if (panel >= 2) {
                mbar_wait(&a_free[ab], ((panel - 2) >> 1) & 1);
                tc_fence_after();
            }
            const uint8_t* arow = sA + ab * A_STAGE_BYTES + row * a_pitch;
            const uint16_t* tbl = sT + ab * (G_MAX * BKW_MAX);
            for (int g = ghalf; g < G; g += 2) {
                const uint16_t* tg = tbl + g * BKW_MAX;
                for (int j = 0; j < bkwp / 16; ++j) {
                    const uint4 t0 = *reinterpret_cast<const uint4*>(tg + j * 16);
                    const uint4 t1 = *reinterpret_cast<const uint4*>(tg + j * 16 + 8);
                    const uint32_t kw[8] = {t0.x, t0.y, t0.z, t0.w, t1.x, t1.y, t1.z, t1.w};
                    uint32_t v[8];
#pragma unroll
                    for (int c = 0; c < 8; ++c) {
                        const uint32_t ka = kw[c] & 0xFFFFu, kb = kw[c] >> 16;
                        const uint32_t wa = *reinterpret_cast<const uint32_t*>(arow + ((ka >> 1) << 2));
                        const uint32_t wb = *reinterpret_cast<const uint32_t*>(arow + ((kb >> 1) << 2));
                        const uint32_t sel = ((ka & 1u) ? 0x32u : 0x10u) | ((kb & 1u) ? 0x7600u : 0x5400u);
                        v[c] = __byte_perm(wa, wb, sel);
                    }
                    tmem_st8(tmem + lane_addr + BN + ab * a_cols + g * (bkwp / 2) + j * 8, v);
                }
            }
            tmem_wait_st();
            tc_fence_before();
            mbar_arrive(&a_full[ab]);
            if (more) {
                store_a(panel + 1);
                store_d(panel + 1);
            }
        }

        // ===================== epilogue: TMEM -> registers -> global =====================
        mbar_wait(acc_full, 0);
        tc_fence_after();
        const int grow = m0 + row;
        const int cols_half = BN / 2;
        for (int cb = 0; cb < cols_half; cb += 16) {
            const int col = ghalf * cols_half + cb;
            uint32_t v[16];
            tmem_ld16(tmem + lane_addr + col, v);
            tmem_wait_ld();
            const int gc = n0 + col;
            if (grow < p.m && gc < p.n) {
                if (p.c_bf16) {
                    uint32_t pk[8];
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        __nv_bfloat162 h = __floats2bfloat162_rn(__uint_as_float(v[2 * i]), __uint_as_float(v[2 * i + 1]));
                        pk[i] = *reinterpret_cast<uint32_t*>(&h);
                    }
                    uint4* dst = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(p.C) + static_cast<int64_t>(grow) * p.n + gc);
                    dst[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
                    dst[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
                } else {
                    uint4* dst = reinterpret_cast<uint4*>(static_cast<float*>(p.C) + static_cast<int64_t>(grow) * p.n + gc);
#pragma unroll
                    for (int i = 0; i < 4; ++i) dst[i] = make_uint4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
                }
            }
        }
        tc_fence_before();
    }
    __syncthreads();
    if (warp == GATHER_WARPS) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

}  // namespace tc

bool tc_bf16_applicable(const void* A, const void* Bv, const void* C, int64_t m, int64_t n, int64_t k, int N, int M,
                        int L) {
    if (!(L == 16 || L == 32 || L == 64 || L == 128)) return false;
    if (M % 8 != 0 || M > tc::BK_MAX || N > tc::BKW_MAX) return false;
    if (n % 8 != 0 || k % 8 != 0) return false;
    if ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(Bv) | reinterpret_cast<uintptr_t>(C)) & 15)
        return false;
    if (m >= (1ll << 31) || n >= (1ll << 31) || k >= (1ll << 31)) return false;
    return true;
}

// Panel geometry: WP whole windows (never straddling one), BK = WP*M <= 128 dense k,
// BKW = WP*N <= 64 compressed rows, preferring BKW % 16 == 0 (no zero-padded MMA steps).
void tc_bf16_geometry(int N, int M, int* wp, int* bk, int* bkw, int* bkw_pad) {
    int best = 1, best_score = -1;
    for (int w = 1; w * M <= tc::BK_MAX && w * N <= tc::BKW_MAX; ++w) {
        const int kw = w * N, pad = (kw + 15) / 16 * 16;
        const int score = kw * 1000 / pad * 100 + kw;  // efficiency first, then size
        if (score > best_score) {
            best_score = score;
            best = w;
        }
    }
    *wp = best;
    *bk = best * M;
    *bkw = best * N;
    *bkw_pad = (*bkw + 15) / 16 * 16;
}

nm_status tc_bf16_launch(const void* A, const void* Bv, const uint8_t* D, void* C, bool c_bf16, int64_t m, int64_t n,
                         int64_t k, int N, int M, int L, cudaStream_t s) {
    using namespace tc;
    Params p{};
    p.A = static_cast<const __nv_bfloat16*>(A);
    p.D = D;
    p.C = C;
    p.m = static_cast<int>(m);
    p.n = static_cast<int>(n);
    p.k = static_cast<int>(k);
    p.N = N;
    p.M = M;
    p.L = L;
    p.q = static_cast<int>(n / L);
    p.c_bf16 = c_bf16 ? 1 : 0;
    tc_bf16_geometry(N, M, &p.wp, &p.bk, &p.bkw, &p.bkw_pad);
    const int windows = static_cast<int>(k / M);
    p.npanels = (windows + p.wp - 1) / p.wp;
    const int64_t w = k / M * N;
    CUtensorMap tmB;
    const int box_cols = L >= 64 ? 64 : L;
    const int sw = box_cols * 2;  // 32 / 64 / 128 B swizzle = the group's row width
    nm_status st = make_tma_2d(&tmB, Bv, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, w, n, p.bkw, box_cols, sw);
    if (st) return st;
    static bool attr = false;
    if (!attr) {
        NM_CUDA_TRY(cudaFuncSetAttribute(spmm_tc_bf16_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES));
        attr = true;
    }
    const dim3 grid(static_cast<unsigned>(ceil_div(n, BN)), static_cast<unsigned>(ceil_div(m, BM)));
    spmm_tc_bf16_kernel<<<grid, THREADS, SMEM_BYTES, s>>>(tmB, p);
    NM_LAUNCH_CHECK("spmm_tc_bf16_kernel");
    return NM_OK;
}

}  // namespace nm
