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
// Warp roles (one 128 x BN output tile per CTA, 1 CTA per SM):
//   warps 0-3   "loader":  dense A panel (128 rows x BK) global -> regs -> padded
//               smem (row pitch BK*2+4 B, so the 32 rows a warp touches at one
//               column hit 32 distinct banks) + the per-panel cell table built
//               from D (index prefetch); double-buffered (Listing 4).
//   warps 4-15  "gather":  per (group, 8-cell block) item: 2 LDS.32 + 1 PRMT per
//               cell (thread = TMEM lane = token row), tcgen05.st.32x32b into a
//               double-buffered TMEM A region.
//   warp 16     "control": TMEM alloc/dealloc; lane 0 issues the TMA loads of the
//               B' panel (one box per group, MN-major, swizzle = L*2 bytes -- the
//               canonical UMMA MN-major layout) and the MMAs; tcgen05.commit ->
//               mbarriers release TMEM A buffers, B stages and the accumulator.
//   warps 0-15  epilogue: tcgen05.ld -> cvt -> st.global.
// Paper structure kept: CTA tile over C with the k loop inside (Listing 1,
// P:241-268), double buffering (Listing 4), per-panel index prefetch
// (P:546).  Everything else is B200-specific.
#include <cuda_bf16.h>

#include <cstdlib>

#include "tcgen05.cuh"

namespace nm {
namespace tc {

constexpr int BM = 128;
constexpr int LOADER_WARPS = 4, GATHER_WARPS = 12;
constexpr int LOADER_THREADS = LOADER_WARPS * 32, GATHER_THREADS = GATHER_WARPS * 32;
constexpr int CONTROL_WARP = LOADER_WARPS + GATHER_WARPS;
constexpr int THREADS = (CONTROL_WARP + 1) * 32;  // 544
constexpr int B_STAGES = 3;
// TMEM A buffers (gathers run up to NAB-1 panels ahead of the MMA) and B' panel rows:
// BN = 128 -> 3 buffers, BKW <= 64; BN = 256 -> 2 buffers, BKW <= 32 (512 TMEM columns).
template <int BN> constexpr int nab() { return BN == 256 ? 2 : 3; }
template <int BN> constexpr int bkw_cap() { return BN == 256 ? 32 : 64; }
constexpr int BK_MAX = 128;   // dense k per panel
constexpr int BKW_MAX = 64;   // compressed rows per panel (padded to a multiple of 16)
constexpr int CELLS_MAX = 256;  // (group, u-pair) cells per panel: G * bkw_pad / 2 <= (512 - BN) / 2
constexpr int A_PITCH_MAX = BK_MAX * 2 + 4;
constexpr int A_STAGE_BYTES = (BM * A_PITCH_MAX + 1023) / 1024 * 1024;  // 33,792 (keeps the next region aligned)
constexpr int TBL_WORDS = 2 * CELLS_MAX;         // [sel | offA << 16][offB] per cell (uint32)
constexpr int TBL_BYTES = TBL_WORDS * 4;
constexpr int LD_UNITS = BM * BK_MAX / 8 / LOADER_THREADS;  // 16-byte units per loader thread: 16
constexpr int A_STAGES = 2;                                    // TMA staging ring for the dense A panel
constexpr int STG_A_BYTES = BM * BK_MAX * 2;                   // 32 KB dense A panel
constexpr int STG_BYTES = STG_A_BYTES + TBL_BYTES;             // + the panel's prepacked cell table

template <int BN>
struct Smem {
    static constexpr int B_STAGE_BYTES = bkw_cap<BN>() * BN * 2;
    static constexpr int B = 0;                               // B_STAGES B' panels (1024-aligned)
    static constexpr int A = B + B_STAGES * B_STAGE_BYTES;    // 2 padded A panels
    static constexpr int STG = A + 2 * A_STAGE_BYTES;         // A_STAGES dense TMA panels (1024-aligned)
    static constexpr int T = STG + A_STAGES * STG_BYTES;      // 2 cell tables
    static constexpr int BAR = T + 2 * TBL_BYTES;             // mbarriers
    static constexpr int NBAR = 2 * B_STAGES + 2 * A_STAGES + 2 * 2 + 2 * nab<BN>() + 1;
    static constexpr int TMEM_SLOT = BAR + NBAR * 8;
    static constexpr int END = TMEM_SLOT + 16;
    static constexpr int BYTES = END + 1024;
};

struct Params {
    const __nv_bfloat16* A;
    const uint32_t* tbl;  // prepacked cell tables [n tiles][npanels][3][CELLS_MAX]
    void* C;
    int m, n, k, N, M, L;
    int q, wp, bk, bkw, bkw_pad, npanels;
    int c_bf16;
};

// ------------------------------------------------------------------ kernel
template <int BN>
__global__ void __launch_bounds__(THREADS, 1)
    spmm_tc_bf16_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                        const Params p) {
    using S = Smem<BN>;
    constexpr int NAB = nab<BN>();
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* sB = smem + S::B;
    uint8_t* sA = smem + S::A;
    uint8_t* sStg = smem + S::STG;
    uint32_t* sT = reinterpret_cast<uint32_t*>(smem + S::T);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S::BAR);
    uint64_t* b_full = bars;                 // [B_STAGES] TMA -> MMA
    uint64_t* b_free = bars + B_STAGES;      // [B_STAGES] MMA -> TMA
    uint64_t* s_full = bars + 2 * B_STAGES;  // [2] loader -> gather (A panel + table in smem)
    uint64_t* s_free = s_full + 2;           // [2] gather -> loader
    uint64_t* a_full = s_free + 2;           // [NAB] gather -> MMA (TMEM A buffer written)
    uint64_t* a_free = a_full + NAB;         // [NAB] MMA -> gather (TMEM A buffer consumed)
    uint64_t* acc_full = a_free + NAB;       // MMA -> epilogue
    uint64_t* g_full = acc_full + 1;         // [A_STAGES] TMA (dense A panel) -> loaders
    uint64_t* g_free = g_full + A_STAGES;    // [A_STAGES] loaders -> TMA
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + S::TMEM_SLOT);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
    const int L = p.L, G = BN / L;
    const int bk = p.bk, bkw = p.bkw, bkwp = p.bkw_pad;
    const int a_pitch = bk * 2 + 4;
    const int cells_g = bkwp / 2;      // cells per group per panel
    const int a_cols = G * cells_g;    // TMEM columns of one A buffer

    if (warp == CONTROL_WARP) {
        if (lane == 0) {
            tma_prefetch_desc(&tmB);
            tma_prefetch_desc(&tmA);
            for (int s = 0; s < B_STAGES; ++s) {
                mbar_init(&b_full[s], 1);
                mbar_init(&b_free[s], 1);
            }
            for (int b = 0; b < 2; ++b) {
                mbar_init(&s_full[b], LOADER_THREADS);
                mbar_init(&s_free[b], GATHER_THREADS);
            }
            for (int b = 0; b < NAB; ++b) {
                mbar_init(&a_full[b], GATHER_THREADS);
                mbar_init(&a_free[b], 1);
            }
            mbar_init(acc_full, 1);
            for (int b = 0; b < A_STAGES; ++b) {
                mbar_init(&g_full[b], 1);
                mbar_init(&g_free[b], LOADER_THREADS);
            }
            fence_mbar_init();
        }
        __syncwarp();
        tmem_alloc(tmem_slot, 512);
    } else {
        // zero the B stages once: rows past the panel's bkw (k padding to 16) stay +0.0
        for (int i = tid; i < B_STAGES * S::B_STAGE_BYTES / 16; i += CONTROL_WARP * 32)
            reinterpret_cast<uint4*>(sB)[i] = make_uint4(0, 0, 0, 0);
        fence_proxy_async_smem();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == CONTROL_WARP) {
        // ===================== control: TMA (B', A panel, cell table) + MMA issue =====================
        // The whole warp runs the loop (warp-uniform values stay in uniform registers);
        // one elected lane issues TMA and MMA instructions.
        const bool leader = elect_one();
        const int rb = (L >= 64 ? 64 : L) * 2;            // bytes per B row inside one atom
        const int atoms = (L * 2 + 127) / 128;           // 64-column atoms per group (L > 64)
        const int gbytes = bkwp * L * 2;                  // one group's B_g region
        const uint32_t layout = rb == 128 ? 2u : rb == 64 ? 4u : 6u;  // SW128 / SW64 / SW32
        const uint32_t sbo = 8u * rb, lbo = static_cast<uint32_t>(bkwp * 128);
        const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) |
                               (static_cast<uint32_t>(L >> 3) << 17) | (static_cast<uint32_t>(BM >> 4) << 24);
        const uint32_t stage_tx = static_cast<uint32_t>(G * atoms * bkw * rb);
        const uint32_t a_tx = static_cast<uint32_t>(BM * bk * 2 + TBL_BYTES);
        const uint32_t* tsrc = p.tbl + static_cast<int64_t>(blockIdx.x) * p.npanels * TBL_WORDS;
        const uint64_t gstep = static_cast<uint64_t>(gbytes >> 4), kstep = static_cast<uint64_t>((16 * rb) >> 4);
        const int nk = bkwp / 16;
        auto issue_b = [&](int panel) {
            if (leader) {
                const int s = panel % B_STAGES;
                mbar_arrive_expect_tx(&b_full[s], stage_tx);
                uint8_t* dst = sB + s * S::B_STAGE_BYTES;
                for (int g = 0; g < G; ++g)
                    for (int a = 0; a < atoms; ++a)
                        tma_load_2d(dst + g * gbytes + a * bkwp * 128, &tmB, &b_full[s], n0 + g * L + a * 64,
                                    panel * bkw);
            }
        };
        auto issue_a = [&](int panel) {
            if (leader) {
                const int s = panel % A_STAGES;
                mbar_arrive_expect_tx(&g_full[s], a_tx);
                tma_load_2d(sStg + s * STG_BYTES, &tmA, &g_full[s], panel * bk, m0);
                bulk_load(sStg + s * STG_BYTES + STG_A_BYTES, tsrc + static_cast<int64_t>(panel) * TBL_WORDS,
                          TBL_BYTES, &g_full[s]);
            }
        };
        for (int i = 0; i < A_STAGES && i < p.npanels; ++i) issue_a(i);
        int a_next = A_STAGES;  // next dense A panel to stage
        for (int i = 0; i < B_STAGES - 1 && i < p.npanels; ++i) issue_b(i);
        for (int panel = 0; panel < p.npanels; ++panel) {
            const int nxt = panel + B_STAGES - 1;
            if (nxt < p.npanels) {
                if (nxt >= B_STAGES) mbar_wait(&b_free[nxt % B_STAGES], ((nxt / B_STAGES) - 1) & 1);
                issue_b(nxt);
            }
            const int s = panel % B_STAGES, ab = panel % NAB;
            // keep the A staging ring full: refill every slot the loaders have released
            auto refill = [&]() {
                while (a_next < p.npanels && mbar_test(&g_free[a_next % A_STAGES], ((a_next / A_STAGES) - 1) & 1)) {
                    issue_a(a_next);
                    ++a_next;
                }
            };
            refill();
            while (!mbar_test(&b_full[s], (panel / B_STAGES) & 1)) refill();
            while (!mbar_test(&a_full[ab], (panel / NAB) & 1)) refill();
            tc_fence_after();
            // descriptors advance by plain adds: +gbytes per group, +16 rows per k-step
            uint64_t dg = smem_desc(smem_u32(sB + s * S::B_STAGE_BYTES), lbo, sbo, layout);
            uint32_t ag = tmem + BN + ab * a_cols, dcol = tmem;
            for (int g = 0; g < G; ++g) {
                uint64_t dk = dg;
                uint32_t ak = ag;
                for (int kk = 0; kk < nk; ++kk) {
                    if (leader) mma_ts(dcol, ak, dk, idesc, (panel | kk) ? 1u : 0u);
                    dk += kstep;
                    ak += 8;
                }
                dg += gstep;
                ag += cells_g;
                dcol += L;
            }
            if (leader) {
                tc_commit(&a_free[ab]);
                tc_commit(&b_free[s]);
            }
            __syncwarp();
        }
        if (leader) tc_commit(acc_full);
        while (a_next < p.npanels) {  // (only if the MMA loop finished first; not expected)
            mbar_wait(&g_free[a_next % A_STAGES], ((a_next / A_STAGES) - 1) & 1);
            issue_a(a_next);
            ++a_next;
        }
        __syncwarp();
    } else if (warp < LOADER_WARPS) {
        // ===================== loaders: staged A panel -> padded smem, D -> cell table =====================
        const int chunks_per_row = bk / 8;
        int a_soff[LD_UNITS], a_doff[LD_UNITS];
#pragma unroll
        for (int i = 0; i < LD_UNITS; ++i) {
            // one warp-instruction covers 4 rows x 8 chunks when a row has a multiple of 8
            // chunks: LDS.128 quarter-warps read 128 contiguous bytes, STS banks
            // (row + 4*chunk + word) mod 32 are all distinct
            const int unit = i * LOADER_THREADS + tid;
            int r, c;
            if ((chunks_per_row & 7) == 0) {
                const int oct = unit >> 5, l = unit & 31, opr = chunks_per_row >> 3;
                r = (oct / opr) * 4 + (l >> 3);
                c = (oct % opr) * 8 + (l & 7);
            } else {
                r = unit / chunks_per_row;
                c = unit - r * chunks_per_row;
            }
            a_soff[i] = r < BM ? r * a_pitch + c * 16 : -1;
            a_doff[i] = r * bk * 2 + c * 16;  // dense TMA panel: rows of bk bf16
        }
        for (int panel = 0; panel < p.npanels; ++panel) {
            const int st = panel & 1, gs = panel % A_STAGES;
            if (panel >= 2) mbar_wait(&s_free[st], ((panel - 2) >> 1) & 1);
            mbar_wait(&g_full[gs], (panel / A_STAGES) & 1);
            const uint8_t* src = sStg + gs * STG_BYTES;
            uint8_t* dst = sA + st * A_STAGE_BYTES;
#pragma unroll
            for (int i = 0; i < LD_UNITS; ++i) {
                if (a_soff[i] >= 0) {
                    const uint4 v = *reinterpret_cast<const uint4*>(src + a_doff[i]);
                    uint32_t* d = reinterpret_cast<uint32_t*>(dst + a_soff[i]);
                    d[0] = v.x;
                    d[1] = v.y;
                    d[2] = v.z;
                    d[3] = v.w;
                }
            }
            // prepacked cell table of the panel -> the gather-side table buffer
            const uint4* ts = reinterpret_cast<const uint4*>(src + STG_A_BYTES);
            uint4* td = reinterpret_cast<uint4*>(sT + st * TBL_WORDS);
            for (int i = tid; i < TBL_BYTES / 16; i += LOADER_THREADS) td[i] = ts[i];
            mbar_arrive(&g_free[gs]);
            // the pad word of each row is the zero source for the k padding (sentinel column bk)
            *reinterpret_cast<uint32_t*>(dst + tid * a_pitch + bk * 2) = 0u;
            mbar_arrive(&s_full[st]);
        }
    } else {
        // ===================== gather: A_g rows -> TMEM =====================
        const int gw = warp - LOADER_WARPS;
        const int quarter = warp & 3, sub = gw >> 2;  // 3 warps per lane quarter
        const int row = quarter * 32 + lane;
        const uint32_t lane_addr = static_cast<uint32_t>(quarter * 32) << 16;
        for (int panel = 0; panel < p.npanels; ++panel) {
            const int st = panel & 1, ab = panel % NAB;
            mbar_wait(&s_full[st], (panel >> 1) & 1);
            if (panel >= NAB) {
                mbar_wait(&a_free[ab], ((panel / NAB) - 1) & 1);
                tc_fence_after();
            }
            const uint8_t* arow = sA + st * A_STAGE_BYTES + row * a_pitch;
            const uint32_t* tA = sT + st * TBL_WORDS;
            const uint32_t* tB = tA + CELLS_MAX;
            const uint32_t tm_a = tmem + lane_addr + BN + ab * a_cols;
            // items = blocks of 8 cells, cell index == TMEM column offset inside the buffer;
            // this warp takes blocks sub, sub+3, ... (cells of group g are [g*cells_g, +cells_g))
            const int ncells = G * cells_g;
            for (int cell0 = sub * 8; cell0 < ncells; cell0 += 24) {
                // word 1 = PRMT selector | offset of kabs(2c)'s word << 16 (PRMT reads only the
                // low 16 selector bits), word 2 = offset of kabs(2c+1)'s word: 4 LDS.128 / 8 cells
                uint32_t sa[8], ob[8];
                *reinterpret_cast<uint4*>(&sa[0]) = *reinterpret_cast<const uint4*>(tA + cell0);
                *reinterpret_cast<uint4*>(&sa[4]) = *reinterpret_cast<const uint4*>(tA + cell0 + 4);
                *reinterpret_cast<uint4*>(&ob[0]) = *reinterpret_cast<const uint4*>(tB + cell0);
                *reinterpret_cast<uint4*>(&ob[4]) = *reinterpret_cast<const uint4*>(tB + cell0 + 4);
                uint32_t v[8];
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    const uint32_t wa = *reinterpret_cast<const uint32_t*>(arow + (sa[c] >> 16));
                    const uint32_t wb = *reinterpret_cast<const uint32_t*>(arow + ob[c]);
                    v[c] = prmt(wa, wb, sa[c]);
                }
                tmem_st8(tm_a + cell0, v);
            }
            tmem_wait_st();
            tc_fence_before();
            mbar_arrive(&a_full[ab]);
            mbar_arrive(&s_free[st]);
        }
    }

    // ===================== epilogue (warps 0-15): TMEM -> registers -> global =====================
    if (warp < CONTROL_WARP) {
        const int quarter = warp & 3, sub = warp >> 2;  // 4 warps per lane quarter
        const uint32_t lane_addr = static_cast<uint32_t>(quarter * 32) << 16;
        const int grow = m0 + quarter * 32 + lane;
        mbar_wait(acc_full, 0);
        tc_fence_after();
        for (int cb = sub * 16; cb < BN; cb += 64) {
            uint32_t v[16];
            tmem_ld16(tmem + lane_addr + cb, v);
            tmem_wait_ld();
            const int gc = n0 + cb;
            if (grow < p.m && gc < p.n) {
                if (p.c_bf16) {
                    uint32_t pk[8];
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        __nv_bfloat162 h = __floats2bfloat162_rn(__uint_as_float(v[2 * i]), __uint_as_float(v[2 * i + 1]));
                        pk[i] = *reinterpret_cast<uint32_t*>(&h);
                    }
                    uint4* dst = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(p.C) +
                                                          static_cast<int64_t>(grow) * p.n + gc);
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
    if (warp == CONTROL_WARP) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

// Offline-style index preprocessing ("reorder the index matrix D" and
// "transform the data layout of D"): for every (column tile, panel) the gather's
// cell table -- per (group g, u-pair c): byte offsets of the A words that hold dense
// columns kabs(2c), kabs(2c+1) inside a padded panel row, and the PRMT selector that
// packs the two bf16 halves.  One contiguous 3 KB block per (tile, panel), fetched
// by a bulk copy next to the A panel.
__global__ void build_cell_table_kernel(const uint8_t* __restrict__ D, uint32_t* __restrict__ tbl, int q, int N,
                                        int M, int L, int BN, int bk, int bkw, int bkw_pad, int npanels, int wtot) {
    const int tile = blockIdx.y, panel = blockIdx.x;
    const int G = BN / L, cells_g = bkw_pad / 2;
    uint32_t* t = tbl + (static_cast<int64_t>(tile) * npanels + panel) * TBL_WORDS;
    const int u0 = panel * bkw;
    for (int e = threadIdx.x; e < CELLS_MAX; e += blockDim.x) {
        const int g = e / cells_g, c = e - g * cells_g;
        const int gg = tile * G + g;
        uint32_t k2[2] = {static_cast<uint32_t>(bk), static_cast<uint32_t>(bk)};  // sentinel -> zero pad word
        if (g < G && gg < q) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int u = 2 * c + h;
                if (u < bkw && u0 + u < wtot)
                    k2[h] = static_cast<uint32_t>((u / N) * M + D[static_cast<int64_t>(u0 + u) * q + gg]);
            }
        }
        const uint32_t sel = ((k2[0] & 1u) ? 0x32u : 0x10u) | ((k2[1] & 1u) ? 0x7600u : 0x5400u);
        t[e] = sel | (((k2[0] >> 1) << 2) << 16);
        t[CELLS_MAX + e] = (k2[1] >> 1) << 2;
    }
}

}  // namespace tc

// Column-tile width: at high sparsity a 128-wide tile re-streams its dense A panel for
// little MMA work per panel, so 256 columns (8 groups) share each A panel; at <= 4:1
// density ratio the 128-wide tile wins (more CTAs, 3 TMEM A buffers).  Measured on B200
// (profiles/r01_summary.md): 16:32 128 > 256; 8:32 and 4:32 256 > 128.
static int tc_bn(int N, int M, int L) {
    const char* e = getenv("NM_TC_BN");  // ablation override
    if (e && (atoi(e) == 128 || atoi(e) == 256) && 256 % L == 0 && (atoi(e) / L) * 16 <= tc::CELLS_MAX) return atoi(e);
    return (L == 32 && 4 * N <= M) ? 256 : 128;
}

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
// BKW = WP*N compressed rows with G * BKW_pad <= 512 - BN TMEM columns for the two A
// buffers, preferring BKW % 16 == 0 (no zero-padded MMA k-steps), then larger panels.
void tc_bf16_geometry(int N, int M, int L, int* wp, int* bk, int* bkw, int* bkw_pad, int* bn) {
    const int BN = tc_bn(N, M, L), G = BN / L;
    const int nab = BN == 256 ? tc::nab<256>() : tc::nab<128>();
    const int bcap = BN == 256 ? tc::bkw_cap<256>() : tc::bkw_cap<128>();
    int cap = 2 * (512 - BN) / (nab * G);
    cap = cap < bcap ? cap : bcap;
    cap = cap / 16 * 16;
    if (G * (cap / 2) > tc::CELLS_MAX) cap = 2 * (tc::CELLS_MAX / G) / 16 * 16;
    int best = 1, best_score = -1;
    for (int w = 1; w * M <= tc::BK_MAX && (w * N + 15) / 16 * 16 <= cap; ++w) {
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
    *bn = BN;
}

bool tc_pair_applicable(int64_t m, int64_t n, int64_t k, int N, int M, int L, int bn, int bkw_pad);
nm_status tc_pair_launch(const void* A, const void* Bv, const uint8_t* D, void* C, bool c_bf16, int64_t m, int64_t n,
                         int64_t k, int N, int M, int L, int wp, int bk, int bkw, int bkwp, int bn, cudaStream_t s);

template <int BN>
static nm_status tc_launch_bn(const tc::Params& p, const CUtensorMap& tmA, const CUtensorMap& tmB, int64_t m, int64_t n,
                              cudaStream_t s) {
    using namespace tc;
    static bool attr = false;
    if (!attr) {
        NM_CUDA_TRY(cudaFuncSetAttribute(spmm_tc_bf16_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         Smem<BN>::BYTES));
        attr = true;
    }
    const dim3 grid(static_cast<unsigned>(ceil_div(n, BN)), static_cast<unsigned>(ceil_div(m, BM)));
    prof_begin(s);
    spmm_tc_bf16_kernel<BN><<<grid, THREADS, Smem<BN>::BYTES, s>>>(tmA, tmB, p);
    prof_end(s);
    note_launch();
    NM_LAUNCH_CHECK("spmm_tc_bf16_kernel");
    return NM_OK;
}

nm_status tc_bf16_launch(const void* A, const void* Bv, const uint8_t* D, void* C, bool c_bf16, int64_t m, int64_t n,
                         int64_t k, int N, int M, int L, cudaStream_t s) {
    using namespace tc;
    Params p{};
    p.A = static_cast<const __nv_bfloat16*>(A);
    p.C = C;
    p.m = static_cast<int>(m);
    p.n = static_cast<int>(n);
    p.k = static_cast<int>(k);
    p.N = N;
    p.M = M;
    p.L = L;
    p.q = static_cast<int>(n / L);
    p.c_bf16 = c_bf16 ? 1 : 0;
    int bn = 128;
    tc_bf16_geometry(N, M, L, &p.wp, &p.bk, &p.bkw, &p.bkw_pad, &bn);
    // token-pair gather (spmm_tc_pair.cu) when its layout constraints hold; NM_TC_PAIR=0 disables
    const char* pe = getenv("NM_TC_PAIR");
    if (!(pe && pe[0] == '0') && tc_pair_applicable(m, n, k, N, M, L, bn, p.bkw_pad))
        return tc_pair_launch(A, Bv, D, C, c_bf16, m, n, k, N, M, L, p.wp, p.bk, p.bkw, p.bkw_pad, bn, s);
    const int windows = static_cast<int>(k / M);
    p.npanels = (windows + p.wp - 1) / p.wp;
    const int64_t w = k / M * N;
    CUtensorMap tmB;
    const int box_cols = L >= 64 ? 64 : L;
    const int sw = box_cols * 2;  // 32 / 64 / 128 B swizzle = the group's row width
    nm_status st = make_tma_2d(&tmB, Bv, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, w, n, p.bkw, box_cols, sw);
    if (st) return st;
    CUtensorMap tmA;  // dense A panel [128 rows][bk] (no swizzle; OOB rows / columns read as zero)
    st = make_tma_2d(&tmA, A, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, m, k, BM, p.bk, 0);
    if (st) return st;
    // cell tables: stream-ordered scratch (the pool caches it across calls)
    const int ntiles = static_cast<int>(ceil_div(n, bn));
    const size_t tbytes = static_cast<size_t>(ntiles) * p.npanels * TBL_BYTES;
    uint32_t* tbl = nullptr;
    st = scratch_alloc(reinterpret_cast<void**>(&tbl), tbytes, s);
    if (st) return st;
    build_cell_table_kernel<<<dim3(p.npanels, ntiles), 256, 0, s>>>(D, tbl, p.q, N, M, L, bn, p.bk, p.bkw, p.bkw_pad,
                                                                      p.npanels, static_cast<int>(w));
    note_launch();
    NM_LAUNCH_CHECK("build_cell_table_kernel");
    p.tbl = tbl;
    st = bn == 256 ? tc_launch_bn<256>(p, tmA, tmB, m, n, s) : tc_launch_bn<128>(p, tmA, tmB, m, n, s);
    NM_CUDA_TRY(cudaFreeAsync(tbl, s));
    return st;
}

}  // namespace nm
