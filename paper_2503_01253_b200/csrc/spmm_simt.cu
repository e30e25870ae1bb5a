// spmm_simt.cu -- fp32 CUDA-core N:M SpMM (the paper's fp32 semantics),
// re-designed for sm_100a.
//
// What is kept from the paper: the hierarchical blocking of Listing 1 (CTA
// tile over C, k-loop inside the CTA, no split-K), the register
// outer-product micro-kernel of Listing 2 / Eq. 6 (8x8 thread tiles,
// P:349-400), index prefetch ahead of the fragment loads (Listing 4)
// and double buffering.
// What is B200-specific: operand panels arrive by TMA (one thread issues,
// mbarrier completion, OOB zero-fill for ragged m / n / k tails); the dense A
// panel lands in the 128-byte-swizzled layout so the index-driven column
// gather (A_s[row][kabs]) is bank-conflict free across the 8 rows a warp
// touches; the per-panel index table D_s is converted once into swizzled byte
// offsets so the inner loop spends one LDS + one XOR per (step, group).
//
// Tile: BM=128 rows x BN=128 columns, 256 threads (8 warps of 64x32), thread
// tile 8 rows x 8 columns (two 4-column chunks 16 apart).  A panel: WP whole
// windows (BK = WP*M <= 64 dense k, never straddling a window), i.e.
// BKW = WP*N <= 32 compressed rows.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"

namespace nm {
namespace simt {

constexpr int BM = 128, BN = 128, BK = 64, BKW = 32, THREADS = 256, STAGES = 2;
constexpr int A_BOX_COLS = 32;                      // 128 B of fp32: the swizzle-128B atom width
constexpr int A_BOX_BYTES = BM * A_BOX_COLS * 4;    // 16 KB
constexpr int A_STAGE_BYTES = BM * BK * 4;          // 32 KB
constexpr int B_STAGE_BYTES = BKW * BN * 4;         // 16 KB
constexpr int MAX_SLOTS = 33;                       // column groups touched by a 128-wide tile, L >= 4
constexpr int KOFF_BYTES = 2 * BKW * MAX_SLOTS * 4;
constexpr int MAX_PANELS_PACKED = 512;               // col_info masks kept in shared memory
constexpr int MASK_BYTES = MAX_PANELS_PACKED * 8;
constexpr int SMEM_BYTES = STAGES * (A_STAGE_BYTES + B_STAGE_BYTES) + KOFF_BYTES + 64 + 1024;
constexpr int SMEM_BYTES_PACKED = SMEM_BYTES + MASK_BYTES;
constexpr int D_PER_THREAD = (BKW * MAX_SLOTS + THREADS - 1) / THREADS;  // 5

struct Params {
    const uint8_t* D;
    float* C;
    const float* AT;        // A^T (k x at_ld), packed mode
    const uint64_t* masks;  // col_info per (column tile, panel): bit kk = dense column kk is needed
    int m, n, k, N, M, L;
    int q, wp, bk, bkw, npanels, nboxA;
    int at_ld;
    // tile schedule (1-D grid, grouped raster: `gm` row tiles x all column tiles per group);
    // the last, partial wave is split along k ("stream-K lite"): tiles >= full_tiles are
    // done by `split` CTAs each, whose partial sums meet in ws and are added in a fixed
    // order by whichever CTA finishes last (deterministic, no atomics on data).
    int ntn, full_tiles, split;
    int ntm, gm;  // row tiles; rows per raster group
    float* ws;
    int* counters;
    // peer-store epilogue (nm_spmm_peers): the C tile goes to cpeer[0 .. npeer) at
    // [row][col_off + col] (row pitch ldc), columns < n_valid only -- the column all-gather of a
    // sharded layer fused into the SpMM's stores over NVLink peer memory.  npeer = 0: C.
    float* cpeer[8];
    int npeer, n_valid;
    int mc;  // 1: cpeer[0] is a multicast (NVLS) address: one multimem.st per float4 reaches every rank
    int64_t ldc, col_off;
    float alpha;  // C = alpha . A B~ (1: the product; M/N: Eq. 1 as printed, nm_spmm_scaled)
    // bit-packed tile-major indices (nm_index_pack, P:288 / P:419) instead of D when non-null:
    // column tile ct's stream at Dw + ct * dwt, entry x = u * dT + t at word x / de, bit (x % de) * db
    const uint32_t* Dw;
    int db, de, dT;
    int64_t dwt;
};

// 16-B store through a multicast (NVLS) address: one instruction, replicated to every bound buffer
__device__ __forceinline__ void mc_store4(float* addr, float a, float b, float c, float d) {
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "f"(a), "f"(b), "f"(c),
                 "f"(d)
                 : "memory");
}

// Byte offset (before the per-row XOR) of dense column kk (0..63) inside an A stage:
// box kk/32, 16-byte chunk (kk%32)/4, word kk%4.
template <int BMT>
__device__ __forceinline__ int a_col_offset(int kk) {
    return ((kk >> 5) * (BMT * A_BOX_COLS * 4)) + (((kk & 31) >> 2) << 4) + ((kk & 3) << 2);
}

// Row-tile geometry: BMT = 128 (8 warps of 64 x 32, 2 CTAs/SM) or 64 (4 warps of 64 x 32, 3 CTAs/SM;
// for sub-wave grids: column shards of a multi-GPU layer, small problems -- the selector's choice).
template <int BMT>
struct SG {
    static constexpr int THREADS = 2 * BMT;
    static constexpr int MINB = BMT == 128 ? 2 : 3;                 // resident CTAs per SM
    static constexpr int A_BOX_BYTES = BMT * A_BOX_COLS * 4;
    static constexpr int A_STAGE_BYTES = BMT * BK * 4;
    static constexpr int SMEM_BYTES = STAGES * (A_STAGE_BYTES + B_STAGE_BYTES) + KOFF_BYTES + 64 + 1024;
    static constexpr int SMEM_BYTES_PACKED = SMEM_BYTES + MASK_BYTES;
    static constexpr int D_PER_THREAD = (BKW * MAX_SLOTS + THREADS - 1) / THREADS;
};

// TWO: the thread's two 4-column chunks may belong to different column groups (L < 32).
// AT:  A arrives transposed (A^T, k x m, written by transpose_kernel): the panel is
//      [BK k-rows][128 m] and a gathered fragment is two LDS.128 of row kabs
//      (8 rows of A); otherwise the panel is [128 m][BK] (swizzled) and a fragment is
//      eight LDS.32 of column kabs.
// PK:  (with AT) the paper's packing for high sparsity (Listing 3): only
//      the dense columns some group of the tile selects (col_info) are
//      fetched -- one 512-B A^T row per warp-wide cp.async, the rows spread over all
//      warps -- into consecutive panel rows, and the indices are remapped to packed
//      positions (reorderingIdx) by a popcount over the col_info mask.
// PEER: the fused exchange's peer-store epilogue (nm_spmm_peers), a separate instantiation so the
// common kernel's code and register allocation stay as they were.
template <int BMT, bool TWO, bool AT, bool PK, bool PEER = false>
__global__ void __launch_bounds__(SG<BMT>::THREADS, SG<BMT>::MINB)
    spmm_simt_f32_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                         const Params p) {
    constexpr int BM = BMT, THREADS = SG<BMT>::THREADS, A_BOX_BYTES = SG<BMT>::A_BOX_BYTES;
    constexpr int A_STAGE_BYTES = SG<BMT>::A_STAGE_BYTES, D_PER_THREAD = SG<BMT>::D_PER_THREAD;
    static_assert(!PK || BMT == 128, "packed mode: one 512-B A^T row per warp-wide cp.async (BM = 128)");
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // 1024-B alignment for the swizzle-128B TMA destination; offset arithmetic on the
    // __shared__ array keeps the shared address space visible to the compiler (LDS, not LD)
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* sA = smem;                                        // STAGES x 32 KB
    uint8_t* sB = smem + STAGES * A_STAGE_BYTES;               // STAGES x 16 KB
    int* koff = reinterpret_cast<int*>(sB + STAGES * B_STAGE_BYTES);  // [2][BKW][MAX_SLOTS]
    uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(koff) + KOFF_BYTES);
    uint64_t* smask = bars + 8;  // [MAX_PANELS_PACKED] (packed mode)

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = BMT == 128 ? (warp & 1) : 0, wn = BMT == 128 ? (warp >> 1) : warp;
    const int t_m = lane & 7, t_n = lane >> 3;
    int tile = blockIdx.x, part = 0, nparts = 1;
    if (tile >= p.full_tiles) {
        part = (tile - p.full_tiles) % p.split;
        tile = p.full_tiles + (tile - p.full_tiles) / p.split;
        nparts = p.split;
    }
    // grouped raster: groups of `gm` row tiles sweep the column tiles with the row index fastest, so
    // the group's A^T panels stay in L2 and each B' panel is read from DRAM once per group (an
    // n-fastest order re-streamed all of B' every ~2 row tiles: 3.3x the algorithmic DRAM bytes)
    int tm, tn;
    {
        const int per = p.gm * p.ntn, grp = tile / per, r = tile - grp * per;
        const int first = grp * p.gm, gsz = min(p.gm, p.ntm - first);
        tm = first + r % gsz;
        tn = r / gsz;
    }
    const int m0 = tm * BM, n0 = tn * BN;
    const int p_begin = part * p.npanels / nparts, p_end = (part + 1) * p.npanels / nparts;
    const int g_first = n0 / p.L;
    const int nslots = min((n0 + BN - 1) / p.L, p.q - 1) - g_first + 1;

    if (tid == 0) {
        if (!PK) tma_prefetch_desc(&tmA);
        tma_prefetch_desc(&tmB);
        // packed mode: + one cp.async.mbarrier.arrive.noinc per thread (the gathered A^T rows)
        for (int s = 0; s < STAGES; ++s) mbar_init(&bars[s], PK ? 1 + THREADS : 1);
        fence_mbar_init();
    }
    if (PK)
        for (int i = tid; i < p.npanels; i += THREADS) smask[i] = p.masks[static_cast<int64_t>(tn) * p.npanels + i];
    __syncthreads();

    const uint32_t stage_tx =
        static_cast<uint32_t>((AT ? p.bk * BM * 4 : p.nboxA * A_BOX_BYTES) + p.bkw * BN * 4);
    // called by thread 0 (tile modes) or by all of warp 0 (packed mode)
    auto issue = [&](int panel) {
        const int s = (panel - p_begin) % STAGES;
        const int k0 = panel * p.bk, u0 = panel * p.bkw;
        if (PK) {
            // every warp: the needed rows among dense columns [8 warp, 8 warp + 8) of the panel,
            // one 512-B A^T row per warp-wide 16-B cp.async (the TMA bulk copy per row was the
            // cost that made packing lose); thread 0 also fetches the B' panel
            const uint64_t mk = smask[panel];
            if (tid == 0) {
                mbar_arrive_expect_tx(&bars[s], static_cast<uint32_t>(p.bkw * BN * 4));
                tma_load_2d(sB + s * B_STAGE_BYTES, &tmB, &bars[s], n0, u0);
            }
            const uint32_t sa = smem_u32(sA + s * A_STAGE_BYTES) + 16u * static_cast<uint32_t>(lane);
            const float* src = p.AT + static_cast<int64_t>(k0) * p.at_ld + m0 + 4 * lane;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int b = 8 * warp + i;
                if ((mk >> b) & 1ull) {
                    const int pos = __popcll(mk & ((1ull << b) - 1ull));
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa + pos * (BM * 4)),
                                 "l"(src + static_cast<int64_t>(b) * p.at_ld)
                                 : "memory");
                }
            }
            asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(&bars[s])) : "memory");
            return;
        }
        mbar_arrive_expect_tx(&bars[s], stage_tx);
        if (AT)
            tma_load_2d(sA + s * A_STAGE_BYTES, &tmA, &bars[s], m0, k0);
        else
            for (int b = 0; b < p.nboxA; ++b)
                tma_load_2d(sA + s * A_STAGE_BYTES + b * A_BOX_BYTES, &tmA, &bars[s], k0 + b * A_BOX_COLS, m0);
        tma_load_2d(sB + s * B_STAGE_BYTES, &tmB, &bars[s], n0, u0);
    };

    // D_s -> byte offsets koff[buf][u][slot] (index prefetch).  The (u, slot)
    // entries a thread handles, their D offsets and window bases are panel-invariant
    // (panels hold whole windows: (u0 + u) / N - t0 == u / N), so they are computed once.
    // d_us = window base << 16 | u << 8 | slot (or -1): one register per entry (register pressure:
    // the fragment double buffer of the inner loop needs the room)
    int dreg[D_PER_THREAD], d_us[D_PER_THREAD];
#pragma unroll
    for (int r = 0; r < D_PER_THREAD; ++r) {
        const int e = tid + r * THREADS;
        const int u = e / nslots, sl = e - u * nslots;
        d_us[r] = (u < p.bkw && sl < nslots) ? ((u / p.N) * p.M << 16 | u << 8 | sl) : -1;
    }
    // the valid entries are a prefix r < nd (e grows with r): the per-panel index loops stop
    // there -- at L >= 32 a panel has only BKW x (BN/L + 1) entries, most threads 0 or 1
    const int nd = min(D_PER_THREAD, max(0, (p.bkw * nslots - tid + THREADS - 1) / THREADS));
    const int wtot = (p.k / p.M) * p.N;
    auto load_d = [&](int panel) {
        const int u0 = panel * p.bkw;
        const int ulim = wtot - u0;  // rows of D left (last panel may be partial)
        if (p.Dw) {  // packed: this column tile's contiguous word stream (g_first = tile * dT)
            const uint32_t* Dt = p.Dw + static_cast<int64_t>(tn) * p.dwt;
            const uint32_t mask = (1u << p.db) - 1u;
#pragma unroll
            for (int r = 0; r < D_PER_THREAD; ++r) {
                if (r >= nd) break;
                const int u = (d_us[r] >> 8) & 255, sl = d_us[r] & 255;
                const int64_t x = static_cast<int64_t>(u0 + u) * p.dT + sl;
                dreg[r] = (u < ulim) ? static_cast<int>((__ldg(Dt + x / p.de) >> ((x % p.de) * p.db)) & mask) : 0;
            }
            return;
        }
        const uint8_t* Dp = p.D + static_cast<int64_t>(u0) * p.q + g_first;
#pragma unroll
        for (int r = 0; r < D_PER_THREAD; ++r) {
            if (r >= nd) break;
            const int u = (d_us[r] >> 8) & 255, sl = d_us[r] & 255;
            dreg[r] = (u < ulim) ? Dp[u * p.q + sl] : 0;
        }
    };
    auto store_d = [&](int panel) {
        int* kb = koff + ((panel - p_begin) & 1) * (BKW * MAX_SLOTS);
        const uint64_t mk = PK ? smask[panel] : 0ull;
#pragma unroll
        for (int r = 0; r < D_PER_THREAD; ++r) {
            if (r >= nd) break;
            {
                const int kk = (d_us[r] >> 16) + dreg[r];  // dense column inside the panel
                const int row = PK ? __popcll(mk & ((1ull << kk) - 1ull)) : kk;  // packed position
                kb[((d_us[r] >> 8) & 255) * MAX_SLOTS + (d_us[r] & 255)] = AT ? row * (BM * 4) : a_col_offset<BMT>(kk);
            }
        }
    };

    if (PK || tid == 0) issue(p_begin);
    load_d(p_begin);
    store_d(p_begin);
    __syncthreads();

    // thread geometry
    const int col0 = wn * 32 + 4 * t_n;  // chunk 0 (chunk 1 at col0 + 16), tile-relative
    // columns past n (ragged tile) read a valid slot; their results are never stored
    const int slot0 = min((n0 + col0) / p.L - g_first, nslots - 1);
    const int slot1 = min((n0 + col0 + 16) / p.L - g_first, nslots - 1);
    const int tmx = AT ? 0 : (t_m << 4);
    const int a_row = AT ? (wm * 64 + 4 * t_m) * 4 : (wm * 64 + t_m) * 128;

    float acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;

    for (int panel = p_begin; panel < p_end; ++panel) {
        const int rel = panel - p_begin, s = rel % STAGES;
        if ((PK || tid == 0) && panel + 1 < p_end) issue(panel + 1);  // freed by the last sync
        if (panel + 1 < p_end) load_d(panel + 1);
        mbar_wait(&bars[s], (rel / STAGES) & 1);

        const int u0 = panel * p.bkw;
        const int bkw = min(p.bkw, (p.k / p.M) * p.N - u0);
        const uint8_t* aS = sA + s * A_STAGE_BYTES + a_row;
        const float* bS = reinterpret_cast<const float*>(sB + s * B_STAGE_BYTES) + col0;
        const int* kS = koff + (rel & 1) * (BKW * MAX_SLOTS);

        // software pipeline: the gathered fragment(s) of row u + 1 (index LDS -> fragment LDS) are
        // loaded while row u's FMAs run, so the index -> gather latency chain is off the FMA path
        auto ld_frag = [&](const uint8_t* ap, float (&a)[8]) {
            if (AT) {
                const float4 x0 = *reinterpret_cast<const float4*>(ap);
                const float4 x1 = *reinterpret_cast<const float4*>(ap + 128);
                a[0] = x0.x, a[1] = x0.y, a[2] = x0.z, a[3] = x0.w;
                a[4] = x1.x, a[5] = x1.y, a[6] = x1.z, a[7] = x1.w;
            } else {
#pragma unroll
                for (int i = 0; i < 8; ++i) a[i] = *reinterpret_cast<const float*>(ap + i * 1024);
            }
        };
        // ping-pong fragment buffers (f*: even rows, g*: odd rows; *1: the second column group when TWO)
        float fa0[8], fa1[8], ga0[8], ga1[8];
        auto ld_row = [&](int u, float (&x0)[8], float (&x1)[8]) {
            const int* krow = kS + u * MAX_SLOTS;
            ld_frag(aS + (krow[slot0] ^ tmx), x0);
            if (TWO) ld_frag(aS + (krow[slot1] ^ tmx), x1);
        };
        // the 8 x 8 outer product as 32 paired FMAs (FFMA2, sm_100: two fp32 FMAs with the A element
        // broadcast, each rounded exactly as fmaf -- the same bits, half the issue slots)
        auto fma_row = [&](int u, const float (&x0)[8], const float (&x1)[8]) {
            const float4 b0 = *reinterpret_cast<const float4*>(bS + u * BN);
            const float4 b1 = *reinterpret_cast<const float4*>(bS + u * BN + 16);
            const float2 b01 = make_float2(b0.x, b0.y), b23 = make_float2(b0.z, b0.w);
            const float2 b45 = make_float2(b1.x, b1.y), b67 = make_float2(b1.z, b1.w);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const float2 y0 = make_float2(x0[i], x0[i]);
                const float2 y1 = TWO ? make_float2(x1[i], x1[i]) : y0;
                float2 c;
                c = __ffma2_rn(y0, b01, make_float2(acc[i][0], acc[i][1])), acc[i][0] = c.x, acc[i][1] = c.y;
                c = __ffma2_rn(y0, b23, make_float2(acc[i][2], acc[i][3])), acc[i][2] = c.x, acc[i][3] = c.y;
                c = __ffma2_rn(y1, b45, make_float2(acc[i][4], acc[i][5])), acc[i][4] = c.x, acc[i][5] = c.y;
                c = __ffma2_rn(y1, b67, make_float2(acc[i][6], acc[i][7])), acc[i][6] = c.x, acc[i][7] = c.y;
            }
        };
        ld_row(0, fa0, fa1);
        int u = 0;
#pragma unroll 1
        for (; u + 1 < bkw; u += 2) {
            ld_row(u + 1, ga0, ga1);
            fma_row(u, fa0, fa1);
            ld_row(min(u + 2, bkw - 1), fa0, fa1);  // the last pair reloads a valid row (unused)
            fma_row(u + 1, ga0, ga1);
        }
        if (u < bkw) fma_row(u, fa0, fa1);  // odd row count (odd N)
        if (panel + 1 < p_end) store_d(panel + 1);
        __syncthreads();
    }

    if (nparts > 1) {
        // split tile: publish this part's partial sums, the last part to arrive adds all
        // parts in order 0..split-1 (fixed order -> bit-reproducible) and stores C
        const int ti = tile - p.full_tiles;
        float4* mine = reinterpret_cast<float4*>(p.ws + (static_cast<int64_t>(ti) * p.split + part) * (BM * BN)) + tid * 16;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            mine[2 * i] = make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
            mine[2 * i + 1] = make_float4(acc[i][4], acc[i][5], acc[i][6], acc[i][7]);
        }
        __threadfence();
        __syncthreads();
        int* last = reinterpret_cast<int*>(bars + 2);
        if (tid == 0) *last = atomicAdd(&p.counters[ti], 1) == p.split - 1;
        __syncthreads();
        if (!*last) return;
        __threadfence();
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
        for (int q2 = 0; q2 < p.split; ++q2) {
            const float4* src =
                reinterpret_cast<const float4*>(p.ws + (static_cast<int64_t>(ti) * p.split + q2) * (BM * BN)) + tid * 16;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const float4 x = __ldcg(src + 2 * i), y = __ldcg(src + 2 * i + 1);
                acc[i][0] += x.x, acc[i][1] += x.y, acc[i][2] += x.z, acc[i][3] += x.w;
                acc[i][4] += y.x, acc[i][5] += y.y, acc[i][6] += y.z, acc[i][7] += y.w;
            }
        }
        if (tid == 0) p.counters[ti] = 0;  // ready for the next launch
    }

    // epilogue: registers -> global (float4 stores, guarded for ragged m / n); alpha after any
    // k-split reduction (x 1.0f is exact)
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] *= p.alpha;
    const int gc0 = n0 + col0;
    if (PEER) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int row = m0 + wm * 64 + (AT ? (i & 3) + 4 * t_m + 32 * (i >> 2) : 8 * i + t_m);
            if (row >= p.m) continue;
            if (p.mc) {  // NVLS: the switch replicates each store into every rank's bound C buffer
                float* crow = p.cpeer[0] + static_cast<int64_t>(row) * p.ldc + p.col_off;
                if (gc0 < p.n_valid) mc_store4(crow + gc0, acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
                if (gc0 + 16 < p.n_valid) mc_store4(crow + gc0 + 16, acc[i][4], acc[i][5], acc[i][6], acc[i][7]);
                continue;
            }
            for (int pi = 0; pi < p.npeer; ++pi) {
                float* crow = p.cpeer[pi] + static_cast<int64_t>(row) * p.ldc + p.col_off;
                if (gc0 < p.n_valid)
                    *reinterpret_cast<float4*>(crow + gc0) = make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
                if (gc0 + 16 < p.n_valid)
                    *reinterpret_cast<float4*>(crow + gc0 + 16) = make_float4(acc[i][4], acc[i][5], acc[i][6], acc[i][7]);
            }
        }
        // the peer stores are visible system-wide before this kernel completes, so the barrier
        // kernel that follows on the stream may publish them with its release flag
        __threadfence_system();
        return;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int row = m0 + wm * 64 + (AT ? (i & 3) + 4 * t_m + 32 * (i >> 2) : 8 * i + t_m);
        if (row >= p.m) continue;
        float* crow = p.C + static_cast<int64_t>(row) * p.n;
        if (gc0 < p.n) *reinterpret_cast<float4*>(crow + gc0) = make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
        if (gc0 + 16 < p.n)
            *reinterpret_cast<float4*>(crow + gc0 + 16) = make_float4(acc[i][4], acc[i][5], acc[i][6], acc[i][7]);
    }
}

}  // namespace simt

// Applicability of the tiled SIMT kernel (else the generic kernel runs).
bool simt_f32_applicable(const void* A, const void* Bv, const void* C, int64_t m, int64_t n, int64_t k, int N, int M,
                         int L) {
    if (L % 4 != 0 || M > simt::BK || N > simt::BKW) return false;
    if (k % 4 != 0 || n % 4 != 0) return false;
    if ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(Bv) | reinterpret_cast<uintptr_t>(C)) & 15)
        return false;
    if (m > (1ll << 31) - simt::BM || n > (1ll << 31) - simt::BN || k >= (1ll << 31)) return false;
    return true;
}

void simt_f32_geometry(int N, int M, int* wp, int* bk, int* bkw) {
    int w = simt::BK / M;
    w = w < simt::BKW / N ? w : simt::BKW / N;
    if (w < 1) w = 1;
    *wp = w;
    *bk = w * M;
    *bkw = w * N;
}

// A (m x k) -> A^T (k x m): 32x32 tiles through padded shared memory, coalesced both ways.
__global__ void __launch_bounds__(256) transpose_kernel(const float* __restrict__ A, float* __restrict__ AT, int m,
                                                       int k, int ld) {
    // 64 x 64 tile, 16-B global accesses on both sides (a warp moves 2 x 256 contiguous bytes);
    // smem rows padded to 65 floats: the 4-token column reads are conflict-free.  k % 4 == 0
    // (SIMT applicability); tokens >= m are written as zeros (never read back into C).
    __shared__ float t[64][65];
    const int k0 = blockIdx.x * 64, m0 = blockIdx.y * 64;
    const int tid = threadIdx.x;
#pragma unroll
    for (int it = 0; it < 4; ++it) {
        const int e = tid + it * 256;
        const int r = e >> 4, c4 = (e & 15) * 4;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (m0 + r < m && k0 + c4 < k) v = *reinterpret_cast<const float4*>(A + static_cast<int64_t>(m0 + r) * k + k0 + c4);
        t[r][c4] = v.x;
        t[r][c4 + 1] = v.y;
        t[r][c4 + 2] = v.z;
        t[r][c4 + 3] = v.w;
    }
    __syncthreads();
#pragma unroll
    for (int it = 0; it < 4; ++it) {
        const int e = tid + it * 256;
        const int kr = e >> 4, q4 = (e & 15) * 4;
        if (k0 + kr < k && m0 + q4 < ld)
            *reinterpret_cast<float4*>(AT + static_cast<int64_t>(k0 + kr) * ld + m0 + q4) =
                make_float4(t[q4][kr], t[q4 + 1][kr], t[q4 + 2][kr], t[q4 + 3][kr]);
    }
}

// col_info: per (column tile, panel) the set of dense panel columns that at
// least one column group of the tile selects, as a 64-bit mask (BK <= 64).
__global__ void build_colinfo_kernel(const uint8_t* __restrict__ D, uint64_t* __restrict__ masks, int q, int N, int M,
                                     int L, int wp, int bkw, int npanels, int wtot) {
    __shared__ unsigned long long mk;
    const int panel = blockIdx.x, tile = blockIdx.y;
    const int g0 = tile * simt::BN / L, g1 = min((tile * simt::BN + simt::BN - 1) / L, q - 1);
    const int ng = g1 - g0 + 1;
    if (threadIdx.x == 0) mk = 0ull;
    __syncthreads();
    const int u0 = panel * bkw, t0 = panel * wp;
    unsigned long long mine = 0ull;
    for (int e = threadIdx.x; e < bkw * ng; e += blockDim.x) {
        const int u = e / ng, g = g0 + e % ng;
        if (u0 + u < wtot) mine |= 1ull << (((u0 + u) / N - t0) * M + D[static_cast<int64_t>(u0 + u) * q + g]);
    }
    atomicOr(&mk, mine);
    __syncthreads();
    if (threadIdx.x == 0) masks[static_cast<int64_t>(tile) * npanels + panel] = mk;
}

template <int BMT, bool TWO, bool AT, bool PK>
static nm_status launch_simt(const CUtensorMap& tmA, const CUtensorMap& tmB, const simt::Params& p, dim3 grid,
                             cudaStream_t s) {
    using namespace simt;
    using G = SG<BMT>;
    const int smem = PK ? G::SMEM_BYTES_PACKED : G::SMEM_BYTES;
    static std::atomic<uint64_t> attr_mask{0};
    if (!attr_once(attr_mask)) {
        NM_CUDA_TRY(cudaFuncSetAttribute(spmm_simt_f32_kernel<BMT, TWO, AT, PK>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        if (!PK)
            NM_CUDA_TRY(cudaFuncSetAttribute(spmm_simt_f32_kernel<BMT, TWO, AT, false, true>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        attr_done(attr_mask);
    }
    prof_begin(s);
    if (!PK && p.npeer)
        spmm_simt_f32_kernel<BMT, TWO, AT, false, true><<<grid, G::THREADS, smem, s>>>(tmA, tmB, p);
    else
        spmm_simt_f32_kernel<BMT, TWO, AT, PK><<<grid, G::THREADS, smem, s>>>(tmA, tmB, p);
    prof_end(s);
    note_launch();
    NM_LAUNCH_CHECK("spmm_simt_f32_kernel");
    return NM_OK;
}

// Row tile of the SIMT kernel (the selector): 64 rows (4 warps, 3 resident CTAs per
// SM) or 128 (8 warps, 2 per SM, with the wave-model split of its tail / sub-wave grid).
//  * tiles64 in (2, 3] x SMs (the 64-row grid fills 0.67-1 round of resident CTAs): 64.  Measured
//    on B200 (profiles/r02j_simt_row_tile.txt, the 100-point dataset r02n vs r02e): 256x13824x5120
//    141 -> 114 us, the cfg3-75 % 8-GPU shard 183 -> 173, 256x12288x4096 203 -> 162,
//    512x6656x6656 322 -> 254.
//  * tiles64 <= 2 x SMs: 128 with its k-split once the compressed k is long (w >= 1024: the split
//    parts amortise their fixed cost; 256x4096x11008 167 vs 209 us, 256x8192x8192 219 vs 228, the
//    cfg2 8-GPU shard 220 vs 225), 64 for short k (1024^3 39.5 vs 47.1, cfg1 20.8 vs 27.2).
//  * larger grids: 128 (m = 256 cfg4-65B 258 vs 280, 2048^3 188 vs 193).
// NM_SIMT_BM=64/128 overrides.
int simt_row_tile(int64_t m, int64_t n, int64_t w) {
    const char* e = getenv("NM_SIMT_BM");
    if (e) return atoi(e) == 64 ? 64 : 128;
    const int64_t tiles64 = ceil_div(m, 64) * ceil_div(n, simt::BN), sms = num_sms();
    if (tiles64 > 3 * sms) return 128;
    if (tiles64 > 2 * sms) return 64;
    return w >= 1024 ? 128 : 64;
}

// Split factor of the SIMT kernel's tile schedule (the selector's wave model): the
// tiles of a partial last wave (multi-wave grids) or of a sub-wave grid (small problems, column
// shards of a multi-GPU layer) run as S CTAs each over S k-ranges, partials added in a fixed
// order by the last arriver.  R = 2 x SMs resident CTAs; with 2 CTAs on an SM each runs at about
// 0.6x the speed of a lone CTA, so a split pays only when it leaves the split CTAs alone on their
// SMs (or nearly) and each part keeps enough rows to amortise its fixed cost:
//   * multi-wave, rem = tiles mod R with 0 < 2 rem <= SMs: S = min(3, SMs / rem);
//   * sub-wave: the largest S <= 4 with tiles x S <= SMs and >= 256 compressed rows per part;
//     else, when SMs < tiles, S = 2 if the CTAs beyond the first R fit half the SMs and each part
//     keeps >= 512 rows;
//   * else 1.
// Measured on B200 (pipelined kernel, profiles/r02c_simt_streamk.txt table 1) this picks the
// fastest S of {1, 2, 3, 4} at all 11 shapes timed (BASELINE tails, m = 256, the 8-GPU shards of
// cfg2 / cfg3 / cfg4, 1024^3 and 2048^3).  NM_SIMT_SPLIT overrides (never for whole waves).
int simt_split_factor(int ntiles, int64_t w, int npanels, int bm) {
    const int sms = num_sms(), resident = 2 * sms;
    if (ntiles <= 0 || npanels < 2 || (ntiles >= resident && ntiles % resident == 0)) return 1;
    const char* e = getenv("NM_SIMT_SPLIT");  // timing studies / tests
    if (e) return std::max(1, std::min(atoi(e), std::min(4, npanels / 2)));
    int S = 1;
    if (bm == 64) {
        // the 64-row tile splits only grids whose split CTAs all run alone on their SMs, with >= 128
        // compressed rows per part: measured (profiles/r02v_simt_small_split.txt) 512x1024x1024
        // 16:32 39.0 -> 31.1 us, 512^3 27.5 -> 25.2; 1024^3 (128 x 2 CTAs > SMs) and cfg1 (w = 128)
        // lose with any split
        for (int c = 4; c >= 2; --c)
            if (static_cast<int64_t>(ntiles) * c <= sms && w / c >= 128) {
                S = c;
                break;
            }
        return std::min(S, std::max(1, npanels / 2));
    }
    if (ntiles >= resident) {
        const int rem = ntiles % resident;
        if (rem > 0 && 2 * rem <= sms) S = std::min(3, sms / rem);
    } else {
        for (int c = 4; c >= 2; --c)
            if (static_cast<int64_t>(ntiles) * c <= sms && w / c >= 256) {
                S = c;
                break;
            }
        if (S == 1 && ntiles > sms && 2 * ntiles - resident <= sms / 2 && w / 2 >= 512) S = 2;
    }
    return std::min(S, std::max(1, npanels / 2));
}

// mode: 0 = A panels straight from A (swizzled [m][k] boxes), 1 = A^T staged (tile TMA),
// 2 = A^T staged + packed col_info loads (high sparsity).  The selector decides.
// At_in (nm_spmm_at): A arrives transposed from the caller (k x lda, lda >= m): staged mode
// without the per-call transpose (the packed mode, which reads whole bm-row segments raw, is off).
nm_status simt_f32_launch(const float* A, const float* Bv, const uint8_t* D, float* C, int64_t m, int64_t n, int64_t k,
                          int N, int M, int L, int mode, cudaStream_t s, const PeerOut* po, float alpha,
                          const uint32_t* Dw, const float* At_in, int64_t lda) {
    using namespace simt;
    Params p{};
    p.D = D;
    if (Dw) {  // bit-packed tile-major indices (needs 128 % L == 0: a CTA tile = whole groups)
        p.Dw = Dw;
        p.db = 1;
        while ((1 << p.db) < M) ++p.db;
        p.de = 32 / p.db;
        p.dT = 128 / L;
        p.dwt = ((k / M * N) * p.dT + p.de - 1) / p.de;
        if (mode == 2) mode = 1;  // the packed col_info mode reads D itself
    }
    p.C = C;
    p.alpha = alpha;
    if (po) {
        p.npeer = po->np;
        for (int i = 0; i < po->np && i < 8; ++i) p.cpeer[i] = static_cast<float*>(po->c[i]);
        p.ldc = po->ldc;
        p.col_off = po->col_off;
        p.n_valid = static_cast<int>(po->n_valid);
        p.mc = po->mc;
    }
    p.m = static_cast<int>(m);
    p.n = static_cast<int>(n);
    p.k = static_cast<int>(k);
    p.N = N;
    p.M = M;
    p.L = L;
    p.q = static_cast<int>(n / L);
    simt_f32_geometry(N, M, &p.wp, &p.bk, &p.bkw);
    const int windows = static_cast<int>(k / M);
    p.npanels = (windows + p.wp - 1) / p.wp;
    p.nboxA = (p.bk + A_BOX_COLS - 1) / A_BOX_COLS;
    const int64_t w = k / M * N;
    if (mode == 2 && p.npanels > MAX_PANELS_PACKED) mode = 1;
    const int bm = simt_row_tile(m, n, k / M * N);
    if (bm == 64 && mode == 2) mode = 1;  // packed mode: 512-B A^T rows (BM = 128)
    if (At_in) mode = 1;
    const bool use_at = mode >= 1;
    const bool packed = mode == 2;
    const int ntiles_n = static_cast<int>(ceil_div(n, BN));
    p.at_ld = static_cast<int>(ceil_div(m, bm) * bm);  // padded so every bm-row A^T segment is in bounds

    CUtensorMap tmA, tmB;
    nm_status st = make_tma_2d(&tmB, Bv, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, w, n, p.bkw, BN, 0);
    if (st) return st;
    float* AT = nullptr;
    uint64_t* masks = nullptr;
    if (At_in) {
        p.AT = At_in;
        st = make_tma_2d_pitched(&tmA, At_in, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, k, m, lda, p.bk, bm, 0);
    } else if (use_at) {
        st = scratch_alloc(reinterpret_cast<void**>(&AT), static_cast<size_t>(k) * p.at_ld * sizeof(float), s);
        if (st) return st;
        const dim3 tg(static_cast<unsigned>(ceil_div(k, 64)), static_cast<unsigned>(ceil_div(p.at_ld, 64)));
        transpose_kernel<<<tg, 256, 0, s>>>(A, AT, static_cast<int>(m), static_cast<int>(k), p.at_ld);
        note_launch();
        NM_LAUNCH_CHECK("transpose_kernel");
        p.AT = AT;
        st = make_tma_2d(&tmA, AT, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, k, p.at_ld, p.bk, bm, 0);
    } else {
        st = make_tma_2d(&tmA, A, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, m, k, bm, A_BOX_COLS, 128);
    }
    if (st) return st;
    if (packed) {
        st = scratch_alloc(reinterpret_cast<void**>(&masks), static_cast<size_t>(ntiles_n) * p.npanels * 8, s);
        if (st) return st;
        build_colinfo_kernel<<<dim3(p.npanels, ntiles_n), 128, 0, s>>>(D, masks, p.q, N, M, L, p.wp, p.bkw, p.npanels,
                                                                       static_cast<int>(w));
        note_launch();
        NM_LAUNCH_CHECK("build_colinfo_kernel");
        p.masks = masks;
    }

    // schedule: full waves of whole tiles, the partial last wave split along k
    p.ntn = ntiles_n;
    p.ntm = static_cast<int>(ceil_div(m, bm));
    {
        const char* ge = getenv("NM_SIMT_GROUP");
        p.gm = ge ? atoi(ge) : 8;
        if (p.gm < 1) p.gm = 1;
        if (p.gm > p.ntm) p.gm = p.ntm;
    }
    const int ntiles = ntiles_n * static_cast<int>(ceil_div(m, bm));
    const int resident = 2 * num_sms();  // 2 CTAs per SM (launch bounds, ~105 KB smem)
    const int rem = ntiles % resident;
    // the wave-model split of the 128-row tile, or the 64-row tile's split of very small grids
    const int split = simt_split_factor(ntiles, w, p.npanels, bm);
    p.split = split;
    p.full_tiles = split > 1 ? ntiles - rem : ntiles;
    float* ws = nullptr;
    int* counters = nullptr;
    if (split > 1) {
        st = scratch_alloc(reinterpret_cast<void**>(&ws), static_cast<size_t>(rem) * split * bm * BN * sizeof(float), s);
        if (!st) st = scratch_alloc(reinterpret_cast<void**>(&counters), static_cast<size_t>(rem) * sizeof(int), s);
        if (st) return st;
        NM_CUDA_TRY(cudaMemsetAsync(counters, 0, static_cast<size_t>(rem) * sizeof(int), s));
        p.ws = ws;
        p.counters = counters;
    }
    const dim3 grid(static_cast<unsigned>(p.full_tiles + (ntiles - p.full_tiles) * split));
    const bool two = L < 32;
    if (packed)
        st = two ? launch_simt<128, true, true, true>(tmA, tmB, p, grid, s)
                 : launch_simt<128, false, true, true>(tmA, tmB, p, grid, s);
    else if (bm == 64)
        st = use_at ? (two ? launch_simt<64, true, true, false>(tmA, tmB, p, grid, s)
                           : launch_simt<64, false, true, false>(tmA, tmB, p, grid, s))
                    : (two ? launch_simt<64, true, false, false>(tmA, tmB, p, grid, s)
                           : launch_simt<64, false, false, false>(tmA, tmB, p, grid, s));
    else if (use_at)
        st = two ? launch_simt<128, true, true, false>(tmA, tmB, p, grid, s)
                 : launch_simt<128, false, true, false>(tmA, tmB, p, grid, s);
    else
        st = two ? launch_simt<128, true, false, false>(tmA, tmB, p, grid, s)
                 : launch_simt<128, false, false, false>(tmA, tmB, p, grid, s);
    if (ws) {
        cudaError_t e1 = cudaFreeAsync(ws, s), e2 = cudaFreeAsync(counters, s);
        if (st == NM_OK && (e1 != cudaSuccess || e2 != cudaSuccess)) st = cuda_fail(e1 != cudaSuccess ? e1 : e2, "cudaFreeAsync");
    }
    if (masks) {
        cudaError_t e = cudaFreeAsync(masks, s);
        if (e != cudaSuccess && st == NM_OK) st = cuda_fail(e, "cudaFreeAsync");
    }
    if (AT) {
        cudaError_t e = cudaFreeAsync(AT, s);
        if (e != cudaSuccess && st == NM_OK) st = cuda_fail(e, "cudaFreeAsync");
    }
    return st;
}

}  // namespace nm
