// spmm_tc_pair.cu -- bf16 N:M SpMM on tcgen05, "token-pair" gather (sm_100a).
//
// Same contraction as spmm_tc.cu (Eq. 1: per column group g, C_g += A_g . B'_g
// with A_g the selected k of every window, one tcgen05.mma M=128 N=L K=16 per group
// and k-step, A_g in TMEM), with a gather that moves two useful bf16 per 4-byte
// shared-memory load instead of one:
//   * loaders rebuild the dense A panel as W[k][pair]: one 32-bit word holds token
//     rows r and r+8 (r in each 16-row block) at column k;
//   * gather warps store with tcgen05.st.16x128b, whose register pair per thread is
//     exactly (lane t/4, lane t/4+8) of a column, so one LDS.32 of W serves both
//     lanes and PRMT with a constant selector splits the pair;
//   * the 4 columns a warp loads at once are chosen (offline, per group and panel:
//     the paper's index reordering slot) so their 4 k-rows fall in
//     different bank quarters (row pitch 288 B = 8 banks mod 32 per k): the loads are
//     conflict-free whenever the k residues allow; B' rows are permuted identically
//     (prepacked B'_perm), so the MMA's K order matches.
#include <cuda_bf16.h>

#include <cstdlib>

#include "tcgen05.cuh"

namespace nm {
namespace tcp {

using namespace nm::tc;

constexpr int BM = 128;
constexpr int LOADER_WARPS = 4, GATHER_WARPS = 12;
constexpr int LOADER_THREADS = LOADER_WARPS * 32, GATHER_THREADS = GATHER_WARPS * 32;
constexpr int CONTROL_WARP = LOADER_WARPS + GATHER_WARPS;
constexpr int THREADS = (CONTROL_WARP + 1) * 32;  // 544
constexpr int B_STAGES = 3, A_STAGES = 2, S_STAGES = 2;
template <int BN> constexpr int nab() { return BN == 256 ? 2 : 3; }
template <int BN> constexpr int bkw_cap() { return BN == 256 ? 32 : 64; }
constexpr int BK_MAX = 128;
constexpr int CELLS_MAX = 256;
constexpr int PAIRS = BM / 2;                 // 64 token pairs per tile
constexpr int W_PITCH = PAIRS * 4 + 32;       // 288 B: k-rows shift 8 banks, so 4 rows mod 4 never collide
constexpr int W_STAGE_BYTES = ((BK_MAX + 1) * W_PITCH + 1023) / 1024 * 1024;  // + zero row (k = bk)
constexpr int TBL_BYTES = CELLS_MAX * 4;      // per cell: W-row byte offset of k_a | of k_b << 16
constexpr int STG_A_BYTES = BM * BK_MAX * 2;  // dense A panel, 128-B swizzled 64-column boxes
constexpr int STG_BYTES = STG_A_BYTES + TBL_BYTES;
constexpr int LD_UNITS = BK_MAX / 8 * 2 * 32 / LOADER_THREADS;  // (8-k chunk, 32-pair half) units: 8

template <int BN>
struct Smem {
    static constexpr int B_STAGE_BYTES = bkw_cap<BN>() * BN * 2;
    static constexpr int B = 0;
    static constexpr int W = B + B_STAGES * B_STAGE_BYTES;
    static constexpr int STG = W + S_STAGES * W_STAGE_BYTES;
    static constexpr int T = STG + A_STAGES * STG_BYTES;
    static constexpr int BAR = T + S_STAGES * TBL_BYTES;
    static constexpr int NBAR = 2 * B_STAGES + 2 * A_STAGES + 2 * S_STAGES + 2 * nab<BN>() + 1;
    static constexpr int TMEM_SLOT = BAR + NBAR * 8;
    static constexpr int BYTES = TMEM_SLOT + 16 + 1024;
};

struct Params {
    const uint32_t* tbl;  // [n tiles][npanels][CELLS_MAX] cell table, order [chunk][i][j]
    void* C;
    int m, n, k, N, M, L;
    int q, bk, bkw, bkw_pad, npanels;
    int c_bf16;
};

template <int BN>
__global__ void __launch_bounds__(THREADS, 1)
    spmm_tc_pair_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                        const Params p) {
    using S = Smem<BN>;
    constexpr int NAB = nab<BN>();
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* sB = smem + S::B;
    uint8_t* sW = smem + S::W;
    uint8_t* sStg = smem + S::STG;
    uint32_t* sT = reinterpret_cast<uint32_t*>(smem + S::T);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S::BAR);
    uint64_t* b_full = bars;
    uint64_t* b_free = b_full + B_STAGES;
    uint64_t* g_full = b_free + B_STAGES;   // staging (TMA) -> loaders
    uint64_t* g_free = g_full + A_STAGES;   // loaders -> staging refill
    uint64_t* s_full = g_free + A_STAGES;   // W + table -> gather
    uint64_t* s_free = s_full + S_STAGES;   // gather -> loaders
    uint64_t* a_full = s_free + S_STAGES;   // TMEM A buffer -> MMA
    uint64_t* a_free = a_full + NAB;        // MMA -> gather
    uint64_t* acc_full = a_free + NAB;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + S::TMEM_SLOT);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
    const int L = p.L, G = BN / L;
    const int bk = p.bk, bkwp = p.bkw_pad;
    const int cells_g = bkwp / 2;
    const int a_cols = G * cells_g;
    const int nbox = (bk + 63) / 64;

    if (warp == CONTROL_WARP) {
        if (lane == 0) {
            tma_prefetch_desc(&tmA);
            tma_prefetch_desc(&tmB);
            for (int s = 0; s < B_STAGES; ++s) {
                mbar_init(&b_full[s], 1);
                mbar_init(&b_free[s], 1);
            }
            for (int s = 0; s < A_STAGES; ++s) {
                mbar_init(&g_full[s], 1);
                mbar_init(&g_free[s], LOADER_THREADS);
            }
            for (int s = 0; s < S_STAGES; ++s) {
                mbar_init(&s_full[s], LOADER_THREADS);
                mbar_init(&s_free[s], GATHER_THREADS);
            }
            for (int s = 0; s < NAB; ++s) {
                mbar_init(&a_full[s], GATHER_THREADS);
                mbar_init(&a_free[s], 1);
            }
            mbar_init(acc_full, 1);
            fence_mbar_init();
        }
        __syncwarp();
        tmem_alloc(tmem_slot, 512);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == CONTROL_WARP) {
        // ===================== control: TMA (B'_perm, A panel, cell table) + MMA =====================
        const bool leader = elect_one();
        const int rb = (L >= 64 ? 64 : L) * 2;
        const int atoms = (L * 2 + 127) / 128;
        const int gbytes = bkwp * L * 2;
        const uint32_t layout = rb == 128 ? 2u : rb == 64 ? 4u : 6u;
        const uint32_t sbo = 8u * rb, lbo = static_cast<uint32_t>(bkwp * 128);
        const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) |
                               (static_cast<uint32_t>(L >> 3) << 17) | (static_cast<uint32_t>(BM >> 4) << 24);
        const uint32_t b_tx = static_cast<uint32_t>(G * atoms * bkwp * rb);
        const uint32_t a_tx = static_cast<uint32_t>(nbox * BM * 128 + TBL_BYTES);
        const uint32_t* tsrc = p.tbl + static_cast<int64_t>(blockIdx.x) * p.npanels * CELLS_MAX;
        const uint64_t gstep = static_cast<uint64_t>(gbytes >> 4), kstep = static_cast<uint64_t>((16 * rb) >> 4);
        const int nk = bkwp / 16;
        auto issue_b = [&](int panel) {
            if (leader) {
                const int s = panel % B_STAGES;
                mbar_arrive_expect_tx(&b_full[s], b_tx);
                uint8_t* dst = sB + s * S::B_STAGE_BYTES;
                for (int g = 0; g < G; ++g)
                    for (int a = 0; a < atoms; ++a)
                        tma_load_2d(dst + g * gbytes + a * bkwp * 128, &tmB, &b_full[s], n0 + g * L + a * 64,
                                    panel * bkwp);
            }
        };
        auto issue_a = [&](int panel) {
            if (leader) {
                const int s = panel % A_STAGES;
                uint8_t* dst = sStg + s * STG_BYTES;
                mbar_arrive_expect_tx(&g_full[s], a_tx);
                for (int b = 0; b < nbox; ++b) tma_load_2d(dst + b * (BM * 128), &tmA, &g_full[s], panel * bk + b * 64, m0);
                bulk_load(dst + STG_A_BYTES, tsrc + static_cast<int64_t>(panel) * CELLS_MAX, TBL_BYTES, &g_full[s]);
            }
        };
        for (int i = 0; i < A_STAGES && i < p.npanels; ++i) issue_a(i);
        int a_next = A_STAGES;
        for (int i = 0; i < B_STAGES - 1 && i < p.npanels; ++i) issue_b(i);
        for (int panel = 0; panel < p.npanels; ++panel) {
            const int nxt = panel + B_STAGES - 1;
            if (nxt < p.npanels) {
                if (nxt >= B_STAGES) mbar_wait(&b_free[nxt % B_STAGES], ((nxt / B_STAGES) - 1) & 1);
                issue_b(nxt);
            }
            const int s = panel % B_STAGES, ab = panel % NAB;
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
        while (a_next < p.npanels) {
            mbar_wait(&g_free[a_next % A_STAGES], ((a_next / A_STAGES) - 1) & 1);
            issue_a(a_next);
            ++a_next;
        }
        __syncwarp();
    } else if (warp < LOADER_WARPS) {
        // ===================== loaders: swizzled dense panel -> W[k][pair] =====================
        // unit = (8-column chunk c, half h): lanes take 32 consecutive pairs pp = 32h + lane;
        // pair pp = rows (r, r + 8), r = 16 * (pp / 8) + pp % 8.  Two LDS.128 (rows r, r+8 at
        // chunk c: the 8 rows r % 8 hit 8 distinct swizzled 16-B positions), 8 PRMT, 8 STS.32
        // into W rows 8c..8c+7 (bank = 8k + pp mod 32: 32 consecutive pairs are distinct).
        const int nchunk = bk / 8;
        for (int panel = 0; panel < p.npanels; ++panel) {
            const int st = panel % S_STAGES, gs = panel % A_STAGES;
            if (panel >= S_STAGES) mbar_wait(&s_free[st], ((panel / S_STAGES) - 1) & 1);
            mbar_wait(&g_full[gs], (panel / A_STAGES) & 1);
            const uint8_t* src = sStg + gs * STG_BYTES;
            uint8_t* W = sW + st * W_STAGE_BYTES;
#pragma unroll
            for (int i = 0; i < LD_UNITS; ++i) {
                const int u = i * LOADER_WARPS + warp;  // warp-uniform unit
                const int c = u >> 1, h = u & 1;
                if (c < nchunk) {
                    const int pp = 32 * h + lane;
                    const int r = 16 * (pp >> 3) + (pp & 7);
                    const uint8_t* a0 = src + (c >> 3) * (BM * 128) + r * 128 + (((c & 7) ^ (r & 7)) << 4);
                    const uint4 x = *reinterpret_cast<const uint4*>(a0);
                    const uint4 y = *reinterpret_cast<const uint4*>(a0 + 8 * 128);
                    uint8_t* w = W + (8 * c) * W_PITCH + pp * 4;
                    const uint32_t xs[4] = {x.x, x.y, x.z, x.w}, ys[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        *reinterpret_cast<uint32_t*>(w + (2 * j) * W_PITCH) = prmt(xs[j], ys[j], 0x5410u);
                        *reinterpret_cast<uint32_t*>(w + (2 * j + 1) * W_PITCH) = prmt(xs[j], ys[j], 0x7632u);
                    }
                }
            }
            // zero row (k = bk) for the padding sentinel, and the panel's cell table
            if (tid < PAIRS) *reinterpret_cast<uint32_t*>(W + bk * W_PITCH + tid * 4) = 0u;
            const uint4* ts = reinterpret_cast<const uint4*>(src + STG_A_BYTES);
            uint4* td = reinterpret_cast<uint4*>(sT + st * CELLS_MAX);
            for (int i = tid; i < TBL_BYTES / 16; i += LOADER_THREADS) td[i] = ts[i];
            mbar_arrive(&g_free[gs]);
            mbar_arrive(&s_full[st]);
        }
    } else {
        // ===================== gather: W pairs -> TMEM (16x128b stores) =====================
        const int gw = warp - LOADER_WARPS;
        const int quarter = warp & 3, sub = gw >> 2;  // 3 gather warps per lane quarter
        const int ti = lane & 3, prow = lane >> 2;
        const int nchunks = a_cols / 16;
        const int nitems = 2 * nchunks;  // (16-row half, 16-column chunk)
        for (int panel = 0; panel < p.npanels; ++panel) {
            const int st = panel % S_STAGES, ab = panel % NAB;
            mbar_wait(&s_full[st], (panel / S_STAGES) & 1);
            if (panel >= NAB) {
                mbar_wait(&a_free[ab], ((panel / NAB) - 1) & 1);
                tc_fence_after();
            }
            const uint8_t* W = sW + st * W_STAGE_BYTES;
            const uint32_t* tb = sT + st * CELLS_MAX;
            for (int it = sub; it < nitems; it += 3) {
                const int h = it & 1, chunk = it >> 1;
                const int pp = (2 * quarter + h) * 8 + prow;
                const uint8_t* wb = W + pp * 4;
                const uint4 e4 = *reinterpret_cast<const uint4*>(tb + chunk * 16 + ti * 4);
                const uint32_t es[4] = {e4.x, e4.y, e4.z, e4.w};
                uint32_t v[8];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const uint32_t wa = *reinterpret_cast<const uint32_t*>(wb + (es[j] & 0xFFFFu));
                    const uint32_t wv = *reinterpret_cast<const uint32_t*>(wb + (es[j] >> 16));
                    v[2 * j] = prmt(wa, wv, 0x5410u);      // row r:     (k_a, k_b)
                    v[2 * j + 1] = prmt(wa, wv, 0x7632u);  // row r + 8: (k_a, k_b)
                }
                tmem_st16x128b_x4(tmem + (static_cast<uint32_t>(quarter * 32 + h * 16) << 16) + BN + ab * a_cols +
                                      chunk * 16,
                                  v);
            }
            tmem_wait_st();
            tc_fence_before();
            mbar_arrive(&a_full[ab]);
            mbar_arrive(&s_free[st]);
        }
    }

    // ===================== epilogue (warps 0-15): TMEM -> registers -> global =====================
    if (warp < CONTROL_WARP) {
        const int quarter = warp & 3, sub = warp >> 2;
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
                        __nv_bfloat162 hh = __floats2bfloat162_rn(__uint_as_float(v[2 * i]), __uint_as_float(v[2 * i + 1]));
                        pk[i] = *reinterpret_cast<uint32_t*>(&hh);
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

// Offline index reordering for one (panel, group): the compacted k order
// pi (B'_perm row u' = B' row pi(u')) is chosen quad by quad so that the 4 "a" and the
// 4 "b" columns of every 4 consecutive cells have distinct (k mod 4) -- the bank
// quarter of W row k -- when the residues allow; padding rows (u >= bkw) act as
// wildcards.  Writes pi and the group's cells of the tile's cell table.
__global__ void pair_perm_kernel(const uint8_t* __restrict__ D, uint8_t* __restrict__ perm,
                                 uint32_t* __restrict__ tbl, int q, int N, int M, int BN, int L, int bk, int bkw,
                                 int bkwp, int npanels, int wtot) {
    const int gidx = blockIdx.x * blockDim.x + threadIdx.x;
    if (gidx >= q * npanels) return;
    const int panel = gidx / q, g = gidx % q;
    const int u0 = panel * bkw;
    int kl[64];       // panel-relative dense column of compressed row u (bk: padding)
    int bucket[5][64];
    int cnt[5] = {0, 0, 0, 0, 0};
    for (int u = 0; u < bkwp; ++u) {
        int k = bk;
        if (u < bkw && u0 + u < wtot) k = (u / N) * M + D[static_cast<int64_t>(u0 + u) * q + g];
        kl[u] = k;
        const int b = k == bk ? 4 : (k & 3);
        bucket[b][cnt[b]++] = u;
    }
    int take[4] = {0, 0, 0, 0}, wtake = 0;
    uint8_t* pm = perm + (static_cast<int64_t>(panel) * q + g) * 64;
    auto pick = [&](unsigned used) -> int {
        // the residue with most items left among unused ones; else a wildcard; else any
        int best = -1, bl = 0;
        for (int r = 0; r < 4; ++r)
            if (!(used >> r & 1u) && cnt[r] - take[r] > bl) best = r, bl = cnt[r] - take[r];
        if (best >= 0) return best;
        if (wtake < cnt[4]) return 4;
        for (int r = 0; r < 4; ++r)
            if (cnt[r] - take[r] > bl) best = r, bl = cnt[r] - take[r];
        return best;
    };
    const int G = BN / L, tile = g / G, gi = g % G, cells_g = bkwp / 2;
    uint32_t* t = tbl + (static_cast<int64_t>(tile) * npanels + panel) * CELLS_MAX;
    for (int qd = 0; qd < bkwp / 8; ++qd) {
        int ua[4], ub[4];
        for (int set = 0; set < 2; ++set) {
            unsigned used = 0;
            for (int i = 0; i < 4; ++i) {
                const int r = pick(used);
                const int u = r == 4 ? bucket[4][wtake++] : bucket[r][take[r]++];
                if (r < 4) used |= 1u << r;
                (set == 0 ? ua : ub)[i] = u;
            }
        }
        for (int i = 0; i < 4; ++i) {
            const int c = qd * 4 + i;  // cell inside the group
            pm[2 * c] = static_cast<uint8_t>(ua[i]);
            pm[2 * c + 1] = static_cast<uint8_t>(ub[i]);
            const int cell = gi * cells_g + c;  // cell inside the tile = TMEM column
            const int chunk = cell >> 4, w = cell & 15;
            t[chunk * 16 + (w & 3) * 4 + (w >> 2)] =
                static_cast<uint32_t>(kl[ua[i]] * W_PITCH) | (static_cast<uint32_t>(kl[ub[i]] * W_PITCH) << 16);
        }
    }
}

// B'_perm[panel * bkwp + u'][j] = B'[panel * bkw + pi_g(u')][j] (zeros for padding rows).
__global__ void pair_bperm_kernel(const __nv_bfloat16* __restrict__ Bv, const uint8_t* __restrict__ perm,
                                  __nv_bfloat16* __restrict__ Bp, int n, int q, int L, int bkw, int bkwp, int npanels,
                                  int wtot) {
    const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;  // 16-byte unit
    const int cpr = n / 8;
    if (e >= static_cast<int64_t>(npanels) * bkwp * cpr) return;
    const int row = static_cast<int>(e / cpr), cc = static_cast<int>(e % cpr);
    const int panel = row / bkwp, up = row % bkwp;
    const int g = (cc * 8) / L;
    const int u = perm[(static_cast<int64_t>(panel) * q + g) * 64 + up];
    uint4 v = make_uint4(0, 0, 0, 0);
    if (u < bkw && panel * bkw + u < wtot)
        v = *reinterpret_cast<const uint4*>(Bv + static_cast<int64_t>(panel * bkw + u) * n + cc * 8);
    *reinterpret_cast<uint4*>(Bp + static_cast<int64_t>(row) * n + cc * 8) = v;
}

}  // namespace tcp

bool tc_pair_applicable(int64_t m, int64_t n, int64_t k, int N, int M, int L, int bn, int bkw_pad) {
    const int G = bn / L;
    return (L == 16 || L == 32 || L == 64 || L == 128) && (G * bkw_pad / 2) % 16 == 0 && bkw_pad <= 64 &&
           M % 8 == 0 && n % 8 == 0 && k % 8 == 0 && m < (1ll << 31);
}

template <int BN>
static nm_status pair_launch_bn(const tcp::Params& p, const CUtensorMap& tmA, const CUtensorMap& tmB, int64_t m,
                                int64_t n, cudaStream_t s) {
    using namespace tcp;
    static bool attr = false;
    if (!attr) {
        NM_CUDA_TRY(cudaFuncSetAttribute(spmm_tc_pair_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         Smem<BN>::BYTES));
        attr = true;
    }
    const dim3 grid(static_cast<unsigned>(ceil_div(n, BN)), static_cast<unsigned>(ceil_div(m, BM)));
    prof_begin(s);
    spmm_tc_pair_kernel<BN><<<grid, THREADS, Smem<BN>::BYTES, s>>>(tmA, tmB, p);
    prof_end(s);
    note_launch();
    NM_LAUNCH_CHECK("spmm_tc_pair_kernel");
    return NM_OK;
}

// Sizes of the weight-side prepack (everything derived from B' and D alone).
void tc_pair_sizes(int64_t n, int64_t k, int N, int M, int L, int wp, int bkwp, int bn, size_t* perm_bytes,
                   size_t* tbl_bytes, size_t* bp_bytes) {
    const int64_t npanels = (k / M + wp - 1) / wp, q = n / L, ntiles = ceil_div(n, bn);
    *perm_bytes = static_cast<size_t>(npanels * q * 64);
    *tbl_bytes = static_cast<size_t>(ntiles * npanels) * tcp::TBL_BYTES;
    *bp_bytes = static_cast<size_t>(npanels * bkwp * n) * sizeof(__nv_bfloat16);
}

// The paper's offline PreProcessing (Listing 3) for the token-pair path:
// per-group k order (perm), cell tables (tbl) and the reordered B' (bp).
nm_status tc_pair_prepack(const void* Bv, const uint8_t* D, int64_t n, int64_t k, int N, int M, int L, int wp, int bk,
                          int bkw, int bkwp, int bn, uint8_t* perm, uint32_t* tbl, void* bp, cudaStream_t s) {
    using namespace tcp;
    const int q = static_cast<int>(n / L);
    const int npanels = static_cast<int>((k / M + wp - 1) / wp);
    const int wtot = static_cast<int>(k / M * N);
    size_t pb, tb, bb;
    tc_pair_sizes(n, k, N, M, L, wp, bkwp, bn, &pb, &tb, &bb);
    NM_CUDA_TRY(cudaMemsetAsync(tbl, 0, tb, s));
    const int nt = npanels * q;
    pair_perm_kernel<<<static_cast<unsigned>(ceil_div(nt, 128)), 128, 0, s>>>(D, perm, tbl, q, N, M, bn, L, bk, bkw,
                                                                             bkwp, npanels, wtot);
    note_launch();
    NM_LAUNCH_CHECK("pair_perm_kernel");
    const int64_t units = static_cast<int64_t>(npanels) * bkwp * (n / 8);
    pair_bperm_kernel<<<static_cast<unsigned>(ceil_div(units, 256)), 256, 0, s>>>(
        static_cast<const __nv_bfloat16*>(Bv), perm, static_cast<__nv_bfloat16*>(bp), static_cast<int>(n), q, L, bkw,
        bkwp, npanels, wtot);
    note_launch();
    NM_LAUNCH_CHECK("pair_bperm_kernel");
    return NM_OK;
}

nm_status tc_pair_run(const void* A, const uint32_t* tbl, const void* bp, void* C, bool c_bf16, int64_t m, int64_t n,
                      int64_t k, int N, int M, int L, int wp, int bk, int bkw, int bkwp, int bn, cudaStream_t s) {
    using namespace tcp;
    Params p{};
    p.C = C;
    p.m = static_cast<int>(m);
    p.n = static_cast<int>(n);
    p.k = static_cast<int>(k);
    p.N = N;
    p.M = M;
    p.L = L;
    p.q = static_cast<int>(n / L);
    p.bk = bk;
    p.bkw = bkw;
    p.bkw_pad = bkwp;
    p.c_bf16 = c_bf16 ? 1 : 0;
    p.npanels = static_cast<int>((k / M + wp - 1) / wp);
    p.tbl = tbl;
    CUtensorMap tmA, tmB;
    const int box_cols = L >= 64 ? 64 : L;
    nm_status st = make_tma_2d(&tmB, bp, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, static_cast<int64_t>(p.npanels) * bkwp, n,
                               bkwp, box_cols, box_cols * 2);
    if (!st) st = make_tma_2d(&tmA, A, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, m, k, BM, 64, 128);
    if (!st) st = bn == 256 ? pair_launch_bn<256>(p, tmA, tmB, m, n, s) : pair_launch_bn<128>(p, tmA, tmB, m, n, s);
    return st;
}

// nm_spmm without a prepacked weight: prepack into pooled scratch, run, release.
nm_status tc_pair_launch(const void* A, const void* Bv, const uint8_t* D, void* C, bool c_bf16, int64_t m, int64_t n,
                         int64_t k, int N, int M, int L, int wp, int bk, int bkw, int bkwp, int bn, cudaStream_t s) {
    size_t pb, tb, bb;
    tc_pair_sizes(n, k, N, M, L, wp, bkwp, bn, &pb, &tb, &bb);
    uint8_t* perm = nullptr;
    uint32_t* tbl = nullptr;
    void* bp = nullptr;
    nm_status st = scratch_alloc(reinterpret_cast<void**>(&perm), pb, s);
    if (!st) st = scratch_alloc(reinterpret_cast<void**>(&tbl), tb, s);
    if (!st) st = scratch_alloc(&bp, bb, s);
    if (st) return st;
    st = tc_pair_prepack(Bv, D, n, k, N, M, L, wp, bk, bkw, bkwp, bn, perm, tbl, bp, s);
    if (!st) st = tc_pair_run(A, tbl, bp, C, c_bf16, m, n, k, N, M, L, wp, bk, bkw, bkwp, bn, s);
    cudaError_t e1 = cudaFreeAsync(bp, s), e2 = cudaFreeAsync(tbl, s), e3 = cudaFreeAsync(perm, s);
    if (st == NM_OK && (e1 != cudaSuccess || e2 != cudaSuccess || e3 != cudaSuccess)) st = cuda_fail(e1, "cudaFreeAsync");
    return st;
}

}  // namespace nm
