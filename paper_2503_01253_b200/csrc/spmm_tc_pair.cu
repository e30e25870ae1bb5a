// spmm_tc_pair.cu -- bf16 N:M SpMM on tcgen05, "token-pair" gather (sm_100a).
//
// Same contraction as spmm_tc.cu (Eq. 1: per column group g, C_g += A_g . B'_g
// with A_g the selected k of every window, one tcgen05.mma M=128 N=L K=16 per group
// and k-step, A_g in TMEM), with a gather that moves two useful bf16 per 4-byte
// shared-memory load instead of one:
//   * A is repacked once per call (pair_pack_a_kernel) into Apair[m/128][k][64 pairs]:
//     one 32-bit word holds token rows r and r+8 (r in each 16-row block) at column k;
//     TMA drops a panel of it straight into shared memory (two 128-B-swizzled boxes of
//     32 pairs), so no warp rebuilds the panel on chip;
//   * gather warps store with tcgen05.st.16x128b, whose register pair per thread is
//     exactly (lane t/4, lane t/4+8) of a column, so one LDS.32 serves both lanes and
//     PRMT with a constant selector splits the pair;
//   * the 4 columns a warp loads at once are chosen (offline, per group and panel: the
//     paper's index reordering slot) so their k rows have distinct
//     (k >> 1) & 3 -- with the 128-B swizzle that puts the 4 loads in 4 different
//     8-bank groups, conflict-free whenever the residues allow; B' rows are permuted
//     identically (prepacked B' images), so the MMA's K order matches.
// Roles: 16 gather warps (also the epilogue), 1 MMA warp, 2 producer warps (A pair panels, B' images).
#include <cuda_bf16.h>

#include <cstdlib>

#include "tcgen05.cuh"

namespace nm {
namespace tcp {

using namespace nm::tc;

constexpr int BM = 128;
constexpr int GATHER_WARPS = 16;
constexpr int MMA_WARP = GATHER_WARPS, A_PRODUCER_WARP = MMA_WARP + 1, B_PRODUCER_WARP = MMA_WARP + 2;
constexpr int THREADS = (B_PRODUCER_WARP + 1) * 32;  // 608
constexpr int B_STAGES = 3, A_STAGES = 4;
template <int BN> constexpr int nab() { return BN == 256 ? 2 : 3; }
template <int BN> constexpr int bkw_cap() { return BN == 256 ? 32 : 64; }
constexpr int BK_MAX = 128;
constexpr int CELLS_MAX = 256;
constexpr int PAIRS = BM / 2;  // 64 token pairs per tile
constexpr int HALF_BYTES = ((BK_MAX + 1) * 128 + 1023) / 1024 * 1024;  // 32 pairs x (bk rows + zero row k = bk)
constexpr int TBL_BYTES = CELLS_MAX * 4;  // per cell: W offset of k_a | of k_b << 16, offset = 128 k + 16 (k & 7)
constexpr int A_STAGE_BYTES = 2 * HALF_BYTES + TBL_BYTES;

template <int BN>
struct Smem {
    static constexpr int B_STAGE_BYTES = bkw_cap<BN>() * BN * 2;
    static constexpr int B = 0;
    static constexpr int A = B + B_STAGES * B_STAGE_BYTES;
    static constexpr int BAR = A + A_STAGES * A_STAGE_BYTES;
    static constexpr int NBAR = 2 * B_STAGES + 2 * A_STAGES + 2 * nab<BN>() + 1;
    static constexpr int TMEM_SLOT = BAR + NBAR * 8;
    static constexpr int BYTES = TMEM_SLOT + 16 + 1024;
};

struct Params {
    const uint32_t* tbl;  // [n tiles][npanels][CELLS_MAX] cell table, order [chunk][i][j]
    const uint8_t* bimg;  // [n tiles][npanels][bkw_pad * BN * 2 B]: B'_perm as the swizzled smem image
    void* C;
    int m, n, k, N, M, L;
    int q, bk, bkw, bkw_pad, npanels;
    int c_bf16;
    int dbg;  // ablation mask (NM_TC_DBG, timing studies only): 1 skip gather, 2 skip MMA, 8 skip A TMA,
              // 16 skip B TMA, 64 timestamps
};

// NM_TC_DBG & 64: CTA (0,0) records clock64 per panel and role into C (timing study only)
#define NM_TS(slot)                                                                                       \
    do {                                                                                                  \
        if ((p.dbg & 64) && blockIdx.x == 0 && blockIdx.y == 0 && lane == 0)                              \
            static_cast<long long*>(p.C)[panel * 12 + (slot)] = clock64();                                \
    } while (0)

template <int BN, int L>
__global__ void __launch_bounds__(THREADS, 1)
    spmm_tc_pair_kernel(const __grid_constant__ CUtensorMap tmA, const Params p) {
    using S = Smem<BN>;
    constexpr int NAB = nab<BN>();
    constexpr int G = BN / L;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* sB = smem + S::B;
    uint8_t* sA = smem + S::A;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S::BAR);
    uint64_t* b_full = bars;                 // B' image landed
    uint64_t* b_free = b_full + B_STAGES;    // MMA done with the B stage
    uint64_t* s_full = b_free + B_STAGES;    // A pair panel + cell table landed
    uint64_t* s_free = s_full + A_STAGES;    // gather done with the A stage
    uint64_t* t_full = s_free + A_STAGES;    // TMEM A buffer written (gather -> MMA)
    uint64_t* t_free = t_full + NAB;         // MMA done with the TMEM A buffer
    uint64_t* acc_full = t_free + NAB;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + S::TMEM_SLOT);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int m0 = blockIdx.y * BM;
    const int bk = p.bk, bkwp = p.bkw_pad;
    const int cells_g = bkwp / 2;
    const int a_cols = G * cells_g;

    if (warp == MMA_WARP) {
        if (lane == 0) {
            tma_prefetch_desc(&tmA);
            for (int s = 0; s < B_STAGES; ++s) {
                mbar_init(&b_full[s], 1);
                mbar_init(&b_free[s], 1);
            }
            for (int s = 0; s < A_STAGES; ++s) {
                mbar_init(&s_full[s], 1);
                mbar_init(&s_free[s], GATHER_WARPS);
            }
            for (int s = 0; s < NAB; ++s) {
                mbar_init(&t_full[s], GATHER_WARPS);
                mbar_init(&t_free[s], 1);
            }
            mbar_init(acc_full, 1);
            fence_mbar_init();
        }
        __syncwarp();
        tmem_alloc(tmem_slot, 512);
    } else if (warp < GATHER_WARPS) {
        // zero row (k = bk) of every half panel: the padding cells' sentinel; TMA writes rows < bk only
        for (int i = tid; i < A_STAGES * 2 * 32; i += GATHER_WARPS * 32) {
            const int st = i >> 6, h = (i >> 5) & 1, w = i & 31;
            *reinterpret_cast<uint32_t*>(sA + st * A_STAGE_BYTES + h * HALF_BYTES + bk * 128 + w * 4) = 0u;
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    // One CTA per SM (shared memory) allocating all 512 columns: the allocation starts at
    // lane 0, column 0.  Using the constant keeps every MMA operand in uniform registers
    // (an address loaded from shared memory is per-lane to the compiler and costs an
    // R2UR per operand per MMA); a different address would be a hardware contract change.
    constexpr uint32_t tmem = 0;
    if (*tmem_slot != tmem) __trap();

    if (warp == MMA_WARP) {
        // ===================== MMA issuer: one tcgen05.mma per (group, 16-k step) =====================
        constexpr int rb = (L >= 64 ? 64 : L) * 2;
        constexpr uint32_t layout = rb == 128 ? 2u : rb == 64 ? 4u : 6u;
        constexpr uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) |
                                   (static_cast<uint32_t>(L >> 3) << 17) | (static_cast<uint32_t>(BM >> 4) << 24);
        constexpr uint64_t kstep = static_cast<uint64_t>((16 * rb) >> 4);
        const uint32_t sbo = 8u * rb, lbo = static_cast<uint32_t>(bkwp * 128);
        const uint64_t gstep = static_cast<uint64_t>((bkwp * L * 2) >> 4);
        const int nk = bkwp / 16;
        const uint64_t d0 = smem_desc(smem_u32(sB), lbo, sbo, layout);
        constexpr uint64_t sstep = static_cast<uint64_t>(S::B_STAGE_BYTES >> 4);
        for (int panel = 0; panel < p.npanels; ++panel) {
            const int s = panel % B_STAGES, ab = panel % NAB;
            mbar_wait(&b_full[s], (panel / B_STAGES) & 1);
            NM_TS(0);
            mbar_wait(&t_full[ab], (panel / NAB) & 1);
            NM_TS(1);
            tc_fence_after();
            if (elect_one() && !(p.dbg & 2)) {
                // all operands are warp-uniform: fully unrolled over the compile-time group
                // count, the k-steps predicated on nk <= 4, so the MMAs issue back to back
                const uint64_t dg = d0 + s * sstep;
                const uint32_t ag = tmem + BN + ab * a_cols;
                const uint32_t acc0 = panel ? 1u : 0u;
#pragma unroll
                for (int g = 0; g < G; ++g) {
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk)
                        if (kk < nk)
                            mma_ts(tmem + g * L, ag + g * cells_g + kk * 8, dg + g * gstep + kk * kstep, idesc,
                                   kk ? 1u : acc0);
                }
            }
            __syncwarp();
            NM_TS(2);
            if (elect_one()) {
                tc_commit(&t_free[ab]);
                tc_commit(&b_free[s]);
            }
            __syncwarp();
        }
        if (elect_one()) tc_commit(acc_full);
        __syncwarp();
    } else if (warp == A_PRODUCER_WARP) {
        // ===================== A producer: TMA of the pair panel + bulk copy of the cell table ==========
        const bool leader = elect_one();
        const uint32_t a_tx = static_cast<uint32_t>(2 * bk * 128 + TBL_BYTES);
        const uint32_t* tsrc = p.tbl + static_cast<int64_t>(blockIdx.x) * p.npanels * CELLS_MAX;
        const int arow0 = blockIdx.y * p.k;  // Apair row of (m block, k = 0)
        for (int panel = 0; panel < p.npanels; ++panel) {
            const int sa = panel % A_STAGES;
            if (panel >= A_STAGES) mbar_wait(&s_free[sa], ((panel / A_STAGES) - 1) & 1);
            if (leader) {
                if (p.dbg & 8) {
                    mbar_arrive(&s_full[sa]);
                } else {
                    uint8_t* dst = sA + sa * A_STAGE_BYTES;
                    mbar_arrive_expect_tx(&s_full[sa], a_tx);
                    tma_load_2d(dst, &tmA, &s_full[sa], 0, arow0 + panel * bk);
                    tma_load_2d(dst + HALF_BYTES, &tmA, &s_full[sa], 32, arow0 + panel * bk);
                    bulk_load(dst + 2 * HALF_BYTES, tsrc + static_cast<int64_t>(panel) * CELLS_MAX, TBL_BYTES,
                              &s_full[sa]);
                }
            }
            __syncwarp();
        }
    } else if (warp == B_PRODUCER_WARP) {
        // ===================== B producer: bulk copy of the B' image =====================
        const bool leader = elect_one();
        const uint32_t b_bytes = static_cast<uint32_t>(bkwp * BN * 2);
        const uint8_t* bsrc = p.bimg + static_cast<int64_t>(blockIdx.x) * p.npanels * b_bytes;
        for (int panel = 0; panel < p.npanels; ++panel) {
            const int sb = panel % B_STAGES;
            if (panel >= B_STAGES) mbar_wait(&b_free[sb], ((panel / B_STAGES) - 1) & 1);
            if (leader) {
                if (p.dbg & 16) {
                    mbar_arrive(&b_full[sb]);
                } else {
                    mbar_arrive_expect_tx(&b_full[sb], b_bytes);
                    bulk_load(sB + sb * S::B_STAGE_BYTES, bsrc + static_cast<int64_t>(panel) * b_bytes, b_bytes,
                              &b_full[sb]);
                }
            }
            __syncwarp();
        }
    } else {
        // ===================== gather: pair words -> TMEM (16x128b stores) =====================
        // item = (16-row half h, 16-column chunk); lane t: pair pp = (2 quarter + h) 8 + t / 4,
        // cell j of the chunk's 4 x 4 block = t % 4 + 4 j; word of (k, pp) in the half panel
        // pp / 32 at 128 k + 16 ((pp % 32) / 4 ^ k % 8) + 4 (pp % 4) = (table entry ^ q16) + 4 (pp % 4).
        const int quarter = warp & 3, sub = warp >> 2;  // 4 gather warps per TMEM lane quarter
        const int ti = lane & 3, prow = lane >> 2;
        const int nchunks = a_cols / 16;
        const int h = sub & 1;
        const int pp = (2 * quarter + h) * 8 + prow;
        const uint32_t q16 = static_cast<uint32_t>(((pp & 31) >> 2) << 4);
        for (int panel = 0; panel < p.npanels; ++panel) {
            const int st = panel % A_STAGES, ab = panel % NAB;
            mbar_wait(&s_full[st], (panel / A_STAGES) & 1);
            if (sub == 0) NM_TS(3);
            if (panel >= NAB) {
                mbar_wait(&t_free[ab], ((panel / NAB) - 1) & 1);
                tc_fence_after();
            }
            if (sub == 0) NM_TS(4);
            const uint8_t* stage = sA + st * A_STAGE_BYTES;
            const uint32_t* tb = reinterpret_cast<const uint32_t*>(stage + 2 * HALF_BYTES);
            const uint8_t* wb = stage + (pp >> 5) * HALF_BYTES + (pp & 3) * 4;
            // this warp's items: fixed half h = sub % 2, chunks sub / 2 + 2 i; two items per
            // step so 16 independent loads are in flight before the first PRMT
            const uint32_t tcol = tmem + (static_cast<uint32_t>(quarter * 32 + h * 16) << 16) + BN + ab * a_cols;
            for (int c = (p.dbg & 1) ? nchunks : (sub >> 1); c < nchunks; c += 4) {
                const bool two = c + 2 < nchunks;
                const uint4 ea = *reinterpret_cast<const uint4*>(tb + c * 16 + ti * 4);
                const uint4 eb = two ? *reinterpret_cast<const uint4*>(tb + (c + 2) * 16 + ti * 4) : ea;
                const uint32_t es[8] = {ea.x, ea.y, ea.z, ea.w, eb.x, eb.y, eb.z, eb.w};
                uint32_t wa[8], wv[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    wa[j] = *reinterpret_cast<const uint32_t*>(wb + ((es[j] & 0xFFFFu) ^ q16));
                    wv[j] = *reinterpret_cast<const uint32_t*>(wb + ((es[j] >> 16) ^ q16));
                }
                uint32_t v[8];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    v[2 * j] = prmt(wa[j], wv[j], 0x5410u);      // row r:     (k_a, k_b)
                    v[2 * j + 1] = prmt(wa[j], wv[j], 0x7632u);  // row r + 8: (k_a, k_b)
                }
                tmem_st16x128b_x4(tcol + c * 16, v);
                if (two) {
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        v[2 * j] = prmt(wa[4 + j], wv[4 + j], 0x5410u);
                        v[2 * j + 1] = prmt(wa[4 + j], wv[4 + j], 0x7632u);
                    }
                    tmem_st16x128b_x4(tcol + (c + 2) * 16, v);
                }
            }
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(&t_full[ab]);
                mbar_arrive(&s_free[st]);
            }
            if (sub == 0) NM_TS(5);
        }
    }

    // ===================== epilogue (gather warps): TMEM -> registers -> global =====================
    if (warp < GATHER_WARPS) {
        const int quarter = warp & 3, sub = warp >> 2;
        const uint32_t lane_addr = static_cast<uint32_t>(quarter * 32) << 16;
        const int grow = m0 + quarter * 32 + lane;
        const int n0 = blockIdx.x * BN;
        mbar_wait(acc_full, 0);
        tc_fence_after();
        for (int cb = sub * 16; cb < BN; cb += 64) {
            uint32_t v[16];
            tmem_ld16(tmem + lane_addr + cb, v);
            tmem_wait_ld();
            const int gc = n0 + cb;
            if (grow < p.m && gc < p.n && !(p.dbg & 64)) {
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
    if (warp == MMA_WARP) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

// A (m x k bf16, row-major) -> Apair[ceil(m/128)][k][64] uint32: word (b, k, pp) = bf16 pair
// (A[128 b + r][k], A[128 b + r + 8][k]), r = 16 (pp / 8) + pp % 8; rows >= m are zero.
// One thread per (block, 8-column chunk, pair): two 16-B loads, eight 4-B stores (a warp
// covers 32 consecutive pairs of one k row: 128-B coalesced stores).
__global__ void pair_pack_a_kernel(const __nv_bfloat16* __restrict__ A, uint32_t* __restrict__ Ap, int m, int k) {
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int kc8 = k / 8;
    const int pp = static_cast<int>(t % PAIRS);
    const int64_t rest = t / PAIRS;
    const int c = static_cast<int>(rest % kc8);
    const int b = static_cast<int>(rest / kc8);
    if (b >= (m + BM - 1) / BM) return;
    const int r = b * BM + 16 * (pp >> 3) + (pp & 7);
    uint4 x = make_uint4(0, 0, 0, 0), y = make_uint4(0, 0, 0, 0);
    if (r < m) x = *reinterpret_cast<const uint4*>(A + static_cast<int64_t>(r) * k + c * 8);
    if (r + 8 < m) y = *reinterpret_cast<const uint4*>(A + static_cast<int64_t>(r + 8) * k + c * 8);
    const uint32_t xs[4] = {x.x, x.y, x.z, x.w}, ys[4] = {y.x, y.y, y.z, y.w};
    uint32_t* dst = Ap + (static_cast<int64_t>(b) * k + c * 8) * PAIRS + pp;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        dst[(2 * j) * PAIRS] = prmt(xs[j], ys[j], 0x5410u);
        dst[(2 * j + 1) * PAIRS] = prmt(xs[j], ys[j], 0x7632u);
    }
}

// byte offset of pair-panel row k before the lane's chunk XOR: 128 k + 16 (k mod 8)
__device__ __forceinline__ uint32_t woff(int k) { return static_cast<uint32_t>(128 * k + 16 * (k & 7)); }

// Offline index reordering for one (panel, group): the compacted k order
// pi (B'_perm row u' = B' row pi(u')) is chosen quad by quad so that the 4 "a" and the
// 4 "b" columns of every 4 consecutive cells have distinct (k >> 1) mod 4 -- the 8-bank
// group row k's swizzle sends a lane quad to -- when the residues allow; padding rows
// (u >= bkw, k = bk: the zero row) act as wildcards.  Writes pi and the group's cells
// of the tile's cell table.
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
        const int b = k == bk ? 4 : ((k >> 1) & 3);
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
                woff(kl[ua[i]]) | (woff(kl[ub[i]]) << 16);
        }
    }
}

// B'_perm as shared-memory images, one contiguous block per (column tile, panel) that a
// single bulk copy drops into a B stage: per group g (and 64-column atom a when L > 64)
// a [bkw_pad rows][min(L,64) columns] MN-major box, 16-B chunks XOR-swizzled with the
// row-address bits exactly as a TMA load with swizzle = row bytes would place them
// (offset bits [4, 4+s) ^= bits [7, 7+s), s = log2(row bytes / 16)).  Row u' of group g
// is B'[panel * bkw + pi_g(u')] (zeros for padding rows and columns >= n).
__global__ void pair_bimg_kernel(const __nv_bfloat16* __restrict__ Bv, const uint8_t* __restrict__ perm,
                                 uint8_t* __restrict__ img, int n, int q, int L, int BN, int bkw, int bkwp, int npanels,
                                 int ntiles, int wtot) {
    const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;  // 16-byte chunk of the image
    const int block16 = bkwp * BN * 2 / 16;
    if (e >= static_cast<int64_t>(ntiles) * npanels * block16) return;
    const int blk = static_cast<int>(e / block16);
    const int o = static_cast<int>(e % block16) * 16;
    const int tile = blk / npanels, panel = blk % npanels;
    const int rb = (L >= 64 ? 64 : L) * 2, atoms = (L * 2 + 127) / 128;
    const int R = bkwp * rb;
    const int reg = o / R, g = reg / atoms, a = reg % atoms, off = o % R;
    const int lin = off ^ (((off >> 7) & ((rb >> 4) - 1)) << 4);
    const int r = lin / rb, e0 = (lin % rb) / 2;
    const int col = tile * BN + g * L + a * 64 + e0;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (col < n) {
        const int u = perm[(static_cast<int64_t>(panel) * q + col / L) * 64 + r];
        if (u < bkw && panel * bkw + u < wtot)
            v = *reinterpret_cast<const uint4*>(Bv + static_cast<int64_t>(panel * bkw + u) * n + col);
    }
    *reinterpret_cast<uint4*>(img + e * 16) = v;
}

}  // namespace tcp

bool tc_pair_applicable(int64_t m, int64_t n, int64_t k, int N, int M, int L, int bn, int bkw_pad) {
    const int G = bn / L;
    return (L == 16 || L == 32 || L == 64 || L == 128) && (G * bkw_pad / 2) % 16 == 0 && bkw_pad <= 64 &&
           M % 8 == 0 && n % 8 == 0 && k % 8 == 0 && m < (1ll << 31);
}

template <int BN, int L>
static nm_status pair_launch_bn(const tcp::Params& p, const CUtensorMap& tmA, int64_t m, int64_t n, cudaStream_t s) {
    using namespace tcp;
    static bool attr = false;
    if (!attr) {
        NM_CUDA_TRY(cudaFuncSetAttribute(spmm_tc_pair_kernel<BN, L>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         Smem<BN>::BYTES));
        attr = true;
    }
    const dim3 grid(static_cast<unsigned>(ceil_div(n, BN)), static_cast<unsigned>(ceil_div(m, BM)));
    prof_begin(s);
    spmm_tc_pair_kernel<BN, L><<<grid, THREADS, Smem<BN>::BYTES, s>>>(tmA, p);
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
    *bp_bytes = static_cast<size_t>(ntiles * npanels * bkwp * bn) * sizeof(__nv_bfloat16);
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
    const int ntiles = static_cast<int>(ceil_div(n, bn));
    const int64_t units = static_cast<int64_t>(ntiles) * npanels * bkwp * bn * 2 / 16;
    pair_bimg_kernel<<<static_cast<unsigned>(ceil_div(units, 256)), 256, 0, s>>>(
        static_cast<const __nv_bfloat16*>(Bv), perm, static_cast<uint8_t*>(bp), static_cast<int>(n), q, L, bn, bkw,
        bkwp, npanels, ntiles, wtot);
    note_launch();
    NM_LAUNCH_CHECK("pair_bimg_kernel");
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
    const char* dbg = std::getenv("NM_TC_DBG");
    p.dbg = dbg ? std::atoi(dbg) : 0;
    p.bimg = static_cast<const uint8_t*>(bp);
    const int64_t mblocks = ceil_div(m, BM);
    uint32_t* ap = nullptr;
    nm_status st = scratch_alloc(reinterpret_cast<void**>(&ap), static_cast<size_t>(mblocks * k * PAIRS * 4), s);
    if (st) return st;
    const int64_t threads = mblocks * (k / 8) * PAIRS;
    pair_pack_a_kernel<<<static_cast<unsigned>(ceil_div(threads, 256)), 256, 0, s>>>(
        static_cast<const __nv_bfloat16*>(A), ap, static_cast<int>(m), static_cast<int>(k));
    note_launch();
    NM_LAUNCH_CHECK("pair_pack_a_kernel");
    CUtensorMap tmA;
    st = make_tma_2d(&tmA, ap, CU_TENSOR_MAP_DATA_TYPE_UINT32, 4, mblocks * k, PAIRS, bk, 32, 128);
    if (!st) {
        const int key = bn * 1000 + L;
        switch (key) {
            case 128016: st = pair_launch_bn<128, 16>(p, tmA, m, n, s); break;
            case 128032: st = pair_launch_bn<128, 32>(p, tmA, m, n, s); break;
            case 128064: st = pair_launch_bn<128, 64>(p, tmA, m, n, s); break;
            case 128128: st = pair_launch_bn<128, 128>(p, tmA, m, n, s); break;
            case 256016: st = pair_launch_bn<256, 16>(p, tmA, m, n, s); break;
            case 256032: st = pair_launch_bn<256, 32>(p, tmA, m, n, s); break;
            case 256064: st = pair_launch_bn<256, 64>(p, tmA, m, n, s); break;
            case 256128: st = pair_launch_bn<256, 128>(p, tmA, m, n, s); break;
            default: st = fail(NM_ERR_UNSUPPORTED, "token-pair kernel: unsupported (BN, L)");
        }
    }
    const cudaError_t e = cudaFreeAsync(ap, s);
    if (st == NM_OK && e != cudaSuccess) st = cuda_fail(e, "cudaFreeAsync");
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
