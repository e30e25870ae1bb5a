// spmm_tc_sp.cu -- bf16 vector-wise N:M SpMM on the sparse tensor cores (tcgen05.mma.sp, sm_100a).
//
// Eq. 1 computed as C^T = B~^T . A^T with the weight as the MMA's sparse A operand:
//   * MMA M = 128 output columns per column half (128 / L groups; H = 1 or 2 halves share a
//     token tile), MMA N = NT tokens (160-256), MMA K = 32 "slots".
//   * Per column tile, the union of the k rows its groups keep (the paper's col_info)
//     is arranged offline into a slot sequence kappa(s) in which every aligned quad of slots holds
//     at most two rows kept by any one group (sp_pack_kernel: the paper's offline index
//     reordering).  Each output column then is 2:4 sparse along the slots, which is
//     exactly what the sparse tensor core contracts at twice the dense rate: per quad, two
//     values of B' plus a 4-bit metadata nibble naming their slots.
//   * The dense operand is the token tile of A gathered by slot: rows kappa(s) of A^T (A
//     transposed once per call), one row segment (NT tokens) per warp-wide 16-B cp.async,
//     written straight into the 128-B-swizzled MN-major layout the MMA reads.  (TMA
//     tile::gather4 does the same with no SM instructions but measured ~80 clk per 4 rows
//     per SM on B200 -- 6x slower than this kernel needs.)
//   * Compressed weights + metadata are prepacked per (column tile, 64-slot stage) as the exact
//     shared-memory images (one bulk copy each; a stage pair's metadata rides with its even
//     stage); metadata goes to TMEM by tcgen05.cp.
// Roles: warps 0-7 gather (8 slot rows each per stage; warp 0 also bulk-copies the weight
// image) and then the epilogue (TMEM -> registers -> smem -> TMA store); warp 8 issues the
// tcgen05.cp + 2 H tcgen05.mma.sp per stage.  Optional: tail split of the last partial wave,
// (the round-2 weight multicast over 2-CTA clusters measured slower and was removed).
#include <cuda_bf16.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>

#include "tc_sp.cuh"

namespace nm {

__global__ void transpose_kernel(const float* __restrict__ A, float* __restrict__ AT, int m, int k, int ld);


namespace tcs {

using namespace nm::tc;

constexpr int GATHER_WARPS = 8;            // also the epilogue warps (TMEM lane quarter = warp % 4)
constexpr int MMA_WARP = GATHER_WARPS;
constexpr int THREADS = (GATHER_WARPS + 1) * 32;
constexpr int TMEM_COLS = 512;

template <int H, int NT_, bool TF = false>
struct Cfg {
    static constexpr int MC = 128 * H;                    // output columns per CTA
    static constexpr int NT = NT_;                        // tokens per CTA (MMA N)
    static constexpr int ATOMS = (NT + El<TF>::TOK_ATOM - 1) / El<TF>::TOK_ATOM;
    static constexpr int B_BYTES = El<TF>::SLOTS * ATOMS * 128;  // token atoms x slot rows x 128 B
    static constexpr int W_BYTES = H * WH_BYTES;          // per (column tile, stage) weight image
    static constexpr int ST0 = (232448 - 1024 - 256) / (W_BYTES + B_BYTES);
    static constexpr int ST = ST0 > 8 ? 8 : ST0;          // pipeline stages (shared-memory bound)
    static constexpr int SMEM_BYTES = ST * (W_BYTES + B_BYTES) + 1024 + 256;
    static constexpr int META_COL = H * NT;               // metadata ring: 4 H columns per stage pair
    // a pair's TMEM columns are rewritten NPAIR pairs later; by then the producer has refilled the
    // smem slot of a stage >= STAGES later, so the MMAs that read them have completed
    static constexpr int NPAIR = (ST + 2) / 2;
    static_assert(NT % 16 == 0 && NT <= 256, "MMA N");
    static_assert(META_COL + 4 * H * NPAIR <= TMEM_COLS, "TMEM budget");
    static_assert(SMEM_BYTES <= 232448, "shared memory budget");
};

// Tokens per CTA (MMA N); NM_SP_NT overrides (ablation).  Choice by a wave model: a tile's time
// ~ its stages x (hand-off floor + MMA work), the MMA work growing with NT, so over the candidate
// token tiles minimise rounds(tiles) x (NT + 64): rounds = full waves of tiles over the SMs plus
// the last partial wave (half a round when it at most half fills the SMs and may be split).  The
// +64 is the per-tile fixed cost in token-equivalents (fit on the A-F study: on small grids NT = 128
// wins at H = 1, profiles/r02e_protocol_summary.txt); at equal cost the earlier candidate wins
// (the order is the measured preference, profiles/r01f_sp_nt_sweep.txt; TMEM caps N at 224 with two
// accumulators and the metadata ring at H = 2).
constexpr int MIN_PART_STAGES = 24;  // a split part keeps >= 24 stages (sp_launch_h, profiles/r02f_sp_split_probe.txt)
static int sp_tokens(int H, int64_t m, int64_t n, int est_stages) {
    const char* e = std::getenv("NM_SP_NT");
    if (e) return std::atoi(e);
    const int64_t sms = num_sms(), col_tiles = (n + 128 * H - 1) / (128 * H);
    static const int c1[] = {256, 192, 128};
    static const int c2[] = {192, 208, 176, 224, 160, 128};
    const int* cand = H == 1 ? c1 : c2;
    const int nc = H == 1 ? 3 : 6;
    int best = cand[0];
    double best_cost = -1;
    for (int i = 0; i < nc; ++i) {
        const int nt = cand[i];
        const int64_t tiles = col_tiles * ((m + nt - 1) / nt), tail = tiles % sms;
        double rounds;
        if (tiles <= sms) {  // one round, shortened by a sub-wave split into S parts
            const int64_t S = std::max<int64_t>(1, std::min<int64_t>({8, sms / tiles, est_stages / MIN_PART_STAGES}));
            rounds = 1.0 / static_cast<double>(S);
        } else {  // full waves + the last partial wave (half a round when it is split in two)
            const bool half = 2 * tail <= sms && est_stages / 2 >= MIN_PART_STAGES;
            rounds = static_cast<double>(tiles / sms) + (tail == 0 ? 0.0 : half ? 0.5 : 1.0);
        }
        const double cost = rounds * (nt + 64);
        if (best_cost < 0 || cost < best_cost - 1e-9) best_cost = cost, best = nt;
    }
    return best;
}

// Column halves per CTA (NM_SP_H=1/2 overrides, ablation).  H = 2 halves the gathered bytes per
// MAC but packs 8 groups per slot sequence instead of 4, whose union needs more slots as the
// sparsity grows: measured on B200 (the A-F study, profiles/r02e_protocol_summary.txt, and the
// BASELINE shapes, profiles/r02g_sp_tmem_weights_ab.txt tw=0 rows) H = 2 wins at 50 % (cfg2 104.5 vs
// 115.2 us, 8192^3 583 vs 755) and 62.5 % (cfg3 109 vs 124), ties at 75 % on cfg3 (103 vs 105) and
// loses there on 4096^3 / 2048x4096x4096 (95 vs 86, 64 vs 46 us), loses at 87.5 % -- so H = 2 iff
// L >= 32 and 3N >= M.
static int sp_halves(int L, int N, int M) {
    const char* e = std::getenv("NM_SP_H");
    if (e && e[0] == '1') return 1;
    if (e && e[0] == '2' && L >= 32) return 2;
    return (L >= 32 && 3 * N >= M) ? 2 : 1;
}

// With the token count known (a per-call prepack: nm_spmm, nm_spmm_host) small grids take H = 1
// below 100 % density: H = 2 then leaves the grid under two waves, and the 2x tiles of H = 1 buy
// more parallelism than its larger unions cost (A-F study: 2048x4096x4096 62.5 % 53 vs 64 us,
// 1024x2048x2048 50 % 20 vs 23 us; profiles/r02e_protocol_summary.txt).
// Stages per tile the selector expects (host, no data): the tile's kept-row union
// k (1 - (1 - N/M)^G) over its G = 128 H / L groups, at least 2 w (two rows per quad / one per
// pair), + 10 % packing slack.
static int sp_est_stages(int64_t k, int N, int M, int L, int H, bool tf) {
    const int G = 128 * H / L;
    const double keep = static_cast<double>(N) / M;
    const double uni = 1.0 - std::pow(1.0 - keep, G);
    const double slots = 1.1 * static_cast<double>(k) * std::max(uni, std::min(1.0, 2.0 * keep));
    return static_cast<int>(slots / (tf ? El<true>::SLOTS : El<false>::SLOTS)) + 1;
}

static int sp_halves_m(int L, int N, int M, int64_t m, int64_t n, int64_t k) {
    const int H = sp_halves(L, N, M);
    // (N = M included: the A-F study at 0 % also prefers H = 1 on grids under two waves, A-E 9-23 %
    // faster, profiles/r02w_protocol_summary.txt)
    if (H != 2 || std::getenv("NM_SP_H")) return H;
    const int nt = sp_tokens(2, m, n, sp_est_stages(k, N, M, L, 2, false));
    const int64_t tiles = ((n + 255) / 256) * ((m + nt - 1) / nt);
    return tiles >= 2 * static_cast<int64_t>(num_sms()) ? 2 : 1;
}


// NM_SP_DBG & 64: CTA (0,0) records clock64 per stage into C (timing study only)
#define SP_TS(st, slot)                                                                                \
    do {                                                                                               \
        if ((p.dbg & 64) && blockIdx.x == 0 && blockIdx.y == 0 && lane == 0)                           \
            static_cast<long long*>(p.C)[(st) * 8 + (slot)] = clock64();                               \
    } while (0)

// TF: fp32 operands on kind::tf32 (El<true>), else bf16 on kind::f16.  PEER: the fused exchange's
// direct-store epilogue into every rank's C (a separate instantiation: the peer loop in the
// common kernel cost 30 % on the tf32 NT = 208 variant through register allocation).
template <int H, int NT_, bool TF, bool PEER = false>
__global__ void __launch_bounds__(THREADS, 1)
    spmm_tc_sp_kernel(const void* __restrict__ At, const __grid_constant__ CUtensorMap tmC,
                      const __grid_constant__ CUtensorMap tmC16, const Params p) {
    using CF = Cfg<H, NT_, TF>;
    using EL = El<TF>;
    constexpr int NT = CF::NT, MC = CF::MC, B_BYTES = CF::B_BYTES, W_BYTES = CF::W_BYTES, STAGES = CF::ST;
    constexpr int SLOTS = EL::SLOTS;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* sB = smem;                               // STAGES x B_BYTES (1024-aligned: 128-B swizzle atoms)
    uint8_t* sW = smem + STAGES * B_BYTES;            // STAGES x H x (A image 64-B swizzle, metadata)
    uint64_t* full = reinterpret_cast<uint64_t*>(sW + STAGES * W_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* acc_full = empty + STAGES;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_full + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned long long t_start = 0;
    long long c_start = 0, c_acc = 0;
    if ((p.dbg & 256) && threadIdx.x == 0) {
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
        c_start = clock64();
    }
    // 1-D grid, token tiles fastest (the CTAs that share a column tile's weight stream run
    // together, so it is read from DRAM once and served from L2 to the others).  The last,
    // partial wave's tiles are split in two stage ranges ("tail split"): part 1 leaves an fp32
    // partial in ws, part 0 adds it in its epilogue (a + b: order-independent, deterministic).
    int tid_lin = blockIdx.x, part = 0, nparts = 1;
    if (tid_lin >= p.full_ctas) {
        nparts = p.split;
        part = (tid_lin - p.full_ctas) % nparts;
        tid_lin = p.full_ctas + (tid_lin - p.full_ctas) / nparts;
    }
    const int tile = tid_lin / p.n_tok;
    const int m0 = (tid_lin % p.n_tok) * NT;
    const int4 ti = p.tinfo[tile];
    const int nst_all = ti.x;
    // pair-aligned stage ranges (a stage pair's metadata stays in one part)
    const int npairs = (nst_all + 1) >> 1;
    const int sa = min(nst_all, 2 * (part * npairs / nparts));
    const int sb = min(nst_all, 2 * ((part + 1) * npairs / nparts));
    const int nst = (p.dbg & 512) ? 0 : sb - sa;  // stages this CTA runs (ring index = st - sa); dbg 512: none
    const int tail_idx = tid_lin - p.full_ctas;

    if (warp == MMA_WARP) {
        if (lane == 0) {
            for (int s = 0; s < STAGES; ++s) {
                mbar_init(&full[s], 1 + 2 * 32);  // two owner warps' copies + the weight copy
                mbar_init(&empty[s], 1);
            }
            mbar_init(acc_full, 1);
            fence_mbar_init();
        }
        __syncwarp();
        tmem_alloc(tmem_slot, TMEM_COLS);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp < GATHER_WARPS) {
        // ============ gather: stage-owning warp pairs ============
        // Warps (g, g + 4) own the stages st == g (mod 4) of this CTA's range and copy half of the
        // stage's slot rows each (bf16: 32 rows of NT tokens, one warp-wide 16-B cp.async per row;
        // tf32: 16 rows x 2 token halves).  A warp thus walks every 4th stage with 32 independent
        // copies per visit, instead of every stage with 8 -- measured on B200 (scripts/ubench_ring2,
        // profiles/r02_ring_layouts.txt) the per-stage ring time drops from ~690 to ~420 clk when
        // stage ownership replaces lock-step sharing.  4 owners <= STAGES, so a wait on empty[s]
        // is never two ring laps behind (no parity aliasing).  Completion: one
        // cp.async.mbarrier.arrive.noinc per thread (full count 2 x 32 + 1: the weight copy).
        static_assert(STAGES >= 4, "four stage owners need a ring of at least four stages");
        const int own = warp & 3, half = warp >> 2;
        constexpr int ROWS = SLOTS / 2;          // slot rows per warp and owned stage (32 / 16)
        constexpr int CPR = TF ? 2 : 1;          // 512-B copies per slot row (token halves for tf32)
        constexpr int NCOPY = ROWS * CPR;        // 32 copies per warp and owned stage
        static_assert(NCOPY == 32, "32 copies per warp and owned stage");
        const uint8_t* wsrc = p.base + static_cast<int64_t>(ti.z) * 1024;
        // this lane's slot row (lane < ROWS) of each owned stage: slot list + stage * SLOTS + half * ROWS + lane
        const int* ssrc = reinterpret_cast<const int*>(p.base + p.slots_off) + ti.y + half * ROWS + (lane % ROWS);
        // per-lane source (A^T + E (m0 + token)) and destination constants; the destination of copy i
        // is dbase[i % 8] + (i / 8) * 8 rows (bf16) or dbase[i % 8] + (i / 8) * 4 rows (tf32)
        const char* src_c[CPR];
        uint32_t srcsz_c[CPR];
        bool on_c[CPR];
#pragma unroll
        for (int h2 = 0; h2 < CPR; ++h2) {
            const int tl = TF ? 128 * h2 + 4 * lane : 8 * lane;  // first token of this lane's 16 B
            on_c[h2] = tl < NT;
            const bool ok = on_c[h2] && m0 + tl < p.mp;
            srcsz_c[h2] = ok ? 16u : 0u;
            src_c[h2] = static_cast<const char*>(At) + EL::E * static_cast<int64_t>(ok ? m0 + tl : 0);
        }
        const uint32_t pitch = static_cast<uint32_t>(p.mp) * EL::E;
        uint32_t dl[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (TF) {  // copy i: row half * 16 + i / 2, token half i % 2; swizzle phase row % 4 = (i / 2) % 4
                const uint32_t j = i / 2, h2 = i % 2;
                dl[i] = static_cast<uint32_t>((4 * h2 + (lane >> 3)) * (SLOTS * 128) + (half * ROWS + j) * 128) +
                        (((static_cast<uint32_t>(lane & 7) >> 1) ^ j) << 5) + ((static_cast<uint32_t>(lane) & 1u) << 4);
            } else {   // copy i: row half * 32 + i; swizzle phase row % 8 = i % 8
                dl[i] = static_cast<uint32_t>((lane >> 3) * (SLOTS * 128) + (half * ROWS + i) * 128) +
                        ((static_cast<uint32_t>(lane & 7) ^ static_cast<uint32_t>(i)) << 4);
            }
        }
        constexpr uint32_t DSTEP = TF ? 4 * 128 : 8 * 128;  // 8 copies further = 4 (tf32) / 8 (bf16) rows
        // slot rows of the next owned stages prefetched in a 4-deep register ring (loop unrolled by
        // 4): a register is consumed 4 owned stages (16 stages) after its load was issued
        constexpr int PF = 4;
        int kq[PF];
#pragma unroll
        for (int u = 0; u < PF; ++u) {
            const int st = own + 4 * u;
            kq[u] = st < nst ? ssrc[(sa + st) * SLOTS] : 0;
        }
        for (int v0 = 0; own + 4 * v0 < nst; v0 += PF) {
#pragma unroll
            for (int u = 0; u < PF; ++u) {
                const int st = own + 4 * (v0 + u);  // local stage (global stage sa + st)
                if (st >= nst) break;
                const int s = st % STAGES;
                // byte offset of this lane's row; padding slots (row k) are zero-filled by the copy
                // (source size 0), so a caller's A^T needs no zero row (nm_spmm_at)
                const uint32_t off = kq[u] < p.k ? static_cast<uint32_t>(kq[u]) * pitch : 0xFFFFFFFFu;
                {
                    const int stn = st + 4 * PF;
                    if (stn < nst) kq[u] = ssrc[(sa + stn) * SLOTS];
                }
                if (st >= STAGES) mbar_wait_dbg(&empty[s], ((st / STAGES) - 1) & 1, p.dbg, 2048, 8192);
                if (half == 0 && lane == 0) {
                    if (p.dbg & 16) {
                        mbar_arrive(&full[s]);
                    } else {
                        // even stages bring the pair's metadata blocks, odd ones only the A images
                        const uint32_t wb = ((sa + st) & 1) ? static_cast<uint32_t>(H * A_BYTES) : W_BYTES;
                        mbar_arrive_expect_tx(&full[s], wb);
                        const uint8_t* wst = wsrc + sp_stage_off(sa + st, H);
                        bulk_load(sW + s * W_BYTES, wst, wb, &full[s]);
                    }
                }
                if (!(p.dbg & 1)) {
                    const uint32_t bstage = smem_u32(sB + s * B_BYTES);
#pragma unroll
                    for (int i = 0; i < NCOPY; ++i) {
                        const uint32_t o = __shfl_sync(0xffffffffu, off, i / CPR);
                        const bool pad = o == 0xFFFFFFFFu;
                        cp_async16_pred(bstage + dl[i % 8] + (i / 8) * DSTEP, src_c[i % CPR] + (pad ? 0u : o),
                                        pad ? 0u : srcsz_c[i % CPR], on_c[i % CPR]);
                    }
                }
                // arrives on full[s] once this thread's copies have landed (counts as one of the
                // barrier's expected arrivals: 2 x 32 + 1)
                cp_async_arrive_noinc(&full[s]);
            }
        }
    } else if (warp == MMA_WARP) {
        // ============ MMA issuer: per stage and half, metadata -> TMEM and two sparse MMAs ============
        // The warp runs the loop converged (all values warp-uniform); one elect per stage issues the
        // metadata copies, MMAs and the commit.  Descriptors of ring slot 0 are built once and
        // advanced by immediate offsets (the 14-bit start-address field never carries: shared
        // memory < 256 KB); ring slot / phase / metadata pair are kept incrementally.
        {
            constexpr uint32_t idesc = (1u << 2) | (1u << 4) | (EL::FMT << 7) | (EL::FMT << 10) | (1u << 16) |
                                       (static_cast<uint32_t>(NT >> 3) << 17) | (static_cast<uint32_t>(128 >> 4) << 24);
            const uint64_t bdesc0 = smem_desc(smem_u32(sB), SLOTS * 128, EL::B_SBO, EL::B_LAYOUT);
            const uint64_t adesc0 = smem_desc(smem_u32(sW), 16, 512, 4);
            const uint64_t edesc0 = smem_desc(smem_u32(sW) + H * A_BYTES, 2048, 128, 0);
            const bool skip_mma = (p.dbg & 2) != 0;
            int s = 0, pi = (sa >> 1) % CF::NPAIR;
            uint32_t ph = 0;
            for (int st = 0; st < nst; ++st) {
                const int gs = sa + st;  // stage index in the tile (pairs: 2i, 2i+1)
                mbar_wait_dbg(&full[s], ph, p.dbg, 1024, 4096);
                tc_fence_after();
                if (elect_one()) {
                    if (!skip_mma) {
                        const uint64_t bo = static_cast<uint64_t>(s * (B_BYTES >> 4));
                        const uint64_t wo = static_cast<uint64_t>(s * (W_BYTES >> 4));
                        const uint32_t pcol = tmem + CF::META_COL + 4 * H * pi;
#pragma unroll
                        for (int h = 0; h < H; ++h) {
                            if (!(gs & 1))  // the pair's metadata arrives with its even stage (sa is even)
                                tmem_cp_128x128b(pcol + 4 * h, edesc0 + wo + (h * E_BYTES >> 4));
#pragma unroll
                            for (int j = 0; j < 2; ++j)
                                mma_sp<TF>(tmem + h * NT, adesc0 + wo + ((h * A_BYTES + 32 * j) >> 4),
                                           bdesc0 + bo + ((EL::B_STEP * j) >> 4), idesc | static_cast<uint32_t>(j),
                                           (st | j) ? 1u : 0u, pcol + 4 * h + 2 * (gs & 1));
                        }
                    }
                    if (p.dbg & 128) mbar_arrive(&empty[s]);       // timing study: plain arrive instead of commit
                    else tc_commit(&empty[s]);
                }
                if (gs & 1) pi = pi + 1 == CF::NPAIR ? 0 : pi + 1;
                if (++s == STAGES) s = 0, ph ^= 1u;
            }
            if (elect_one()) tc_commit(acc_full);
            __syncwarp();
        }
    }

    if (warp < GATHER_WARPS) {
        // ============ epilogue: TMEM lane = output column, TMEM column = token ============
        const bool odd = lane & 1;
        if (warp == 0) SP_TS(nst, 6);
        mbar_wait(acc_full, 0);
        tc_fence_after();
        if (warp == 0) SP_TS(nst, 7);
        if ((p.dbg & 256) && threadIdx.x == 0) c_acc = clock64();
        const int qw = warp & 3;
        // split tiles (nparts > 1): the first nparts - 1 CTAs of a tile to finish publish their fp32
        // partials in ws; the last one (by ticket) waits for them -- they hold tickets, so they are
        // running: no co-residency assumption -- and adds all parts in the fixed order 0 .. nparts-1
        // (bit-reproducible whichever CTA is last), then stores C
        bool publish = false;
        if (nparts > 1) {
            volatile uint32_t* s_flag = tmem_slot + 1;
            if (warp == 0 && lane == 0) *s_flag = atomicAdd(p.counters + 2 * tail_idx, 1) < nparts - 1 ? 1u : 0u;
            named_bar_sync(1, 32 * GATHER_WARPS);
            publish = *s_flag != 0;
        }
        if (publish) {
            // ws[tile][part] is [NT][MC] (token-major): for each token the warp's 32 lanes write 128
            // contiguous bytes
            float* w = p.ws + (static_cast<int64_t>(tail_idx) * nparts + part) * MC * NT;
#pragma unroll 1
            for (int h = 0; h < H; ++h)
#pragma unroll 1
                for (int t0 = (warp >> 2) * 32; t0 < NT; t0 += 64) {
                    uint32_t v[32];
                    if (nst > 0) {
                        tmem_ld32(tmem + (static_cast<uint32_t>(qw * 32) << 16) + h * NT + t0, v);
                        tmem_wait_ld();
                    } else {
#pragma unroll
                        for (int i = 0; i < 32; ++i) v[i] = 0u;
                    }
                    const int nv = NT - t0 < 32 ? NT - t0 : 32;
                    float* dst = w + static_cast<int64_t>(t0) * MC + h * 128 + qw * 32 + lane;
#pragma unroll
                    for (int i = 0; i < 32; ++i)
                        if (i < nv) dst[static_cast<int64_t>(i) * MC] = __uint_as_float(v[i]);
                }
            __threadfence();
            named_bar_sync(1, 32 * GATHER_WARPS);
            if (warp == 0 && lane == 0) red_release_add(p.counters + 2 * tail_idx + 1, 1);
        } else if (p.tma_c) {
            if (nparts > 1) {
                if (warp == 0 && lane == 0) {  // one poller with back-off
                    unsigned long long t0g, tn;
                    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0g));
                    while (ld_acquire(p.counters + 2 * tail_idx + 1) < nparts - 1) {
                        __nanosleep(256);
                        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tn));
                        if (tn - t0g > 20000000000ull) __trap();  // 20 s: a lost partial is a bug, fail loudly
                    }
                }
                named_bar_sync(1, 32 * GATHER_WARPS);
                __threadfence();
            }
            const float* wpart = nparts > 1 ? p.ws + static_cast<int64_t>(tail_idx) * nparts * MC * NT : nullptr;
            // staged: each 32-token chunk of the [NT][MC] C tile is assembled in the (now idle)
            // stage ring, then one TMA tensor store writes it (clipped at m, n).  Warps 0-3 take
            // the even chunks, 4-7 the odd ones; lane = column, so a warp's 32 stores per token row
            // are 64 / 128 contiguous bytes.
            const int eb = p.c_bf16 ? 2 : 4;
            const int rowb = MC * eb;
            const uint32_t tbase = tmem + (static_cast<uint32_t>(qw * 32) << 16);
            // (chunk, half) items j = 0 .. J - 1 of this warp: t0 = (warp / 4 + 2 (j / H)) 32, h = j % H.
            // The TMEM load of item j + 1 is issued before item j is converted and staged, so its
            // latency overlaps the stores (tcgen05.wait::ld then waits for it); two register sets.
            const int J = H * (((NT + 31) / 32 - (warp >> 2) + 1) / 2);
            auto item_t0 = [&](int j) { return ((warp >> 2) + 2 * (j / H)) * 32; };
            auto stage = [&](uint32_t (&v)[32], int j) {
                const int t0 = item_t0(j), h = j % H;
                uint8_t* buf = smem + (t0 / 32) * 32 * rowb;
                if (wpart) {  // sum of the parts in the order 0 .. nparts-1 (this CTA's own from TMEM)
                    const int nv = NT - t0 < 32 ? NT - t0 : 32;
                    float a[32];
#pragma unroll
                    for (int i = 0; i < 32; ++i) a[i] = 0.f;
#pragma unroll 1
                    for (int q2 = 0; q2 < nparts; ++q2) {
                        if (q2 == part) {
#pragma unroll
                            for (int i = 0; i < 32; ++i) a[i] += __uint_as_float(v[i]);
                        } else {
                            const float* src = wpart + static_cast<int64_t>(q2) * MC * NT + static_cast<int64_t>(t0) * MC +
                                               h * 128 + qw * 32 + lane;
#pragma unroll
                            for (int i = 0; i < 32; ++i)
                                if (i < nv) a[i] += __ldcg(src + static_cast<int64_t>(i) * MC);
                        }
                    }
#pragma unroll
                    for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(a[i]);
                }
#pragma unroll
                for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * p.alpha);
                uint8_t* cb = buf + (h * 128 + qw * 32 + lane) * eb;
                // NT % 32 == 16 (176, 208 tokens): the last chunk holds 16 tokens of this tile
                const int rows = NT - t0 < 32 ? NT - t0 : 32;
                if (p.c_bf16) {
#pragma unroll
                    for (int i = 0; i < 32; ++i)
                        if (i < rows)
                            *reinterpret_cast<__nv_bfloat16*>(cb + i * rowb) = __float2bfloat16_rn(__uint_as_float(v[i]));
                } else {
#pragma unroll
                    for (int i = 0; i < 32; ++i)
                        if (i < rows) *reinterpret_cast<uint32_t*>(cb + i * rowb) = v[i];
                }
                if (h == H - 1) {  // the chunk is complete in shared memory: one TMA store
                    fence_proxy_async_smem();
                    named_bar_sync(1 + (warp >> 2), 128);
                    if (qw == 0 && lane == 0 && !(p.dbg & (8 | 64 | 256))) {
                        tma_store_2d(NT - t0 < 32 ? &tmC16 : &tmC, buf, tile * MC, m0 + t0);
                        bulk_commit();
                    }
                }
            };
            auto load = [&](uint32_t (&v)[32], int j) {
                if (nst > 0) {
                    tmem_ld32(tbase + (j % H) * NT + item_t0(j), v);
                } else {
#pragma unroll
                    for (int i = 0; i < 32; ++i) v[i] = 0u;
                }
            };
            uint32_t va[32], vb[32];
            if (J > 0) {
                load(va, 0);
                tmem_wait_ld();
            }
#pragma unroll 1
            for (int j = 0; j < J; j += 2) {
                if (j + 1 < J) load(vb, j + 1);
                stage(va, j);
                tmem_wait_ld();
                if (j + 1 >= J) break;
                if (j + 2 < J) load(va, j + 2);
                stage(vb, j + 1);
                tmem_wait_ld();
            }
            if (qw == 0 && lane == 0) bulk_wait_read0();
        } else {
#pragma unroll 1
        for (int h = 0; h < H; ++h) {
            const int col = tile * MC + h * 128 + qw * 32 + lane;        // this lane's output column
            const int pc = tile * MC + h * 128 + qw * 32 + (lane & ~1);  // column pair base
#pragma unroll 1
            for (int t0 = (warp >> 2) * 32; t0 < NT; t0 += 32 * (GATHER_WARPS / 4)) {
                uint32_t v[32];
                if (nst > 0) {
                    tmem_ld32(tmem + (static_cast<uint32_t>(qw * 32) << 16) + h * NT + t0, v);
                    tmem_wait_ld();
                } else {
#pragma unroll
                    for (int i = 0; i < 32; ++i) v[i] = 0u;
                }
#pragma unroll
                for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * p.alpha);
                // destinations: C itself, or (PEER, fused exchange) every rank's C at col_off + col
                const int npeer = PEER ? p.npeer : 1;
                const int64_t ldc = PEER ? p.ldc : p.n, coff = PEER ? p.col_off : 0;
                const int ncol = PEER ? p.n_valid : p.n;
                if (p.c_bf16) {
                    // lanes (2p, 2p+1) swap so each stores a bf16 pair (columns pc, pc+1): even lane token i, odd i+1
#pragma unroll
                    for (int i = 0; i < 32; i += 2) {
                        const uint32_t x = odd ? v[i] : v[i + 1];
                        const uint32_t y = __shfl_xor_sync(0xffffffffu, x, 1);
                        const float lo = __uint_as_float(odd ? y : v[i]);
                        const float hi = __uint_as_float(odd ? v[i + 1] : y);
                        const int tl = t0 + i + (odd ? 1 : 0), t = m0 + tl;  // tl < NT: stay inside the tile
                        if (tl < NT && t < p.m && pc < ncol && !(p.dbg & (8 | 64))) {
                            __nv_bfloat162 hh = __floats2bfloat162_rn(lo, hi);
                            for (int pi = 0; pi < npeer; ++pi)
                                *reinterpret_cast<__nv_bfloat162*>(static_cast<__nv_bfloat16*>(PEER ? p.cpeer[pi] : p.C) +
                                                                   static_cast<int64_t>(t) * ldc + coff + pc) = hh;
                        }
                    }
                } else {
#pragma unroll
                    for (int i = 0; i < 32; ++i) {
                        const int t = m0 + t0 + i;
                        if (t0 + i < NT && t < p.m && col < ncol && !(p.dbg & (8 | 64)))
                            for (int pi = 0; pi < npeer; ++pi)
                                static_cast<float*>(PEER ? p.cpeer[pi] : p.C)[static_cast<int64_t>(t) * ldc + coff + col] =
                                    __uint_as_float(v[i]);
                    }
                }
            }
        }
        }
        if (PEER) __threadfence_system();  // peer stores visible before the kernel completes
        tc_fence_before();
        if (warp == 0) SP_TS(nst, 0);
    }
    __syncthreads();
    if (warp == MMA_WARP) {
        tc_fence_after();
        tmem_dealloc(tmem, TMEM_COLS);
    }
    if ((p.dbg & 256) && threadIdx.x == 0) {  // timeline study: [start ns, end ns, smid, stages, clk: start, accumulators done, end]
        unsigned long long t_end;
        uint32_t smid;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        long long* o = static_cast<long long*>(p.C) + 8 * static_cast<int64_t>(blockIdx.x);
        o[0] = static_cast<long long>(t_start);
        o[1] = static_cast<long long>(t_end);
        o[2] = smid;
        o[3] = nst;
        o[4] = c_start;
        o[5] = c_acc;
        o[6] = clock64();
        o[7] = 0;
    }
}

// A (m x k bf16, row-major) -> At (k x mp, mp = m rounded up to 8): 64 x 64 tiles through shared memory.
__global__ void __launch_bounds__(256) transpose_bf16_kernel(const __nv_bfloat16* __restrict__ A,
                                                            __nv_bfloat16* __restrict__ At, int m, int k, int mp) {
    // 64 tokens x 64 k per block.  Token pairs (2p, 2p+1) travel as one 32-bit word: a thread
    // loads 8 k of rows 2p and 2p+1 (two 16-B loads; a warp covers 4 pairs x 128 B: coalesced),
    // PRMT builds the 8 (row 2p, row 2p+1) words, 8 smem stores (columns XOR-swizzled by 4 (k/8)
    // words: conflict-free); the output side reads 16 B (8 tokens) of a k row per LDS.128 and
    // writes it with one 16-B store.
    __shared__ __align__(16) uint32_t t2[64][36];  // [k][token pair], rows padded to 144 B
    const int k0 = blockIdx.x * 64, r0 = blockIdx.y * 64;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (blockIdx.x == 0 && blockIdx.y == 0)  // row k: the zero row the padding slots read
        for (int c = tid * 8; c < mp; c += 256 * 8)
            *reinterpret_cast<uint4*>(At + static_cast<int64_t>(k) * mp + c) = make_uint4(0, 0, 0, 0);
    {
        const int c = lane & 7, p = 4 * warp + (lane >> 3);  // 8-k chunk, token pair
        const int r = r0 + 2 * p, kc = k0 + 8 * c;
        uint4 x = make_uint4(0, 0, 0, 0), y = make_uint4(0, 0, 0, 0);
        if (kc < k) {
            if (r < m) x = *reinterpret_cast<const uint4*>(A + static_cast<int64_t>(r) * k + kc);
            if (r + 1 < m) y = *reinterpret_cast<const uint4*>(A + static_cast<int64_t>(r + 1) * k + kc);
        }
        const uint32_t xs[4] = {x.x, x.y, x.z, x.w}, ys[4] = {y.x, y.y, y.z, y.w};
        const int col = p ^ (4 * c);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            uint32_t lo, hi;
            asm("prmt.b32 %0, %1, %2, 0x5410;" : "=r"(lo) : "r"(xs[i]), "r"(ys[i]));
            asm("prmt.b32 %0, %1, %2, 0x7632;" : "=r"(hi) : "r"(xs[i]), "r"(ys[i]));
            t2[8 * c + 2 * i][col] = lo;
            t2[8 * c + 2 * i + 1][col] = hi;
        }
    }
    __syncthreads();
#pragma unroll
    for (int it = 0; it < 2; ++it) {
        const int e = tid + it * 256;
        const int kr = e >> 3, q = e & 7;  // k row, 8-token chunk
        if (k0 + kr < k && r0 + 8 * q < mp)
            *reinterpret_cast<uint4*>(At + static_cast<int64_t>(k0 + kr) * mp + r0 + 8 * q) =
                *reinterpret_cast<const uint4*>(&t2[kr][(4 * q) ^ (4 * ((kr >> 3) & 7))]);
    }
}

// ------------------------------------------------------------------------- offline prepack
// Slot packing (the paper's offline PreProcessing slot, Listing 3), one thread per
// (column tile, k chunk of KC rows, KC a multiple of M): item = k row of the chunk kept by at
// least one of the tile's G groups, type = G-bit membership mask.  Packing unit = PG slots with
// at most PG / 2 rows of any one group: quads (PG = 4, bf16 2:4) or pairs (PG = 2, tf32 1:2).
// First complementary pairs (t, ~t) (two per quad, one per pair: every group at exactly PG / 2);
// then greedy: fill each unit with the heaviest type that still fits, ties to the type with the
// most items left.  Every unit takes >= PG / 2 items, so a chunk needs at most 2 |U_c| + 4 slots.
// Chunks pack independently (each ends with at most one partial quad) so the prepack runs on
// tiles x chunks threads; sp_compact_kernel concatenates them.
__host__ __device__ inline int sp_chunk_rows(int M) { return (1024 + M - 1) / M * M; }

__global__ void sp_pack_kernel(const uint8_t* __restrict__ D, int* __restrict__ tmp_slots,
                               uint8_t* __restrict__ tmp_type, int* __restrict__ chunk_cnt, int* __restrict__ qbuf,
                               int n, int k, int N, int M, int L, int H, int nchunks, int PG) {
    const int gid = blockIdx.x * blockDim.x + threadIdx.x;
    const int MC = 128 * H;
    const int ntiles = (n + MC - 1) / MC;
    if (gid >= ntiles * nchunks) return;
    const int tile = gid / nchunks, c = gid % nchunks;
    const int KC = sp_chunk_rows(M);
    const int r0 = c * KC, r1 = min(k, r0 + KC), rows = r1 - r0;
    const int q = n / L, G = MC / L, g0 = tile * G;
    const int gcount = min(G, q - g0);
    const int T = 1 << G;
    int* qk = qbuf + static_cast<int64_t>(gid) * KC;                         // chunk rows, bucketed by type
    int* sl = tmp_slots + static_cast<int64_t>(gid) * (2 * KC + 4);           // this chunk's slots
    uint8_t* ty = tmp_type + static_cast<int64_t>(gid) * (2 * KC + 4);
    // membership masks of the chunk's rows (kept in sl[] while bucketing)
    for (int i = 0; i < rows; ++i) sl[i] = 0;
    for (int gi = 0; gi < gcount; ++gi)
        for (int t = r0 / M; t < r1 / M; ++t)
            for (int s = 0; s < N; ++s) sl[t * M + D[static_cast<int64_t>(t * N + s) * q + g0 + gi] - r0] |= 1 << gi;
    int start[257], head[256];
    for (int t = 0; t <= T; ++t) start[t] = 0;
    for (int i = 0; i < rows; ++i) start[sl[i] + 1]++;
    for (int t = 0; t < T; ++t) start[t + 1] += start[t];
    for (int t = 0; t < T; ++t) head[t] = start[t];
    for (int i = 0; i < rows; ++i) qk[head[sl[i]]++] = r0 + i;
    for (int t = 0; t < T; ++t) head[t] = start[t];
    int remaining = rows - (start[1] - start[0]);
    int ns = 0;
    // 1) complementary pairs (t, ~t): each pair puts every group at exactly one row, so two pairs
    //    make a perfect quad (every group at two) -- measured in simulation 3-9 % fewer slots than
    //    the greedy alone at 50-75 % sparsity
    const int full = (1 << gcount) - 1;
    int pend_a = -1, pend_b = -1, pend_ta = 0, pend_tb = 0;
    for (int t = 1; t < T; ++t) {
        const int u = full ^ t;
        if (u == 0 || t >= u || (t & ~full)) continue;
        int np = min(start[t + 1] - head[t], start[u + 1] - head[u]);
        for (; np > 0; --np) {
            const int ra = qk[head[t]++], rb = qk[head[u]++];
            remaining -= 2;
            if (PG == 2) {  // a perfect pair on its own
                sl[ns] = ra, ty[ns] = static_cast<uint8_t>(t), ++ns;
                sl[ns] = rb, ty[ns] = static_cast<uint8_t>(u), ++ns;
            } else if (pend_a < 0) {
                pend_a = ra, pend_b = rb, pend_ta = t, pend_tb = u;
            } else {
                sl[ns] = pend_a, ty[ns] = static_cast<uint8_t>(pend_ta), ++ns;
                sl[ns] = pend_b, ty[ns] = static_cast<uint8_t>(pend_tb), ++ns;
                sl[ns] = ra, ty[ns] = static_cast<uint8_t>(t), ++ns;
                sl[ns] = rb, ty[ns] = static_cast<uint8_t>(u), ++ns;
                pend_a = -1;
            }
        }
    }
    if (pend_a >= 0) {  // an odd pair: one quad with two padding slots
        sl[ns] = pend_a, ty[ns] = static_cast<uint8_t>(pend_ta), ++ns;
        sl[ns] = pend_b, ty[ns] = static_cast<uint8_t>(pend_tb), ++ns;
        sl[ns] = k, ty[ns] = 0, ++ns;
        sl[ns] = k, ty[ns] = 0, ++ns;
    }
    // 2) greedy on the rest
    while (remaining > 0) {
        uint32_t once = 0, twice = 0;
        int placed = 0;
        for (int sidx = 0; sidx < PG; ++sidx) {
            int best = -1, bkey = -1;
            const uint32_t full_groups = PG == 4 ? twice : once;  // groups already at PG / 2 rows
            for (int t = 1; t < T; ++t) {
                const int left = start[t + 1] - head[t];
                if (left == 0 || (static_cast<uint32_t>(t) & full_groups)) continue;
                const int key = (__popc(t) << 20) + left;
                if (key > bkey) bkey = key, best = t;
            }
            if (best < 0) break;
            sl[ns] = qk[head[best]++];
            ty[ns] = static_cast<uint8_t>(best);
            ++ns;
            twice |= once & static_cast<uint32_t>(best);
            once |= static_cast<uint32_t>(best);
            --remaining;
            ++placed;
        }
        for (; placed < PG; ++placed) {
            sl[ns] = k;  // padding slot: the zero row k of A^T
            ty[ns] = 0;
            ++ns;
        }
    }
    chunk_cnt[gid] = ns;
}

// The same packing, one warp per (column tile, chunk), producing exactly the slot lists of
// sp_pack_kernel (same bucket order, same pairs, same greedy choices and tie-breaks), ~40x
// faster: the chunk's rows live in shared memory, rows are bucketed by a stable warp-wide
// scatter (__match_any_sync ranks, rows in ascending order), the complementary pairs are
// emitted lane-parallel, and each greedy pick is a warp max-reduction over the 2^G types
// (key = popcount << 11 | items left, ties to the smaller type).  sp_pack_kernel stays as the
// sequential reference (NM_SP_PACK_SEQ=1; the GPU tests compare the two byte for byte).
constexpr int PACK_KC_MAX = 1280;  // >= sp_chunk_rows(M) for M <= 256
__global__ void __launch_bounds__(32) sp_pack_warp_kernel(const uint8_t* __restrict__ D, int* __restrict__ tmp_slots,
                                                          uint8_t* __restrict__ tmp_type, int* __restrict__ chunk_cnt,
                                                          int n, int k, int N, int M, int L, int H, int nchunks, int PG) {
    __shared__ int s_type[PACK_KC_MAX], s_qk[PACK_KC_MAX], s_start[257], s_head[256], s_off[257];
    const int gid = blockIdx.x, lane = threadIdx.x;
    const int MC = 128 * H;
    const int tile = gid / nchunks, c = gid % nchunks;
    const int KC = sp_chunk_rows(M);
    const int r0 = c * KC, r1 = min(k, r0 + KC), rows = r1 - r0;
    const int q = n / L, G = MC / L, g0 = tile * G;
    const int gcount = min(G, q - g0);
    const int T = 1 << G;
    const int full = (1 << gcount) - 1;
    int* sl = tmp_slots + static_cast<int64_t>(gid) * (2 * KC + 4);
    uint8_t* ty = tmp_type + static_cast<int64_t>(gid) * (2 * KC + 4);
    const unsigned all = 0xffffffffu;
    // 1) membership masks (OR is order-independent)
    for (int i = lane; i < rows; i += 32) s_type[i] = 0;
    for (int t = lane; t <= T; t += 32) s_start[t] = 0;
    __syncwarp();
    const int nwin = rows / M, per_g = nwin * N;
    for (int e = lane; e < gcount * per_g; e += 32) {
        const int gi = e / per_g, rem = e - gi * per_g, tw = rem / N, sidx = rem - tw * N;
        const int t = r0 / M + tw;
        atomicOr(&s_type[t * M + D[static_cast<int64_t>(t * N + sidx) * q + g0 + gi] - r0], 1 << gi);
    }
    __syncwarp();
    // 2) bucket sizes and starts
    for (int i = lane; i < rows; i += 32) atomicAdd(&s_start[s_type[i] + 1], 1);
    __syncwarp();
    if (lane == 0)
        for (int t = 0; t < T; ++t) s_start[t + 1] += s_start[t];
    __syncwarp();
    for (int t = lane; t < T; t += 32) s_head[t] = s_start[t];
    __syncwarp();
    // 3) stable scatter: rows in ascending order within each bucket
    const unsigned lt = (1u << lane) - 1u;
    for (int b0 = 0; b0 < rows; b0 += 32) {
        const int i = b0 + lane;
        const int tt = i < rows ? s_type[i] : -1;
        const unsigned peers = __match_any_sync(all, tt);
        if (tt >= 0) {
            s_qk[s_head[tt] + __popc(peers & lt)] = r0 + i;
        }
        __syncwarp();
        if (tt >= 0 && (peers & lt) == 0) s_head[tt] += __popc(peers);
        __syncwarp();
    }
    for (int t = lane; t < T; t += 32) s_head[t] = s_start[t];
    __syncwarp();
    // 4) complementary pairs (t, ~t), t ascending: offsets by a (short, sequential) scan
    for (int t = lane; t < T; t += 32) {
        const int u = full ^ t;
        int np = 0;
        if (t >= 1 && u != 0 && t < u && !(t & ~full))
            np = min(s_start[t + 1] - s_start[t], s_start[u + 1] - s_start[u]);
        s_off[t] = np;
    }
    __syncwarp();
    if (lane == 0) {
        int acc = 0;
        for (int t = 0; t < T; ++t) {
            const int np = s_off[t];
            s_off[t] = acc;
            acc += np;
        }
        s_off[T] = acc;
    }
    __syncwarp();
    const int npairs = s_off[T];
    for (int t = 1; t < T; ++t) {
        const int np = s_off[t + 1] - s_off[t];  // t's pairs (u = full ^ t), 0 unless t < u
        if (np == 0) continue;
        const int u = full ^ t;
        for (int j = lane; j < np; j += 32) {
            const int o = 2 * (s_off[t] + j);
            sl[o] = s_qk[s_start[t] + j], ty[o] = static_cast<uint8_t>(t);
            sl[o + 1] = s_qk[s_start[u] + j], ty[o + 1] = static_cast<uint8_t>(u);
        }
        __syncwarp();
        if (lane == 0) s_head[t] += np, s_head[u] += np;
        __syncwarp();
    }
    int ns = 2 * npairs;
    if (PG == 4 && (npairs & 1)) {  // an odd pair: its quad gets two padding slots
        if (lane == 0) sl[ns] = k, ty[ns] = 0, sl[ns + 1] = k, ty[ns + 1] = 0;
        ns += 2;
    }
    int remaining = rows - (s_start[1] - s_start[0]) - 2 * npairs;
    // 5) greedy, one warp max-reduction per pick; lane owns types lane + 32 j
    int left[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const int t = lane + 32 * j;
        left[j] = (t >= 1 && t < T) ? s_start[t + 1] - s_head[t] : 0;
    }
    while (remaining > 0) {
        uint32_t once = 0, twice = 0;
        int placed = 0;
        for (int sidx = 0; sidx < PG; ++sidx) {
            const uint32_t blocked = PG == 4 ? twice : once;
            uint32_t mine = 0;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const uint32_t t = static_cast<uint32_t>(lane + 32 * j);
                if (left[j] > 0 && !(t & blocked)) {
                    const uint32_t key = ((static_cast<uint32_t>(__popc(t)) << 11 | static_cast<uint32_t>(left[j])) << 8) |
                                         (255u - t);
                    mine = key > mine ? key : mine;
                }
            }
            const uint32_t best_key = __reduce_max_sync(all, mine);
            if (best_key == 0) break;
            const int best = 255 - static_cast<int>(best_key & 255u);
            if ((best & 31) == lane) left[best >> 5]--;
            if (lane == 0) {
                sl[ns] = s_qk[s_head[best]++];
                ty[ns] = static_cast<uint8_t>(best);
            }
            ++ns;
            twice |= once & static_cast<uint32_t>(best);
            once |= static_cast<uint32_t>(best);
            --remaining;
            ++placed;
        }
        if (lane == 0)
            for (int pi = placed; pi < PG; ++pi) sl[ns + pi - placed] = k, ty[ns + pi - placed] = 0;
        ns += PG - placed;
    }
    if (lane == 0) chunk_cnt[gid] = ns;
}

// Concatenate a tile's chunk slot lists (one block per tile), pad to whole stages of SLOTS slots.
__global__ void sp_compact_kernel(const int* __restrict__ tmp_slots, const uint8_t* __restrict__ tmp_type,
                                  const int* __restrict__ chunk_cnt, int* __restrict__ slots, uint8_t* __restrict__ stype,
                                  int* __restrict__ nstages, int k, int M, int nchunks, int smax, int SLOTS) {
    const int tile = blockIdx.x;
    const int KC = sp_chunk_rows(M);
    int* sl = slots + static_cast<int64_t>(tile) * smax;
    uint8_t* ty = stype + static_cast<int64_t>(tile) * smax;
    int off = 0;
    for (int c = 0; c < nchunks; ++c) {
        const int gid = tile * nchunks + c;
        const int cnt = chunk_cnt[gid];
        for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
            sl[off + i] = tmp_slots[static_cast<int64_t>(gid) * (2 * KC + 4) + i];
            ty[off + i] = tmp_type[static_cast<int64_t>(gid) * (2 * KC + 4) + i];
        }
        off += cnt;
    }
    const int padded = (off + SLOTS - 1) / SLOTS * SLOTS;
    for (int i = off + threadIdx.x; i < padded; i += blockDim.x) {
        sl[i] = k;
        ty[i] = 0;
    }
    if (threadIdx.x == 0) nstages[tile] = padded / SLOTS;
}

// Weight images: one thread per (tile, stage, output row r of the tile).  Per packing unit (16 per
// stage: quads for bf16, pairs for tf32): the slots whose row the thread's group keeps -> PG / 2
// compressed values (A image, 64-B swizzled K-major) + the metadata nibble at the TMEM position of
// (row r, chunk) for tcgen05.mma.sp (the same for kind::f16 and kind::tf32):
//   lane = r%8 + 8 (chunk/4 of the MMA) + 16 (r/16), bit = 16 ((r/8)%2) + 4 (chunk%4);
// nibble: bf16 slot index of value 0 | slot index of value 1 << 2; tf32 0x4 (slot 0) / 0xE (slot 1).
// tf32 values are rounded to tf32 (RNA) here, offline; the MMA reads the top 19 bits.
__device__ __forceinline__ void sp_store_val(uint8_t* p, float v, bool tf) {
    if (tf) {
        uint32_t r;
        asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(v));
        *reinterpret_cast<uint32_t*>(p) = r;
    } else {
        *reinterpret_cast<__nv_bfloat16*>(p) = __float2bfloat16_rn(v);
    }
}

template <bool TF>
__global__ void sp_image_kernel(const void* __restrict__ Bv_, const uint8_t* __restrict__ D,
                                const int* __restrict__ slots, const uint8_t* __restrict__ stype,
                                const int* __restrict__ nstages, const int4* __restrict__ tinfo, uint8_t* __restrict__ base,
                                int n, int k, int N, int M, int L, int smax, int max_stages, int H) {
    const int64_t gid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int MC = 128 * H;
    const int r = static_cast<int>(gid % MC);
    const int64_t ts = gid / MC;
    const int st = static_cast<int>(ts % max_stages);
    const int tile = static_cast<int>(ts / max_stages);
    const int ntiles = (n + MC - 1) / MC;
    if (tile >= ntiles || st >= nstages[tile]) return;
    const int q = n / L;
    const int j = tile * MC + r;
    const int g = j / L, gi = r / L;
    const bool live = j < n;
    const int hf = r / 128;
    uint8_t* timg = base + static_cast<int64_t>(tinfo[tile].z) * 1024;  // the tile's compact image block
    uint8_t* img = timg + sp_stage_off(st, H) + hf * A_BYTES;
    // metadata of the pair (st & ~1, st | 1) lives in the even stage's E block of this half
    uint32_t* meta = reinterpret_cast<uint32_t*>(timg + sp_stage_off(st & ~1, H) + H * A_BYTES + hf * E_BYTES);
    constexpr int SLOTS = El<TF>::SLOTS, PG = El<TF>::PG, NV = PG / 2, E = El<TF>::E;
    const int* sl = slots + static_cast<int64_t>(tile) * smax + st * SLOTS;
    const uint8_t* ty = stype + static_cast<int64_t>(tile) * smax + st * SLOTS;
    for (int qd = 0; qd < SLOTS / PG; ++qd) {
        int pos[2] = {-1, -1};
        int npos = 0;
        for (int i = 0; i < PG; ++i)
            if (live && npos < NV && ((ty[PG * qd + i] >> gi) & 1)) pos[npos++] = i;
        // fill unused value positions with distinct unused slots (value 0)
        for (int i = 0; npos < NV && i < PG; ++i)
            if (i != pos[0]) pos[npos++] = i;
        if (NV == 2 && pos[0] > pos[1]) {
            const int t = pos[0];
            pos[0] = pos[1];
            pos[1] = t;
        }
        for (int e = 0; e < NV; ++e) {
            float v = 0.f;
            const int kk = sl[PG * qd + pos[e]];
            if (live && kk < k && ((ty[PG * qd + pos[e]] >> gi) & 1)) {
                const int t = kk / M, off = kk % M;
                int lo = 0, hi = N - 1;  // D ascending within the window (R7)
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (D[static_cast<int64_t>(t * N + mid) * q + g] < off) lo = mid + 1;
                    else hi = mid;
                }
                const int64_t vi = static_cast<int64_t>(t * N + lo) * n + j;
                v = TF ? static_cast<const float*>(Bv_)[vi] : __bfloat162float(static_cast<const __nv_bfloat16*>(Bv_)[vi]);
            }
            const int pidx = NV * qd + e;  // compressed element of the row (32 bf16 / 16 tf32)
            const int b = E * pidx;
            const int rr = r % 128;
            const int off = (rr / 8) * 512 + (rr % 8) * 64 + ((((b >> 4) ^ ((rr % 8) >> 1)) & 3) << 4) + (b & 15);
            sp_store_val(img + off, v, TF);
        }
        const int rr = r % 128;
        const int mma = qd / 8, c = qd % 8;
        const int ln = (rr % 8) + 8 * (c / 4) + 16 * (rr / 16);
        const int bit = 16 * ((rr / 8) % 2) + 4 * (c % 4);
        const uint32_t nib = TF ? (pos[0] ? 0xEu : 0x4u) : static_cast<uint32_t>(pos[0] | (pos[1] << 2));
        atomicOr(&meta[ln * 4 + 2 * (st & 1) + mma], nib << bit);
    }
}

// Compact layout of the prepacked weight (one thread): per tile its stage count, first slot,
// image block offset and size (1 KB units, images start 1 KB-aligned after the slot lists), and the
// exact buffer size in the header.  Tiles are few (n / 128H), so one thread suffices.
__global__ void sp_layout_kernel(const int* __restrict__ nstages, int4* __restrict__ tinfo, int64_t* __restrict__ header,
                                 int ntiles, int H, int SLOTS, int64_t slots_off) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    int64_t nslots = 0;
    for (int t = 0; t < ntiles; ++t) nslots += static_cast<int64_t>(nstages[t]) * SLOTS;
    int64_t img_kb = (slots_off + nslots * 4 + 1023) / 1024;
    int64_t sl = 0;
    for (int t = 0; t < ntiles; ++t) {
        const int nst = nstages[t];
        const int64_t kb = sp_stage_off(nst, H) / 1024;
        tinfo[t] = make_int4(nst, static_cast<int>(sl), static_cast<int>(img_kb), static_cast<int>(kb));
        sl += static_cast<int64_t>(nst) * SLOTS;
        img_kb += kb;
    }
    header[0] = img_kb * 1024;  // exact bytes of the prepacked buffer
    header[1] = ntiles;
    header[2] = H;
}

// A tile's slot list (scratch, smax per tile) -> its compact position (one block per tile).
__global__ void sp_slots_copy_kernel(const int* __restrict__ slots, const int4* __restrict__ tinfo, int* __restrict__ out,
                                     int smax, int SLOTS) {
    const int tile = blockIdx.x;
    const int4 ti = tinfo[tile];
    const int cnt = ti.x * SLOTS;
    for (int i = threadIdx.x; i < cnt; i += blockDim.x) out[ti.y + i] = slots[static_cast<int64_t>(tile) * smax + i];
}

}  // namespace tcs

bool tc_sp_applicable(int64_t m, int64_t n, int64_t k, int N, int M, int L) {
    (void)m;
    (void)N;
    return (L == 16 || L == 32 || L == 64 || L == 128) && n % 2 == 0 && k > 0 && k < (1 << 30) && M <= 256;
}

// Geometry of a prepacked weight (H column halves per tile, SLOTS slots per stage).
struct SpGeom {
    int H, SLOTS, PG, ntiles, KC, nchunks;
    int64_t smax, max_stages, slots_off;
};
static SpGeom sp_geom(int64_t n, int64_t k, int N, int M, int L, bool tf, int H) {
    using namespace tcs;
    SpGeom g{};
    g.H = H > 0 ? H : sp_halves(L, N, M);
    g.SLOTS = tf ? El<true>::SLOTS : El<false>::SLOTS;
    g.PG = tf ? El<true>::PG : El<false>::PG;
    g.ntiles = static_cast<int>((n + 128 * g.H - 1) / (128 * g.H));
    g.KC = sp_chunk_rows(M);
    g.nchunks = static_cast<int>((k + g.KC - 1) / g.KC);
    g.smax = ((2 * k + 4 * g.nchunks) + g.SLOTS - 1) / g.SLOTS * g.SLOTS;  // >= sum of chunk bounds
    g.max_stages = g.smax / g.SLOTS;
    g.slots_off = (256 + 16 * static_cast<int64_t>(g.ntiles) + 255) / 256 * 256;
    return g;
}
static size_t al256(size_t b) { return (b + 255) / 256 * 256; }

// Retained prepacked buffer: [header 256 B: exact bytes, ntiles, H | tinfo ntiles x int4 | slots |
// images (1 KB-aligned)].  The exact size depends on the slot counts (data); this is the bound.
size_t tc_sp_prepack_bytes(int64_t n, int64_t k, int N, int M, int L, bool tf) {
    const SpGeom g = sp_geom(n, k, N, M, L, tf, 0);
    return static_cast<size_t>(g.slots_off + (g.ntiles * g.smax * 4 + 1023) / 1024 * 1024 +
                               g.ntiles * tcs::sp_stage_off(static_cast<int>(g.max_stages), g.H));
}

// Pack scratch (library pool, released after the prepack): chunk buckets, chunk slot lists and
// types, chunk counts, per-tile slot lists / types / stage counts, tinfo, header.
static size_t sp_scratch_bytes(const SpGeom& g) {
    const int64_t units = static_cast<int64_t>(g.ntiles) * g.nchunks;
    return al256(units * g.KC * 4) + al256(units * (2 * g.KC + 4) * 5) + al256(units * 4) +
           al256(g.ntiles * g.smax * 4) + al256(g.ntiles * g.smax) + al256(g.ntiles * 4) + al256(g.ntiles * 16) + 256;
}

// Zero the metadata blocks (the image kernel ORs nibbles into them): one block per (tile, pair).
__global__ void sp_meta_zero_kernel(const int4* __restrict__ tinfo, uint8_t* __restrict__ base, int H, int max_pairs) {
    using namespace tcs;
    const int tile = blockIdx.x / max_pairs, pr = blockIdx.x % max_pairs;
    const int4 ti = tinfo[tile];
    if (2 * pr >= ti.x) return;
    uint4* e = reinterpret_cast<uint4*>(base + static_cast<int64_t>(ti.z) * 1024 + sp_stage_off(2 * pr, H) + H * A_BYTES);
    for (int i = threadIdx.x; i < H * E_BYTES / 16; i += blockDim.x) e[i] = make_uint4(0, 0, 0, 0);
}

// The paper's offline PreProcessing (Listing 3) for the slot kernels: slot packing of
// every column tile's kept rows, then the compact weight images.  exact (host, may be null): the
// exact buffer size, which synchronizes s; with query_only nothing is written to buf.
nm_status tc_sp_prepack(const void* Bv, const uint8_t* D, int64_t n, int64_t k, int N, int M, int L, bool tf, int H,
                        void* buf, int64_t buf_bytes, int64_t* exact, bool query_only, cudaStream_t s) {
    using namespace tcs;
    const SpGeom g = sp_geom(n, k, N, M, L, tf, H);
    const int64_t units = static_cast<int64_t>(g.ntiles) * g.nchunks;
    void* scr = nullptr;
    nm_status st = scratch_alloc(&scr, sp_scratch_bytes(g), s);
    if (st) return st;
    uint8_t* sb = static_cast<uint8_t*>(scr);
    int* qk = reinterpret_cast<int*>(sb);
    sb += al256(units * g.KC * 4);
    int* tsl = reinterpret_cast<int*>(sb);
    uint8_t* tty = sb + units * (2 * g.KC + 4) * 4;
    sb += al256(units * (2 * g.KC + 4) * 5);
    int* ccnt = reinterpret_cast<int*>(sb);
    sb += al256(units * 4);
    int* slots = reinterpret_cast<int*>(sb);
    sb += al256(g.ntiles * g.smax * 4);
    uint8_t* stype = sb;
    sb += al256(g.ntiles * g.smax);
    int* nst = reinterpret_cast<int*>(sb);
    sb += al256(g.ntiles * 4);
    int4* tinfo = reinterpret_cast<int4*>(sb);
    sb += al256(g.ntiles * 16);
    int64_t* header = reinterpret_cast<int64_t*>(sb);
    cudaError_t e = cudaSuccess;
    auto done = [&](nm_status r) {
        cudaFreeAsync(scr, s);
        return r;
    };
    const char* seq = std::getenv("NM_SP_PACK_SEQ");
    if (seq && seq[0] == '1')
        sp_pack_kernel<<<static_cast<unsigned>(ceil_div(units, 32)), 32, 0, s>>>(
            D, tsl, tty, ccnt, qk, static_cast<int>(n), static_cast<int>(k), N, M, L, g.H, g.nchunks, g.PG);
    else
        sp_pack_warp_kernel<<<static_cast<unsigned>(units), 32, 0, s>>>(D, tsl, tty, ccnt, static_cast<int>(n),
                                                                      static_cast<int>(k), N, M, L, g.H, g.nchunks, g.PG);
    note_launch();
    if ((e = cudaGetLastError()) != cudaSuccess) return done(cuda_fail(e, "sp_pack_kernel"));
    sp_compact_kernel<<<static_cast<unsigned>(g.ntiles), 256, 0, s>>>(tsl, tty, ccnt, slots, stype, nst,
                                                                     static_cast<int>(k), M, g.nchunks,
                                                                     static_cast<int>(g.smax), g.SLOTS);
    note_launch();
    sp_layout_kernel<<<1, 32, 0, s>>>(nst, tinfo, header, g.ntiles, g.H, g.SLOTS, g.slots_off);
    note_launch();
    if ((e = cudaGetLastError()) != cudaSuccess) return done(cuda_fail(e, "sp_layout_kernel"));
    int64_t need = -1;
    if (exact || query_only) {
        if ((e = cudaMemcpyAsync(&need, header, 8, cudaMemcpyDeviceToHost, s)) != cudaSuccess ||
            (e = cudaStreamSynchronize(s)) != cudaSuccess)
            return done(cuda_fail(e, "nm_prepack size"));
        if (exact) *exact = need;
        if (query_only) return done(NM_OK);
        if (buf_bytes < need) return done(fail(NM_ERR_NULL, "nm_prepack: buffer smaller than the prepacked weight (" +
                                                                std::to_string(need) + " bytes, nm_prepack_size)"));
    }
    uint8_t* b = static_cast<uint8_t*>(buf);
    // header + tinfo, then the slot region zeroed (so alignment gaps are deterministic) and filled
    const int64_t zero_to = std::min<int64_t>(buf_bytes, g.slots_off + g.ntiles * g.smax * 4);
    if ((e = cudaMemsetAsync(b, 0, static_cast<size_t>(zero_to), s)) != cudaSuccess ||
        (e = cudaMemcpyAsync(b, header, 24, cudaMemcpyDeviceToDevice, s)) != cudaSuccess ||
        (e = cudaMemcpyAsync(b + 256, tinfo, static_cast<size_t>(g.ntiles) * 16, cudaMemcpyDeviceToDevice, s)) !=
            cudaSuccess)
        return done(cuda_fail(e, "nm_prepack layout"));
    sp_slots_copy_kernel<<<static_cast<unsigned>(g.ntiles), 256, 0, s>>>(slots, tinfo, reinterpret_cast<int*>(b + g.slots_off),
                                                                        static_cast<int>(g.smax), g.SLOTS);
    note_launch();
    const int max_pairs = static_cast<int>((g.max_stages + 1) / 2);
    sp_meta_zero_kernel<<<static_cast<unsigned>(static_cast<int64_t>(g.ntiles) * max_pairs), 128, 0, s>>>(tinfo, b, g.H,
                                                                                                          max_pairs);
    note_launch();
    const int64_t threads = static_cast<int64_t>(g.ntiles) * g.max_stages * 128 * g.H;
    auto img = tf ? sp_image_kernel<true> : sp_image_kernel<false>;
    img<<<static_cast<unsigned>(ceil_div(threads, 128)), 128, 0, s>>>(
        Bv, D, slots, stype, nst, tinfo, b, static_cast<int>(n), static_cast<int>(k), N, M, L, static_cast<int>(g.smax),
        static_cast<int>(g.max_stages), g.H);
    note_launch();
    if ((e = cudaGetLastError()) != cudaSuccess) return done(cuda_fail(e, "sp_image_kernel"));
    return done(NM_OK);
}

template <int H, int NT, bool TF>
static nm_status sp_launch_h(const void* at, tcs::Params p, int64_t m, int64_t n, int est_stages, cudaStream_t s) {
    using namespace tcs;
    using CF = Cfg<H, NT, TF>;
    static std::atomic<uint64_t> attr_mask{0};
    if (!attr_once(attr_mask)) {
        NM_CUDA_TRY(cudaFuncSetAttribute(spmm_tc_sp_kernel<H, NT, TF>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, CF::SMEM_BYTES));
        NM_CUDA_TRY(cudaFuncSetAttribute(spmm_tc_sp_kernel<H, NT, TF, true>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, CF::SMEM_BYTES));
        attr_done(attr_mask);
    }
    // C through TMA stores when its rows are 16-B aligned (the staged tile, NT/32 chunks of
    // 32 x MC elements, must fit in the stage ring it reuses)
    CUtensorMap tmC, tmC16;
    const int eb = p.c_bf16 ? 2 : 4;
    p.tma_c = 0;
    const char* te = std::getenv("NM_SP_TMA_C");
    if (!p.npeer && !(te && te[0] == '0') && (n * eb) % 16 == 0 && (reinterpret_cast<uintptr_t>(p.C) & 15) == 0 &&
        (NT + 31) / 32 * 32 * CF::MC * eb <= CF::ST * (CF::B_BYTES + CF::W_BYTES)) {
        const CUtensorMapDataType dt = p.c_bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
        if (make_tma_2d(&tmC, p.C, dt, eb, m, n, 32, CF::MC, 0) == NM_OK &&
            make_tma_2d(&tmC16, p.C, dt, eb, m, n, 16, CF::MC, 0) == NM_OK)
            p.tma_c = 1;
    }
    if (!p.tma_c) {
        memset(&tmC, 0, sizeof(tmC));
        memset(&tmC16, 0, sizeof(tmC16));
    }
    // tail split (NM_SP_TAIL=0 disables): the tiles of a partial last wave that at most half
    // fills the SMs run as two half-range CTAs each
    p.n_tok = static_cast<int>(ceil_div(m, CF::NT));
    const int64_t tiles = ceil_div(n, CF::MC) * p.n_tok;
    const int64_t sms = num_sms();
    // Split stage ranges (pair-aligned) over several CTAs per tile, partials added in a fixed order:
    //  * a grid below one wave (small problems, column shards of a multi-GPU layer): every tile in
    //    S = sms / tiles parts (<= 8, >= MIN_PART_STAGES stages per part, est_stages = the host's
    //    estimate);
    //  * a partial last wave that at most half fills the SMs: its tiles in 2 parts ("tail split").
    // NM_SP_SPLIT=S forces S for those tiles; NM_SP_TAIL=0 disables splitting.
    const char* te2 = std::getenv("NM_SP_TAIL");
    const char* se = std::getenv("NM_SP_SPLIT");
    const bool can_split = p.tma_c && !(te2 && te2[0] == '0');
    int64_t split_tiles = 0;
    int S = 1;
    // Every part must keep >= 24 stages: measured on B200 (profiles/r02f_sp_split_probe.txt) shorter
    // parts lose to their fixed costs (1024^3 16:32 in 2 parts of ~8 stages: 25.6 vs 18.4 us unsplit;
    // 2048x5120x5120 4:32 tail in parts of ~18: 56.6 vs 53.5 us), longer ones gain 1-4 % (cfg2 tail,
    // the 8-GPU column shards of cfg2 / cfg3).
    if (can_split && tiles < sms) {
        split_tiles = tiles;
        S = static_cast<int>(std::min<int64_t>(8, sms / tiles));
        S = std::max(1, std::min(S, est_stages / MIN_PART_STAGES));
    } else if (can_split && tiles % sms > 0 && 2 * (tiles % sms) <= sms) {
        split_tiles = tiles % sms;
        S = est_stages / 2 >= MIN_PART_STAGES ? 2 : 1;
    }
    if (se && split_tiles > 0) S = std::max(1, std::min(16, std::atoi(se)));  // forced (tests, studies)
    if (S <= 1) split_tiles = 0, S = 1;
    p.full_ctas = static_cast<int>(tiles - split_tiles);
    p.split = S;
    p.ws = nullptr;
    p.counters = nullptr;
    if (split_tiles > 0) {
        nm_status st = scratch_alloc(reinterpret_cast<void**>(&p.ws),
                                     static_cast<size_t>(split_tiles) * S * CF::MC * NT * 4, s);
        if (!st) st = scratch_alloc(reinterpret_cast<void**>(&p.counters), static_cast<size_t>(split_tiles) * 8, s);
        if (st) return st;
        NM_CUDA_TRY(cudaMemsetAsync(p.counters, 0, static_cast<size_t>(split_tiles) * 8, s));
    }
    const unsigned grid = static_cast<unsigned>(p.full_ctas + split_tiles * S);
    prof_begin(s);
    if (p.npeer)
        spmm_tc_sp_kernel<H, NT, TF, true><<<grid, THREADS, CF::SMEM_BYTES, s>>>(at, tmC, tmC16, p);
    else
        spmm_tc_sp_kernel<H, NT, TF><<<grid, THREADS, CF::SMEM_BYTES, s>>>(at, tmC, tmC16, p);
    prof_end(s);
    note_launch();
    const cudaError_t e = cudaGetLastError();
    if (p.ws) cudaFreeAsync(p.ws, s);
    if (p.counters) cudaFreeAsync(p.counters, s);
    if (e != cudaSuccess) return cuda_fail(e, "spmm_tc_sp_kernel");
    return NM_OK;
}

template <bool TF>
static nm_status sp_dispatch(int H, int nt, const void* at, const tcs::Params& p, int64_t m, int64_t n, int est,
                             cudaStream_t s) {
    switch (H * 1000 + nt) {
        case 2192: return sp_launch_h<2, 192, TF>(at, p, m, n, est, s);
        case 2128: return sp_launch_h<2, 128, TF>(at, p, m, n, est, s);
        case 2160: return sp_launch_h<2, 160, TF>(at, p, m, n, est, s);
        case 2224: return sp_launch_h<2, 224, TF>(at, p, m, n, est, s);
        case 2176: return sp_launch_h<2, 176, TF>(at, p, m, n, est, s);
        case 2208: return sp_launch_h<2, 208, TF>(at, p, m, n, est, s);
        case 1256: return sp_launch_h<1, 256, TF>(at, p, m, n, est, s);
        case 1128: return sp_launch_h<1, 128, TF>(at, p, m, n, est, s);
        case 1192: return sp_launch_h<1, 192, TF>(at, p, m, n, est, s);
        default: return fail(NM_ERR_UNSUPPORTED, "spmm_tc_sp: unsupported (H, NT)");
    }
}


// One SpMM on a prepacked weight (buf from tc_sp_prepack with H column halves per tile).
nm_status tc_sp_run(const void* A, const void* buf, int H, void* C, bool c_bf16, int64_t m, int64_t n, int64_t k, int N,
                    int M, int L, bool tf, cudaStream_t s, const PeerOut* po, float alpha, const void* At_in,
                    int64_t lda) {
    using namespace tcs;
    const SpGeom g = sp_geom(n, k, N, M, L, tf, H);
    const uint8_t* b = static_cast<const uint8_t*>(buf);
    const int64_t mp = At_in ? lda : (m + 7) / 8 * 8;  // A^T row pitch (elements)
    const int eb = tf ? 4 : 2;
    void* at = nullptr;
    if (static_cast<uint64_t>(k + 1) * static_cast<uint64_t>(mp) * static_cast<uint64_t>(eb) >= (1ull << 32))
        return fail(NM_ERR_UNSUPPORTED, "spmm_tc_sp: A^T larger than 4 GiB (32-bit row offsets)");
    nm_status st = NM_OK;
    cudaError_t e = cudaSuccess;
    if (At_in) {  // nm_spmm_at: the caller's A^T (padding slots are zero-filled by the gather)
        at = const_cast<void*>(At_in);
    } else {
    // k + 1 rows: row k is zero (padding slots also zero-fill in the gather; kept for the tf32 path)
    st = scratch_alloc(&at, static_cast<size_t>((k + 1) * mp) * eb, s);
    if (st) return st;
    const dim3 tg(static_cast<unsigned>(ceil_div(k, 64)), static_cast<unsigned>(ceil_div(mp, 64)));
    if (tf) {
        // fp32 A^T by the SIMT path's transpose (tokens >= m written as zeros), then the zero row k
        transpose_kernel<<<tg, 256, 0, s>>>(static_cast<const float*>(A), static_cast<float*>(at), static_cast<int>(m),
                                            static_cast<int>(k), static_cast<int>(mp));
        note_launch();
        e = cudaGetLastError();
        if (e == cudaSuccess)
            e = cudaMemsetAsync(static_cast<float*>(at) + k * mp, 0, static_cast<size_t>(mp) * 4, s);
    } else {
        transpose_bf16_kernel<<<tg, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(A), static_cast<__nv_bfloat16*>(at),
                                                 static_cast<int>(m), static_cast<int>(k), static_cast<int>(mp));
        note_launch();
        e = cudaGetLastError();
    }
    if (e != cudaSuccess) st = cuda_fail(e, "spmm_tc_sp transpose");
    }
    if (!st) {
        Params p{};
        p.base = b;
        p.tinfo = reinterpret_cast<const int4*>(b + 256);
        p.slots_off = g.slots_off;
        p.C = C;
        p.m = static_cast<int>(m);
        p.n = static_cast<int>(n);
        p.k = static_cast<int>(k);
        p.mp = static_cast<int>(mp);
        p.c_bf16 = c_bf16 ? 1 : 0;
        const char* dbg = std::getenv("NM_SP_DBG");
        p.dbg = dbg ? std::atoi(dbg) : 0;
        p.alpha = alpha;
        if (po) {
            p.npeer = po->np;
            for (int i = 0; i < po->np && i < 8; ++i) p.cpeer[i] = po->c[i];
            p.ldc = po->ldc;
            p.col_off = po->col_off;
            p.n_valid = static_cast<int>(po->n_valid);
        }
        const int est = tcs::sp_est_stages(k, N, M, L, g.H, tf);
        const int nt = sp_tokens(g.H, m, n, est);
        st = tf ? sp_dispatch<true>(g.H, nt, at, p, m, n, est, s) : sp_dispatch<false>(g.H, nt, at, p, m, n, est, s);
    }
    if (!At_in) {
        e = cudaFreeAsync(at, s);
        if (st == NM_OK && e != cudaSuccess) st = cuda_fail(e, "cudaFreeAsync");
    }
    return st;
}

// nm_plan_query: the geometry nm_spmm (a per-call prepack) would use; nm_spmm_prepacked keeps the
// H of its prepack (tcs::sp_halves, chosen without m)
void tc_sp_geometry(int64_t m, int64_t n, int64_t k, int N, int M, int L, int* halves, int* tokens) {
    *halves = tcs::sp_halves_m(L, N, M, m, n, k);
    *tokens = tcs::sp_tokens(*halves, m, n, tcs::sp_est_stages(k, N, M, L, *halves, false));
}

int tc_sp_halves(int N, int M, int L) { return tcs::sp_halves(L, N, M); }
int tc_sp_halves_m(int N, int M, int L, int64_t m, int64_t n, int64_t k) { return tcs::sp_halves_m(L, N, M, m, n, k); }

// nm_spmm without a prepacked weight: prepack into pooled scratch (the size bound, no sync), run,
// release.
nm_status tc_sp_launch(const void* A, const void* Bv, const uint8_t* D, void* C, bool c_bf16, int64_t m, int64_t n,
                       int64_t k, int N, int M, int L, bool tf, cudaStream_t s, float alpha, const void* At_in,
                       int64_t lda) {
    void* buf = nullptr;
    const size_t bytes = tc_sp_prepack_bytes(n, k, N, M, L, tf);
    const int H = tcs::sp_halves_m(L, N, M, m, n, k);  // per-call prepack: the token count is known
    nm_status st = scratch_alloc(&buf, bytes, s);
    if (st) return st;
    st = tc_sp_prepack(Bv, D, n, k, N, M, L, tf, H, buf, static_cast<int64_t>(bytes), nullptr, false, s);
    if (!st) st = tc_sp_run(A, buf, H, C, c_bf16, m, n, k, N, M, L, tf, s, nullptr, alpha, At_in, lda);
    const cudaError_t e = cudaFreeAsync(buf, s);
    if (st == NM_OK && e != cudaSuccess) st = cuda_fail(e, "cudaFreeAsync");
    return st;
}

}  // namespace nm
