// spmm_tc_sp2.cu -- the slot-packed sparse contraction of spmm_tc_sp.cu (Eq. 1; DESIGN.md
// 5.2) on CTA pairs: tcgen05.mma.sp.cta_group::2, persistent.
//
// C^T = B~^T . A^T per column tile of 256 output columns (the H = 2 prepack: one slot sequence for
// the tile's 256 / L groups, the paper's col_info union) and token tile of 256 tokens:
//   * one MMA covers M = 256 columns x N = 256 tokens x K = 32 slots; CTA rank r of the pair holds
//     weight half r (128 columns: its A-operand rows and metadata) and tokens [128 r, 128 r + 128)
//     of the gathered B operand, and receives the accumulator of its 128 columns in its own TMEM.
//     Per SM this halves the shared-memory traffic of the token operand per MAC against the one-CTA
//     kernel (which reads its gathered token tile once per 128-column half) -- the one-CTA kernel
//     is bound by shared-memory bytes per stage;
//   * 128-slot stages (two prepack stages: A images even | odd, the even stage's metadata block =
//     both stages' metadata), so every ring round trip carries 4 MMAs;
//   * gather: 8 warps, stage-owning pairs (warps g, g + 4 own the stages = g mod 4, 64 slot rows
//     each, two 256-B row segments per warp-wide 16-B cp.async), weight images by bulk copies;
//     the peer's completion reaches the leader's full barrier through a relay warp (cp.async
//     completions arrive only on CTA-local barriers);
//   * the leader's warp 8 issues tcgen05.cp (metadata) + the MMAs and commits to both CTAs' empty
//     barriers (multicast); after a unit's last stage it commits the accumulator to both CTAs;
//   * 4 epilogue warps per CTA drain TMEM (tcgen05.ld, lane = output column) straight to global C
//     (no shared-memory staging: shared memory is the bound resource of the main loop) while the
//     gather warps already fill the ring for the next unit; the MMA warp waits for both CTAs'
//     epilogues (acc_empty) before the first MMA of the next unit;
//   * persistent clusters walk the units round-robin: full tiles, then the split parts of the
//     tiles of a partial last wave (pair-aligned stage ranges, partials added in the fixed order
//     0 .. S-1 by the last arriver: bit-reproducible, no co-residency assumption).
#include <cuda_bf16.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>

#include "tc_sp.cuh"

namespace nm {
namespace tcs2 {

using namespace nm::tc;
using namespace nm::tcs;

constexpr int NT2 = 256;           // tokens per pair (MMA N)
constexpr int TPC = NT2 / 2;       // tokens per CTA
constexpr int GW = 8;              // gather warps
constexpr int MW = 8;              // MMA issuer (leader) / relay (peer)
constexpr int EW0 = 9;             // epilogue warps EW0 .. EW0 + 3
constexpr int THREADS2 = (EW0 + 4) * 32;
constexpr int MR = 8;              // metadata ring (4 TMEM columns per stage) >= STAGES + 1
constexpr int TMEM_COLS2 = 512;

template <bool TF>
struct G2 {
    static constexpr int SL = 2 * El<TF>::SLOTS;              // slots per stage (two prepack stages)
    static constexpr int ATOMS = TPC / El<TF>::TOK_ATOM;      // 128-B token atoms per slot row
    static constexpr int B_BYTES = SL * ATOMS * 128;          // gathered token tile per stage (32 KB)
    static constexpr int W_BYTES = 2 * A_BYTES + E_BYTES;     // [A even | A odd | E] of this CTA's half
    static constexpr int ST = 4;                              // ring stages (= the 4 stage owners)
    static constexpr int SMEM = ST * (B_BYTES + W_BYTES) + 1024 + 256;
    static_assert(SMEM <= 232448, "shared memory budget");
    static_assert(NT2 + 4 * MR <= TMEM_COLS2, "TMEM budget");
};

__device__ __forceinline__ void mbar_arrive_remote(uint64_t* bar, uint32_t cta) {
    asm volatile(
        "{\n\t.reg .b32 ra;\n\tmapa.shared::cluster.u32 ra, %0, %1;\n\t"
        "mbarrier.arrive.release.cluster.shared::cluster.b64 _, [ra];\n\t}" ::"r"(smem_u32(bar)),
        "r"(cta)
        : "memory");
}
__device__ __forceinline__ void mbar_spin(uint64_t* bar, uint32_t parity) {
    while (!mbar_test(bar, parity)) {
    }
}
__device__ __forceinline__ uint64_t gtime() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
// NM_SP_DBG & 64: cluster 0 records %globaltimer (ns) per stage g < 64 into C as [g][slot] (16 slots):
// 0/1 leader owner before / after its empty wait, 2 leader owner after its copies are issued,
// 4/5 peer owner before / after empty wait, 6 peer owner issued, 8 relay saw peer full,
// 10 MMA saw full, 11 MMA committed
#define TS2(g, slot)                                                                                   \
    do {                                                                                               \
        if ((p.dbg & 64) && cid == 0 && (g) < 64) static_cast<long long*>(p.C)[(g) * 16 + (slot)] = gtime(); \
    } while (0)
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
    uint32_t ok = 0;
    while (!ok)
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
}
template <bool TF>
__device__ __forceinline__ void mma_sp2(uint32_t d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc,
                                        uint32_t emeta) {
    if (TF)
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.sp.cta_group::2.kind::tf32 [%0], %1, %2, [%5], %3, p;\n\t}" ::"r"(d),
            "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc), "r"(emeta)
            : "memory");
    else
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.sp.cta_group::2.kind::f16 [%0], %1, %2, [%5], %3, p;\n\t}" ::"r"(d),
            "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc), "r"(emeta)
            : "memory");
}
__device__ __forceinline__ void tmem_cp2_128x128b(uint32_t taddr, uint64_t sdesc) {
    asm volatile("tcgen05.cp.cta_group::2.128x128b [%0], %1;" ::"r"(taddr), "l"(sdesc) : "memory");
}
__device__ __forceinline__ void tc_commit2_mc(uint64_t* bar, uint16_t mask) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"(mask)
        : "memory");
}

// A work unit: (column tile, token tile, part of a split tile) and its stage range in 128-slot
// stages: b0 .. b0 + nb - 1, prepack stages 2b (always) and 2b + 1 (iff 2b + 1 < sb).
struct Unit {
    int tile, m0, part, nparts, tail_idx, b0, nb, sb;
};
__device__ __forceinline__ Unit unit_of(const Params& p, int u) {
    Unit x;
    int lin = u;
    x.part = 0;
    x.nparts = 1;
    if (lin >= p.full_ctas) {
        x.nparts = p.split;
        x.part = (lin - p.full_ctas) % p.split;
        lin = p.full_ctas + (lin - p.full_ctas) / p.split;
    }
    x.tile = lin / p.n_tok;
    x.m0 = (lin % p.n_tok) * NT2;
    x.tail_idx = lin - p.full_ctas;
    const int nst_all = __ldg(&p.tinfo[x.tile].x);
    const int npairs = (nst_all + 1) >> 1;
    const int sa = min(nst_all, 2 * (x.part * npairs / x.nparts));
    x.sb = min(nst_all, 2 * ((x.part + 1) * npairs / x.nparts));
    x.b0 = sa >> 1;
    x.nb = (p.dbg & 512) ? 0 : (x.sb - sa + 1) >> 1;
    return x;
}

template <bool TF>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS2, 1)
    spmm_tc_sp2_kernel(const void* __restrict__ At, const Params p) {
    using GG = G2<TF>;
    using EL = El<TF>;
    constexpr int SL = GG::SL, B_BYTES = GG::B_BYTES, W_BYTES = GG::W_BYTES, STAGES = GG::ST;
    static_assert(!TF, "the tf32 pair variant is not built yet");
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* sB = smem;                     // STAGES x B_BYTES (1024-aligned: 128-B swizzle atoms)
    uint8_t* sW = smem + STAGES * B_BYTES;  // STAGES x [A even 8 KB | A odd 8 KB | metadata 2 KB]
    uint64_t* full = reinterpret_cast<uint64_t*>(sW + STAGES * W_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* acc_full = empty + STAGES;
    uint64_t* acc_empty = acc_full + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 1);
    volatile uint32_t* s_flag = tmem_slot + 1;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_rank();
    const bool leader = rank == 0;
    const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;

    if (warp == MW) {
        if (lane == 0) {
            for (int s = 0; s < STAGES; ++s) {
                // two owner warps' copies (2 x 32 noinc arrivals) + the weight copy; the leader's
                // barrier also takes the peer's relay arrive
                mbar_init(&full[s], 2 * 32 + 1 + (leader ? 1 : 0));
                mbar_init(&empty[s], 1);  // the leader's multicast commit
            }
            mbar_init(acc_full, 1);
            mbar_init(acc_empty, 2 * 4);  // both CTAs' 4 epilogue warps (the leader's barrier counts)
            fence_mbar_init();
        }
        __syncwarp();
        // both CTAs, the same warp (a pair allocation)
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(TMEM_COLS2)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    cluster_sync_all();  // barriers initialised and TMEM allocated in both CTAs
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp < GW) {
        // ============ gather: this CTA's 128 tokens of every slot row ============
        // Warps (o, o + 4) own the stages g = o (mod 4) (ring slot o); warp half h copies rows
        // 64 h .. 64 h + 63 (h = 1: the odd prepack stage) as 32 warp-wide cp.async of two rows each
        // (lanes 0-15 row 2i, 16-31 row 2i + 1; lane chunk c = 8 tokens, atom c / 8).
        static_assert(STAGES == 4, "four stage owners");
        const int own = warp & 3, half = warp >> 2, hi = lane >> 4, c = lane & 15;
        const uint32_t pitch = static_cast<uint32_t>(p.mp) * 2u;
        uint32_t dl[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int r = half * 64 + 2 * i + hi;
            dl[i] = static_cast<uint32_t>((c >> 3) * (SL * 128) + r * 128) +
                    ((static_cast<uint32_t>(c & 7) ^ static_cast<uint32_t>(r & 7)) << 4);
        }
        const int* slots = reinterpret_cast<const int*>(p.base + p.slots_off);
        int g = 0;  // running stage counter over all units of this cluster
        for (int u = cid; u < p.n_units; u += ncl) {
            const Unit x = unit_of(p, u);
            const int4 ti = __ldg(&p.tinfo[x.tile]);
            const int tok = x.m0 + static_cast<int>(rank) * TPC + 8 * c;
            const bool tok_ok = tok < p.mp;
            const uint32_t srcsz = tok_ok ? 16u : 0u;
            const char* src = static_cast<const char*>(At) + 2 * static_cast<int64_t>(tok_ok ? tok : 0);
            const int* ssrc = slots + ti.y + half * 64 + lane;
            const uint8_t* wsrc = p.base + static_cast<int64_t>(ti.z) * 1024;
            // this warp's first owned stage of the unit and its slot rows (one owned stage ahead)
            int bl = (own - g) & 3;
            int k0 = 0, k1 = 0;
            if (bl < x.nb && (half == 0 || 2 * (x.b0 + bl) + 1 < x.sb)) {
                k0 = ssrc[(x.b0 + bl) * SL];
                k1 = ssrc[(x.b0 + bl) * SL + 32];
            }
            for (; bl < x.nb; bl += 4) {
                const int gg = g + bl;
                const int b = x.b0 + bl;
                const bool odd = 2 * b + 1 < x.sb;
                const bool rows_on = half == 0 || odd;
                const uint32_t o0 = static_cast<uint32_t>(k0) * pitch, o1 = static_cast<uint32_t>(k1) * pitch;
                {  // prefetch the next owned stage's slot rows
                    const int bn = bl + 4;
                    if (bn < x.nb && (half == 0 || 2 * (x.b0 + bn) + 1 < x.sb)) {
                        k0 = ssrc[(x.b0 + bn) * SL];
                        k1 = ssrc[(x.b0 + bn) * SL + 32];
                    }
                }
                const int s = gg & 3;
                if (half == 0 && lane == 0) TS2(gg, 4 * rank + 0);
                if (gg >= STAGES) {
                    if (p.dbg & 2048) mbar_spin(&empty[s], ((gg >> 2) - 1) & 1);
                    else mbar_wait(&empty[s], ((gg >> 2) - 1) & 1);
                }
                if (half == 0 && lane == 0) TS2(gg, 4 * rank + 1);
                if (half == 0 && lane == 0) {
                    if (p.dbg & 16) {
                        mbar_arrive(&full[s]);
                    } else {
                        const uint8_t* we = wsrc + sp_stage_off(2 * b, 2);
                        uint8_t* wd = sW + s * W_BYTES;
                        mbar_arrive_expect_tx(&full[s], static_cast<uint32_t>(A_BYTES + E_BYTES + (odd ? A_BYTES : 0)));
                        bulk_load(wd, we + rank * A_BYTES, A_BYTES, &full[s]);
                        bulk_load(wd + 2 * A_BYTES, we + 2 * A_BYTES + rank * E_BYTES, E_BYTES, &full[s]);
                        if (odd) bulk_load(wd + A_BYTES, wsrc + sp_stage_off(2 * b + 1, 2) + rank * A_BYTES, A_BYTES, &full[s]);
                    }
                }
                if (rows_on && !(p.dbg & 1)) {
                    const uint32_t bst = smem_u32(sB + s * B_BYTES);
#pragma unroll
                    for (int i = 0; i < 32; ++i) {
                        const uint32_t o = __shfl_sync(0xffffffffu, i < 16 ? o0 : o1, (2 * i + hi) & 31);
                        cp_async16(bst + dl[i & 3] + (i >> 2) * 1024, src + o, srcsz);
                    }
                }
                cp_async_arrive_noinc(&full[s]);
                if (half == 0 && lane == 0) TS2(gg, 4 * rank + 2);
            }
            g += x.nb;
        }
    } else if (warp == MW) {
        if (leader) {
            // ============ MMA issuer: per stage the metadata copy + 4 (2 on an odd tail) sparse MMAs ============
            constexpr uint32_t idesc = (1u << 2) | (1u << 4) | (EL::FMT << 7) | (EL::FMT << 10) | (1u << 16) |
                                       (static_cast<uint32_t>(NT2 >> 3) << 17) | (static_cast<uint32_t>(256 >> 4) << 24);
            const uint64_t bdesc0 = smem_desc(smem_u32(sB), SL * 128, EL::B_SBO, EL::B_LAYOUT);
            const uint64_t adesc0 = smem_desc(smem_u32(sW), 16, 512, 4);
            const uint64_t edesc0 = smem_desc(smem_u32(sW) + 2 * A_BYTES, 2048, 128, 0);
            const bool skip_mma = (p.dbg & 2) != 0;
            int g = 0, ue = 0;
            for (int u = cid; u < p.n_units; u += ncl, ++ue) {
                const Unit x = unit_of(p, u);
                if (ue > 0) {  // both CTAs' epilogues have drained the previous unit's accumulator
                    mbar_wait_cluster(acc_empty, (ue - 1) & 1);
                    tc_fence_after();
                }
                for (int bl = 0; bl < x.nb; ++bl, ++g) {
                    const int s = g & 3;
                    const bool odd = 2 * (x.b0 + bl) + 1 < x.sb;
                    if (p.dbg & 1024) {
                        while (!mbar_test(&full[s], (g >> 2) & 1)) {
                        }
                        asm volatile("fence.acq_rel.cluster;" ::: "memory");
                    } else {
                        mbar_wait_cluster(&full[s], (g >> 2) & 1);
                    }
                    if (lane == 0) TS2(g, 10);
                    tc_fence_after();
                    if (elect_one()) {
                        if (!skip_mma) {
                            const uint64_t bo = static_cast<uint64_t>(s * (B_BYTES >> 4));
                            const uint64_t wo = static_cast<uint64_t>(s * (W_BYTES >> 4));
                            const uint32_t mcol = tmem + NT2 + 4 * (g % MR);
                            tmem_cp2_128x128b(mcol, edesc0 + wo);
#pragma unroll
                            for (int j = 0; j < 4; ++j)
                                if ((j < 2 || odd) && !((p.dbg & 4096) && j > 0))  // dbg 4096: one MMA per stage
                                    mma_sp2<TF>(tmem, adesc0 + wo + (((j >> 1) * A_BYTES + 32 * (j & 1)) >> 4),
                                                bdesc0 + bo + ((EL::B_STEP * j) >> 4), idesc | static_cast<uint32_t>(j & 1),
                                                (bl | j) ? 1u : 0u, mcol + 2 * (j >> 1));
                        }
                        if (p.dbg & 128) {  // timing study: plain arrives instead of the commit
                            mbar_arrive(&empty[s]);
                            mbar_arrive_remote(&empty[s], 1);
                        } else {
                            tc_commit2_mc(&empty[s], 0x3);
                        }
                    }
                    if (lane == 0) TS2(g, 11);
                    __syncwarp();
                }
                if (elect_one()) tc_commit2_mc(acc_full, 0x3);
                __syncwarp();
            }
        } else {
            // ============ relay: this CTA's stage s is complete -> arrive on the leader's full[s] ============
            int g = 0;
            for (int u = cid; u < p.n_units; u += ncl) {
                const Unit x = unit_of(p, u);
                for (int bl = 0; bl < x.nb; ++bl, ++g) {
                    if (p.dbg & 1024) mbar_spin(&full[g & 3], (g >> 2) & 1);
                    else mbar_wait(&full[g & 3], (g >> 2) & 1);
                    if (lane == 0) TS2(g, 8);
                    if (lane == 0) mbar_arrive_remote(&full[g & 3], 0);
                    __syncwarp();
                }
            }
        }
    } else {
        // ============ epilogue: TMEM lane = output column, TMEM column = token; direct stores ============
        const int qw = warp & 3;  // TMEM lane quarter of this warp
        const bool odd_lane = lane & 1;
        const uint32_t tbase = tmem + (static_cast<uint32_t>(qw * 32) << 16);
        int ue = 0;
        for (int u = cid; u < p.n_units; u += ncl, ++ue) {
            const Unit x = unit_of(p, u);
            mbar_wait(acc_full, ue & 1);
            tc_fence_after();
            const int col = x.tile * 256 + static_cast<int>(rank) * 128 + qw * 32 + lane;
            const int pc = col & ~1;
            const int cidx = 2 * (x.tail_idx * 2 + static_cast<int>(rank));  // split counters of this half
            bool publish = false;
            if (x.nparts > 1) {
                if (warp == EW0 && lane == 0) *s_flag = atomicAdd(p.counters + cidx, 1) < x.nparts - 1 ? 1u : 0u;
                named_bar_sync(2, 128);
                publish = *s_flag != 0;
            }
            const int64_t part_stride = static_cast<int64_t>(2) * 128 * NT2;  // floats per (tile, part)
            float* wbase = x.nparts > 1 ? p.ws + static_cast<int64_t>(x.tail_idx) * x.nparts * part_stride +
                                              static_cast<int64_t>(rank) * 128 * NT2
                                        : nullptr;
            if (!publish && x.nparts > 1) {
                if (warp == EW0 && lane == 0) {
                    unsigned long long t0g, tn;
                    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0g));
                    while (ld_acquire(p.counters + cidx + 1) < x.nparts - 1) {
                        __nanosleep(256);
                        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tn));
                        if (tn - t0g > 20000000000ull) __trap();  // 20 s: a lost partial is a bug
                    }
                }
                named_bar_sync(2, 128);
                __threadfence();
            }
#pragma unroll 1
            for (int t0 = 0; t0 < NT2; t0 += 32) {
                uint32_t v[32];
                if (x.nb > 0) {
                    tmem_ld32(tbase + t0, v);
                    tmem_wait_ld();
                } else {
#pragma unroll
                    for (int i = 0; i < 32; ++i) v[i] = 0u;
                }
                if (publish) {  // token-major [NT2][128] partial of this half
                    float* w = wbase + x.part * part_stride + static_cast<int64_t>(t0) * 128 + qw * 32 + lane;
#pragma unroll
                    for (int i = 0; i < 32; ++i) w[i * 128] = __uint_as_float(v[i]);
                    continue;
                }
                if (wbase) {  // sum of the parts in the order 0 .. nparts-1
                    float a[32];
#pragma unroll
                    for (int i = 0; i < 32; ++i) a[i] = 0.f;
#pragma unroll 1
                    for (int q2 = 0; q2 < x.nparts; ++q2) {
                        if (q2 == x.part) {
#pragma unroll
                            for (int i = 0; i < 32; ++i) a[i] += __uint_as_float(v[i]);
                        } else {
                            const float* w = wbase + q2 * part_stride + static_cast<int64_t>(t0) * 128 + qw * 32 + lane;
#pragma unroll
                            for (int i = 0; i < 32; ++i) a[i] += __ldcg(w + i * 128);
                        }
                    }
#pragma unroll
                    for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(a[i]);
                }
#pragma unroll
                for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * p.alpha);
                if (p.dbg & (8 | 64)) continue;
                if (p.c_bf16) {
                    // lanes (2q, 2q+1) swap so each stores a bf16 pair (columns pc, pc+1): even lane token i, odd i+1
#pragma unroll
                    for (int i = 0; i < 32; i += 2) {
                        const uint32_t xv = odd_lane ? v[i] : v[i + 1];
                        const uint32_t yv = __shfl_xor_sync(0xffffffffu, xv, 1);
                        const float lo = __uint_as_float(odd_lane ? yv : v[i]);
                        const float hi = __uint_as_float(odd_lane ? v[i + 1] : yv);
                        const int t = x.m0 + t0 + i + (odd_lane ? 1 : 0);
                        if (t < p.m && pc < p.n)
                            *reinterpret_cast<__nv_bfloat162*>(static_cast<__nv_bfloat16*>(p.C) +
                                                               static_cast<int64_t>(t) * p.n + pc) =
                                __floats2bfloat162_rn(lo, hi);
                    }
                } else {
#pragma unroll
                    for (int i = 0; i < 32; ++i) {
                        const int t = x.m0 + t0 + i;
                        if (t < p.m && col < p.n)
                            static_cast<float*>(p.C)[static_cast<int64_t>(t) * p.n + col] = __uint_as_float(v[i]);
                    }
                }
            }
            // the accumulator is drained: release it to the leader's MMA issuer
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if (leader) mbar_arrive(acc_empty);
                else mbar_arrive_remote(acc_empty, 0);
            }
            if (publish) {
                __threadfence();
                named_bar_sync(2, 128);
                if (warp == EW0 && lane == 0) red_release_add(p.counters + cidx + 1, 1);
            }
        }
    }
    tc_fence_before();
    cluster_sync_all();  // every MMA / commit touching either CTA has completed
    if (warp == MW) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS2) : "memory");
    }
}

}  // namespace tcs2

// Pair kernel applicability: bf16 operands, the H = 2 prepack (256-column tiles), no peer stores;
// opt-in (NM_SP_PAIR=1).  Measured on B200 it is slower than the one-CTA kernel at every BASELINE
// shape (cfg2 144 vs 100 us, 8192^3 854 vs 578 us; profiles/r02b_sp_pair_ablation.txt): both are
// bound by the latency of the stage hand-off, not by shared-memory bytes, and the pair adds a
// hop (the peer's relay) to every stage while carrying only 1.33x the MMA time per stage.
bool tc_sp2_enabled(bool tf, int H) {
    if (tf || H != 2) return false;
    const char* e = std::getenv("NM_SP_PAIR");
    return e && e[0] == '1';
}

// Launch on a prepacked weight (p from tc_sp_run: base, tinfo, slots_off, C, dims, dbg, alpha).
nm_status tc_sp2_launch(const void* at, tcs::Params p, int64_t m, int64_t n, int est_stages, cudaStream_t s) {
    using namespace tcs2;
    using GG = G2<false>;
    static std::atomic<uint64_t> attr_mask{0};
    if (!attr_once(attr_mask)) {
        NM_CUDA_TRY(cudaFuncSetAttribute(spmm_tc_sp2_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, GG::SMEM));
        attr_done(attr_mask);
    }
    p.tma_c = 0;
    p.n_tok = static_cast<int>(ceil_div(m, NT2));
    const int64_t tiles = ceil_div(n, 256) * p.n_tok;
    const int64_t pairs = num_sms() / 2;
    // split: a grid below one wave of pairs -> every tile in S parts (>= 4 stage pairs each);
    // a partial last wave that at most half fills the pairs -> its tiles in 2 parts.  NM_SP_SPLIT
    // forces S; NM_SP_TAIL=0 disables splitting.
    const char* te = std::getenv("NM_SP_TAIL");
    const char* se = std::getenv("NM_SP_SPLIT");
    const bool can_split = !(te && te[0] == '0');
    int64_t split_tiles = 0;
    int S = 1;
    if (can_split && tiles < pairs) {
        split_tiles = tiles;
        S = static_cast<int>(std::min<int64_t>(8, pairs / tiles));
        S = std::max(1, std::min(S, est_stages / 8));
    } else if (can_split && tiles % pairs > 0 && 2 * (tiles % pairs) <= pairs) {
        split_tiles = tiles % pairs;
        S = 2;
    }
    if (se && split_tiles > 0) S = std::max(1, std::min(16, std::atoi(se)));
    if (S <= 1) split_tiles = 0, S = 1;
    p.full_ctas = static_cast<int>(tiles - split_tiles);
    p.split = S;
    p.n_units = static_cast<int>(p.full_ctas + split_tiles * S);
    p.ws = nullptr;
    p.counters = nullptr;
    if (split_tiles > 0) {
        nm_status st = scratch_alloc(reinterpret_cast<void**>(&p.ws),
                                     static_cast<size_t>(split_tiles) * S * 2 * 128 * NT2 * 4, s);
        if (!st) st = scratch_alloc(reinterpret_cast<void**>(&p.counters), static_cast<size_t>(split_tiles) * 2 * 2 * 4, s);
        if (st) return st;
        NM_CUDA_TRY(cudaMemsetAsync(p.counters, 0, static_cast<size_t>(split_tiles) * 2 * 2 * 4, s));
    }
    const int64_t clusters = std::min<int64_t>(pairs, p.n_units);
    prof_begin(s);
    spmm_tc_sp2_kernel<false><<<static_cast<unsigned>(2 * clusters), THREADS2, GG::SMEM, s>>>(at, p);
    prof_end(s);
    note_launch();
    const cudaError_t e = cudaGetLastError();
    if (p.ws) cudaFreeAsync(p.ws, s);
    if (p.counters) cudaFreeAsync(p.counters, s);
    if (e != cudaSuccess) return cuda_fail(e, "spmm_tc_sp2_kernel");
    return NM_OK;
}

}  // namespace nm
