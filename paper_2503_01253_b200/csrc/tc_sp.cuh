// tc_sp.cuh -- definitions of the slot-packed sparse tensor-core kernels (spmm_tc_sp.cu, one CTA
// per tile; the round-2 CTA-pair variant was measured slower and removed): element types, the
// prepacked weight-image geometry, launch parameters and inline-PTX helpers (written from the
// PTX ISA).
#pragma once

#include <cuda_bf16.h>

#include "tcgen05.cuh"

namespace nm {
namespace tcs {

using namespace nm::tc;

// Geometry.  H = column halves per CTA: each half is one MMA M = 128 with its own accumulator,
// weight image and metadata, and both halves share the gathered token tile (the slot sequence
// is packed over all 128 H / L groups), so the gathered bytes per MAC halve at H = 2.
// H = 2 (L >= 32): 256 columns x 192 tokens; H = 1 (L = 16, where 256 columns would be 16
// groups): 128 columns x 256 tokens.
// Element types.  bf16 (kind::f16): 2:4 along the slots, 64 slots per stage (2 MMAs of K = 32),
// quads of slots share a metadata nibble.  tf32 (kind::tf32, fp32 operands): 1:2 along the
// slots, 32 slots per stage (2 MMAs of K = 16), pairs of slots share a nibble (0x4: the pair's
// first slot, 0xE: its second -- established on the GPU by scripts/ubench_sp_tf32.cu).  Both
// give 64-B weight-image rows and the same bytes per stage; the tf32 token tile is MN-major with
// the 32-B-atom 128-B swizzle (descriptor layout 1: 32-B chunks XOR k % 4, 4-row groups).
template <bool TF>
struct El {
    static constexpr int E = TF ? 4 : 2;                // operand bytes
    static constexpr int SLOTS = TF ? 32 : 64;          // slots per stage
    static constexpr int PG = TF ? 2 : 4;               // slots per metadata group
    static constexpr int TOK_ATOM = 128 / E;            // tokens per 128-B swizzled row
    static constexpr uint32_t B_SBO = TF ? 512 : 1024;  // k-direction stride of the swizzle groups
    static constexpr uint32_t B_LAYOUT = TF ? 1 : 2;    // 128B_BASE32B / 128B
    static constexpr uint32_t B_STEP = (SLOTS / 2) * 128;  // one MMA's K slots of the token tile
    static constexpr uint32_t FMT = TF ? 2 : 1;         // instruction-descriptor a/b format
};
constexpr int A_BYTES = 8192;              // per half: 128 rows x 64 B (32 bf16 / 16 tf32), 64-B swizzle
constexpr int E_BYTES = 128 * 16;          // per half: metadata of a stage PAIR, 128 TMEM lanes x 16 B
                                           // (words 0, 1: the even stage's two MMAs; 2, 3: the odd stage's)
constexpr int WH_BYTES = A_BYTES + E_BYTES;
// Weight image of one (column tile, stage): [A_0 .. A_{H-1} | E_0 .. E_{H-1}]; the E blocks are
// present (and copied) only for even stages and carry the metadata of the stage pair, so an odd
// stage moves H x A_BYTES and the metadata costs 1 KB per half and stage instead of 2.
// Byte offset of stage st inside a tile's compact image block: even stages carry the pair's
// metadata (H x (A + E)), odd stages only the A images (H x A).
__host__ __device__ constexpr int64_t sp_stage_off(int st, int H) {
    return static_cast<int64_t>(st >> 1) * H * (2 * A_BYTES + E_BYTES) + static_cast<int64_t>(st & 1) * H * (A_BYTES + E_BYTES);
}

struct Params {
    // compact prepacked weight (tc_sp_prepack): tinfo[tile] = {stages, first slot, image offset / 1 KB,
    // image bytes / 1 KB}; slots (row of A^T per slot, k = padding: the zero row) at base + slots_off;
    // a tile's stage images at base + 1 KB x tinfo.z, stage st at sp_stage_off(st, H)
    const uint8_t* base;
    const int4* tinfo;
    int64_t slots_off;
    void* C;
    int m, n, k, mp, c_bf16;
    int tma_c;  // 1: C tile staged in shared memory and written by TMA stores (tmC valid)
    int n_tok;       // token tiles (1-D grid: token tile fastest)
    int full_ctas;   // CTAs [0, full_ctas) do one whole tile; the rest split each remaining tile into
    int split;       // `split` stage ranges (pair-aligned)
    float* ws;       // split tiles: fp32 partials [tile - full tiles][part][NT][MC] (token-major)
    int* counters;   // split tiles: [2 x (tile - full tiles)] = {tickets, partials published} (zeroed per launch)
    int dbg;  // NM_SP_DBG (timing studies only): 1 skip gathers, 2 skip MMAs, 8 skip C stores, 16 skip weights,
              // 64 per-stage clock64 trace, 128 plain arrive for commits (no MMA), 256 per-CTA timeline
    // fused column all-gather (nm_spmm_prepacked_peers): the direct-store epilogue writes every C
    // element to cpeer[0 .. npeer) at [token][col_off + col] (row pitch ldc), columns < n_valid
    void* cpeer[8];
    int npeer, n_valid;
    int64_t ldc, col_off;
    float alpha;  // C = alpha . A B~ (nm_spmm_scaled); applied after the tail-split addition
};

// mbarrier wait variants (timing studies of the stage hand-off, NM_SP_DBG 1024 / 2048 / 4096):
// try_wait with an explicit suspend-time hint (ns), and a pure test_wait spin
__device__ __forceinline__ void mbar_wait_hint(uint64_t* bar, uint32_t parity, uint32_t ns) {
    uint32_t ok = 0;
    while (!ok)
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(smem_u32(bar)), "r"(parity), "r"(ns)
            : "memory");
}
__device__ __forceinline__ void mbar_wait_dbg(uint64_t* bar, uint32_t parity, int dbg, int hint_bit, int spin_bit) {
    if (dbg & spin_bit) {
        while (!mbar_test(bar, parity)) {
        }
    } else if (dbg & hint_bit) {
        mbar_wait_hint(bar, parity, 32);
    } else {
        mbar_wait(bar, parity);
    }
}

// 16-B global -> shared copy (L2 only); src_bytes = 0 zero-fills the destination
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, uint32_t src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}
// predicated form (no branch around the copy)
__device__ __forceinline__ void cp_async16_pred(uint32_t dst, const void* src, uint32_t src_bytes, bool on) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %3, 0;\n\t"
        "@p cp.async.cg.shared.global [%0], [%1], 16, %2;\n\t}" ::"r"(dst),
        "l"(src), "r"(src_bytes), "r"(static_cast<uint32_t>(on))
        : "memory");
}
__device__ __forceinline__ void cp_async_arrive_noinc(uint64_t* bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int c0, int c1) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(map),
                 "r"(smem_u32(src)), "r"(c0), "r"(c1)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void named_bar_sync(int id, int threads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

template <bool TF>
__device__ __forceinline__ void mma_sp(uint32_t d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc,
                                       uint32_t emeta) {
    if (TF)
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.sp.cta_group::1.kind::tf32 [%0], %1, %2, [%5], %3, p;\n\t}" ::"r"(d),
            "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc), "r"(emeta)
            : "memory");
    else
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.sp.cta_group::1.kind::f16 [%0], %1, %2, [%5], %3, p;\n\t}" ::"r"(d),
            "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc), "r"(emeta)
            : "memory");
}

__device__ __forceinline__ void tmem_cp_128x128b(uint32_t taddr, uint64_t sdesc) {
    asm volatile("tcgen05.cp.cta_group::1.128x128b [%0], %1;" ::"r"(taddr), "l"(sdesc) : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr)
        : "memory");
}

__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void red_release_add(int* p, int v) {
    asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

}  // namespace tcs
}  // namespace nm
