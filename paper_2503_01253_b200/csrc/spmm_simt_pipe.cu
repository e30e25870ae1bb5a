// spmm_simt_pipe.cu -- fp32 CUDA-core N:M SpMM, deep-pipelined variant (sm_100a).
//
// Same arithmetic as spmm_simt.cu (the paper's fp32 semantics; register
// outer products of Listing 2 / Eq. 6 with 8x8 thread tiles) with a B200 data
// path built for the high-sparsity regime, where a panel carries little FFMA
// work per byte loaded:
//   * one 128 x 256 output tile per CTA, 512 threads (16 warps of 64 x 32), one CTA
//     per SM, so the shared-memory budget buys pipeline depth instead of a second CTA;
//   * an S-stage ring (S = 3 at 50 %, up to 6 at 87.5 %) of {A^T panel (TMA, BK k-rows
//     x 128 m), B' panel (TMA), prepacked index table (bulk copy)} with full/empty
//     mbarriers: no __syncthreads in the k loop, panels land S-1 ahead;
//   * the index table of each (column tile, panel) -- the byte offset of the A^T row
//     every (compressed row u, column group) gathers -- is built once per call by
//     build_simt_table_kernel (the paper's offline index preprocessing slot,
//     P:416-419), so the k loop does no index arithmetic beyond one LDS.U16.
// A^T comes from transpose_kernel (spmm_simt.cu), row pitch padded to 128.
#include "common.cuh"

namespace nm {

__global__ void transpose_kernel(const float* __restrict__ A, float* __restrict__ AT, int m, int k, int ld);

namespace simt3 {

constexpr int BM = 128, BN = 256, BK = 64, BKW = 32, THREADS = 512, WARPS = 16;
constexpr int A_BYTES = BK * BM * 4;  // 32 KB
constexpr int MAX_STAGES = 6;
constexpr int SMEM_LIMIT = 227 * 1024;

struct Params {
    const uint16_t* tbl;  // [n tiles][npanels][tbl_elems] A^T-row byte offsets
    float* C;
    int m, n, k, N, M, L;
    int q, bk, bkw, npanels;
    int slots, tbl_elems, tbl_bytes, stage_bytes, stages;
};

// SL: row stride of the index table (column groups a 256-wide tile can touch + 1);
// compile-time so the inner loop's table address is a shift-add.  TWO: L < 32.
template <int SL, bool TWO>
__global__ void __launch_bounds__(THREADS, 1)
    spmm_simt_pipe_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                          const Params p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + p.stages * p.stage_bytes);
    uint64_t* empty = full + MAX_STAGES;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp & 1, wn = warp >> 1;
    const int t_m = lane & 7, t_n = lane >> 3;
    const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
    const int g_first = n0 / p.L;
    const int nslots = min((n0 + BN - 1) / p.L, p.q - 1) - g_first + 1;
    const int b_bytes = p.bkw * BN * 4;
    const uint32_t tx = static_cast<uint32_t>(A_BYTES + b_bytes + p.tbl_bytes);
    const uint16_t* tsrc = p.tbl + static_cast<int64_t>(blockIdx.x) * p.npanels * p.tbl_elems;

    if (tid == 0) {
        tma_prefetch_desc(&tmA);
        tma_prefetch_desc(&tmB);
        for (int s = 0; s < p.stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], WARPS);
        }
        fence_mbar_init();
    }
    __syncthreads();

    auto issue = [&](int panel) {  // thread 0
        const int s = panel % p.stages;
        uint8_t* st = smem + s * p.stage_bytes;
        mbar_arrive_expect_tx(&full[s], tx);
        tma_load_2d(st, &tmA, &full[s], m0, panel * p.bk);
        tma_load_2d(st + A_BYTES, &tmB, &full[s], n0, panel * p.bkw);
        bulk_load(st + A_BYTES + b_bytes, tsrc + static_cast<int64_t>(panel) * p.tbl_elems, p.tbl_bytes, &full[s]);
    };
    if (tid == 0)
        for (int j = 0; j < p.stages && j < p.npanels; ++j) issue(j);

    const int col0 = wn * 32 + 4 * t_n;  // chunk 0 (chunk 1 at col0 + 16), tile-relative
    const int slot0 = min((n0 + col0) / p.L - g_first, nslots - 1);
    const int slot1 = min((n0 + col0 + 16) / p.L - g_first, nslots - 1);
    const int a_row = (wm * 64 + 4 * t_m) * 4;
    const int wtot = (p.k / p.M) * p.N;

    float acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;

    for (int panel = 0; panel < p.npanels; ++panel) {
        const int s = panel % p.stages;
        mbar_wait(&full[s], (panel / p.stages) & 1);
        const uint8_t* st = smem + s * p.stage_bytes;
        const uint8_t* aS = st + a_row;
        const float* bS = reinterpret_cast<const float*>(st + A_BYTES) + col0;
        const uint16_t* kS = reinterpret_cast<const uint16_t*>(st + A_BYTES + b_bytes);
        const int bkw = min(p.bkw, wtot - panel * p.bkw);

        float a0[8], a1[8];
#pragma unroll 2
        for (int u = 0; u < bkw; ++u) {
            const uint16_t* krow = kS + u * SL;
            const uint8_t* ap0 = aS + krow[slot0];
            const float4 b0 = *reinterpret_cast<const float4*>(bS + u * BN);
            const float4 b1 = *reinterpret_cast<const float4*>(bS + u * BN + 16);
            {
                const float4 x0 = *reinterpret_cast<const float4*>(ap0);
                const float4 x1 = *reinterpret_cast<const float4*>(ap0 + 128);
                a0[0] = x0.x, a0[1] = x0.y, a0[2] = x0.z, a0[3] = x0.w;
                a0[4] = x1.x, a0[5] = x1.y, a0[6] = x1.z, a0[7] = x1.w;
            }
            if (TWO) {
                const uint8_t* ap1 = aS + krow[slot1];
                const float4 x0 = *reinterpret_cast<const float4*>(ap1);
                const float4 x1 = *reinterpret_cast<const float4*>(ap1 + 128);
                a1[0] = x0.x, a1[1] = x0.y, a1[2] = x0.z, a1[3] = x0.w;
                a1[4] = x1.x, a1[5] = x1.y, a1[6] = x1.z, a1[7] = x1.w;
            } else {
#pragma unroll
                for (int i = 0; i < 8; ++i) a1[i] = a0[i];
            }
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                acc[i][0] = fmaf(a0[i], b0.x, acc[i][0]);
                acc[i][1] = fmaf(a0[i], b0.y, acc[i][1]);
                acc[i][2] = fmaf(a0[i], b0.z, acc[i][2]);
                acc[i][3] = fmaf(a0[i], b0.w, acc[i][3]);
                acc[i][4] = fmaf(a1[i], b1.x, acc[i][4]);
                acc[i][5] = fmaf(a1[i], b1.y, acc[i][5]);
                acc[i][6] = fmaf(a1[i], b1.z, acc[i][6]);
                acc[i][7] = fmaf(a1[i], b1.w, acc[i][7]);
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        // producer: refill this stage with panel + stages once all 16 warps released it
        if (tid == 0 && panel + p.stages < p.npanels) {
            mbar_wait(&empty[s], (panel / p.stages) & 1);
            issue(panel + p.stages);
        }
    }

    const int gc0 = n0 + col0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int row = m0 + wm * 64 + (i & 3) + 4 * t_m + 32 * (i >> 2);
        if (row >= p.m) continue;
        float* crow = p.C + static_cast<int64_t>(row) * p.n;
        if (gc0 < p.n) *reinterpret_cast<float4*>(crow + gc0) = make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
        if (gc0 + 16 < p.n)
            *reinterpret_cast<float4*>(crow + gc0 + 16) = make_float4(acc[i][4], acc[i][5], acc[i][6], acc[i][7]);
    }
}

// Index preprocessing: entry (u, slot) of (column tile, panel) = byte
// offset in the A^T panel of dense column kabs(u, group) = (u / N) * M + D[u0 + u][g].
__global__ void build_simt_table_kernel(const uint8_t* __restrict__ D, uint16_t* __restrict__ tbl, int q, int N, int M,
                                        int L, int bkw, int npanels, int slots, int tbl_elems, int wtot) {
    const int panel = blockIdx.x, tile = blockIdx.y;
    const int g_first = tile * BN / L;
    uint16_t* t = tbl + (static_cast<int64_t>(tile) * npanels + panel) * tbl_elems;
    const int u0 = panel * bkw;
    for (int e = threadIdx.x; e < tbl_elems; e += blockDim.x) {
        const int u = e / slots, sl = e - u * slots;
        const int g = g_first + sl;
        int v = 0;
        if (u < bkw && u0 + u < wtot && g < q) v = ((u / N) * M + D[static_cast<int64_t>(u0 + u) * q + g]) * (BM * 4);
        t[e] = static_cast<uint16_t>(v);
    }
}

}  // namespace simt3

template <int SL, bool TWO>
static nm_status launch_pipe(const CUtensorMap& tmA, const CUtensorMap& tmB, const simt3::Params& p, dim3 grid, int smem,
                             cudaStream_t s) {
    // set per call (an ablation-only path; the attribute is per device and smem varies per shape)
    NM_CUDA_TRY(cudaFuncSetAttribute(simt3::spmm_simt_pipe_kernel<SL, TWO>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     smem));
    prof_begin(s);
    simt3::spmm_simt_pipe_kernel<SL, TWO><<<grid, simt3::THREADS, smem, s>>>(tmA, tmB, p);
    prof_end(s);
    note_launch();
    NM_LAUNCH_CHECK("spmm_simt_pipe_kernel");
    return NM_OK;
}

bool simt_pipe_applicable(int64_t m, int64_t n, int64_t k, int N, int M, int L) {
    return L % 4 == 0 && M <= simt3::BK && N <= simt3::BKW && k % 4 == 0 && n % 4 == 0 && m % 4 == 0 &&
           m < (1ll << 31) && n < (1ll << 31) && k < (1ll << 31);
}

nm_status simt_pipe_launch(const float* A, const float* Bv, const uint8_t* D, float* C, int64_t m, int64_t n, int64_t k,
                           int N, int M, int L, cudaStream_t s) {
    using namespace simt3;
    Params p{};
    p.C = C;
    p.m = static_cast<int>(m);
    p.n = static_cast<int>(n);
    p.k = static_cast<int>(k);
    p.N = N;
    p.M = M;
    p.L = L;
    p.q = static_cast<int>(n / L);
    int wp = BK / M;
    wp = wp < BKW / N ? wp : BKW / N;
    if (wp < 1) wp = 1;
    p.bk = wp * M;
    p.bkw = wp * N;
    const int windows = static_cast<int>(k / M);
    p.npanels = (windows + wp - 1) / wp;
    p.slots = L >= 32 ? 9 : L >= 16 ? 17 : L >= 8 ? 33 : 65;  // >= ceil(BN / L) + 1 groups per tile
    p.tbl_elems = (p.bkw * p.slots + 7) / 8 * 8;  // 16-byte multiple
    p.tbl_bytes = p.tbl_elems * 2;
    p.stage_bytes = (A_BYTES + p.bkw * BN * 4 + p.tbl_bytes + 1023) / 1024 * 1024;
    p.stages = (SMEM_LIMIT - 1024 - 2 * MAX_STAGES * 8) / p.stage_bytes;
    p.stages = p.stages > MAX_STAGES ? MAX_STAGES : p.stages;
    if (p.stages < 2) return fail(NM_ERR_UNSUPPORTED, "simt pipe: shared memory too small");
    const int smem = p.stages * p.stage_bytes + 2 * MAX_STAGES * 8 + 1024;
    const int64_t w = k / M * N;
    const int at_ld = static_cast<int>(ceil_div(m, BM) * BM);
    const int ntiles_n = static_cast<int>(ceil_div(n, BN));

    float* AT = nullptr;
    uint16_t* tbl = nullptr;
    nm_status st = scratch_alloc(reinterpret_cast<void**>(&AT), static_cast<size_t>(k) * at_ld * sizeof(float), s);
    if (st) return st;
    st = scratch_alloc(reinterpret_cast<void**>(&tbl), static_cast<size_t>(ntiles_n) * p.npanels * p.tbl_bytes, s);
    if (st) return st;
    const dim3 tg(static_cast<unsigned>(ceil_div(k, 64)), static_cast<unsigned>(ceil_div(at_ld, 64)));
    transpose_kernel<<<tg, 256, 0, s>>>(A, AT, static_cast<int>(m), static_cast<int>(k), at_ld);
    note_launch();
    NM_LAUNCH_CHECK("transpose_kernel");
    build_simt_table_kernel<<<dim3(p.npanels, ntiles_n), 256, 0, s>>>(D, tbl, p.q, N, M, L, p.bkw, p.npanels, p.slots,
                                                                       p.tbl_elems, static_cast<int>(w));
    note_launch();
    NM_LAUNCH_CHECK("build_simt_table_kernel");
    p.tbl = tbl;

    CUtensorMap tmA, tmB;
    st = make_tma_2d(&tmA, AT, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, k, at_ld, p.bk, BM, 0);
    if (!st) st = make_tma_2d(&tmB, Bv, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, w, n, p.bkw, BN, 0);
    if (!st) {
        const dim3 grid(static_cast<unsigned>(ntiles_n), static_cast<unsigned>(ceil_div(m, BM)));
        switch (p.slots) {
            case 9: st = launch_pipe<9, false>(tmA, tmB, p, grid, smem, s); break;
            case 17: st = launch_pipe<17, true>(tmA, tmB, p, grid, smem, s); break;
            case 33: st = launch_pipe<33, true>(tmA, tmB, p, grid, smem, s); break;
            default: st = launch_pipe<65, true>(tmA, tmB, p, grid, smem, s); break;
        }
    }
    cudaError_t e1 = cudaFreeAsync(tbl, s), e2 = cudaFreeAsync(AT, s);
    if (st == NM_OK && e1 != cudaSuccess) st = cuda_fail(e1, "cudaFreeAsync");
    if (st == NM_OK && e2 != cudaSuccess) st = cuda_fail(e2, "cudaFreeAsync");
    return st;
}

}  // namespace nm
