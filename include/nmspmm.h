/*
 * nmspmm.h -- C ABI of libnmspmm.so: B200-native (sm_100a) vector-wise N:M
 * sparse matrix multiplication, after NM-SpMM (arXiv 2503.01253).
 *
 * Citations: "P:<line>" = PAPER.md line (+ section / equation), "S:<line>" =
 * SPEC.md line; readings Rn are listed in DESIGN.md "Readings of the paper".
 *
 * Notation (Sec. II-A): C (m x n) = A (m x k) . B~ (k x n), where B~
 * is B pruned vector-wise N:M along k: in every window of M consecutive
 * length-L row vectors of one column group, N are kept.  Storage:
 *   B' ("values") : w x n, w = k*N/M, row u = the (u mod N)-th kept vector of
 *                   window floor(u/N), ascending offset (R7);
 *   D  ("idx")    : w x q uint8, q = n/L, offset of that vector in its window.
 * The product is Eq. 1 with readings R1-R4 (window base
 * floor(u/N)*M, sum u = 0..w-1, floor(j/L), no M/N prefactor):
 *   C[i][j] = sum_{u=0}^{w-1} A[i][floor(u/N)*M + D[u][floor(j/L)]] * B'[u][j].
 *
 * Conventions for every entry point:
 *  - all matrices are row-major and contiguous; every data pointer is a
 *    DEVICE pointer owned by the caller (the library keeps no pointer after
 *    return and allocates no persistent memory);
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default
 *    stream); calls are stream-ordered and asynchronous unless stated;
 *  - argument errors are returned synchronously, before any launch; device
 *    faults surface at the next synchronisation (CUDA semantics);
 *  - no exceptions or aborts cross the ABI; nm_last_error() gives a
 *    thread-local message for the last non-OK status of the calling thread;
 *  - there is no CPU fallback: without a CUDA device every compute entry
 *    point returns NM_ERR_CUDA.
 */
#ifndef NMSPMM_H_
#define NMSPMM_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    NM_OK = 0,
    NM_ERR_INVALID_CONFIG = 1,  /* !(1 <= N <= M <= 256) or L < 1 (uint8 D, R8)        */
    NM_ERR_SHAPE = 2,           /* k % M, n % L, negative dims (caller pads, R9)            */
    NM_ERR_ALIGNMENT = 3,       /* a pointer the chosen kernel needs 16-B aligned is not         */
    NM_ERR_NONFINITE = 4,       /* NaN in B during compress (score undefined, R6)                 */
    NM_ERR_UNSUPPORTED = 5,     /* dtype / math / shape combination without a kernel              */
    NM_ERR_INVALID_INDICES = 6, /* nm_validate found an entry >= M or not strictly increasing      */
    NM_ERR_CUDA = 7,            /* CUDA runtime error (message in nm_last_error)                  */
    NM_ERR_NULL = 8             /* a required pointer is NULL                                      */
} nm_status;

typedef enum { NM_F32 = 0, NM_BF16 = 1 } nm_dtype;

typedef enum {
    NM_MATH_AUTO = 0,     /* selector decides (nm_plan_query)                                 */
    NM_MATH_F32_SIMT = 1, /* fp32 FFMA on CUDA cores: the paper's fp32 semantics     */
    NM_MATH_TF32_TC = 2,  /* tcgen05 kind::tf32, fp32 accumulate in TMEM (R11)                */
    NM_MATH_BF16_TC = 3   /* tcgen05 kind::f16 (bf16 operands), fp32 accumulate in TMEM      */
} nm_math;

/* Selector output (P:150 blocking parameters re-cut for B200). */
typedef struct {
    int32_t math;         /* nm_math actually used                                             */
    int32_t kernel;       /* kernel id; 0 = generic                             */
    int32_t bm, bn, bk;   /* CTA tile: rows of A, columns of C, dense k per panel (mult. of M)  */
    int32_t bkw;          /* compressed rows per panel = bk*N/M                                 */
    int32_t stages;       /* smem pipeline depth                                               */
    int32_t grid;         /* CTAs launched                                                     */
    int32_t threads;      /* threads per CTA                                                   */
    int32_t smem_bytes;   /* dynamic shared memory per CTA                                     */
    double flops;         /* 2*m*n*w (kept MACs only)                                   */
    double bytes;         /* algorithmic HBM bytes: A + B' + D + C                             */
    double t_compute_us;  /* roofline estimates from the peaks passed in (or built-in nominal)   */
    double t_memory_us;
    int32_t bound;        /* 0 = compute (FMA or tensor), 1 = HBM                               */
    int32_t split;        /* k-range parts per tile of the split tiles (the partial last wave, or  */
                          /* every tile of a sub-wave grid); 1 = none                           */
    int32_t split_tiles;  /* tiles run as `split` CTAs each                                    */
    double waves;         /* CTAs launched / resident CTA slots (selector's wave model)          */
} nm_plan;

/* Library version string, e.g. "nmspmm 0.1 sm_100a". */
const char* nm_version(void);

/* Thread-local message for the last non-OK status returned on this thread. */
const char* nm_last_error(void);

/* Checks 1 <= N <= M <= 256 and L >= 1.  Host only. */
nm_status nm_check_config(int N, int M, int L);

/*
 * nm_compress -- magnitude pruning + compression (readings R6, R7, R10, R11).
 *   B      : k x n, dtype b_dt (NM_F32 or NM_BF16), device.
 *   values : w x n, dtype v_dt, device, written.  v_dt == b_dt is a bit copy;
 *            NM_F32 -> NM_BF16 rounds to nearest even; NM_BF16 -> NM_F32 widens.
 *   idx    : w x q uint8, device, written.
 * For every window t and group g: score_r = sum_{c<L} x^2 (x = B[t*M+r][g*L+c]),
 * formed in fp64 with products and sums rounded in ascending c, no FMA; the N
 * largest scores are kept, ties to the smaller offset; offsets written
 * ascending.  Bit-exact with the CPU oracle.
 * SYNCHRONOUS: returns after the work on `stream` has finished, because a NaN
 * in B is reported as NM_ERR_NONFINITE (outputs are then unspecified).
 */
nm_status nm_compress(const void* B, nm_dtype b_dt, int64_t k, int64_t n, int N, int M, int L,
                      void* values, nm_dtype v_dt, uint8_t* idx, void* stream);

/*
 * nm_decompress -- B~ (k x n, dtype v_dt): +0.0 everywhere except
 * B~[t*M + idx[t*N+s][g]][g*L+c] = values[t*N+s][g*L+c].
 * Entries of idx >= M are skipped (use nm_validate first).  Asynchronous.
 */
nm_status nm_decompress(const void* values, nm_dtype v_dt, const uint8_t* idx, int64_t k, int64_t n,
                        int N, int M, int L, void* B_out, void* stream);

/*
 * nm_validate -- S:93-101.  *first_bad_host (host pointer) receives -1 if every
 * entry is < M and strictly increasing inside its window, else the smallest
 * row-major flat index u*q+g of a violating entry; the return value is then
 * NM_ERR_INVALID_INDICES.  SYNCHRONOUS on `stream`.
 */
nm_status nm_validate(const uint8_t* idx, int64_t k, int64_t n, int N, int M, int L,
                      int64_t* first_bad_host, void* stream);

/*
 * nm_spmm -- C = A . decompress(values, idx) (Eq. 1 with R1-R4).
 *   A      : m x k, dtype ab_dt, device;   values : w x n, dtype ab_dt;
 *   idx    : w x q uint8 (must be valid; not re-checked on the hot path);
 *   C      : m x n, dtype c_dt, device, overwritten.
 *   ab_dt / c_dt / math:  NM_F32 + NM_MATH_F32_SIMT   -> fp32 FFMA, c_dt NM_F32
 *                         NM_F32 + NM_MATH_TF32_TC    -> opt-in: fp32 operands on the tf32 sparse tensor
 *                                                        cores (A read at tf32 precision, B' rounded to
 *                                                        tf32 offline, fp32 accumulate, c_dt NM_F32) by the
 *                                                        slot kernel with 1:2 slot pairs; needs L in
 *                                                        {16,32,64,128}, k % 8 == 0, A 16-B and C 4-B
 *                                                        aligned, else NM_ERR_UNSUPPORTED.  AUTO on fp32
 *                                                        never picks it (it changes the numerics).
 *                         NM_BF16 + NM_MATH_BF16_TC   -> bf16 on the tensor cores, fp32 accumulate,
 *                                                        c_dt NM_BF16 (RNE) or NM_F32: the sparse-
 *                                                        tensor-core kernel (tcgen05.mma.sp over the
 *                                                        offline slot packing) when L is 16/32/64/128,
 *                                                        k % 8 == 0, A 16-B and C 4-B aligned; else
 *                                                        the fp32 SIMT kernel on exact fp32 copies of
 *                                                        A and values (scratch from the library pool;
 *                                                        C rounded to bf16 after the fp32 sum; needs
 *                                                        the SIMT shape rules below and A / values
 *                                                        16-B aligned, else NM_ERR_ALIGNMENT); else
 *                                                        the generic kernel (one thread per element)
 *                         NM_MATH_AUTO                -> selector (nm_plan_query)
 * bf16 / tf32 without a prepack re-pack the weight on every call (ms); use
 * nm_prepack (nm_prepack_ex for tf32) / nm_spmm_prepacked for repeated products with one weight.
 * No atomics on data: where a tile's k range is split over CTAs (grids below one wave, the
 * partial last wave of the slot kernels) the partials are added in a fixed order, so results
 * are bit-reproducible run to run for a given shape (R13).
 * m == 0 or n == 0 is a no-op returning NM_OK.  Asynchronous.
 */
nm_status nm_spmm(const void* A, const void* values, const uint8_t* idx, void* C, int64_t m, int64_t n,
                  int64_t k, int N, int M, int L, nm_dtype ab_dt, nm_dtype c_dt, nm_math math,
                  void* stream);

/*
 * nm_spmm_scaled -- Eq. 1 as printed: C = alpha . A . decompress(values, idx), the
 * paper's approximation C' of the unpruned product being alpha = M/N (R1 reads the product
 * path unscaled: nm_spmm == nm_spmm_scaled with alpha = 1).  alpha is applied in fp32 to the
 * fp32 accumulators inside the epilogue of the SIMT and sparse-tensor-core kernels (after any
 * split-k / tail-split addition, before the bf16 rounding); the generic kernel is followed by
 * one in-place scaling pass over C (for a bf16
 * C: a second rounding, exact when alpha is a power of two).  Otherwise as nm_spmm.
 */
nm_status nm_spmm_scaled(const void* A, const void* values, const uint8_t* idx, void* C, int64_t m, int64_t n,
                         int64_t k, int N, int M, int L, nm_dtype ab_dt, nm_dtype c_dt, nm_math math, float alpha,
                         void* stream);

/*
 * nm_spmm_host -- the same product with HOST operands (end-to-end path):
 * copies A, values, idx from host memory (pinned for async copies) into the
 * caller's device workspace, runs nm_spmm, copies C back to C_host.  On the fp32
 * SIMT path and the bf16 / tf32 slot kernels with m >= 1024 the rows of A / C go in
 * nch + 1 chunks sized 1 : 2 : .. : 2 : 1 (nch = 4; 8 on the fp32 SIMT path once m >= 2048;
 * NM_HOST_CHUNKS=1..8 overrides) so that the copies of one chunk overlap the SpMM of another (two
 * library-created copy streams, destroyed before return; the slot kernels prepack the
 * weight once per call into pooled scratch first); other paths copy, compute and copy
 * back in sequence.
 * Workspace `dev_ws` must hold nm_spmm_host_ws_bytes(...) bytes (device).
 * SYNCHRONOUS (returns after C_host is written).
 */
int64_t nm_spmm_host_ws_bytes(int64_t m, int64_t n, int64_t k, int N, int M, int L, nm_dtype ab_dt,
                              nm_dtype c_dt);
nm_status nm_spmm_host(const void* A_host, const void* values_host, const uint8_t* idx_host,
                       void* C_host, int64_t m, int64_t n, int64_t k, int N, int M, int L,
                       nm_dtype ab_dt, nm_dtype c_dt, nm_math math, void* dev_ws, void* stream);

/*
 * nm_plan_query -- the selector's decision for a problem (S9 of SURVEY 8(a)),
 * without launching.  peak_flops / peak_hbm_bytes_per_s: the roofline
 * denominators (<= 0 selects built-in nominal B200 numbers).  Host only;
 * needs a device only to read the SM count (148 assumed if none).
 */
nm_status nm_plan_query(int64_t m, int64_t n, int64_t k, int N, int M, int L, nm_dtype ab_dt,
                        nm_math math, double peak_flops, double peak_hbm_bytes_per_s, nm_plan* out);

/*
 * nm_unshard_columns -- multi-GPU assembly.  The q = n/L column
 * groups are split over G ranks, rank r owning groups [floor(r*q/G),
 * floor((r+1)*q/G)); every rank's slice is padded to nr >= L*ceil(q/G)
 * columns.  src is the all-gathered [G][m][nr] buffer (device), dst the
 * m x n row-major result (device); padding columns are dropped.
 * elem_bytes is 2 (bf16) or 4 (fp32).  Asynchronous.
 */
nm_status nm_unshard_columns(const void* src, void* dst, int64_t G, int64_t m, int64_t nr, int64_t n, int L,
                             int elem_bytes, void* stream);

/*
 * Weight prepack -- the paper's offline PreProcessing step (Listing 3, P:470-475:
 * queryColInfo / reoderingIdx / transformLayout), done once per weight.  For the
 * sparse-tensor-core slot kernels (bf16: kind 2; tf32: kind 3) it computes, from B' and D
 * alone: per column tile of 128 H output columns the union of the k rows its groups keep (the
 * paper's col_info) packed into 2:4-compatible slot quads (bf16) or 1:2 pairs (tf32),
 * the slot list (row of A^T per slot) and the exact shared-memory images of the compressed
 * weights + sparse-MMA metadata per 64- (bf16) / 32-slot (tf32) stage.  The buffer is compact:
 *   [header 256 B | per tile {stages, first slot, image offset, image size} | slot lists |
 *    stage images (even stages: H x (8 KB weights + 2 KB metadata of the stage pair), odd: H x 8 KB)]
 * fp32 weights on the SIMT kernel with 128 % L == 0 get kind 4: the index matrix bit-packed and
 * tile-major (nm_index_pack below), read by the kernel instead of D.
 * Other weights keep using `values` / `idx` directly (kind 0, no buffer).
 *   nm_prepack_bytes[_ex]: a data-independent UPPER BOUND of the buffer (0 for kind 0; -1 on bad
 *                      args).  Host only.
 *   nm_prepack_size  : the EXACT buffer size for this weight (*bytes; 0 for kind 0): runs the slot
 *                      packing on `stream` and SYNCHRONIZES it.  Device pointers values / idx.
 *   nm_prepack[_ex]  : fills `buf` (device, caller-owned, buf_bytes >= nm_prepack_size; a buffer
 *                      below the bound makes the call check the exact size, synchronizing) and the
 *                      host descriptor `*out`; `values` and `idx` must stay alive and unmodified
 *                      while `*out` is used.  Asynchronous on `stream` otherwise.
 *   nm_spmm_prepacked: C (m x n, c_dt) = A (m x k) . decompress(values, idx), same semantics and
 *                      parity as nm_spmm (A's dtype must be the weight's).  Asynchronous.
 */
typedef struct {
    int32_t magic;   /* 0x4B504D4E ("NMPK") once filled */
    int32_t kind;    /* 0 = plain (values/idx used directly),
                        2 = sparse-tensor-core slot prepack, bf16 (whole buffer at `bperm`),
                        3 = the same for tf32 (fp32 weights, nm_prepack_ex with NM_MATH_TF32_TC),
                        4 = fp32 SIMT weight with bit-packed tile-major indices (nm_index_pack
                            words at `tbl`; 128 % L == 0) */
    int32_t dtype, N, M, L;
    int64_t n, k;
    int32_t bn;      /* kind 2/3: output columns per tile (128 H) */
    int32_t wp, bk, bkw, bkw_pad;  /* reserved (0) */
    int32_t npanels; /* kind 2/3: column tiles */
    const void* values;
    const uint8_t* idx;
    void* perm;      /* reserved (NULL) */
    void* tbl;       /* kind 4: the packed index words */
    void* bperm;     /* kind 2/3: the prepacked buffer */
} nm_prepacked;

int64_t nm_prepack_bytes(int64_t n, int64_t k, int N, int M, int L, nm_dtype dt);
nm_status nm_prepack(const void* values, const uint8_t* idx, int64_t n, int64_t k, int N, int M, int L, nm_dtype dt,
                     void* buf, int64_t buf_bytes, nm_prepacked* out, void* stream);
nm_status nm_spmm_prepacked(const void* A, const nm_prepacked* w, void* C, int64_t m, nm_dtype c_dt, void* stream);

/* nm_spmm_at / nm_spmm_prepacked_at -- the same product with A supplied TRANSPOSED (feature-major
 * activations): At is k x lda row-major, At[kk * lda + i] = A[i][kk], lda >= m (the columns
 * m .. lda-1 are never used in C).  Both kernels consume A^T internally (the SIMT kernel stages
 * A^T panels, the slot kernels gather rows of A^T), so this form skips the per-call transpose
 * (Eq. 1 unchanged; results identical to nm_spmm / nm_spmm_prepacked bit for bit).
 *   At : device, 16-B aligned, lda * element size a multiple of 16 B; C : m x n row-major.
 *   Paths: fp32 -> the SIMT kernel (staged A^T mode); bf16 / tf32 -> the slot kernels (padding
 *   slots are zero-filled by the gather, no zero row needed).  Other selections (the generic
 *   kernel, bf16 on the SIMT kernel) return NM_ERR_UNSUPPORTED; misalignment NM_ERR_ALIGNMENT;
 *   lda < m NM_ERR_SHAPE.  Asynchronous on `stream`. */
nm_status nm_spmm_at(const void* At, int64_t lda, const void* values, const uint8_t* idx, void* C, int64_t m, int64_t n,
                     int64_t k, int N, int M, int L, nm_dtype ab_dt, nm_dtype c_dt, nm_math math, void* stream);
nm_status nm_spmm_prepacked_at(const void* At, int64_t lda, const nm_prepacked* w, void* C, int64_t m, nm_dtype c_dt,
                               void* stream);
/* The same with the math the prepacked weight will run with: nm_prepack == nm_prepack_ex(...,
 * NM_MATH_AUTO, ...).  dt NM_F32 + NM_MATH_TF32_TC gives kind 3 (tf32 slot images, 1:2 slot
 * pairs, values rounded to tf32) when the tf32 path applies to the weight's shape, else kind 0;
 * nm_spmm_prepacked on kind 3 runs the tf32 kernel (c_dt must be NM_F32) and reports
 * NM_ERR_UNSUPPORTED where nm_spmm with NM_MATH_TF32_TC would. */
int64_t nm_prepack_bytes_ex(int64_t n, int64_t k, int N, int M, int L, nm_dtype dt, nm_math math);
nm_status nm_prepack_size(const void* values, const uint8_t* idx, int64_t n, int64_t k, int N, int M, int L,
                          nm_dtype dt, nm_math math, int64_t* bytes, void* stream);
nm_status nm_prepack_ex(const void* values, const uint8_t* idx, int64_t n, int64_t k, int N, int M, int L, nm_dtype dt,
                        nm_math math, void* buf, int64_t buf_bytes, nm_prepacked* out, void* stream);
/* The same for an expected token count m_hint (> 0; 0 = unknown, the calls above): the slot
 * prepacks (kinds 2 / 3) then choose their column halves H as nm_spmm does for that m -- H = 1 when
 * H = 2 would leave the grid under two waves (small m, the column shards of a multi-GPU layer;
 * DESIGN.md 6) -- so nm_spmm_prepacked on m tokens runs the tile nm_spmm would.  Any m may still be
 * passed to nm_spmm_prepacked.  The size and the fill must use the same m_hint. */
nm_status nm_prepack_size_m(const void* values, const uint8_t* idx, int64_t n, int64_t k, int N, int M, int L,
                            nm_dtype dt, nm_math math, int64_t m_hint, int64_t* bytes, void* stream);
nm_status nm_prepack_m(const void* values, const uint8_t* idx, int64_t n, int64_t k, int N, int M, int L, nm_dtype dt,
                       nm_math math, int64_t m_hint, void* buf, int64_t buf_bytes, nm_prepacked* out, void* stream);

/*
 * Bit-packed indices (an index needs only ceil(log2 M) bits) in the tile-major layout of
 * the paper's transformLayout (Listing 3: fewer global memory transactions): b =
 * max(1, ceil(log2 M)) bits per entry, e = floor(32 / b) entries per 32-bit word; the q column
 * groups are cut into tiles of T = 128 / L groups (needs 128 % L == 0; one SIMT CTA tile of 128
 * output columns); a tile's entries x = u*T + t (row u < w, group t < T) form Wt = ceil(w*T / e)
 * consecutive words, entry x in word tile*Wt + x / e at bit (x % e) * b (groups >= q and unused
 * bits are 0).  Bit-exact with the oracle's index_pack (R28).
 *   nm_index_packed_words : words of the packed form (-1 on bad args / 128 % L != 0).  Host only.
 *   nm_index_pack / unpack: D (w x q uint8, device) <-> words (device).  Asynchronous.
 */
int64_t nm_index_packed_words(int64_t k, int64_t n, int N, int M, int L);
nm_status nm_index_pack(const uint8_t* idx, int64_t k, int64_t n, int N, int M, int L, uint32_t* words, void* stream);
nm_status nm_index_unpack(const uint32_t* words, int64_t k, int64_t n, int N, int M, int L, uint8_t* idx,
                          void* stream);

/*
 * Fused multi-GPU exchange of the column-sharded layer.  Column j of C
 * depends only on A, B'[:, j], D[:, j / L] (Eq. 1), so rank r of G computes the columns
 * of its group shard and, instead of an all-gather + unshard pass, the SpMM epilogue stores
 * them straight into every rank's C buffer through peer mappings (NVLink); a flag barrier in
 * peer memory then orders the ranks, stream-ordered, no host synchronisation.
 *
 *   nm_ipc_get_handle : CUDA IPC handle (64 bytes, written to `handle`) of the allocation that
 *                       contains device pointer `dptr`, and dptr's byte offset in it.
 *   nm_ipc_open_handle: maps another process's handle; *dptr = its base + offset.  (A
 *                       process cannot open its own handle: use the local pointer.)
 *   nm_ipc_close      : unmaps (dptr, offset as returned by nm_ipc_open_handle).
 *   nm_spmm_peers     : C_p[i][col_off + j] = (A . decompress(values, idx))[i][j] for every p <
 *                       G, i < m, j < n_valid (the shard's unpadded columns; nr = its padded
 *                       width, values w x nr, idx w x nr/L); C_p are device pointers valid in
 *                       this process (own buffer or IPC-mapped peers), row pitch ldc floats.
 *                       fp32 operands on the SIMT kernel (16-B aligned, ldc, col_off and
 *                       n_valid multiples of 4), else NM_ERR_UNSUPPORTED / NM_ERR_SHAPE.
 *                       Asynchronous.
 *   nm_peer_barrier   : flag_peers[p] = rank p's int[G] flag array (mapped here); publishes
 *                       `epoch` in every rank's flags[rank] (system-scope release after the
 *                       stream's earlier work, i.e. after this rank's peer stores) and waits on
 *                       the stream until every rank has published `epoch` in ours.  Epochs
 *                       must increase by one per call on all ranks; a rank that never arrives
 *                       makes the kernel trap after NM_PEER_TIMEOUT_MS (environment, default
 *                       120000 ms of wall time) instead of hanging.  1 <= G <= 8.
 */
nm_status nm_ipc_get_handle(const void* dptr, void* handle, int64_t* offset);
nm_status nm_ipc_open_handle(const void* handle, int64_t offset, void** dptr);
nm_status nm_ipc_close(void* dptr, int64_t offset);
nm_status nm_spmm_peers(const void* A, const void* values, const uint8_t* idx, void* const* C_peers, int G,
                        int64_t ldc, int64_t col_off, int64_t n_valid, int64_t m, int64_t nr, int64_t k, int N,
                        int M, int L, void* stream);
nm_status nm_peer_barrier(void* const* flag_peers, int G, int rank, int epoch, void* stream);
/* The same for a prepacked shard (nm_prepack / nm_prepack_ex): kind 0 with fp32 values and an
 * fp32 C -> nm_spmm_peers (any other kind-0 weight: NM_ERR_UNSUPPORTED); kind 2 (bf16) / 3
 * (tf32, c_dt NM_F32) -> the sparse-tensor-core slot kernel with its direct-store epilogue
 * writing every C element to all G buffers (c_dt bf16 or fp32; C pointers, ldc and col_off 4-B
 * aligned, A 16-B aligned, k % 8 == 0; a bf16 C needs an even n_valid).  Asynchronous. */
nm_status nm_spmm_prepacked_peers(const void* A, const nm_prepacked* w, void* const* C_peers, int G, int64_t ldc,
                                  int64_t col_off, int64_t n_valid, int64_t m, nm_dtype c_dt, void* stream);

/*
 * NVLS multicast C ("an NVLS multicast epilogue (multimem.st into a symmetric-memory
 * C) so tiles land on all peers as they retire"; the assembly of the column-sharded layer, north
 * star).  A multicast object spans the G ranks' devices; each rank binds its own physical C buffer
 * to it and maps two views of it: the multicast address (a store through it reaches every bound
 * buffer, replicated by the NVSwitch) and the unicast address of its own replica.
 *   nm_mc_supported  : *supported = 1 iff the current device supports multicast objects and this
 *                      process can create one (a trial object; with one visible GPU of a multi-GPU
 *                      node the driver refuses: CUDA_ERROR_INVALID_VALUE).
 *   nm_mc_create     : rank 0 (or a single process): a multicast object of >= bytes per device for
 *                      num_devices devices (1..8); *mc = its handle, *mc_bytes = the size rounded up to
 *                      the recommended granularity (use it everywhere below).  Exportable as a fabric
 *                      handle when num_devices > 1.
 *   nm_mc_export / nm_mc_import : the 64-byte fabric handle of the object (rank 0 exports, the other
 *                      ranks import; the bytes travel over any channel, e.g. torch.distributed).
 *   nm_mc_add_device : add the current device (every rank, before any rank binds).
 *   nm_mc_bind_map   : allocate this device's buffer (mc_bytes), bind it, map *uc_ptr (this replica)
 *                      and *mc_ptr (the multicast view); *mem = the physical allocation's handle.
 *   nm_mc_free       : unmap, unbind and release everything nm_mc_* created here (synchronizes).
 *   nm_spmm_mc       : nm_spmm_peers with one destination, the multicast address: the SIMT kernel's
 *                      epilogue writes each float4 of its [m x n_valid] shard once with multimem.st
 *                      at C_mc[i][col_off + j] (row pitch ldc floats); every rank's replica receives
 *                      it.  Same geometry requirements as nm_spmm_peers.  Completion across ranks:
 *                      nm_peer_barrier.  Asynchronous.
 * Errors: NM_ERR_UNSUPPORTED without multicast support or driver entry points; NM_ERR_CUDA with the
 * driver's CUresult in nm_last_error().
 */
nm_status nm_mc_supported(int* supported);
nm_status nm_mc_create(int64_t bytes, int num_devices, uint64_t* mc, int64_t* mc_bytes);
nm_status nm_mc_export(uint64_t mc, void* fabric_handle);
nm_status nm_mc_import(const void* fabric_handle, uint64_t* mc);
nm_status nm_mc_add_device(uint64_t mc);
nm_status nm_mc_bind_map(uint64_t mc, int64_t mc_bytes, uint64_t* mem, void** uc_ptr, void** mc_ptr);
nm_status nm_mc_free(uint64_t mc, uint64_t mem, void* uc_ptr, void* mc_ptr, int64_t mc_bytes);
nm_status nm_spmm_mc(const void* A, const void* values, const uint8_t* idx, void* C_mc, int64_t ldc, int64_t col_off,
                     int64_t n_valid, int64_t m, int64_t nr, int64_t k, int N, int M, int L, void* stream);

/*
 * nm_profile_begin / nm_profile_end -- launch accounting for measurement
 * (bench.py).  Between the two calls the library counts every kernel it
 * launches and records a CUDA event pair on the launching stream around each
 * dominant SpMM kernel.  nm_profile_end synchronises on the last event and
 * returns the summed duration of those kernels (*kernel_ms, their number in
 * *kernel_count) and the total launch count (*launches); any pointer may be
 * NULL.  Process-wide state, not intended for concurrent profiling sessions.
 */
nm_status nm_profile_begin(void);
nm_status nm_profile_end(double* kernel_ms, int64_t* kernel_count, int64_t* launches);

#ifdef __cplusplus
}
#endif
#endif /* NMSPMM_H_ */
