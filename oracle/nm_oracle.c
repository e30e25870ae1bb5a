/*
 * nm_oracle.c -- plain, slow, obviously-correct CPU oracle for vector-wise
 * N:M sparse matrix multiplication (NM-SpMM, arXiv 2503.01253).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or helper with the CUDA path
 * (paper_2503_01253_b200/csrc); neither side includes the other.
 *
 * Citations: "P:<line>" = /root/reference/PAPER.md line, "S:<line>" =
 * SPEC.md line, plus the section / equation.  Readings of garbled or silent
 * passages are the numbered items of DESIGN.md "Readings" (R1..R22).
 *
 * Notation (Sec. II-A): C (m x n) = A (m x k) . B (k x n)   [R5];
 * B is pruned vector-wise N:M along k: in every window of M consecutive
 * length-L row vectors of one column group, N are kept.  B' (w x n) holds the
 * kept vectors, D (w x q) their offsets inside the window; w = k*N/M,
 * q = n/L (k % M == 0 and n % L == 0, the caller pads: P:94, R9).
 *
 * Precision: scores and products are formed in fp64 (every fp32 or bf16
 * square / product is exact in fp64); sums are sequential in the stated
 * order.  Build with -ffp-contract=off so no FMA contraction changes a sum.
 *
 * Pins: tests/test_oracle_pins.py (worked examples of S:69, S:79, S:90,
 * S:159; brute force C(M,N) search for M <= 8; closed forms; invariants).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define NMO_OK 0
#define NMO_ERR_INVALID_CONFIG 1
#define NMO_ERR_SHAPE 2
#define NMO_ERR_NONFINITE 4
#define NMO_ERR_INVALID_INDICES 6

/* ------------------------------------------------------------------ */
/* bf16 <-> fp32 (bf16 = upper 16 bits of an IEEE binary32)           */
/* ------------------------------------------------------------------ */
static float bf16_to_f32(uint16_t h) {
    uint32_t u = ((uint32_t)h) << 16;
    float f;
    memcpy(&f, &u, 4);
    return f;
}

/* Round-to-nearest-even fp32 -> bf16 (R11: bf16 values are RNE of the input). */
uint16_t nmo_f32_to_bf16_rne(float f) {
    uint32_t u;
    memcpy(&u, &f, 4);
    if ((u & 0x7F800000u) == 0x7F800000u && (u & 0x007FFFFFu) != 0u)
        return (uint16_t)((u >> 16) | 0x0040u); /* quiet NaN, keep sign */
    uint32_t lsb = (u >> 16) & 1u;
    u += 0x7FFFu + lsb;
    return (uint16_t)(u >> 16);
}

float nmo_bf16_to_f32(uint16_t h) { return bf16_to_f32(h); }

static double load_elem(const void* p, int is_bf16, int64_t i) {
    if (is_bf16) return (double)bf16_to_f32(((const uint16_t*)p)[i]);
    return (double)((const float*)p)[i];
}

/* ------------------------------------------------------------------ */
/* Configuration check: 1 <= N <= M <= 256, L >= 1 (uint8 D, R8). */
/* ------------------------------------------------------------------ */
int nmo_check_config(int N, int M, int L) {
    if (N < 1 || M < N || M > 256 || L < 1) return NMO_ERR_INVALID_CONFIG;
    return NMO_OK;
}

int nmo_check_shape(int64_t k, int64_t n, int N, int M, int L) {
    int s = nmo_check_config(N, M, L);
    if (s) return s;
    if (k < 0 || n < 0 || k % M != 0 || n % L != 0) return NMO_ERR_SHAPE; /* P:94, R9 */
    return NMO_OK;
}

/* ------------------------------------------------------------------ */
/* compress ("select N vectors from every M vector along k"):     */
/* For window t and column group g, score_r = sum_{c=0}^{L-1} x^2 with */
/* x = B[t*M + r][g*L + c], accumulated in fp64 in ascending c (R6).   */
/* Keep the N offsets of largest score; ties -> smaller offset (R6).   */
/* Kept offsets are written ascending (R7) into D[t*N + s][g] and the  */
/* kept vectors into B'[t*N + s][g*L .. g*L+L-1] (bit copy, or RNE to  */
/* bf16 when v_bf16 and the input is fp32, R11).                       */
/* A NaN anywhere in B -> NMO_ERR_NONFINITE (score undefined, R6).      */
/* ------------------------------------------------------------------ */
int nmo_compress(const void* B, int b_bf16, int64_t k, int64_t n, int N, int M, int L,
                 void* values, int v_bf16, uint8_t* D) {
    int s = nmo_check_shape(k, n, N, M, L);
    if (s) return s;
    for (int64_t i = 0; i < k * n; ++i)
        if (isnan(load_elem(B, b_bf16, i))) return NMO_ERR_NONFINITE;
    const int64_t windows = k / M, q = n / L;
    double* score = (double*)malloc(sizeof(double) * (size_t)M);
    int* order = (int*)malloc(sizeof(int) * (size_t)M);
    int* kept = (int*)malloc(sizeof(int) * (size_t)N);
    for (int64_t t = 0; t < windows; ++t) {
        for (int64_t g = 0; g < q; ++g) {
            /* 1. scores */
            for (int r = 0; r < M; ++r) {
                double acc = 0.0;
                for (int c = 0; c < L; ++c) {
                    double x = load_elem(B, b_bf16, (t * M + r) * n + g * L + c);
                    double sq = x * x;
                    acc = acc + sq;
                }
                score[r] = acc;
            }
            /* 2. order offsets by (score desc, offset asc): insertion sort */
            for (int r = 0; r < M; ++r) order[r] = r;
            for (int a = 1; a < M; ++a) {
                int cur = order[a];
                int b = a - 1;
                while (b >= 0 && (score[order[b]] < score[cur] ||
                                  (score[order[b]] == score[cur] && order[b] > cur))) {
                    order[b + 1] = order[b];
                    --b;
                }
                order[b + 1] = cur;
            }
            /* 3. first N, re-sorted ascending by offset */
            for (int j = 0; j < N; ++j) kept[j] = order[j];
            for (int a = 1; a < N; ++a) {
                int cur = kept[a];
                int b = a - 1;
                while (b >= 0 && kept[b] > cur) {
                    kept[b + 1] = kept[b];
                    --b;
                }
                kept[b + 1] = cur;
            }
            /* 4. write D and B' */
            for (int j = 0; j < N; ++j) {
                int64_t u = t * N + j;
                D[u * q + g] = (uint8_t)kept[j];
                for (int c = 0; c < L; ++c) {
                    int64_t src = (t * M + kept[j]) * n + g * L + c;
                    int64_t dst = u * n + g * L + c;
                    if (v_bf16) {
                        uint16_t h = b_bf16 ? ((const uint16_t*)B)[src]
                                            : nmo_f32_to_bf16_rne(((const float*)B)[src]);
                        ((uint16_t*)values)[dst] = h;
                    } else {
                        float f = b_bf16 ? bf16_to_f32(((const uint16_t*)B)[src])
                                         : ((const float*)B)[src];
                        ((float*)values)[dst] = f;
                    }
                }
            }
        }
    }
    free(score);
    free(order);
    free(kept);
    return NMO_OK;
}

/* ------------------------------------------------------------------ */
/* decompress (inverse of P:93): B~ = +0.0 everywhere, then   */
/* B~[t*M + D[t*N+s][g]][g*L + c] = B'[t*N+s][g*L + c].                */
/* Output has the dtype of the values.                                 */
/* ------------------------------------------------------------------ */
int nmo_decompress(const void* values, int v_bf16, const uint8_t* D, int64_t k, int64_t n,
                   int N, int M, int L, void* Bout) {
    int s = nmo_check_shape(k, n, N, M, L);
    if (s) return s;
    const int64_t w = k / M * N, q = n / L;
    size_t esz = v_bf16 ? 2 : 4;
    memset(Bout, 0, (size_t)(k * n) * esz);
    for (int64_t u = 0; u < w; ++u) {
        int64_t t = u / N;
        for (int64_t g = 0; g < q; ++g) {
            int d = D[u * q + g];
            if (d >= M) return NMO_ERR_INVALID_INDICES;
            for (int c = 0; c < L; ++c) {
                int64_t src = u * n + g * L + c;
                int64_t dst = (t * M + d) * n + g * L + c;
                if (v_bf16)
                    ((uint16_t*)Bout)[dst] = ((const uint16_t*)values)[src];
                else
                    ((float*)Bout)[dst] = ((const float*)values)[src];
            }
        }
    }
    return NMO_OK;
}

/* ------------------------------------------------------------------ */
/* validate: returns -1 if every entry is < M and strictly  */
/* increasing inside its window; else the first (row-major) flat index */
/* u*q + g of a violating entry.  Returns -2 on a bad configuration.   */
/* ------------------------------------------------------------------ */
int64_t nmo_validate(const uint8_t* D, int64_t k, int64_t n, int N, int M, int L) {
    if (nmo_check_shape(k, n, N, M, L)) return -2;
    const int64_t w = k / M * N, q = n / L;
    for (int64_t u = 0; u < w; ++u) {
        for (int64_t g = 0; g < q; ++g) {
            int d = D[u * q + g];
            if (d >= M) return u * q + g;
            if (u % N != 0 && D[(u - 1) * q + g] >= d) return u * q + g;
        }
    }
    return -1;
}

static int omp_threads(int nthreads) {
#ifdef _OPENMP
    return nthreads > 0 ? nthreads : omp_get_max_threads();
#else
    (void)nthreads;
    return 1;
#endif
}

int nmo_num_threads(int nthreads) { return omp_threads(nthreads); }

/* ------------------------------------------------------------------ */
/* O2: direct sparse loop, Eq. 1 corrected (R1-R4):           */
/*   C[i][j] = sum_{u=0}^{w-1} A[i][floor(u/N)*M + D[u][floor(j/L)]]   */
/*             * B'[u][j]                                              */
/* unscaled (R4), fp64 products, sequential fp64 sum in ascending u.   */
/* rows == NULL: all m rows; else only rows[0..nrows) (sampled check), */
/* output row r of C is rows[r].                                       */
/* ------------------------------------------------------------------ */
int nmo_spmm_sparse_f64(const void* A, int a_bf16, const void* values, int v_bf16, const uint8_t* D,
                        int64_t m, int64_t n, int64_t k, int N, int M, int L, const int64_t* rows,
                        int64_t nrows, double* C, int nthreads) {
    int s = nmo_check_shape(k, n, N, M, L);
    if (s) return s;
    const int64_t w = k / M * N, q = n / L;
    const int64_t R = rows ? nrows : m;
    int nt = omp_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 1) num_threads(nt)
    for (int64_t r = 0; r < R; ++r) {
        const int64_t i = rows ? rows[r] : r;
        double* acc = C + r * n;
        for (int64_t j = 0; j < n; ++j) acc[j] = 0.0;
        for (int64_t u = 0; u < w; ++u) {
            const int64_t base = (u / N) * M;
            for (int64_t g = 0; g < q; ++g) {
                const double a = load_elem(A, a_bf16, i * k + base + D[u * q + g]);
                for (int c = 0; c < L; ++c) {
                    const int64_t j = g * L + c;
                    const double prod = a * load_elem(values, v_bf16, u * n + j);
                    acc[j] = acc[j] + prod;
                }
            }
        }
    }
    return NMO_OK;
}

/* O2s: Eq. 1 as printed, WITH the M/N factor: C'[i][j] =   */
/* (M/N) * sum_u A[i][(u/N)M + D[u][j/L]] * B'[u][j] (the paper's      */
/* approximation of the unpruned C; R1 reads the product     */
/* path unscaled, nm_spmm_scaled exposes the factor as alpha).  The    */
/* sum in fp64, ascending u; the factor applied once, in fp64.         */
int nmo_spmm_eq1_scaled_f64(const void* A, int a_bf16, const void* values, int v_bf16, const uint8_t* D,
                            int64_t m, int64_t n, int64_t k, int N, int M, int L, double* C, int nthreads) {
    int s = nmo_check_shape(k, n, N, M, L);
    if (s) return s;
    const int64_t w = k / M * N, q = n / L;
    const double scale = (double)M / (double)N;
    int nt = omp_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 1) num_threads(nt)
    for (int64_t i = 0; i < m; ++i) {
        for (int64_t j = 0; j < n; ++j) {
            const int64_t g = j / L;
            double sum = 0.0;
            for (int64_t u = 0; u < w; ++u) {
                const double a = load_elem(A, a_bf16, i * k + (u / N) * M + D[u * q + g]);
                sum = sum + a * load_elem(values, v_bf16, u * n + j);
            }
            C[i * n + j] = scale * sum;
        }
    }
    return NMO_OK;
}

/* O2f: the same sum with a 32-bit float accumulator, ascending u     */
/* (SPEC's spmm_naive semantics).                              */
int nmo_spmm_sparse_f32seq(const void* A, int a_bf16, const void* values, int v_bf16,
                           const uint8_t* D, int64_t m, int64_t n, int64_t k, int N, int M, int L,
                           float* C, int nthreads) {
    int s = nmo_check_shape(k, n, N, M, L);
    if (s) return s;
    const int64_t w = k / M * N, q = n / L;
    int nt = omp_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 1) num_threads(nt)
    for (int64_t i = 0; i < m; ++i) {
        float* acc = C + i * n;
        for (int64_t j = 0; j < n; ++j) acc[j] = 0.0f;
        for (int64_t u = 0; u < w; ++u) {
            const int64_t base = (u / N) * M;
            for (int64_t g = 0; g < q; ++g) {
                const float a = (float)load_elem(A, a_bf16, i * k + base + D[u * q + g]);
                for (int c = 0; c < L; ++c) {
                    const int64_t j = g * L + c;
                    const float prod = a * (float)load_elem(values, v_bf16, u * n + j);
                    acc[j] = acc[j] + prod;
                }
            }
        }
    }
    return NMO_OK;
}

/* ------------------------------------------------------------------ */
/* Dense triple loop C = A . B (row-major, m x k times k x n); used as  */
/* O1 on B = decompress(B', D).  fp64 products, ascending p sum.        */
/* ------------------------------------------------------------------ */
int nmo_gemm_dense_f64(const void* A, int a_bf16, const void* B, int b_bf16, int64_t m, int64_t n,
                       int64_t k, double* C, int nthreads) {
    int nt = omp_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 1) num_threads(nt)
    for (int64_t i = 0; i < m; ++i) {
        double* acc = C + i * n;
        for (int64_t j = 0; j < n; ++j) acc[j] = 0.0;
        for (int64_t p = 0; p < k; ++p) {
            const double a = load_elem(A, a_bf16, i * k + p);
            for (int64_t j = 0; j < n; ++j) {
                const double prod = a * load_elem(B, b_bf16, p * n + j);
                acc[j] = acc[j] + prod;
            }
        }
    }
    return NMO_OK;
}

/* O1f: dense loop with a 32-bit float accumulator. */
int nmo_gemm_dense_f32seq(const void* A, int a_bf16, const void* B, int b_bf16, int64_t m,
                          int64_t n, int64_t k, float* C, int nthreads) {
    int nt = omp_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 1) num_threads(nt)
    for (int64_t i = 0; i < m; ++i) {
        float* acc = C + i * n;
        for (int64_t j = 0; j < n; ++j) acc[j] = 0.0f;
        for (int64_t p = 0; p < k; ++p) {
            const float a = (float)load_elem(A, a_bf16, i * k + p);
            for (int64_t j = 0; j < n; ++j) {
                const float prod = a * (float)load_elem(B, b_bf16, p * n + j);
                acc[j] = acc[j] + prod;
            }
        }
    }
    return NMO_OK;
}

/* ------------------------------------------------------------------ */
/* Eq. 2: W[i][j] = |C'[i][j] - C[i][j]| / (m*n), verbatim. */
/* ------------------------------------------------------------------ */
int nmo_confusion(const double* Capprox, const double* Cexact, int64_t m, int64_t n, double* W) {
    const double mn = (double)m * (double)n;
    for (int64_t i = 0; i < m * n; ++i) W[i] = fabs(Capprox[i] - Cexact[i]) / mn;
    return NMO_OK;
}

/* ------------------------------------------------------------------ */
/* Bit-packed, tile-major index matrix ("each element requires   */
/* only log2 M bits"; P:419 / Listing 3 transformLayout "transform the */
/* data layout of matrix D to reduce the number of global memory       */
/* transactions").  The layout (R28) written out plainly:    */
/*   b = bits per entry = max(1, ceil(log2 M)); e = floor(32 / b)      */
/*   entries per 32-bit word (no entry straddles a word);              */
/*   the q column groups are cut into tiles of T = 128 / L groups      */
/*   (the 128 output columns of one CTA tile; 128 % L == 0);           */
/*   a tile's entries are numbered x = u*T + t (row u < w, t < T) and  */
/*   stored in Wt = ceil(w*T / e) words: word P[tile*Wt + x/e] holds   */
/*   D[u][tile*T + t] in bits [(x%e)*b, (x%e)*b + b)                   */
/*   (groups >= q and unused bits: 0).                                 */
/* So a tile's whole index stream (all w rows) is one contiguous run.  */
/* ------------------------------------------------------------------ */
int nmo_index_bits(int M) {
    int b = 1;
    while ((1 << b) < M) ++b;
    return b;
}

int64_t nmo_index_packed_words(int64_t k, int64_t n, int N, int M, int L) {
    if (nmo_check_shape(k, n, N, M, L) || 128 % L) return -1;
    const int64_t w = k / M * N, q = n / L, T = 128 / L;
    const int e = 32 / nmo_index_bits(M);
    const int64_t ntiles = (q + T - 1) / T, Wt = (w * T + e - 1) / e;
    return ntiles * Wt;
}

int nmo_index_pack(const uint8_t* D, int64_t k, int64_t n, int N, int M, int L, uint32_t* P) {
    const int64_t nw = nmo_index_packed_words(k, n, N, M, L);
    if (nw < 0) return NMO_ERR_SHAPE;
    const int64_t w = k / M * N, q = n / L, T = 128 / L;
    const int b = nmo_index_bits(M), e = 32 / b;
    const int64_t ntiles = (q + T - 1) / T, Wt = (w * T + e - 1) / e;
    for (int64_t i = 0; i < nw; ++i) P[i] = 0u;
    for (int64_t tile = 0; tile < ntiles; ++tile)
        for (int64_t u = 0; u < w; ++u)
            for (int64_t t = 0; t < T; ++t) {
                const int64_t g = tile * T + t, x = u * T + t;
                if (g < q) P[tile * Wt + x / e] |= (uint32_t)D[u * q + g] << ((x % e) * b);
            }
    return NMO_OK;
}

int nmo_index_unpack(const uint32_t* P, int64_t k, int64_t n, int N, int M, int L, uint8_t* D) {
    if (nmo_index_packed_words(k, n, N, M, L) < 0) return NMO_ERR_SHAPE;
    const int64_t w = k / M * N, q = n / L, T = 128 / L;
    const int b = nmo_index_bits(M), e = 32 / b;
    const int64_t Wt = (w * T + e - 1) / e;
    const uint32_t mask = (1u << b) - 1u;
    for (int64_t u = 0; u < w; ++u)
        for (int64_t g = 0; g < q; ++g) {
            const int64_t tile = g / T, x = u * T + g % T;
            D[u * q + g] = (uint8_t)((P[tile * Wt + x / e] >> ((x % e) * b)) & mask);
        }
    return NMO_OK;
}
