// common.cuh -- shared device/host helpers of libnmspmm.so (sm_100a only).
// PTX wrappers for mbarrier / TMA / tcgen05 are written here from the PTX ISA;
// no CUTLASS/CuTe code is used.
#pragma once

#include <cuda.h>  // CUtensorMap type only (driver entry point fetched at run time)
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <string>

#include "../../include/nmspmm.h"

namespace nm {

// ---------------------------------------------------------------- host status
void set_error(const std::string& msg);
nm_status fail(nm_status s, const std::string& msg);
nm_status cuda_fail(cudaError_t e, const char* what);

#define NM_CUDA_TRY(expr)                                   \
    do {                                                    \
        cudaError_t _e = (expr);                            \
        if (_e != cudaSuccess) return ::nm::cuda_fail(_e, #expr); \
    } while (0)

#define NM_LAUNCH_CHECK(what)                                     \
    do {                                                          \
        cudaError_t _e = cudaGetLastError();                      \
        if (_e != cudaSuccess) return ::nm::cuda_fail(_e, what);  \
    } while (0)

int num_sms();         // SM count of the current device (cached per device; 148 on B200)
int current_device();  // cudaGetDevice, -1 on error
nm_status require_device();  // NM_OK iff a device of compute capability 10.0 is current
// Once-per-device guards for cudaFuncSetAttribute (MaxDynamicSharedMemorySize is a per-device
// setting): attr_once(mask) is true once attr_done(mask) ran on the current device.  Racing
// threads may both set the attribute, which is idempotent.
bool attr_once(std::atomic<uint64_t>& mask);
void attr_done(std::atomic<uint64_t>& mask);
nm_status scratch_alloc(void** p, size_t bytes, cudaStream_t s);  // library-owned stream-ordered pool

// Launch accounting for nm_profile_begin/end: every kernel launch of the product
// path calls note_launch(); the dominant SpMM kernel is bracketed by
// prof_begin/prof_end, which record CUDA events on its stream while profiling is on.
void note_launch();
void prof_begin(cudaStream_t s);
void prof_end(cudaStream_t s);

// Peer-store destinations of the fused column all-gather (nm_spmm_peers,
// nm_spmm_prepacked_peers): up to 8 ranks'
// C buffers (device pointers valid in this process: own or IPC-opened), row pitch ldc,
// this shard's first global column col_off, its n_valid real (unpadded) columns.
struct PeerOut {
    void* c[8];
    int np;
    int64_t ldc, col_off, n_valid;
    int mc = 0;  // 1: c[0] is a multicast (NVLS) address, written once with multimem.st (nm_spmm_mc)
};

// TMA descriptor encoding (cuTensorMapEncodeTiled fetched via cudaGetDriverEntryPoint).
// 2-D row-major tensor [rows][cols] of elem_bytes elements; box [box_rows][box_cols].
// swizzle: 0 none, 128 = 128-byte swizzle.  OOB elements are zero-filled.
nm_status make_tma_2d(CUtensorMap* map, const void* base, CUtensorMapDataType dt, int elem_bytes,
                      int64_t rows, int64_t cols, int box_rows, int box_cols, int swizzle);

// Same with an explicit row pitch (elements) >= cols.
nm_status make_tma_2d_pitched(CUtensorMap* map, const void* base, CUtensorMapDataType dt, int elem_bytes, int64_t rows,
                              int64_t cols, int64_t pitch_elems, int box_rows, int box_cols, int swizzle);

// --------------------------------------------------------------- device PTX
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}

// non-blocking probe (no suspend), for polling loops that interleave several waits
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    while (!mbar_try_wait(bar, parity)) {
    }
}

__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(map) : "memory");
}

// 2-D TMA tile load: coordinates (c0 = innermost / column, c1 = row).
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
        "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}

// 1-D bulk copy global -> shared (16-B aligned, size multiple of 16), completes on an mbarrier.
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

__host__ __device__ __forceinline__ int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace nm
