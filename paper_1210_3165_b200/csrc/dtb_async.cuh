// dtb_async.cuh -- device helpers shared by the sliding-window kernels (sm_100a): 1-D bulk
// copies through the TMA engine with mbarrier completion, L2 eviction policies, named
// barriers with immediate ids, byte permutes, dp4a forms and the (segmented) row address.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <cstdio>

#include "dtb_slide.cuh"

namespace dtb {

// prmt.b32 with the raw selector (sign-replicate mode available: nibble bit 3 set copies the
// sign bit of the selected byte into all 8 bits; __byte_perm masks selectors to 3 bits).
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
    uint32_t d;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
    return d;
}

// DTB_DEBUG_BOUNDS=1: trap on any out-of-range shared-memory index (debug builds; the pool's
// compute-sanitizer is unavailable, tests/test_fast_path_gpu.py runs once under this build).
#ifndef DTB_DEBUG_BOUNDS
#define DTB_DEBUG_BOUNDS 0
#endif
#if DTB_DEBUG_BOUNDS
#define DTB_CHECK(cond)                                                                       \
    do {                                                                                      \
        if (!(cond)) {                                                                        \
            printf("DTB_CHECK failed %s:%d block (%d,%d,%d) thread %d\n", __FILE__, __LINE__, \
                   blockIdx.x, blockIdx.y, blockIdx.z, threadIdx.x);                           \
            __trap();                                                                         \
        }                                                                                     \
    } while (0)
#else
#define DTB_CHECK(cond) ((void)0)
#endif

// Address of global row g (in0 = the single buffer's row-0 origin).  Segmented inputs pick
// the segment holding g; the pointer may be a peer GPU's memory (NVLink), which the bulk
// copies and loads below read in place.
// SEG is a compile-time kernel variant: the single-buffer kernels keep the plain address
// arithmetic (a runtime segment test in the producer's path measured 8% slower on C4).
template <bool SEG>
__device__ __forceinline__ const uint8_t* row_at(const SlideParams& p, const uint8_t* in0, int g) {
    if (!SEG) return in0 + (int64_t)g * p.pitch;
    const int i = g >= p.seg_lo[2] ? 2 : (g >= p.seg_lo[1] ? 1 : 0);
    return p.seg_ptr[i] + (int64_t)(g - p.seg_lo[i]) * p.seg_pitch[i];
}

// ---- asynchronous row staging: cp.async.bulk (TMA engine, no tensor map) + mbarrier
__device__ __forceinline__ uint32_t smem_u32(const void* ptr) {
    return (uint32_t)__cvta_generic_to_shared(ptr);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n}" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1], %2, [%3], %4;"
        ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy) : "memory");
}
// 3-D tiled tensor copy (tensor map in param space): box {x, y, z} of the map -> dst, bytes
// outside the tensor are zero-filled; completion on the mbarrier's tx count (full box bytes).
__device__ __forceinline__ void tma_load_3d(void* dst, const void* tmap, int x, int y, int z, uint64_t* bar,
                                            uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3, %4}], [%5], %6;"
        ::"r"(smem_u32(dst)), "l"(tmap), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar)), "l"(policy) : "memory");
}
// the same with shared-window addresses (no generic -> shared conversion at the call site)
__device__ __forceinline__ void mbar_expect_tx_a(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait_a(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n}" ::"r"(bar), "r"(parity) : "memory");
}
__device__ __forceinline__ void tma_load_3d_a(uint32_t dst, const void* tmap, int x, int y, int z, uint32_t bar,
                                              uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3, %4}], [%5], %6;"
        ::"r"(dst), "l"(tmap), "r"(x), "r"(y), "r"(z), "r"(bar), "l"(policy) : "memory");
}
// L2 eviction priorities: a row is read three times (entering, centre r steps later, leaving
// 2r+1 steps later); keep it resident on the first two reads, let it go on the last.
__device__ __forceinline__ uint64_t make_policy(int kind) {
    uint64_t p;
    if (kind == 2) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    else if (kind == 1) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    else asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
    return p;
}

// Barrier ids are immediates (a register id makes ptxas reserve all 16 barriers, which caps
// resident CTAs per SM); callers pass (base, buffer) and we branch to constant ids.
template <int ID>
__device__ __forceinline__ void nbar_sync_c(int count) {
    asm volatile("bar.sync %0, %1;" ::"n"(ID), "r"(count) : "memory");
}
template <int ID>
__device__ __forceinline__ void nbar_arrive_c(int count) {
    asm volatile("bar.arrive %0, %1;" ::"n"(ID), "r"(count) : "memory");
}
__device__ __forceinline__ void nbar_sync(int id, int count) {
    switch (id) {
        case 1: nbar_sync_c<1>(count); break;
        case 2: nbar_sync_c<2>(count); break;
        case 3: nbar_sync_c<3>(count); break;
        case 4: nbar_sync_c<4>(count); break;
        case 5: nbar_sync_c<5>(count); break;
        default: nbar_sync_c<6>(count); break;
    }
}
__device__ __forceinline__ void nbar_arrive(int id, int count) {
    switch (id) {
        case 1: nbar_arrive_c<1>(count); break;
        case 2: nbar_arrive_c<2>(count); break;
        case 3: nbar_arrive_c<3>(count); break;
        case 4: nbar_arrive_c<4>(count); break;
        case 5: nbar_arrive_c<5>(count); break;
        default: nbar_arrive_c<6>(count); break;
    }
}
__device__ __forceinline__ void mbar_arrive_cnt(uint64_t* bar, uint32_t cnt) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(cnt) : "memory");
}

// acc - (sum of the four bytes of x): dp4a with unsigned a and signed (-1) b bytes
__device__ __forceinline__ uint32_t dp4a_sub(uint32_t x, uint32_t acc) {
    uint32_t d;
    asm("dp4a.u32.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(x), "r"(0xFFFFFFFFu), "r"(acc));
    return d;
}

// Sequence of pipeline items for one CTA: warm-up rows g0..g1 (entering row only), then
// main row steps y = ya..yb-1 (entering row y+r, leaving row y-r-1, centre row y).
struct Items {
    int g0, nwarm, ya, n;
};

// named-barrier ids of the warp-specialized kernels (0 is __syncthreads)
enum { BAR_COLS = 1, BAR_READY0 = 2, BAR_FREE0 = 4, BAR_WARM = 6 };

}  // namespace dtb
