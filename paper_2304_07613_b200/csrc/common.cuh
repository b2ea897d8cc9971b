// common.cuh -- small device helpers shared by the sm_100a kernels of libsten.
// (Product path only; nothing here is shared with oracle/.)
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#ifndef STEN_DEVICE_INLINE
#define STEN_DEVICE_INLINE __device__ __forceinline__
#endif

namespace sten {

typedef uint16_t bf16_t;   // raw bf16 bits; widened exactly with << 16

STEN_DEVICE_INLINE int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }
STEN_DEVICE_INLINE int64_t max64(int64_t a, int64_t b) { return a > b ? a : b; }

STEN_DEVICE_INLINE float to_f32(float x) { return x; }
STEN_DEVICE_INLINE float to_f32(bf16_t x) { return __uint_as_float(uint32_t(x) << 16); }

// fp32 -> bf16 round-to-nearest-even (finite inputs; NaN stays NaN)
STEN_DEVICE_INLINE bf16_t f32_to_bf16_rne(float x) {
    return __bfloat16_as_ushort(__float2bfloat16_rn(x));
}

template <typename T> STEN_DEVICE_INLINE T from_f32(float x);
template <> STEN_DEVICE_INLINE float from_f32<float>(float x) { return x; }
template <> STEN_DEVICE_INLINE bf16_t from_f32<bf16_t>(float x) { return f32_to_bf16_rne(x); }

// ---- cp.async (LDGSTS) helpers ---------------------------------------------------------
STEN_DEVICE_INLINE uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// 16-byte async copy global -> shared; bytes beyond src_bytes (0..16) are zero-filled.
STEN_DEVICE_INLINE void cp_async16(void* smem, const void* gmem, int src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(smem)),
                 "l"(gmem), "r"(src_bytes));
}
STEN_DEVICE_INLINE void cp_async8(void* smem, const void* gmem, int src_bytes) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(smem)),
                 "l"(gmem), "r"(src_bytes));
}
STEN_DEVICE_INLINE void cp_async4(void* smem, const void* gmem, int src_bytes) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(smem_u32(smem)),
                 "l"(gmem), "r"(src_bytes));
}
// the mbarrier receives one arrive when all prior cp.async of this thread have landed
// (.noinc: that arrive counts against the barrier's initial arrival count)
STEN_DEVICE_INLINE void cp_async_mbar_arrive_noinc(uint64_t* bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
// same, but the barrier's pending count is raised at issue and lowered when the copies land
// (net zero arrivals: the phase cannot complete before the copies)
STEN_DEVICE_INLINE void cp_async_mbar_arrive(uint64_t* bar) {
    asm volatile("cp.async.mbarrier.arrive.shared::cta.b64 [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
STEN_DEVICE_INLINE void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
STEN_DEVICE_INLINE void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

STEN_DEVICE_INLINE float4 lds128(const void* p) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];\n"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "r"(smem_u32(p)));
    return v;
}

// 16-byte shared load from a 32-bit shared-window address; not volatile, so the
// compiler may schedule it freely between the barriers that order the buffer.
STEN_DEVICE_INLINE float4 lds128_addr(uint32_t addr) {
    float4 v;
    asm("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];\n"
        : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
        : "r"(addr));
    return v;
}

STEN_DEVICE_INLINE uint32_t lds32_addr(uint32_t addr) {
    uint32_t v;
    asm("ld.shared.b32 %0, [%1];\n" : "=r"(v) : "r"(addr));
    return v;
}

// ---- mbarrier + TMA (cp.async.bulk.tensor) helpers ---------------------------------------
STEN_DEVICE_INLINE void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
STEN_DEVICE_INLINE void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
STEN_DEVICE_INLINE void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
STEN_DEVICE_INLINE void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
STEN_DEVICE_INLINE void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
STEN_DEVICE_INLINE void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
STEN_DEVICE_INLINE void mbar_wait(uint64_t* bar, uint32_t phase) {
    // try_wait with a suspend-time hint: the waiting warp sleeps instead of spinning on issue slots
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
        "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(bar)),
        "r"(phase), "r"(0x989680)
        : "memory");
}
// 2-D tiled TMA load of box {x..x+bx, y..y+by} (x innermost) into shared memory;
// out-of-bounds elements are zero-filled; completion is signalled on `bar`.
STEN_DEVICE_INLINE void tma_load_2d(void* smem_dst, const void* tmap, uint64_t* bar, int x, int y) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];\n" ::"r"(
            smem_u32(smem_dst)),
        "l"(tmap), "r"(smem_u32(bar)), "r"(x), "r"(y)
        : "memory");
}

STEN_DEVICE_INLINE void tma_load_3d(void* smem_dst, const void* tmap, uint64_t* bar, int x, int y, int z) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], "
        "[%2];\n" ::"r"(smem_u32(smem_dst)),
        "l"(tmap), "r"(smem_u32(bar)), "r"(x), "r"(y), "r"(z)
        : "memory");
}

STEN_DEVICE_INLINE void tma_load_4d(void* smem_dst, const void* tmap, uint64_t* bar, int c0, int c1, int c2, int c3) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], "
        "[%2];\n" ::"r"(smem_u32(smem_dst)),
        "l"(tmap), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
        : "memory");
}
STEN_DEVICE_INLINE void tma_load_5d(void* smem_dst, const void* tmap, uint64_t* bar, int c0, int c1, int c2, int c3,
                                    int c4) {
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6, %7}], "
        "[%2];\n" ::"r"(smem_u32(smem_dst)),
        "l"(tmap), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
        : "memory");
}

}  // namespace sten
