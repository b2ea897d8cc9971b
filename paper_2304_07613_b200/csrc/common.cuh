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
STEN_DEVICE_INLINE void cp_async4(void* smem, const void* gmem, int src_bytes) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(smem_u32(smem)),
                 "l"(gmem), "r"(src_bytes));
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

}  // namespace sten
