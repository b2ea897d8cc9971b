// masked_api.cu -- C ABI of the NEXT-2 masked-linear weight gradient (include/sten.h):
// sten_sddmm_grouped_nm.
#include "sten.h"

#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include "common.cuh"
#include "masked.cuh"

using namespace sten;

namespace {

inline bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

template <typename T, typename TC, int RR>
sten_status launch_sddmm_rr(const SddmmArgs& a, cudaStream_t st) {
    const SddmmGeom g = sddmm_geom(a.n, a.m, RR, int(sizeof(T)));
    auto kern = sddmm_grouped_nm_kernel<T, TC, RR>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(g.smem)) != cudaSuccess)
        return STEN_ERR_CUDA;
    dim3 grid(unsigned((a.Kp + g.kpc - 1) / g.kpc), unsigned((a.M + g.rows - 1) / g.rows));
    kern<<<grid, 256, g.smem, st>>>(a);
    return cudaGetLastError() == cudaSuccess ? STEN_OK : STEN_ERR_CUDA;
}

template <typename T, typename TC>
sten_status launch_sddmm(const SddmmArgs& a, int rr, cudaStream_t st) {
    if (rr == 4) return launch_sddmm_rr<T, TC, 4>(a, st);
    if (rr == 2) return launch_sddmm_rr<T, TC, 2>(a, st);
    return launch_sddmm_rr<T, TC, 1>(a, st);
}

}  // namespace

extern "C" {

sten_status sten_sddmm_grouped_nm(sten_nmg f, sten_dtype ab_dt, const void* G, int64_t M, int64_t N, int64_t ldg,
                                  const void* B, int64_t K, int64_t ldb, const uint8_t* idx, void* dV,
                                  sten_dtype c_dt, void* stream) {
    if (f.n < 1 || f.m > 16 || f.n >= f.m || f.g < 1) return STEN_ERR_INVALID_ARG;
    if (!(f.m == 2 || f.m == 4 || f.m == 6 || f.m == 8 || f.m == 10 || f.m == 12 || f.m == 16))
        return STEN_ERR_UNSUPPORTED;
    if ((ab_dt != STEN_F32 && ab_dt != STEN_BF16) || (c_dt != STEN_F32 && c_dt != STEN_BF16))
        return STEN_ERR_INVALID_ARG;
    if (M < 0 || K < 0 || N < 0 || M % f.g != 0 || K % f.m != 0 || ldg < N || ldb < N) return STEN_ERR_SHAPE;
    if ((M * N > 0 && !G) || (K * N > 0 && !B) || (M * K > 0 && (!idx || !dV))) return STEN_ERR_INVALID_ARG;
    const int64_t es = ab_dt == STEN_F32 ? 4 : 2;
    if (M * N > 0 && (!al16(G) || (ldg * es) % 16 != 0)) return STEN_ERR_UNSUPPORTED;
    if (K * N > 0 && (!al16(B) || (ldb * es) % 16 != 0)) return STEN_ERR_UNSUPPORTED;
    SddmmArgs a;
    memset(&a, 0, sizeof(a));
    a.G = G; a.B = B; a.idx = idx; a.dV = dV;
    a.M = M; a.K = K; a.N = N; a.ldg = ldg; a.ldb = ldb;
    a.KB = K / f.m; a.Kp = a.KB * f.n;
    a.n = f.n; a.m = f.m; a.g = f.g;
    if (M == 0 || a.Kp == 0) return STEN_OK;
    const int rr = f.g % 4 == 0 ? 4 : f.g % 2 == 0 ? 2 : 1;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (ab_dt == STEN_F32)
        return c_dt == STEN_F32 ? launch_sddmm<float, float>(a, rr, st) : launch_sddmm<float, bf16_t>(a, rr, st);
    return c_dt == STEN_F32 ? launch_sddmm<bf16_t, float>(a, rr, st) : launch_sddmm<bf16_t, bf16_t>(a, rr, st);
}

}  // extern "C"
