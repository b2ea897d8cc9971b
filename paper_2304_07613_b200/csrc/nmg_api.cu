// nmg_api.cu -- C ABI of the chunked n:m:g format (include/sten.h, "Chunked n:m:g"):
// argument validation, pattern table, kernel instantiation and launch.
#include "sten.h"

#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "nmg.cuh"

using namespace sten;

namespace {

inline cudaStream_t nmg_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }
inline bool nmg_dtype_ok(int d) { return d == STEN_F32 || d == STEN_BF16; }
inline size_t nmg_dt_size(sten_dtype d) { return d == STEN_F32 ? 4 : 2; }
inline sten_status nmg_last_cuda() { return cudaGetLastError() == cudaSuccess ? STEN_OK : STEN_ERR_CUDA; }

// format + shape checks shared by the three calls; fills the kernel arguments
sten_status nmg_setup(sten_nmg f, int dt, int64_t M, int64_t K, NmgArgs* a) {
    if (f.n < 1 || f.n >= f.m || f.m > 16 || f.g < 1 || !nmg_dtype_ok(dt)) return STEN_ERR_INVALID_ARG;
    const int C = nmg_binom(f.m, f.n);
    if (C > kNmgMaxPatterns) return STEN_ERR_UNSUPPORTED;
    const int64_t L = int64_t(C) * f.g;
    if (L > 65535 || L * C > 2048) return STEN_ERR_UNSUPPORTED;
    if (M < 0 || K < 0 || M % f.m != 0 || K % L != 0) return STEN_ERR_SHAPE;
    a->n = f.n; a->m = f.m; a->g = f.g; a->C = C; a->L = int(L);
    a->M = M; a->K = K; a->NC = K / L; a->RB = M / f.m;
    a->pat = nmg_revolving_door(f.m, f.n);
    return STEN_OK;
}

template <typename TAB, typename TC, int NN, int MM>
sten_status launch_nmg_spmm(const NmgSpmmArgs& a0, cudaStream_t st) {
    NmgSpmmArgs a = a0;
    a.cps = a.L >= 32 ? 1 : (32 + a.L - 1) / a.L;                   // >= 32 B rows per K-stage
    if (a.cps > a.NC) a.cps = int(a.NC > 0 ? a.NC : 1);
    while (a.cps > 1 && kNmgStages * nmg_spmm_stage_bytes<TAB>(a.cps * a.L, NN) > 113 * 1024) --a.cps;
    size_t smem = kNmgStages * nmg_spmm_stage_bytes<TAB>(a.cps * a.L, NN);
    const size_t tile = size_t(kNmgSpmmWarps) * MM * kNmgBN * 4;    // split-K partial tile (fp32)
    const int64_t gx = (a.N + kNmgBN - 1) / kNmgBN, gy = (a.RB + kNmgSpmmWarps - 1) / kNmgSpmmWarps;
    // split-K (cluster z) until about two CTAs per SM: S <= 8 (portable cluster), <= chunks
    // (measured on the C2 shapes: the smallest S reaching two CTAs per SM beats both the largest
    // one-wave S and ~4 CTAs per SM)
    int S = 1;
    while (S < 8 && gx * gy * S < 2 * 148 && a.NC >= 2 * (S + 1)) ++S;
    a.split = S;
    if (S > 1 && smem < tile) smem = tile;
    if (smem > 227 * 1024) return STEN_ERR_UNSUPPORTED;
    auto kern = nmg_spmm_kernel<TAB, TC, NN, MM>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)) != cudaSuccess)
        return STEN_ERR_CUDA;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(gx), unsigned(gy), unsigned(S));
    cfg.blockDim = dim3(kNmgSpmmWarps * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 1;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = unsigned(S);
    cfg.attrs = attr;
    cfg.numAttrs = S > 1 ? 1 : 0;
    if (cudaLaunchKernelEx(&cfg, kern, a) != cudaSuccess) return STEN_ERR_CUDA;
    return nmg_last_cuda();
}

template <typename TAB, typename TC>
sten_status dispatch_nmg_spmm(int n, int m, const NmgSpmmArgs& a, cudaStream_t st) {
    if (n == 1 && m == 2) return launch_nmg_spmm<TAB, TC, 1, 2>(a, st);
    if (n == 1 && m == 4) return launch_nmg_spmm<TAB, TC, 1, 4>(a, st);
    if (n == 2 && m == 4) return launch_nmg_spmm<TAB, TC, 2, 4>(a, st);
    if (n == 1 && m == 8) return launch_nmg_spmm<TAB, TC, 1, 8>(a, st);
    // the paper's Fig.-5 format (3:6) and the 75 / 90 % points of the C2 sweep: more
    // patterns per chunk (20 / 28 / 10) -> a longer straight-line chunk body
    if (n == 3 && m == 6) return launch_nmg_spmm<TAB, TC, 3, 6>(a, st);
    if (n == 2 && m == 8) return launch_nmg_spmm<TAB, TC, 2, 8>(a, st);
    if (n == 1 && m == 10) return launch_nmg_spmm<TAB, TC, 1, 10>(a, st);
    return STEN_ERR_UNSUPPORTED;
}

__global__ void nmg_zero_kernel(void* C, int64_t M, int64_t N, int64_t ldc, int esz) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= M * N) return;
    const int64_t r = i / N, c = i - r * N;
    if (esz == 4) static_cast<float*>(C)[r * ldc + c] = 0.0f;
    else static_cast<uint16_t*>(C)[r * ldc + c] = 0;
}

}  // namespace

extern "C" {

sten_status sten_nmg_sparsify(sten_nmg f, sten_dtype dt, const void* W, int64_t M, int64_t K, int64_t ldw,
                              void* values, uint16_t* idx, void* stream) {
    return sten_nmg_sparsify_ex(f, dt, W, M, K, ldw, values, idx, 0, stream);
}

sten_status sten_nmg_sparsify_ex(sten_nmg f, sten_dtype dt, const void* W, int64_t M, int64_t K, int64_t ldw,
                                 void* values, uint16_t* idx, int32_t method, void* stream) {
    NmgArgs a = {};
    sten_status s = nmg_setup(f, dt, M, K, &a);
    if (s) return s;
    if (method < 0 || method > 2) return STEN_ERR_INVALID_ARG;
    a.method = method;
    if (ldw < K) return STEN_ERR_SHAPE;
    if (M * K > 0 && (!W || !values || !idx)) return STEN_ERR_INVALID_ARG;
    if (M == 0 || K == 0) return STEN_OK;
    a.W = W; a.ldw = ldw; a.values = values; a.idx = idx;
    const int64_t chunks = a.RB * a.NC;
    const size_t smem = size_t(kNmgWarpsPerCta) * nmg_warp_smem(a.L, a.C, a.m, int(nmg_dt_size(dt)));
    const unsigned grid = unsigned((chunks + kNmgWarpsPerCta - 1) / kNmgWarpsPerCta);
    cudaStream_t st = nmg_stream(stream);
    const int NI = a.L * a.C;
    const int kpl = NI <= 64 ? 2 : NI <= 128 ? 4 : NI <= 192 ? 6 : 8;
    auto go = [&](auto kern) -> sten_status {
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem))) return STEN_ERR_CUDA;
        kern<<<grid, kNmgWarpsPerCta * 32, smem, st>>>(a);
        return nmg_last_cuda();
    };
    if (dt == STEN_F32) {
        switch (kpl) {
            case 2: return go(nmg_sparsify_kernel<float, 2>);
            case 4: return go(nmg_sparsify_kernel<float, 4>);
            case 6: return go(nmg_sparsify_kernel<float, 6>);
            default: return go(nmg_sparsify_kernel<float, 8>);
        }
    }
    switch (kpl) {
        case 2: return go(nmg_sparsify_kernel<uint16_t, 2>);
        case 4: return go(nmg_sparsify_kernel<uint16_t, 4>);
        case 6: return go(nmg_sparsify_kernel<uint16_t, 6>);
        default: return go(nmg_sparsify_kernel<uint16_t, 8>);
    }
}

sten_status sten_nmg_densify(sten_nmg f, sten_dtype dt, const void* values, const uint16_t* idx, int64_t M,
                             int64_t K, void* W_out, int64_t ldw, void* stream) {
    NmgArgs a = {};
    sten_status s = nmg_setup(f, dt, M, K, &a);
    if (s) return s;
    if (ldw < K) return STEN_ERR_SHAPE;
    if (M * K > 0 && (!W_out || !values || !idx)) return STEN_ERR_INVALID_ARG;
    if (M == 0 || K == 0) return STEN_OK;
    a.values_in = values; a.idx_in = idx; a.ldw = ldw;
    const int64_t threads = a.RB * a.NC * a.L;
    const unsigned grid = unsigned((threads + 255) / 256);
    cudaStream_t st = nmg_stream(stream);
    if (dt == STEN_F32) nmg_densify_kernel<float><<<grid, 256, 0, st>>>(a, static_cast<float*>(W_out));
    else nmg_densify_kernel<uint16_t><<<grid, 256, 0, st>>>(a, static_cast<uint16_t*>(W_out));
    return nmg_last_cuda();
}

sten_status sten_nmg_spmm(sten_nmg f, sten_dtype ab_dt, const void* values, const uint16_t* idx, int64_t M,
                          int64_t K, const void* B, int64_t ldb, int64_t N, void* C, int64_t ldc,
                          sten_dtype c_dt, void* stream) {
    NmgArgs fa = {};
    sten_status s = nmg_setup(f, ab_dt, M, K, &fa);
    if (s) return s;
    if (!nmg_dtype_ok(c_dt)) return STEN_ERR_INVALID_ARG;
    if (N < 0 || ldb < N || ldc < N) return STEN_ERR_SHAPE;
    if ((M * K > 0 && (!values || !idx)) || (K * N > 0 && !B) || (M * N > 0 && !C)) return STEN_ERR_INVALID_ARG;
    const bool compiled = (f.n == 1 && (f.m == 2 || f.m == 4 || f.m == 8 || f.m == 10)) ||
                          (f.n == 2 && (f.m == 4 || f.m == 8)) || (f.n == 3 && f.m == 6);
    if (!compiled) return STEN_ERR_UNSUPPORTED;
    // idx / values are staged with 4-byte cp.async (L is even for every compiled format)
    if ((reinterpret_cast<uintptr_t>(idx) & 3u) != 0 || (reinterpret_cast<uintptr_t>(values) & 3u) != 0)
        return STEN_ERR_UNSUPPORTED;
    const size_t sab = nmg_dt_size(ab_dt);
    if (K * N > 0 && ((reinterpret_cast<uintptr_t>(B) & 15u) != 0 || (ldb * int64_t(sab)) % 16 != 0))
        return STEN_ERR_UNSUPPORTED;
    if (M == 0 || N == 0) return STEN_OK;
    cudaStream_t st = nmg_stream(stream);
    if (K == 0) {
        nmg_zero_kernel<<<unsigned((M * N + 255) / 256), 256, 0, st>>>(C, M, N, ldc, int(nmg_dt_size(c_dt)));
        return nmg_last_cuda();
    }
    NmgSpmmArgs a = {};
    a.values = values; a.idx = idx; a.B = B; a.C = C;
    a.M = M; a.K = K; a.N = N; a.ldb = ldb; a.ldc = ldc; a.NC = fa.NC; a.RB = fa.RB;
    a.g = f.g; a.L = fa.L;
    a.c_vec = (reinterpret_cast<uintptr_t>(C) & 15u) == 0 && (ldc * int64_t(nmg_dt_size(c_dt))) % 16 == 0;
    if (ab_dt == STEN_F32)
        return c_dt == STEN_F32 ? dispatch_nmg_spmm<float, float>(f.n, f.m, a, st)
                                : dispatch_nmg_spmm<float, uint16_t>(f.n, f.m, a, st);
    return c_dt == STEN_F32 ? dispatch_nmg_spmm<uint16_t, float>(f.n, f.m, a, st)
                            : dispatch_nmg_spmm<uint16_t, uint16_t>(f.n, f.m, a, st);
}

}  // extern "C"
