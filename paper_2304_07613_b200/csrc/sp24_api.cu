// sp24_api.cu -- C ABI of K6 (2:4 structured-sparse tensor-core path, include/sten.h):
// sten_sp24_packed_size, sten_sp24_pack, sten_spmm_sp24.
#include "sten.h"

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "common.cuh"
#include "tma_host.h"
#include "spmm_sp24.cuh"

using namespace sten;

namespace {

inline bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

inline int num_sms() {
    static int n = 0;          // device property, immutable after the first query
    if (n == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

template <typename TC, int MB, int BN, int ST>
sten_status launch_sp24(Sp24Args a, cudaStream_t st) {
    using Cfg = Sp24Cfg<MB, BN, ST>;
    CUtensorMap tmA, tmB, tmC;
    memset(&tmA, 0, sizeof(tmA));
    memset(&tmB, 0, sizeof(tmB));
    memset(&tmC, 0, sizeof(tmC));
    {   // v24 [M128][Kc] bf16: box [kABoxRows rows][32 stored k], 64-byte swizzle (the K-major A operand)
        const uint64_t dims[2] = {uint64_t(a.Kc), uint64_t(sp24_m128(a.M))};
        const uint64_t strides[1] = {uint64_t(a.Kc) * 2};
        const uint32_t box[2] = {32u, uint32_t(Cfg::kABoxRows)};
        if (!make_tmap_nd(&tmA, a.v24, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dims, strides, box,
                          CU_TENSOR_MAP_SWIZZLE_64B))
            return STEN_ERR_CUDA;
    }
    {   // B [K][ldb] bf16: box [64 k rows][64 tokens], 128-byte swizzle (the MN-major B operand);
        // rows >= K and tokens >= N are zero-filled
        const uint64_t dims[2] = {uint64_t(a.N), uint64_t(a.K)};
        const uint64_t strides[1] = {uint64_t(a.ldb) * 2};
        const uint32_t box[2] = {64u, 64u};
        if (!make_tmap_nd(&tmB, a.B, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dims, strides, box,
                          CU_TENSOR_MAP_SWIZZLE_128B))
            return STEN_ERR_CUDA;
    }
    {   // C [M][ldc]: TMA store boxes [32 rows][32 tokens] from the epilogue staging tiles (clipped at M, N)
        const uint64_t dims[2] = {uint64_t(a.N), uint64_t(a.M)};
        const uint64_t strides[1] = {uint64_t(a.ldc) * sizeof(TC)};
        const uint32_t box[2] = {32u, 32u};
        if (!make_tmap_nd(&tmC, a.C, sizeof(TC) == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                          2, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_NONE))
            return STEN_ERR_CUDA;
    }
    a.nkt = int(sp24_k128(a.K) / 64);
    a.row_tiles = int((a.M + Cfg::kBM - 1) / Cfg::kBM);
    a.col_tiles = int((a.N + BN - 1) / BN);
    const int ntiles = a.row_tiles * a.col_tiles;
    auto kern = spmm_sp24_kernel<TC, MB, BN, ST>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(Cfg::kSmem)) != cudaSuccess)
        return STEN_ERR_CUDA;
    cudaLaunchConfig_t cfg;
    memset(&cfg, 0, sizeof(cfg));
    cfg.gridDim = dim3(unsigned(ntiles < num_sms() ? ntiles : num_sms()));     // persistent: one CTA per SM
    cfg.blockDim = dim3(Cfg::kThreads);
    cfg.dynamicSmemBytes = Cfg::kSmem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, kern, a, tmA, tmB, tmC) != cudaSuccess) return STEN_ERR_CUDA;
    return STEN_OK;
}

// 2-SM variant (tile 6): clusters of 2 CTAs, 256 x 256 pair tiles, one pair per 2 SMs (persistent)
template <typename TC, int ST>
sten_status launch_sp24_2sm(Sp24Args a, cudaStream_t st) {
    using Cfg = Sp24Cfg2<ST>;
    CUtensorMap tmA, tmB, tmC, tmE;
    memset(&tmA, 0, sizeof(tmA));
    memset(&tmB, 0, sizeof(tmB));
    memset(&tmC, 0, sizeof(tmC));
    memset(&tmE, 0, sizeof(tmE));
    {   // v24 [M128][Kc]: box [128 rows][64 stored k], 128-byte swizzle
        const uint64_t dims[2] = {uint64_t(a.Kc), uint64_t(sp24_m128(a.M))};
        const uint64_t strides[1] = {uint64_t(a.Kc) * 2};
        const uint32_t box[2] = {64u, 128u};
        if (!make_tmap_nd(&tmA, a.v24, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dims, strides, box,
                          CU_TENSOR_MAP_SWIZZLE_128B))
            return STEN_ERR_CUDA;
    }
    {   // B [K][ldb]: box [128 k][64 tokens], 128-byte swizzle
        const uint64_t dims[2] = {uint64_t(a.N), uint64_t(a.K)};
        const uint64_t strides[1] = {uint64_t(a.ldb) * 2};
        const uint32_t box[2] = {64u, 128u};
        if (!make_tmap_nd(&tmB, a.B, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dims, strides, box,
                          CU_TENSOR_MAP_SWIZZLE_128B))
            return STEN_ERR_CUDA;
    }
    {   // C [M][ldc]: TMA store boxes [32 rows][32 tokens]
        const uint64_t dims[2] = {uint64_t(a.N), uint64_t(a.M)};
        const uint64_t strides[1] = {uint64_t(a.ldc) * sizeof(TC)};
        const uint32_t box[2] = {32u, 32u};
        if (!make_tmap_nd(&tmC, a.C, sizeof(TC) == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                          2, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_NONE))
            return STEN_ERR_CUDA;
    }
    {   // metadata image [M128/128 * KT][128 lanes][4 u32]: box {4, 128, 1} = one (block, K-tile) image
        const uint64_t dims[3] = {4, 128, uint64_t(sp24_m128(a.M) / 128 * a.KT)};
        const uint64_t strides[2] = {16, 2048};
        const uint32_t box[3] = {4u, 128u, 1u};
        if (!make_tmap_nd(&tmE, a.meta, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, dims, strides, box,
                          CU_TENSOR_MAP_SWIZZLE_NONE))
            return STEN_ERR_CUDA;
    }
    a.row_tiles = int((a.M + Cfg::kBM - 1) / Cfg::kBM);
    a.col_tiles = int((a.N + Cfg::kBN - 1) / Cfg::kBN);
    const int ntiles = a.row_tiles * a.col_tiles;
    auto kern = spmm_sp24_2sm_kernel<TC, ST>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(Cfg::kSmem)) != cudaSuccess)
        return STEN_ERR_CUDA;
    const int pairs = ntiles < num_sms() / 2 ? ntiles : num_sms() / 2;
    cudaLaunchConfig_t cfg;
    memset(&cfg, 0, sizeof(cfg));
    cfg.gridDim = dim3(unsigned(2 * pairs));
    cfg.blockDim = dim3(Cfg::kThreads);
    cfg.dynamicSmemBytes = Cfg::kSmem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    if (cudaLaunchKernelEx(&cfg, kern, a, tmA, tmB, tmC, tmE) != cudaSuccess) return STEN_ERR_CUDA;
    return STEN_OK;
}

template <typename TC>
sten_status launch_sp24_tile(const Sp24Args& a, int tile, cudaStream_t st) {
    switch (tile) {
        case 1: return launch_sp24<TC, 2, 192, 4>(a, st);
        case 2: return launch_sp24<TC, 2, 128, 5>(a, st);
        case 3: return launch_sp24<TC, 3, 128, 4>(a, st);
        case 4: return launch_sp24<TC, 1, 256, 4>(a, st);
        case 5: return launch_sp24<TC, 1, 128, 6>(a, st);
        case 6: return launch_sp24_2sm<TC, 3>(a, st);
        default: return STEN_ERR_UNSUPPORTED;
    }
}

}  // namespace

extern "C" {

sten_status sten_sp24_packed_size(sten_nmg f, int64_t M, int64_t K, int64_t* v24_bytes, int64_t* meta_bytes) {
    if (!v24_bytes || !meta_bytes) return STEN_ERR_INVALID_ARG;
    if (f.n < 1 || f.n >= f.m || f.m > 16 || f.g < 1) return STEN_ERR_INVALID_ARG;
    if (M < 0 || K < 0 || M % f.g != 0 || K % f.m != 0) return STEN_ERR_SHAPE;
    if (!sp24_compatible(f.n, f.m)) return STEN_ERR_UNSUPPORTED;
    *v24_bytes = sp24_m128(M) * (sp24_k128(K) / 2) * 2;
    *meta_bytes = sp24_m128(M) / 128 * (sp24_k128(K) / 128) * 2048;
    return STEN_OK;
}

sten_status sten_sp24_pack(sten_nmg f, sten_dtype dt, const void* values, const uint8_t* idx, int64_t M, int64_t K,
                           void* v24, uint32_t* meta, void* stream) {
    int64_t vb, mbytes;
    sten_status s = sten_sp24_packed_size(f, M, K, &vb, &mbytes);
    if (s) return s;
    if (dt != STEN_BF16) return STEN_ERR_UNSUPPORTED;
    if (M * K > 0 && (!values || !idx)) return STEN_ERR_INVALID_ARG;
    if (vb > 0 && (!v24 || !meta)) return STEN_ERR_INVALID_ARG;
    if ((reinterpret_cast<uintptr_t>(v24) & 3u) != 0 || (reinterpret_cast<uintptr_t>(meta) & 3u) != 0)
        return STEN_ERR_UNSUPPORTED;
    if (vb == 0) return STEN_OK;
    const int64_t words = mbytes / 4;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const unsigned grid = unsigned((words + 255) / 256);
    const bf16_t* V = static_cast<const bf16_t*>(values);
    bf16_t* O = static_cast<bf16_t*>(v24);
    if (f.n == 1) sp24_pack_kernel<1><<<grid, 256, 0, st>>>(V, idx, M, K, 1, f.m, f.g, O, meta);
    else sp24_pack_kernel<2><<<grid, 256, 0, st>>>(V, idx, M, K, 2, f.m, f.g, O, meta);
    return cudaGetLastError() == cudaSuccess ? STEN_OK : STEN_ERR_CUDA;
}

sten_status sten_spmm_sp24(const void* v24, const uint32_t* meta, int64_t M, int64_t K, const void* B, int64_t ldb,
                           int64_t N, void* C, int64_t ldc, sten_dtype c_dt, int32_t tile, void* stream) {
    return sten_spmm_sp24_epilogue(v24, meta, M, K, B, ldb, N, C, ldc, c_dt, nullptr, 0, nullptr, 0, tile, stream);
}

sten_status sten_spmm_sp24_epilogue(const void* v24, const uint32_t* meta, int64_t M, int64_t K, const void* B,
                                    int64_t ldb, int64_t N, void* C, int64_t ldc, sten_dtype c_dt, const float* bias,
                                    int32_t act, const void* residual, int64_t ldr, int32_t tile, void* stream) {
    if (act < 0 || act > 2) return STEN_ERR_INVALID_ARG;
    if (residual && (ldr < N || residual == C)) return residual == C ? STEN_ERR_INVALID_ARG : STEN_ERR_SHAPE;
    if (M < 0 || K < 0 || N < 0 || ldb < N || ldc < N) return STEN_ERR_SHAPE;
    if (c_dt != STEN_F32 && c_dt != STEN_BF16) return STEN_ERR_INVALID_ARG;
    if ((M * K > 0 && (!v24 || !meta)) || (K * N > 0 && !B) || (M * N > 0 && !C)) return STEN_ERR_INVALID_ARG;
    // default: the 2-SM pair kernel when K is long enough to amortise its per-tile epilogue (one D
    // buffer per pair), else the 256 x 192 1-SM tile (measured on C3)
    if (tile == 0) tile = K >= 2048 ? 6 : 1;
    if (tile < 1 || tile > 6) return STEN_ERR_UNSUPPORTED;
    if (K * N > 0 && (!al16(B) || (ldb * 2) % 16 != 0)) return STEN_ERR_UNSUPPORTED;
    if (M * K > 0 && (!al16(v24) || !al16(meta))) return STEN_ERR_UNSUPPORTED;
    if (M * N > 0 && (!al16(C) || (ldc * (c_dt == STEN_F32 ? 4 : 2)) % 16 != 0)) return STEN_ERR_UNSUPPORTED;
    if (M == 0 || N == 0) return STEN_OK;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (K == 0) {
        if (cudaMemset2DAsync(C, size_t(ldc) * (c_dt == STEN_F32 ? 4 : 2), 0, size_t(N) * (c_dt == STEN_F32 ? 4 : 2),
                              size_t(M), st) != cudaSuccess)
            return STEN_ERR_CUDA;
        return STEN_OK;
    }
    Sp24Args a;
    memset(&a, 0, sizeof(a));
    a.v24 = v24; a.meta = meta; a.B = B; a.C = C;
    a.M = M; a.K = K; a.N = N; a.ldb = ldb; a.ldc = ldc;
    a.KT = sp24_k128(K) / 128;
    a.Kc = sp24_k128(K) / 2;
    const size_t sc = c_dt == STEN_F32 ? 4 : 2;
    a.c_vec = al16(C) && (size_t(ldc) * sc) % 16 == 0;
    a.bias = bias;
    a.act = act;
    a.residual = residual;
    a.ldr = ldr;
    if (const char* e = getenv("STEN_SP24_EXP")) a.exp = atoi(e);     // debug timing experiments only
    return c_dt == STEN_F32 ? launch_sp24_tile<float>(a, tile, st) : launch_sp24_tile<bf16_t>(a, tile, st);
}

}  // extern "C"
