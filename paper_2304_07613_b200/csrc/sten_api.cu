// sten_api.cu -- the C ABI declared in include/sten.h: argument validation,
// plan selection, kernel instantiation and launch on the caller's stream.
#include "sten.h"

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <vector>

#include "common.cuh"
#include "tma_host.h"
#include "sparsify.cuh"
#include "spmm_simt.cuh"
#include "spmm_mma.cuh"
#include "spmm_tc.cuh"

using namespace sten;

namespace {

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

inline size_t dt_size(sten_dtype d) { return d == STEN_F32 ? 4 : 2; }

inline bool dtype_ok(int d) { return d == STEN_F32 || d == STEN_BF16; }

inline bool m_supported(int m) {
    return m == 2 || m == 4 || m == 6 || m == 8 || m == 10 || m == 12 || m == 16;
}

sten_status check_format(sten_nmg f) {
    if (f.n < 1 || f.m > 16 || f.n >= f.m || f.g < 1) return STEN_ERR_INVALID_ARG;
    if (!m_supported(f.m)) return STEN_ERR_UNSUPPORTED;
    return STEN_OK;
}

sten_status check_shape(sten_nmg f, int64_t M, int64_t K) {
    if (M < 0 || K < 0) return STEN_ERR_SHAPE;
    if (M % f.g != 0 || K % f.m != 0) return STEN_ERR_SHAPE;
    return STEN_OK;
}

inline sten_status last_cuda() {
    return cudaGetLastError() == cudaSuccess ? STEN_OK : STEN_ERR_CUDA;
}

inline unsigned grid1d(int64_t threads) { return unsigned((threads + 255) / 256); }

// ---------------------------------------------------------------------------------------------
// K1 / K2 dispatch on (dtype, m)
// ---------------------------------------------------------------------------------------------
template <typename T, int MB, int NK>
void launch_sparsify_nk(const void* W, int64_t ldw, int64_t G, int64_t KB, sten_nmg f, void* values,
                        int64_t Kp, uint8_t* idx, int aligned, cudaStream_t st) {
    sparsify_grouped_nm_kernel<T, MB, NK><<<unsigned((G * KB + kSpBatchThreads - 1) / kSpBatchThreads),
                                            kSpBatchThreads, 0, st>>>(
        static_cast<const T*>(W), ldw, G, KB, f.n, f.g, static_cast<T*>(values), Kp, idx, aligned);
}

template <typename T, int MB>
void launch_sparsify(const void* W, int64_t ldw, int64_t G, int64_t KB, sten_nmg f, void* values,
                     int64_t Kp, uint8_t* idx, int aligned, cudaStream_t st) {
    // one vector store per row (n in {1, 2, 4}) when the bases are aligned to the vector width;
    // every row offset (r Kp + kb n) and idx offset ((G KB + kb) n) is a multiple of n
    auto ok = [&](int nk) {
        const uintptr_t va = reinterpret_cast<uintptr_t>(values), ia = reinterpret_cast<uintptr_t>(idx);
        return f.n == nk && va % (size_t(nk) * sizeof(T)) == 0 && ia % size_t(nk) == 0;
    };
    if (ok(1)) launch_sparsify_nk<T, MB, 1>(W, ldw, G, KB, f, values, Kp, idx, aligned, st);
    else if (ok(2)) launch_sparsify_nk<T, MB, 2>(W, ldw, G, KB, f, values, Kp, idx, aligned, st);
    else if constexpr (MB > 4) {
        if (ok(4)) launch_sparsify_nk<T, MB, 4>(W, ldw, G, KB, f, values, Kp, idx, aligned, st);
        else launch_sparsify_nk<T, MB, 0>(W, ldw, G, KB, f, values, Kp, idx, aligned, st);
    } else launch_sparsify_nk<T, MB, 0>(W, ldw, G, KB, f, values, Kp, idx, aligned, st);
}

template <typename T>
bool dispatch_sparsify(int m, const void* W, int64_t ldw, int64_t G, int64_t KB, sten_nmg f,
                       void* values, int64_t Kp, uint8_t* idx, int aligned, cudaStream_t st) {
    switch (m) {
        case 2: launch_sparsify<T, 2>(W, ldw, G, KB, f, values, Kp, idx, aligned, st); return true;
        case 4: launch_sparsify<T, 4>(W, ldw, G, KB, f, values, Kp, idx, aligned, st); return true;
        case 6: launch_sparsify<T, 6>(W, ldw, G, KB, f, values, Kp, idx, aligned, st); return true;
        case 8: launch_sparsify<T, 8>(W, ldw, G, KB, f, values, Kp, idx, aligned, st); return true;
        case 10: launch_sparsify<T, 10>(W, ldw, G, KB, f, values, Kp, idx, aligned, st); return true;
        case 12: launch_sparsify<T, 12>(W, ldw, G, KB, f, values, Kp, idx, aligned, st); return true;
        case 16: launch_sparsify<T, 16>(W, ldw, G, KB, f, values, Kp, idx, aligned, st); return true;
    }
    return false;
}

template <typename T, int MB>
void launch_densify(const void* values, const uint8_t* idx, int64_t M, int64_t KB, sten_nmg f,
                    int64_t Kp, void* W, int64_t ldw, bool aligned, cudaStream_t st) {
    densify_grouped_nm_kernel<T, MB><<<grid1d(M * KB), 256, 0, st>>>(
        static_cast<const T*>(values), idx, M, KB, f.n, f.g, Kp, static_cast<T*>(W), ldw, aligned);
}

template <typename T>
bool dispatch_densify(int m, const void* values, const uint8_t* idx, int64_t M, int64_t KB,
                      sten_nmg f, int64_t Kp, void* W, int64_t ldw, bool aligned, cudaStream_t st) {
    switch (m) {
        case 2: launch_densify<T, 2>(values, idx, M, KB, f, Kp, W, ldw, aligned, st); return true;
        case 4: launch_densify<T, 4>(values, idx, M, KB, f, Kp, W, ldw, aligned, st); return true;
        case 6: launch_densify<T, 6>(values, idx, M, KB, f, Kp, W, ldw, aligned, st); return true;
        case 8: launch_densify<T, 8>(values, idx, M, KB, f, Kp, W, ldw, aligned, st); return true;
        case 10: launch_densify<T, 10>(values, idx, M, KB, f, Kp, W, ldw, aligned, st); return true;
        case 12: launch_densify<T, 12>(values, idx, M, KB, f, Kp, W, ldw, aligned, st); return true;
        case 16: launch_densify<T, 16>(values, idx, M, KB, f, Kp, W, ldw, aligned, st); return true;
    }
    return false;
}

// ---------------------------------------------------------------------------------------------
// SpMM dispatch
// ---------------------------------------------------------------------------------------------
int simt_rows_per_warp(int g) {
    if (g % 8 == 0) return 8;
    if (g % 4 == 0) return 4;
    if (g % 2 == 0) return 2;
    return 1;
}

// SIMT tile variants (plan.tile), every one with 64 fp32 accumulators per consumer lane
// (warps = consumers + 1 producer):
//   1: 8 warps,  TN = 8, BM = 56,  BN = 256 (fp32) / 256 (bf16)  -- 2 CTAs / SM
//   2: 16 warps, TN = 8, BM = 120, BN = 256                      -- 1 CTA / SM
//   3: 16 warps, TN = 4, BM = 240, BN = 128 (fp32 only)          -- 1 CTA / SM
// and two narrow tiles for small grids (more CTAs per output without split-K), fp32 only:
//   4: 8 warps,  TN = 4, BM = 112, BN = 128 (64 accumulators)    -- 2 CTAs / SM
//   5: 8 warps,  TN = 4, BM = 56,  BN = 128 (32 accumulators)    -- 2 CTAs / SM
//   6: 8 warps,  TN = 4, BM = 56,  BN = 128 (32 accumulators)    -- 3 CTAs / SM (21 consumer warps)
//   7: 12 warps, TN = 4, BM = 88,  BN = 128 (32 accumulators)    -- 2 CTAs / SM (22 consumer warps)
struct SimtTile { int warps, tn, bm, per_sm; };
constexpr SimtTile kSimtTiles[8] = {{0, 0, 0, 0},   {8, 8, 56, 2}, {16, 8, 120, 1}, {16, 4, 240, 1},
                                    {8, 4, 112, 2}, {8, 4, 56, 2}, {8, 4, 56, 3},   {12, 4, 88, 2}};
constexpr int kSimtNumTiles = 7;
constexpr int kMaxSplit = 8;              // portable thread-block cluster size
#ifndef STEN_SLAB_COST
#define STEN_SLAB_COST 6.0
#endif

inline bool simt_tile_ok(int tile, sten_dtype ab) {
    if (tile < 1 || tile > kSimtNumTiles) return false;
    return !(tile >= 3 && ab == STEN_BF16);
}

// Shared-memory budget per CTA: tiles 1, 4, 5 run two CTAs per SM, tiles 2/3 one.
constexpr size_t kSmemPerSM = 233472;                                    // 228 KB
inline size_t simt_smem_budget(int tile) {
    const int per_sm = kSimtTiles[tile].per_sm;
    return per_sm == 1 ? 232448 : kSmemPerSM / per_sm - 1024;
}

// m-blocks per K-slab for the SIMT kernel: the largest multiple of 4/gcd(n,4) whose
// STAGES-deep ring fits the CTA's shared-memory budget (B slab <= 256 rows, TMA box limit).
int simt_slab_blocks(sten_nmg f, sten_dtype ab, int tile) {
    const int q = 4 / gcd_int(f.n, 4);
    const int rg = simt_rows_per_warp(f.g);
    const int warps = kSimtTiles[tile].warps, bm = kSimtTiles[tile].bm;
    const int esz = ab == STEN_F32 ? 4 : 2;
    const int bn = 32 * kSimtTiles[tile].tn;
    const int nsub = bm / rg;
    (void)warps;
    int best = q;
    for (int kbs = q; kbs * f.m <= 256 && kbs * f.n <= 64; kbs += q) {
        const SimtLayout L(bm, bn, nsub, esz, 3, kbs, f.n, f.m);
        if (L.total > simt_smem_budget(tile)) break;
        best = kbs;
    }
    return best;
}

// tensor maps of one SIMT problem (B slab box, values box) and its shared-memory size
template <typename TAB, int RG, int TN, int SUB, int WARPS>
sten_status prep_simt(SpmmArgs& a, CUtensorMap* tmB, CUtensorMap* tmV, size_t* smem) {
    using Cfg = SimtCfg<TAB, RG, TN, SUB, WARPS>;
    const SimtSmem<TAB, RG, TN, SUB, WARPS> L(a.kbs, a.n, a.m);
    if (L.total > 227 * 1024) return STEN_ERR_UNSUPPORTED;
    const CUtensorMapDataType tdt = sizeof(TAB) == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
    constexpr size_t s = sizeof(TAB);
    memset(tmB, 0, sizeof(*tmB));
    memset(tmV, 0, sizeof(*tmV));
    if (!make_tmap_2d(tmB, a.B, tdt, uint64_t(a.N), uint64_t(a.K), uint64_t(a.ldb) * s, Cfg::kBN, uint32_t(L.bk)))
        return STEN_ERR_CUDA;
    // values as a 3-D tensor {KU, M, Kp/KU} (strides Kp*s, KU*s) so the box lands as [ksp/KU][BM][KU];
    // needs 16-byte inner boxes and strides, else the kernel stages values with cp.async
    constexpr int KU = Cfg::kKU;
    a.v_tma = KU * s == 16 && (size_t(a.Kp) * s) % 16 == 0 && aligned16(a.values) &&
              make_tmap_3d(tmV, a.values, tdt, uint64_t(KU), uint64_t(a.M), uint64_t(a.Kp / KU),
                           uint64_t(a.Kp) * s, uint64_t(KU) * s, uint32_t(KU), Cfg::kBM, uint32_t(L.ksp / KU));
    *smem = L.total;
    return STEN_OK;
}

template <typename TAB, typename TC, int RG, int TN, int SUB, int WARPS, int MINB = (WARPS == 8 ? 2 : 1)>
sten_status launch_simt_cfg(SpmmArgs a, cudaStream_t st) {
    using Cfg = SimtCfg<TAB, RG, TN, SUB, WARPS>;
    CUtensorMap tmB, tmV;
    size_t smem_bytes = 0;
    sten_status ps = prep_simt<TAB, RG, TN, SUB, WARPS>(a, &tmB, &tmV, &smem_bytes);
    if (ps) return ps;
    struct { size_t total; } L = {smem_bytes};
    auto kern = spmm_simt_kernel<TAB, TC, RG, TN, SUB, WARPS, MINB>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(L.total)) != cudaSuccess)
        return STEN_ERR_CUDA;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned((a.N + Cfg::kBN - 1) / Cfg::kBN), unsigned((a.M + Cfg::kBM - 1) / Cfg::kBM),
                       unsigned(a.split));
    cfg.blockDim = dim3(Cfg::kThreads);                        // consumers + the producer warp
    cfg.dynamicSmemBytes = L.total;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    int na = 0;
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;   // PDL: overlap the prologue with
    attr[na].val.programmaticStreamSerializationAllowed = 1;            // the previous kernel (sparsify)
    ++na;
    if (a.split > 1) {
        attr[na].id = cudaLaunchAttributeClusterDimension;
        attr[na].val.clusterDim.x = 1;
        attr[na].val.clusterDim.y = 1;
        attr[na].val.clusterDim.z = unsigned(a.split);
        ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    if (cudaLaunchKernelEx(&cfg, kern, a, tmB, tmV) != cudaSuccess) return STEN_ERR_CUDA;
    return last_cuda();
}

// grouped launch of `count` fp32 problems sharing the kernel variant (sten_spmm_grouped_nm_batched)
template <int RG, int TN, int SUB, int WARPS, int MINB = (WARPS == 8 ? 2 : 1)>
sten_status launch_simt_batch_cfg(SpmmArgs* as, int count, cudaStream_t st) {
    using Cfg = SimtCfg<float, RG, TN, SUB, WARPS>;
    SpmmBatch bt;                  // the kernel parameter (copied at launch; no library state)
    memset(&bt, 0, sizeof(bt));
    size_t smem_max = 0;
    int tiles = 0;
    for (int p = 0; p < count; ++p) {
        size_t sm = 0;
        sten_status ps = prep_simt<float, RG, TN, SUB, WARPS>(as[p], &bt.tmB[p], &bt.tmV[p], &sm);
        if (ps) return ps;
        bt.a[p] = as[p];
        const int ntx = int((as[p].N + Cfg::kBN - 1) / Cfg::kBN), nty = int((as[p].M + Cfg::kBM - 1) / Cfg::kBM);
        bt.tile0[p] = tiles;
        bt.ntx[p] = ntx;
        tiles += ntx * nty * as[p].split;
        smem_max = std::max(smem_max, sm);
    }
    bt.tile0[count] = tiles;
    bt.count = count;
    if (tiles == 0) return STEN_OK;
    auto kern = spmm_simt_batched_kernel<float, float, RG, TN, SUB, WARPS, MINB>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem_max)) != cudaSuccess)
        return STEN_ERR_CUDA;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(tiles));
    cfg.blockDim = dim3(Cfg::kThreads);
    cfg.dynamicSmemBytes = smem_max;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;   // PDL: the prologue overlaps the
    attr[0].val.programmaticStreamSerializationAllowed = 1;            // sparsifier's tail
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, kern, bt) != cudaSuccess) return STEN_ERR_CUDA;
    return last_cuda();
}

// mixed grouped launch: tile 2 (variant 0) and tile 3 (variant 1) problems in one launch
template <int RG>
sten_status launch_simt_batch_mixed(SpmmArgs* as, const int* tiles_of, int count, cudaStream_t st) {
    constexpr int SUB8 = 8 / RG;
    using CfgA = SimtCfg<float, RG, 8, SUB8, 16>;
    using CfgB = SimtCfg<float, RG, 4, 2 * SUB8, 16>;
    SpmmBatch bt;
    memset(&bt, 0, sizeof(bt));
    size_t smem_max = 0;
    int tiles = 0;
    for (int p = 0; p < count; ++p) {
        size_t sm = 0;
        const bool vb = tiles_of[p] == 3;
        sten_status ps = vb ? prep_simt<float, RG, 4, 2 * SUB8, 16>(as[p], &bt.tmB[p], &bt.tmV[p], &sm)
                            : prep_simt<float, RG, 8, SUB8, 16>(as[p], &bt.tmB[p], &bt.tmV[p], &sm);
        if (ps) return ps;
        bt.a[p] = as[p];
        const int bm = vb ? CfgB::kBM : CfgA::kBM, bn = vb ? CfgB::kBN : CfgA::kBN;
        const int ntx = int((as[p].N + bn - 1) / bn), nty = int((as[p].M + bm - 1) / bm);
        bt.tile0[p] = tiles;
        bt.ntx[p] = ntx;
        bt.var[p] = vb ? 1 : 0;
        tiles += ntx * nty * as[p].split;
        smem_max = std::max(smem_max, sm);
    }
    bt.tile0[count] = tiles;
    bt.count = count;
    if (tiles == 0) return STEN_OK;
    auto kern = spmm_simt_batched2_kernel<float, float, RG, 8, SUB8, 4, 2 * SUB8, 16>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem_max)) != cudaSuccess)
        return STEN_ERR_CUDA;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(tiles));
    cfg.blockDim = dim3(16 * 32);
    cfg.dynamicSmemBytes = smem_max;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, kern, bt) != cudaSuccess) return STEN_ERR_CUDA;
    return last_cuda();
}

template <int RG>
sten_status launch_simt_batch_rg(SpmmArgs* as, int count, int tile, cudaStream_t st) {
    constexpr int SUB8 = 8 / RG;
    switch (tile) {
        case 1: return launch_simt_batch_cfg<RG, 8, SUB8, 8>(as, count, st);
        case 2: return launch_simt_batch_cfg<RG, 8, SUB8, 16>(as, count, st);
        case 3: return launch_simt_batch_cfg<RG, 4, 2 * SUB8, 16>(as, count, st);
    }
    return STEN_ERR_UNSUPPORTED;
}

template <typename TAB, typename TC, int RG>
sten_status launch_simt_rg(const SpmmArgs& a, int tile, cudaStream_t st) {
    constexpr int SUB8 = 8 / RG;                 // TN = 8: RG * 8 * SUB8 = 64 accumulators
    switch (tile) {
        case 1: return launch_simt_cfg<TAB, TC, RG, 8, SUB8, 8>(a, st);
        case 2: return launch_simt_cfg<TAB, TC, RG, 8, SUB8, 16>(a, st);
        case 3:
            if constexpr (sizeof(TAB) == 4) return launch_simt_cfg<TAB, TC, RG, 4, 2 * SUB8, 16>(a, st);
            else return STEN_ERR_UNSUPPORTED;
        case 4:
            if constexpr (sizeof(TAB) == 4) return launch_simt_cfg<TAB, TC, RG, 4, 2 * SUB8, 8>(a, st);
            else return STEN_ERR_UNSUPPORTED;
        case 5:
            if constexpr (sizeof(TAB) == 4) return launch_simt_cfg<TAB, TC, RG, 4, SUB8, 8>(a, st);
            else return STEN_ERR_UNSUPPORTED;
        case 6:
            if constexpr (sizeof(TAB) == 4) return launch_simt_cfg<TAB, TC, RG, 4, SUB8, 8, 3>(a, st);
            else return STEN_ERR_UNSUPPORTED;
        case 7:
            if constexpr (sizeof(TAB) == 4) return launch_simt_cfg<TAB, TC, RG, 4, SUB8, 12, 2>(a, st);
            else return STEN_ERR_UNSUPPORTED;
    }
    return STEN_ERR_UNSUPPORTED;
}

template <typename TAB, typename TC>
sten_status launch_simt(const SpmmArgs& a, int tile, cudaStream_t st) {
    switch (simt_rows_per_warp(a.g)) {
        case 8: return launch_simt_rg<TAB, TC, 8>(a, tile, st);
        case 4: return launch_simt_rg<TAB, TC, 4>(a, tile, st);
        case 2: return launch_simt_rg<TAB, TC, 2>(a, tile, st);
        default: return launch_simt_rg<TAB, TC, 1>(a, tile, st);
    }
}

template <typename TC>
__global__ void zero_fill_kernel(TC* C, int64_t M, int64_t N, int64_t ldc) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= M * N) return;
    const int64_t r = i / N, c = i - r * N;
    C[r * ldc + c] = TC(0);
}

constexpr int kNumSMs = 148;

// Pick split_k in [1, max_split] for `tiles` output tiles of `slots` resident CTAs
// per wave over KB m-blocks: minimise waves(S) * ceil(KB/S) * t_kb + reduce(S).
int choose_split(int64_t tiles, int64_t slots, int64_t KB, int max_split, double t_kb_clk,
                 double reduce_clk) {
    int best = 1;
    double best_t = 1e300;
    for (int S = 1; S <= max_split && S <= KB; ++S) {
        const double waves = double((tiles * S + slots - 1) / slots);
        const double t = waves * double((KB + S - 1) / S) * t_kb_clk + (S > 1 ? reduce_clk : 0.0);
        if (t < best_t * 0.97) { best_t = t; best = S; }
    }
    return best;
}

sten_status plan_auto(sten_nmg f, sten_dtype ab, int64_t M, int64_t K, int64_t N, sten_dtype c,
                      sten_spmm_plan* p) {
    (void)c;
    memset(p, 0, sizeof(*p));
    const int64_t KB = K / f.m;
    const double d = double(f.n) / f.m;
    if (ab == STEN_BF16 && tc_supported(f.g) && KB % 8 == 0 && K > 0 &&
        ((M + 255) / 256) * ((N + 127) / 128) >= kNumSMs) {
        // K5 tcgen05 (no split-K): needs at least one full wave of 256 x 128 tiles; largest RB | g
        p->algo = STEN_ALGO_TCGEN05;
        p->tile = f.g % 64 == 0 ? 3 : f.g % 32 == 0 ? 2 : 1;
        p->split_k = 1;
        return STEN_OK;
    }
    if (ab == STEN_BF16 && mma_supported(f.g)) {
        p->algo = STEN_ALGO_MMA_SYNC;
        p->tile = f.g % 16 == 0 ? 2 : 1;
        const int64_t bm = 256, bn = 128;
        const int64_t tiles = ((M + bm - 1) / bm) * ((N + bn - 1) / bn);
        const double t_kb = double(bm * bn * f.n) / 700.0;      // clk per m-block per CTA (~700 MAC/clk/SM)
        const double red = double(bm * bn * 4) / 15.0;          // DSMEM reduce of the tile
        p->split_k = choose_split(tiles, kNumSMs, KB, kMaxSplit, t_kb, red);
        return STEN_OK;
    }
    p->algo = STEN_ALGO_SIMT;
    // Cost model (cycles) over tile x split, calibrated on B200 (tools/sweep.py):
    //   per-CTA FMA rate: min(measured steady-state rate, L2 share / bytes per FMA)
    //   CTA time = ceil(KB/S) m-blocks of work + fixed prologue/epilogue + DSMEM reduce (S > 1)
    //   kernel   = waves * CTA time, waves = ceil(tiles * S / resident CTAs)
    const double esz = ab == STEN_F32 ? 4.0 : 2.0;
    const double base_rate[4] = {0.0, 32.0, 70.0, 56.0};            // FMA/clk per CTA at 2:4
    const double l2_bytes_per_clk_sm = 34.0;                          // ~10 TB/s over 148 SMs
    double best_t = 1e300;
    int best_tile = 1, best_split = 1;
    for (int tile = 1; tile <= 3; ++tile) {
        if (!simt_tile_ok(tile, ab)) continue;
        const double bm = kSimtTiles[tile].bm, bn = 32.0 * kSimtTiles[tile].tn;
        const int per_sm = tile == 1 ? 2 : 1;
        const double bytes_per_fma = esz / (bm * d) + esz / bn;
        const double rate = std::min(base_rate[tile], l2_bytes_per_clk_sm / per_sm / bytes_per_fma);
        const int64_t tiles = ((M + int64_t(bm) - 1) / int64_t(bm)) * ((N + int64_t(bn) - 1) / int64_t(bn));
        const int64_t slots = int64_t(kNumSMs) * per_sm;
        for (int S = 1; S <= kMaxSplit && S <= KB; ++S) {
            const double waves = double((tiles * S + slots - 1) / slots);
            const double work = double((KB + S - 1) / S) * bm * bn * f.n / rate;
            const double red = S > 1 ? bm * bn * 4.0 / 15.0 : 0.0;
            const double t = waves * (work + 4000.0 + red);
            if (t < best_t * 0.98) { best_t = t; best_tile = tile; best_split = S; }
        }
    }
    p->tile = best_tile;
    p->split_k = best_split;
    return STEN_OK;
}

sten_status spmm_impl(sten_nmg f, sten_dtype ab_dt, const void* values, const uint8_t* idx, int64_t M,
                      int64_t K, const void* B, int64_t ldb, int64_t N, void* C, int64_t ldc,
                      sten_dtype c_dt, const sten_spmm_plan* plan_in, cudaStream_t st,
                      void* const* C_peers = nullptr, int npeers = 0, int64_t col0 = 0,
                      const float* bias = nullptr, int act = 0, const void* residual = nullptr,
                      int64_t ldr = 0) {
    sten_status s = check_format(f);
    if (s) return s;
    if (!dtype_ok(ab_dt) || !dtype_ok(c_dt)) return STEN_ERR_INVALID_ARG;
    if ((s = check_shape(f, M, K))) return s;
    if (N < 0 || ldb < N || ldc < N) return STEN_ERR_SHAPE;
    // a buffer may be NULL only when it is empty
    if ((M * K > 0 && (!values || !idx)) || (K * N > 0 && !B) || (M * N > 0 && !C)) return STEN_ERR_INVALID_ARG;
    const size_t sab = dt_size(ab_dt), sc = dt_size(c_dt);
    if (K * N > 0 && (!aligned16(B) || (ldb * int64_t(sab)) % 16 != 0)) return STEN_ERR_UNSUPPORTED;
    if ((reinterpret_cast<uintptr_t>(idx) & 3u) != 0) return STEN_ERR_UNSUPPORTED;
    sten_spmm_plan plan;
    plan_auto(f, ab_dt, M, K, N, c_dt, &plan);
    if (plan.algo == STEN_ALGO_TCGEN05 && !aligned16(values) && (!plan_in || plan_in->algo == STEN_ALGO_AUTO)) {
        // automatic choice only: tcgen05 TMA-loads the values, which needs a 16-byte aligned base
        plan.algo = STEN_ALGO_MMA_SYNC;
        plan.tile = f.g % 16 == 0 ? 2 : 1;
        plan.split_k = 1;
    }
    if (plan_in) {
        if (plan_in->algo != STEN_ALGO_AUTO && plan_in->algo != plan.algo) {
            plan.algo = plan_in->algo;
            plan.tile = plan.algo == STEN_ALGO_SIMT ? 1 : (f.g % 16 == 0 ? 2 : 1);
            if (plan.algo == STEN_ALGO_TCGEN05) {
                plan.tile = f.g % 64 == 0 ? 3 : f.g % 32 == 0 ? 2 : 1;
                plan.split_k = 1;
            }
        }
        if (plan_in->tile > 0) plan.tile = plan_in->tile;
        if (plan_in->split_k > 0) plan.split_k = plan_in->split_k;
    }
    if (plan.algo == STEN_ALGO_MMA_SYNC && (ab_dt != STEN_BF16 || !mma_supported(f.g)))
        return STEN_ERR_UNSUPPORTED;
    if (plan.algo == STEN_ALGO_TCGEN05) {
        // tile t -> RB = 8 << t rows per MMA (16/32/64), RB | g; one K partition (no split-K)
        if (ab_dt != STEN_BF16 || !tc_supported(f.g) || plan.tile < 1 || plan.tile > 3 ||
            f.g % (8 << plan.tile) != 0 || plan.split_k != 1)
            return STEN_ERR_UNSUPPORTED;
    }
    if (plan.algo != STEN_ALGO_SIMT && plan.algo != STEN_ALGO_MMA_SYNC && plan.algo != STEN_ALGO_TCGEN05)
        return STEN_ERR_UNSUPPORTED;
    if (plan.algo == STEN_ALGO_SIMT && (!simt_tile_ok(plan.tile, ab_dt) || plan.split_k > kMaxSplit))
        return STEN_ERR_UNSUPPORTED;
    if (plan.algo == STEN_ALGO_MMA_SYNC && !(plan.tile == 1 || (plan.tile == 2 && f.g % 16 == 0)))
        return STEN_ERR_UNSUPPORTED;
    if (plan.split_k < 1 || plan.split_k > kMaxSplit) return STEN_ERR_UNSUPPORTED;
    if (M == 0 || N == 0) return STEN_OK;
    if (K == 0) {
        if (c_dt == STEN_F32) zero_fill_kernel<float><<<grid1d(M * N), 256, 0, st>>>(static_cast<float*>(C), M, N, ldc);
        else zero_fill_kernel<bf16_t><<<grid1d(M * N), 256, 0, st>>>(static_cast<bf16_t*>(C), M, N, ldc);
        return last_cuda();
    }

    SpmmArgs a;
    memset(&a, 0, sizeof(a));
    a.values = values; a.idx = idx; a.B = B; a.C = C;
    a.M = M; a.K = K; a.N = N; a.ldb = ldb; a.ldc = ldc;
    a.n = f.n; a.m = f.m; a.g = f.g;
    a.KB = K / f.m; a.Kp = a.KB * f.n;
    a.c_vec = aligned16(C) && (ldc * int64_t(sc)) % 16 == 0;
    a.bias = bias;
    a.act = act;
    a.residual = residual;
    a.ldr = ldr;
    if (npeers > 0) {
        // fused all-gather: every peer buffer receives this rank's columns [col0, col0 + N)
        a.npeer = npeers;
        a.c_vec = (ldc * int64_t(sc)) % 16 == 0;
        for (int p = 0; p < npeers; ++p) {
            a.C_peer[p] = static_cast<char*>(C_peers[p]) + col0 * int64_t(sc);
            a.c_vec = a.c_vec && aligned16(a.C_peer[p]);
        }
    }

    if (plan.algo == STEN_ALGO_SIMT) {
        a.v_async = (a.Kp % 4 == 0) && ((reinterpret_cast<uintptr_t>(values) & (4 * sab - 1)) == 0);
        a.idx_bytes = (M / f.g) * a.KB * f.n;
        a.kbs = simt_slab_blocks(f, ab_dt, plan.tile);
        // split-K parts are balanced runs of whole slabs (sizes differ by at most one slab)
        const int64_t slabs = (a.KB + a.kbs - 1) / a.kbs;
        a.split = int(slabs < plan.split_k ? slabs : plan.split_k);
        a.kb_per_split = ((slabs + a.split - 1) / a.split) * a.kbs;   // largest part (informational)
        if (ab_dt == STEN_F32) s = c_dt == STEN_F32 ? launch_simt<float, float>(a, plan.tile, st)
                                                    : launch_simt<float, bf16_t>(a, plan.tile, st);
        else s = c_dt == STEN_F32 ? launch_simt<bf16_t, float>(a, plan.tile, st)
                                  : launch_simt<bf16_t, bf16_t>(a, plan.tile, st);
        return s;
    }

    if ((npeers > 0 || bias || act || residual) && plan.algo != STEN_ALGO_SIMT) return STEN_ERR_UNSUPPORTED;
    if (plan.algo == STEN_ALGO_TCGEN05) {
        // B slabs are TMA-loaded in groups of 8 m-blocks (K % 8m == 0); values rows by TMA
        // (16-byte aligned base; the row stride K' = n KB is then a multiple of 16 bytes)
        if (a.KB % 8 != 0 || !aligned16(values)) return STEN_ERR_UNSUPPORTED;
        a.v_async = true;
        a.idx_bytes = (M / f.g) * a.KB * f.n;
        return c_dt == STEN_F32 ? launch_tc<float>(a, plan.tile, st) : launch_tc<bf16_t>(a, plan.tile, st);
    }
    // mma.sync path (split-K partials reduced over the cluster inside the kernel)
    a.v_async = (a.Kp % 8 == 0) && aligned16(values);
    a.idx_bytes = (M / f.g) * a.KB * f.n;
    return c_dt == STEN_F32 ? launch_mma<float>(a, plan.tile, plan.split_k, st)
                            : launch_mma<bf16_t>(a, plan.tile, plan.split_k, st);
}

}  // namespace

extern "C" {

sten_status sten_sparsify_grouped_nm(sten_nmg f, sten_dtype dt, const void* W, int64_t M, int64_t K,
                                     int64_t ldw, void* values, uint8_t* idx, void* stream) {
    sten_status s = check_format(f);
    if (s) return s;
    if (!dtype_ok(dt)) return STEN_ERR_INVALID_ARG;
    if ((s = check_shape(f, M, K))) return s;
    if (ldw < K) return STEN_ERR_SHAPE;
    if (M * K > 0 && (!W || !values || !idx)) return STEN_ERR_INVALID_ARG;
    const int64_t G = M / f.g, KB = K / f.m, Kp = KB * f.n;
    if (G == 0 || KB == 0) return STEN_OK;
    // 2: 32-byte aligned block starts (256-bit loads when m*s is a multiple of 32), 1: 16-byte
    const int64_t ldw_bytes = ldw * int64_t(dt_size(dt));
    const uintptr_t wa = reinterpret_cast<uintptr_t>(W);
    const int aligned = (wa % 32 == 0 && ldw_bytes % 32 == 0) ? 2 : (wa % 16 == 0 && ldw_bytes % 16 == 0) ? 1 : 0;
    cudaStream_t st = as_stream(stream);
    bool ok = dt == STEN_F32 ? dispatch_sparsify<float>(f.m, W, ldw, G, KB, f, values, Kp, idx, aligned, st)
                             : dispatch_sparsify<bf16_t>(f.m, W, ldw, G, KB, f, values, Kp, idx, aligned, st);
    if (!ok) return STEN_ERR_UNSUPPORTED;
    return last_cuda();
}

sten_status sten_sparsify_grouped_nm_batched(int32_t count, const sten_sparsify_problem* probs, sten_dtype dt,
                                             void* stream) {
    if (count < 1 || count > kMaxSparsifyBatch || !probs) return STEN_ERR_INVALID_ARG;
    if (!dtype_ok(dt)) return STEN_ERR_INVALID_ARG;
    // validate everything before any launch (no partial writes on an argument error)
    int nkc[kMaxSparsifyBatch], al[kMaxSparsifyBatch];
    for (int p = 0; p < count; ++p) {
        const sten_sparsify_problem& q = probs[p];
        sten_status s = check_format(q.f);
        if (s) return s;
        if ((s = check_shape(q.f, q.M, q.K))) return s;
        if (q.ldw < q.K) return STEN_ERR_SHAPE;
        if (q.M * q.K > 0 && (!q.W || !q.values || !q.idx)) return STEN_ERR_INVALID_ARG;
        if ((q.M / q.f.g) * (q.K / q.f.m) > int64_t(0x7fffffff)) return STEN_ERR_UNSUPPORTED;
        const int64_t ldw_bytes = q.ldw * int64_t(dt_size(dt));
        const uintptr_t wa = reinterpret_cast<uintptr_t>(q.W);
        al[p] = (wa % 32 == 0 && ldw_bytes % 32 == 0) ? 2 : (wa % 16 == 0 && ldw_bytes % 16 == 0) ? 1 : 0;
        const uintptr_t va = reinterpret_cast<uintptr_t>(q.values), ia = reinterpret_cast<uintptr_t>(q.idx);
        auto vec_ok = [&](int nk) { return q.f.n == nk && va % (size_t(nk) * dt_size(dt)) == 0 && ia % size_t(nk) == 0; };
        nkc[p] = vec_ok(1) ? 1 : vec_ok(2) ? 2 : 0;
    }
    cudaStream_t st = as_stream(stream);
    // ONE launch for every problem; the lean instantiation when every problem has a lean body
    SparsifyBatch bt;
    memset(&bt, 0, sizeof(bt));
    int64_t blocks = 0;
    bool lean = true;
    for (int p = 0; p < count; ++p) {
        const sten_sparsify_problem& q = probs[p];
        const int64_t G = q.M / q.f.g, KB = q.K / q.f.m;
        if (G * KB == 0) continue;
        const int c = bt.count++;
        bt.W[c] = q.W; bt.values[c] = q.values; bt.idx[c] = q.idx;
        bt.ldw[c] = q.ldw; bt.G[c] = G; bt.KB[c] = KB; bt.Kp[c] = KB * q.f.n;
        bt.n[c] = q.f.n; bt.g[c] = q.f.g; bt.aligned[c] = al[p];
        bt.m[c] = q.f.m; bt.nk[c] = nkc[p];
        bt.block0[c] = int(blocks);
        blocks += (G * KB + kSpBatchThreads - 1) / kSpBatchThreads;
        lean = lean && sparsify_lean_ok(q.f.m, nkc[p], al[p]);
    }
    if (bt.count == 0) return STEN_OK;
    if (blocks > int64_t(0x7fffffff)) return STEN_ERR_UNSUPPORTED;
    bt.block0[bt.count] = int(blocks);
    const unsigned grid = unsigned(blocks);
    if (dt == STEN_F32) {
        if (lean) sparsify_grouped_nm_batched_kernel<float, 1><<<grid, kSpBatchThreads, 0, st>>>(bt);
        else sparsify_grouped_nm_batched_kernel<float, 0><<<grid, kSpBatchThreads, 0, st>>>(bt);
    } else {
        if (lean) sparsify_grouped_nm_batched_kernel<bf16_t, 1><<<grid, kSpBatchThreads, 0, st>>>(bt);
        else sparsify_grouped_nm_batched_kernel<bf16_t, 0><<<grid, kSpBatchThreads, 0, st>>>(bt);
    }
    return last_cuda();
}

sten_status sten_spmm_grouped_nm_allgather(sten_nmg f, sten_dtype ab_dt, const void* values, const uint8_t* idx,
                                           int64_t M, int64_t K, const void* B, int64_t ldb, int64_t N,
                                           void* const* C_peers, int32_t npeers, int64_t col0, int64_t ldc,
                                           sten_dtype c_dt, const sten_spmm_plan* plan, void* stream) {
    if (!C_peers || npeers < 1 || npeers > kMaxPeers || col0 < 0) return STEN_ERR_INVALID_ARG;
    for (int p = 0; p < npeers; ++p)
        if (!C_peers[p]) return STEN_ERR_INVALID_ARG;
    if (ldc < col0 + N) return STEN_ERR_SHAPE;
    // the fused epilogue is the SIMT kernel's; AUTO resolves to it
    sten_spmm_plan pl;
    memset(&pl, 0, sizeof(pl));
    if (plan) pl = *plan;
    if (pl.algo == STEN_ALGO_AUTO) pl.algo = STEN_ALGO_SIMT;
    if (pl.algo != STEN_ALGO_SIMT) return STEN_ERR_UNSUPPORTED;
    if (M > 0 && N > 0 && K == 0) return STEN_ERR_UNSUPPORTED;       // no fused zero-fill path
    return spmm_impl(f, ab_dt, values, idx, M, K, B, ldb, N, C_peers[0], ldc, c_dt, &pl, as_stream(stream),
                     C_peers, npeers, col0);
}

sten_status sten_spmm_grouped_nm_bias_act(sten_nmg f, sten_dtype ab_dt, const void* values, const uint8_t* idx,
                                          int64_t M, int64_t K, const void* B, int64_t ldb, int64_t N, void* C,
                                          int64_t ldc, sten_dtype c_dt, const float* bias, int32_t act,
                                          const sten_spmm_plan* plan, void* stream) {
    if (act < 0 || act > 2) return STEN_ERR_INVALID_ARG;
    sten_spmm_plan pl;
    memset(&pl, 0, sizeof(pl));
    if (plan) pl = *plan;
    if (pl.algo == STEN_ALGO_AUTO) pl.algo = STEN_ALGO_SIMT;       // the fused epilogue is the SIMT kernel's
    if (pl.algo != STEN_ALGO_SIMT) return STEN_ERR_UNSUPPORTED;
    if (M > 0 && N > 0 && K == 0) return STEN_ERR_UNSUPPORTED;       // no fused zero-fill path
    return spmm_impl(f, ab_dt, values, idx, M, K, B, ldb, N, C, ldc, c_dt, &pl, as_stream(stream), nullptr, 0, 0,
                     bias, act);
}

sten_status sten_spmm_grouped_nm_epilogue(sten_nmg f, sten_dtype ab_dt, const void* values, const uint8_t* idx,
                                          int64_t M, int64_t K, const void* B, int64_t ldb, int64_t N, void* C,
                                          int64_t ldc, sten_dtype c_dt, const float* bias, int32_t act,
                                          const void* residual, int64_t ldr, const sten_spmm_plan* plan,
                                          void* stream) {
    if (act < 0 || act > 2) return STEN_ERR_INVALID_ARG;
    if (residual && ldr < N) return STEN_ERR_SHAPE;
    if (residual && residual == C) return STEN_ERR_INVALID_ARG;          // outputs must not overlap inputs
    sten_spmm_plan pl;
    memset(&pl, 0, sizeof(pl));
    if (plan) pl = *plan;
    if (pl.algo == STEN_ALGO_AUTO) pl.algo = STEN_ALGO_SIMT;
    if (pl.algo != STEN_ALGO_SIMT) return STEN_ERR_UNSUPPORTED;
    if (M > 0 && N > 0 && K == 0) return STEN_ERR_UNSUPPORTED;
    return spmm_impl(f, ab_dt, values, idx, M, K, B, ldb, N, C, ldc, c_dt, &pl, as_stream(stream), nullptr, 0, 0,
                     bias, act, residual, ldr);
}

}  // extern "C"

namespace {

// BM / BN of the batched tiles (tile 1: 8 warps, tile 2: 16 warps; TN = 8, RG * SUB = 8 rows per warp)
inline void batch_tile_dims(int tile, int* bm, int* bn) {
    *bm = kSimtTiles[tile].bm;
    *bn = 32 * kSimtTiles[tile].tn;
}

// Validate the problems and fill their kernel arguments; splits[p] (0 = auto) -> a.split.
// Auto: every problem's K is cut into parts of about the same number of FMAs, so that the units of
// all problems together give ~3 units per resident CTA slot (the block scheduler balances them).
// the tile of problem p in a grouped launch: the caller's, or (tile 0) per problem: the 240-row,
// 128-token tile (3x longer K-slabs) for m >= 8 n sparsity, the 120 x 256 tile otherwise
inline int batch_tile_of(const sten_spmm_problem& q, int tile) {
    if (tile) return tile;
    return q.f.m >= 8 * q.f.n ? 3 : 2;
}

sten_status batch_setup(int32_t count, const sten_spmm_problem* probs, const int32_t* splits, int32_t tile,
                        SpmmArgs* as, int64_t* ws_floats, int64_t* ctr_words) {
    if (count < 1 || count > kMaxBatch || !probs) return STEN_ERR_INVALID_ARG;
    if (tile != 0 && tile != 1 && tile != 2 && tile != 3) return STEN_ERR_UNSUPPORTED;
    int bm, bn;
    const int rg = simt_rows_per_warp(probs[0].f.g);
    double tot = 0;
    for (int p = 0; p < count; ++p) {
        const sten_spmm_problem& q = probs[p];
        const sten_nmg f = q.f;
        sten_status s = check_format(f);
        if (s) return s;
        if ((s = check_shape(f, q.M, q.K))) return s;
        if (q.N < 0 || q.ldb < q.N || q.ldc < q.N) return STEN_ERR_SHAPE;
        if ((q.M * q.K > 0 && (!q.values || !q.idx)) || (q.K * q.N > 0 && !q.B) || (q.M * q.N > 0 && !q.C))
            return STEN_ERR_INVALID_ARG;
        if (simt_rows_per_warp(f.g) != rg) return STEN_ERR_UNSUPPORTED;    // one kernel variant per launch
        if (q.K == 0 && q.M * q.N > 0) return STEN_ERR_UNSUPPORTED;
        if (q.K * q.N > 0 && (!aligned16(q.B) || (q.ldb * 4) % 16 != 0)) return STEN_ERR_UNSUPPORTED;
        if ((reinterpret_cast<uintptr_t>(q.idx) & 3u) != 0) return STEN_ERR_UNSUPPORTED;
        if (splits && (splits[p] < 0 || splits[p] > kMaxSplit)) return STEN_ERR_UNSUPPORTED;
        SpmmArgs& a = as[p];
        memset(&a, 0, sizeof(a));
        a.values = q.values; a.idx = q.idx; a.B = q.B; a.C = q.C;
        a.M = q.M; a.K = q.K; a.N = q.N; a.ldb = q.ldb; a.ldc = q.ldc;
        a.n = f.n; a.m = f.m; a.g = f.g;
        a.KB = q.K / f.m; a.Kp = a.KB * f.n;
        a.c_vec = aligned16(q.C) && (q.ldc * 4) % 16 == 0;
        a.v_async = (a.Kp % 4 == 0) && ((reinterpret_cast<uintptr_t>(q.values) & 15u) == 0);
        a.idx_bytes = (q.M / f.g) * a.KB * f.n;
        const int pt = batch_tile_of(q, tile);
        batch_tile_dims(pt, &bm, &bn);
        a.kbs = simt_slab_blocks(f, STEN_F32, pt);
        a.split = 1;
        a.kb_per_split = a.KB;
        const double tiles = double((q.N + bn - 1) / bn) * double((q.M + bm - 1) / bm);
        tot += tiles * double(bm) * bn * double(a.Kp);
    }
    const double slots = double(kNumSMs) * kSimtTiles[batch_tile_of(probs[0], tile)].per_sm;
    double upc = 1.5;                                              // units per resident CTA slot (measured)
    if (const char* e = getenv("STEN_GROUP_UNITS")) upc = atof(e);  // (tuning experiments only)
    const double unit = tot / (upc * slots);                       // target FMAs per unit
    int64_t wsf = 0, ctrw = 0;
    for (int p = 0; p < count; ++p) {
        SpmmArgs& a = as[p];
        batch_tile_dims(batch_tile_of(probs[p], tile), &bm, &bn);
        const int64_t slabs = (a.KB + a.kbs - 1) / a.kbs;
        int S = splits ? splits[p] : 0;
        if (S == 0) {
            const double tile_fma = double(bm) * bn * double(a.Kp);
            S = int(std::min<double>(kMaxSplit, std::max(1.0, std::floor(tile_fma / unit + 0.5))));
        }
        a.split = int(std::max<int64_t>(1, std::min<int64_t>(S, slabs)));
        a.kb_per_split = ((slabs + a.split - 1) / a.split) * a.kbs;
        if (a.split > 1 && a.M > 0 && a.N > 0) {
            const int64_t tiles = ((a.N + bn - 1) / bn) * ((a.M + bm - 1) / bm);
            wsf += tiles * a.split * int64_t(bm) * bn;
            ctrw += tiles;
        }
    }
    *ws_floats = wsf;
    *ctr_words = (ctrw + 31) / 32 * 32;
    return STEN_OK;
}

}  // namespace

extern "C" {

sten_status sten_spmm_batched_workspace_size(int32_t count, const sten_spmm_problem* probs, const int32_t* splits,
                                             int32_t tile, int64_t* bytes) {
    if (!bytes) return STEN_ERR_INVALID_ARG;
    SpmmArgs as[kMaxBatch];
    int64_t wsf = 0, ctrw = 0;
    sten_status s = batch_setup(count, probs, splits, tile, as, &wsf, &ctrw);
    if (s) return s;
    *bytes = ctrw * 4 + wsf * 4;
    return STEN_OK;
}

sten_status sten_spmm_grouped_nm_batched_ex(int32_t count, const sten_spmm_problem* probs, const int32_t* splits,
                                            int32_t tile, void* workspace, int64_t workspace_bytes, void* stream) {
    SpmmArgs as[kMaxBatch];
    int64_t wsf = 0, ctrw = 0;
    sten_status s = batch_setup(count, probs, splits, tile, as, &wsf, &ctrw);
    if (s) return s;
    if (wsf > 0) {
        if (!workspace) return STEN_ERR_INVALID_ARG;
        if (workspace_bytes < ctrw * 4 + wsf * 4 || !aligned16(workspace)) return STEN_ERR_SHAPE;
        // counters first (zero on entry, left at zero), then each split problem's partial tiles
        unsigned* ctr = static_cast<unsigned*>(workspace);
        float* ws = reinterpret_cast<float*>(static_cast<char*>(workspace) + ctrw * 4);
        int bm, bn;
        for (int p = 0; p < count; ++p) {
            SpmmArgs& a = as[p];
            batch_tile_dims(batch_tile_of(probs[p], tile), &bm, &bn);
            if (a.split <= 1 || a.M == 0 || a.N == 0) continue;
            const int64_t tiles = ((a.N + bn - 1) / bn) * ((a.M + bm - 1) / bm);
            a.ws = ws;
            a.ctr = ctr;
            ws += tiles * a.split * int64_t(bm) * bn;
            ctr += tiles;
        }
    }
    // longest unit first: the block scheduler then fills the tail with short units.  A unit's time
    // ~ its kept k plus a fixed cost per K-slab (barrier round trip, idx words, row addresses: ~6 kept
    // k, from the per-class efficiencies of section 14), so 1:10 units (4 kept per slab) count longer
    // than their K' alone says
    int order[kMaxBatch];
    for (int p = 0; p < count; ++p) order[p] = p;
    auto unit_cost = [&](int x) {
        const double slabs = double((as[x].KB + as[x].kbs - 1) / as[x].kbs);
        return (double(as[x].Kp) + STEN_SLAB_COST * slabs) / as[x].split;
    };
    std::stable_sort(order, order + count, [&](int x, int y) { return unit_cost(x) > unit_cost(y); });
    SpmmArgs sorted[kMaxBatch];
    int tiles_of[kMaxBatch];
    int live = 0;
    for (int p = 0; p < count; ++p)
        if (as[order[p]].M > 0 && as[order[p]].N > 0) {
            tiles_of[live] = batch_tile_of(probs[order[p]], tile);
            sorted[live++] = as[order[p]];
        }
    if (live == 0) return STEN_OK;
    const int rg = simt_rows_per_warp(probs[0].f.g);
    cudaStream_t st = as_stream(stream);
    bool mixed = false;
    for (int p = 1; p < live; ++p) mixed |= tiles_of[p] != tiles_of[0];
    if (mixed) {
        switch (rg) {
            case 8: return launch_simt_batch_mixed<8>(sorted, tiles_of, live, st);
            case 4: return launch_simt_batch_mixed<4>(sorted, tiles_of, live, st);
            case 2: return launch_simt_batch_mixed<2>(sorted, tiles_of, live, st);
            default: return launch_simt_batch_mixed<1>(sorted, tiles_of, live, st);
        }
    }
    switch (rg) {
        case 8: return launch_simt_batch_rg<8>(sorted, live, tiles_of[0], st);
        case 4: return launch_simt_batch_rg<4>(sorted, live, tiles_of[0], st);
        case 2: return launch_simt_batch_rg<2>(sorted, live, tiles_of[0], st);
        default: return launch_simt_batch_rg<1>(sorted, live, tiles_of[0], st);
    }
}

sten_status sten_spmm_grouped_nm_batched(int32_t count, const sten_spmm_problem* probs, int32_t tile,
                                         void* stream) {
    // whole K per CTA (no workspace): every split is 1
    int32_t ones[kMaxBatch];
    for (int p = 0; p < kMaxBatch; ++p) ones[p] = 1;
    if (count < 1 || count > kMaxBatch) return STEN_ERR_INVALID_ARG;
    if (tile == 0) tile = 1;
    if (tile != 1 && tile != 2) return STEN_ERR_UNSUPPORTED;
    return sten_spmm_grouped_nm_batched_ex(count, probs, ones, tile, nullptr, 0, stream);
}

sten_status sten_resparsify_same_format(sten_nmg f, sten_dtype dt, const void* W, int64_t M, int64_t K,
                                        int64_t ldw, const uint8_t* idx, void* values, void* stream) {
    return sten_mask_check_repack(f, dt, W, M, K, ldw, idx, values, nullptr, stream);
}

sten_status sten_mask_check_repack(sten_nmg f, sten_dtype dt, const void* W, int64_t M, int64_t K, int64_t ldw,
                                   const uint8_t* idx, void* values, int64_t* outside, void* stream) {
    sten_status s = check_format(f);
    if (s) return s;
    if (!dtype_ok(dt)) return STEN_ERR_INVALID_ARG;
    if ((s = check_shape(f, M, K))) return s;
    if (ldw < K) return STEN_ERR_SHAPE;
    if (M * K > 0 && (!W || !values || !idx)) return STEN_ERR_INVALID_ARG;
    const int64_t KB = K / f.m, Kp = KB * f.n;
    if (outside && (reinterpret_cast<uintptr_t>(outside) & 7u) != 0) return STEN_ERR_UNSUPPORTED;
    if (M == 0 || KB == 0) {
        if (outside && cudaMemsetAsync(outside, 0, sizeof(int64_t), as_stream(stream)) != cudaSuccess)
            return STEN_ERR_CUDA;
        return STEN_OK;
    }
    const int64_t ldw_bytes = ldw * int64_t(dt_size(dt));
    const uintptr_t wa = reinterpret_cast<uintptr_t>(W);
    const int aligned = (wa % 32 == 0 && ldw_bytes % 32 == 0) ? 2 : (wa % 16 == 0 && ldw_bytes % 16 == 0) ? 1 : 0;
    cudaStream_t st = as_stream(stream);
    unsigned long long* cnt = reinterpret_cast<unsigned long long*>(outside);
    if (cnt && cudaMemsetAsync(cnt, 0, sizeof(int64_t), st) != cudaSuccess) return STEN_ERR_CUDA;
    const unsigned grid = grid1d(M * KB);
#define STEN_SF_CASE(MBV)                                                                                      \
    case MBV:                                                                                                 \
        if (dt == STEN_F32)                                                                                   \
            same_format_grouped_nm_kernel<float, MBV><<<grid, 256, 0, st>>>(                                  \
                static_cast<const float*>(W), ldw, M, KB, f.n, f.g, idx, static_cast<float*>(values), Kp, aligned, cnt); \
        else                                                                                                  \
            same_format_grouped_nm_kernel<bf16_t, MBV><<<grid, 256, 0, st>>>(                                 \
                static_cast<const bf16_t*>(W), ldw, M, KB, f.n, f.g, idx, static_cast<bf16_t*>(values), Kp, aligned, cnt); \
        break;
    switch (f.m) {
        STEN_SF_CASE(2) STEN_SF_CASE(4) STEN_SF_CASE(6) STEN_SF_CASE(8) STEN_SF_CASE(10) STEN_SF_CASE(12)
        STEN_SF_CASE(16)
        default: return STEN_ERR_UNSUPPORTED;
    }
#undef STEN_SF_CASE
    return last_cuda();
}

sten_status sten_densify(sten_nmg f, sten_dtype dt, const void* values, const uint8_t* idx, int64_t M,
                         int64_t K, void* W_out, int64_t ldw, void* stream) {
    sten_status s = check_format(f);
    if (s) return s;
    if (!dtype_ok(dt)) return STEN_ERR_INVALID_ARG;
    if ((s = check_shape(f, M, K))) return s;
    if (ldw < K) return STEN_ERR_SHAPE;
    if (M * K > 0 && (!values || !idx || !W_out)) return STEN_ERR_INVALID_ARG;
    const int64_t KB = K / f.m, Kp = KB * f.n;
    if (M == 0 || KB == 0) return STEN_OK;
    const bool aligned = aligned16(W_out) && (ldw * int64_t(dt_size(dt))) % 16 == 0;
    cudaStream_t st = as_stream(stream);
    bool ok = dt == STEN_F32 ? dispatch_densify<float>(f.m, values, idx, M, KB, f, Kp, W_out, ldw, aligned, st)
                             : dispatch_densify<bf16_t>(f.m, values, idx, M, KB, f, Kp, W_out, ldw, aligned, st);
    if (!ok) return STEN_ERR_UNSUPPORTED;
    return last_cuda();
}

sten_status sten_spmm_plan_query(sten_nmg f, sten_dtype ab_dt, int64_t M, int64_t K, int64_t N,
                                 sten_dtype c_dt, sten_spmm_plan* plan) {
    sten_status s = check_format(f);
    if (s) return s;
    if (!plan || !dtype_ok(ab_dt) || !dtype_ok(c_dt)) return STEN_ERR_INVALID_ARG;
    if ((s = check_shape(f, M, K))) return s;
    if (N < 0) return STEN_ERR_SHAPE;
    return plan_auto(f, ab_dt, M, K, N, c_dt, plan);
}

sten_status sten_spmm_grouped_nm_ex(sten_nmg f, sten_dtype ab_dt, const void* values, const uint8_t* idx,
                                    int64_t M, int64_t K, const void* B, int64_t ldb, int64_t N, void* C,
                                    int64_t ldc, sten_dtype c_dt, const sten_spmm_plan* plan, void* stream) {
    return spmm_impl(f, ab_dt, values, idx, M, K, B, ldb, N, C, ldc, c_dt, plan, as_stream(stream));
}

sten_status sten_spmm_grouped_nm(sten_nmg f, sten_dtype ab_dt, const void* values, const uint8_t* idx,
                                 int64_t M, int64_t K, const void* B, int64_t ldb, int64_t N, void* C,
                                 int64_t ldc, sten_dtype c_dt, void* stream) {
    return spmm_impl(f, ab_dt, values, idx, M, K, B, ldb, N, C, ldc, c_dt, nullptr, as_stream(stream));
}

// ---- end-to-end host entry point --------------------------------------------------------------
static inline int64_t round16(int64_t b) { return (b + 15) & ~int64_t(15); }

int64_t sten_sparse_linear_host_workspace_size(sten_nmg f, sten_dtype ab_dt, int64_t M, int64_t K,
                                               int64_t N, sten_dtype c_dt) {
    if (check_format(f) || check_shape(f, M, K) || N < 0 || !dtype_ok(ab_dt) || !dtype_ok(c_dt)) return -1;
    const int64_t s = int64_t(dt_size(ab_dt));
    const int64_t Kp = K / f.m * f.n;
    const int64_t ldb = (N * s + 15) / 16 * 16 / s;
    const int64_t ldc = (N * int64_t(dt_size(c_dt)) + 15) / 16 * 16 / int64_t(dt_size(c_dt));
    return round16(M * K * s) + round16(M * Kp * s) + round16(M / f.g * (K / f.m) * f.n) +
           round16(K * ldb * s) + round16(M * ldc * int64_t(dt_size(c_dt)));
}

static sten_status host_linear_check(sten_nmg f, sten_dtype ab_dt, const void* W_host, int64_t M, int64_t K,
                                     int64_t ldw, const void* B_host, int64_t ldb, int64_t N, void* C_host,
                                     int64_t ldc, sten_dtype c_dt, void* workspace, int64_t workspace_bytes) {
    sten_status s = check_format(f);
    if (s) return s;
    if (!dtype_ok(ab_dt) || !dtype_ok(c_dt)) return STEN_ERR_INVALID_ARG;
    if (!W_host || !B_host || !C_host || !workspace) return STEN_ERR_INVALID_ARG;
    if ((s = check_shape(f, M, K))) return s;
    if (N < 0 || ldw < K || ldb < N || ldc < N) return STEN_ERR_SHAPE;
    const int64_t need = sten_sparse_linear_host_workspace_size(f, ab_dt, M, K, N, c_dt);
    if (need < 0 || workspace_bytes < need || !aligned16(workspace)) return STEN_ERR_INVALID_ARG;
    return STEN_OK;
}

// the three stages of one host linear: H2D of W and B on `in`, sparsify + SpMM on `cmp` after `in`'s
// copies, D2H of C on `out` after the kernels (in == cmp == out: the single-stream call)
static sten_status host_linear_stages(sten_nmg f, sten_dtype ab_dt, const void* W_host, int64_t M, int64_t K,
                                      int64_t ldw, const void* B_host, int64_t ldb, int64_t N, void* C_host,
                                      int64_t ldc, sten_dtype c_dt, void* workspace, cudaStream_t in,
                                      cudaStream_t cmp, cudaStream_t out) {
    const int64_t sab = int64_t(dt_size(ab_dt)), sc = int64_t(dt_size(c_dt));
    const int64_t Kp = K / f.m * f.n;
    const int64_t dldb = (N * sab + 15) / 16 * 16 / sab;
    const int64_t dldc = (N * sc + 15) / 16 * 16 / sc;
    char* p = static_cast<char*>(workspace);
    void* dW = p;             p += round16(M * K * sab);
    void* dV = p;             p += round16(M * Kp * sab);
    uint8_t* dI = reinterpret_cast<uint8_t*>(p); p += round16(M / f.g * (K / f.m) * f.n);
    void* dB = p;             p += round16(K * dldb * sab);
    void* dC = p;
    // pitched copy, or ONE linear copy when both sides are dense (the copy engines move a 2-D copy
    // row by row; measured: the C2 step's copies take ~15 % longer as 2-D copies of 3-12 KB rows)
    auto copy2d = [](void* dst, size_t dpitch, const void* src, size_t spitch, size_t width, size_t height,
                     cudaMemcpyKind kind, cudaStream_t st) -> bool {
        if (dpitch == width && spitch == width)
            return cudaMemcpyAsync(dst, src, width * height, kind, st) == cudaSuccess;
        return cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, height, kind, st) == cudaSuccess;
    };
    auto hand_over = [](cudaStream_t from, cudaStream_t to) -> bool {
        if (from == to) return true;
        cudaEvent_t ev;
        if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) return false;
        const bool ok = cudaEventRecord(ev, from) == cudaSuccess && cudaStreamWaitEvent(to, ev, 0) == cudaSuccess;
        cudaEventDestroy(ev);                      // released once the recorded work completes
        return ok;
    };
    if (M * K > 0 && !copy2d(dW, size_t(K * sab), W_host, size_t(ldw * sab), size_t(K * sab), size_t(M),
                             cudaMemcpyHostToDevice, in))
        return STEN_ERR_CUDA;
    if (K * N > 0 && !copy2d(dB, size_t(dldb * sab), B_host, size_t(ldb * sab), size_t(N * sab), size_t(K),
                             cudaMemcpyHostToDevice, in))
        return STEN_ERR_CUDA;
    if (!hand_over(in, cmp)) return STEN_ERR_CUDA;
    sten_status s;
    if ((s = sten_sparsify_grouped_nm(f, ab_dt, dW, M, K, K, dV, dI, cmp))) return s;
    if ((s = spmm_impl(f, ab_dt, dV, dI, M, K, dB, dldb, N, dC, dldc, c_dt, nullptr, cmp))) return s;
    if (!hand_over(cmp, out)) return STEN_ERR_CUDA;
    if (M * N > 0 && !copy2d(C_host, size_t(ldc * sc), dC, size_t(dldc * sc), size_t(N * sc), size_t(M),
                             cudaMemcpyDeviceToHost, out))
        return STEN_ERR_CUDA;
    return STEN_OK;
}

static sten_status sparse_linear_host_impl(sten_nmg f, sten_dtype ab_dt, const void* W_host, int64_t M, int64_t K,
                                          int64_t ldw, const void* B_host, int64_t ldb, int64_t N, void* C_host,
                                          int64_t ldc, sten_dtype c_dt, void* workspace, int64_t workspace_bytes,
                                          void* stream, bool sync) {
    sten_status s = host_linear_check(f, ab_dt, W_host, M, K, ldw, B_host, ldb, N, C_host, ldc, c_dt, workspace,
                                      workspace_bytes);
    if (s) return s;
    cudaStream_t st = as_stream(stream);
    if ((s = host_linear_stages(f, ab_dt, W_host, M, K, ldw, B_host, ldb, N, C_host, ldc, c_dt, workspace, st, st,
                                st)))
        return s;
    if (sync && cudaStreamSynchronize(st) != cudaSuccess) return STEN_ERR_CUDA;
    return STEN_OK;
}

sten_status sten_sparse_linear_host_pipelined_async(int32_t count, const sten_host_linear_problem* probs,
                                                    sten_dtype ab_dt, sten_dtype c_dt, void* copy_in, void* compute,
                                                    void* copy_out) {
    if (count < 1 || count > 64 || !probs) return STEN_ERR_INVALID_ARG;
    for (int p = 0; p < count; ++p) {
        const sten_host_linear_problem& q = probs[p];
        const sten_status s = host_linear_check(q.f, ab_dt, q.W_host, q.M, q.K, q.ldw, q.B_host, q.ldb, q.N, q.C_host,
                                                q.ldc, c_dt, q.workspace, q.workspace_bytes);
        if (s) return s;
    }
    const cudaStream_t in = as_stream(copy_in), cmp = as_stream(compute), out = as_stream(copy_out);
    for (int p = 0; p < count; ++p) {
        const sten_host_linear_problem& q = probs[p];
        const sten_status s = host_linear_stages(q.f, ab_dt, q.W_host, q.M, q.K, q.ldw, q.B_host, q.ldb, q.N,
                                                 q.C_host, q.ldc, c_dt, q.workspace, in, cmp, out);
        if (s) return s;
    }
    return STEN_OK;
}

sten_status sten_sparse_linear_host(sten_nmg f, sten_dtype ab_dt, const void* W_host, int64_t M, int64_t K,
                                    int64_t ldw, const void* B_host, int64_t ldb, int64_t N, void* C_host,
                                    int64_t ldc, sten_dtype c_dt, void* workspace, int64_t workspace_bytes,
                                    void* stream) {
    return sparse_linear_host_impl(f, ab_dt, W_host, M, K, ldw, B_host, ldb, N, C_host, ldc, c_dt, workspace,
                                   workspace_bytes, stream, true);
}

sten_status sten_sparse_linear_host_async(sten_nmg f, sten_dtype ab_dt, const void* W_host, int64_t M, int64_t K,
                                          int64_t ldw, const void* B_host, int64_t ldb, int64_t N, void* C_host,
                                          int64_t ldc, sten_dtype c_dt, void* workspace, int64_t workspace_bytes,
                                          void* stream) {
    return sparse_linear_host_impl(f, ab_dt, W_host, M, K, ldw, B_host, ldb, N, C_host, ldc, c_dt, workspace,
                                   workspace_bytes, stream, false);
}

const char* sten_status_string(sten_status s) {
    switch (s) {
        case STEN_OK: return "STEN_OK";
        case STEN_ERR_INVALID_ARG: return "STEN_ERR_INVALID_ARG";
        case STEN_ERR_SHAPE: return "STEN_ERR_SHAPE";
        case STEN_ERR_UNSUPPORTED: return "STEN_ERR_UNSUPPORTED";
        case STEN_ERR_CUDA: return "STEN_ERR_CUDA";
    }
    return "STEN_ERR_UNKNOWN";
}

const char* sten_algo_name(int32_t algo) {
    switch (algo) {
        case STEN_ALGO_AUTO: return "auto";
        case STEN_ALGO_SIMT: return "simt";
        case STEN_ALGO_MMA_SYNC: return "mma_sync";
        case STEN_ALGO_TCGEN05: return "tcgen05";
    }
    return "unknown";
}

int32_t sten_spmm_launch_count(const sten_spmm_plan* plan) {
    (void)plan;   // every algorithm reduces split-K partials inside its kernel (cluster DSMEM)
    return 1;
}

sten_status sten_spmm_autotune(sten_nmg f, sten_dtype ab_dt, const void* values, const uint8_t* idx, int64_t M,
                               int64_t K, const void* B, int64_t ldb, int64_t N, void* C, int64_t ldc,
                               sten_dtype c_dt, int32_t reps, void* stream, sten_spmm_plan* best) {
    if (!best || reps < 1) return STEN_ERR_INVALID_ARG;
    cudaStream_t st = as_stream(stream);
    sten_spmm_plan auto_plan;
    sten_status s = check_format(f);
    if (s) return s;
    if (!dtype_ok(ab_dt) || !dtype_ok(c_dt)) return STEN_ERR_INVALID_ARG;
    if ((s = check_shape(f, M, K))) return s;
    plan_auto(f, ab_dt, M, K, N, c_dt, &auto_plan);
    // the AUTO call itself validates every argument; an error here is the caller's
    if ((s = spmm_impl(f, ab_dt, values, idx, M, K, B, ldb, N, C, ldc, c_dt, nullptr, st))) return s;
    std::vector<sten_spmm_plan> cand;
    auto add = [&](int algo, int tile, int split) {
        sten_spmm_plan p;
        memset(&p, 0, sizeof(p));
        p.algo = algo; p.tile = tile; p.split_k = split;
        cand.push_back(p);
    };
    add(STEN_ALGO_AUTO, 0, 0);
    for (int tile = 1; tile <= kSimtNumTiles; ++tile)
        for (int split = 1; split <= kMaxSplit; ++split) add(STEN_ALGO_SIMT, tile, split);
    if (ab_dt == STEN_BF16) {
        for (int tile = 1; tile <= 2; ++tile)
            for (int split = 1; split <= kMaxSplit; ++split) add(STEN_ALGO_MMA_SYNC, tile, split);
        for (int tile = 1; tile <= 3; ++tile) add(STEN_ALGO_TCGEN05, tile, 1);
    }
    cudaEvent_t e0, e1;
    if (cudaEventCreate(&e0) != cudaSuccess) return STEN_ERR_CUDA;
    if (cudaEventCreate(&e1) != cudaSuccess) { cudaEventDestroy(e0); return STEN_ERR_CUDA; }
    float best_ms = 3.0e38f;
    sten_spmm_plan best_plan = auto_plan;
    sten_status rc = STEN_OK;
    for (const sten_spmm_plan& p : cand) {
        const sten_spmm_plan* pp = p.algo == STEN_ALGO_AUTO ? nullptr : &p;
        if (spmm_impl(f, ab_dt, values, idx, M, K, B, ldb, N, C, ldc, c_dt, pp, st) != STEN_OK) {
            cudaGetLastError();     // an unsupported variant: skip it
            continue;
        }
        float t_min = 3.0e38f;
        for (int r = 0; r < reps; ++r) {
            cudaEventRecord(e0, st);
            spmm_impl(f, ab_dt, values, idx, M, K, B, ldb, N, C, ldc, c_dt, pp, st);
            cudaEventRecord(e1, st);
            if (cudaEventSynchronize(e1) != cudaSuccess) { rc = STEN_ERR_CUDA; break; }
            float ms = 0.0f;
            cudaEventElapsedTime(&ms, e0, e1);
            t_min = std::min(t_min, ms);
        }
        if (rc) break;
        if (t_min < best_ms) {
            best_ms = t_min;
            best_plan = p.algo == STEN_ALGO_AUTO ? auto_plan : p;
        }
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (rc) return rc;
    *best = best_plan;
    return STEN_OK;
}

int32_t sten_version(void) { return 1; }

#ifdef STEN_TIMING
// debug builds only: copy the per-CTA phase timestamps of the last SpMM launches
int sten_debug_timing(void* host_out, int max_ctas) {
    return cudaMemcpyFromSymbol(host_out, g_sten_timing, size_t(max_ctas) * 8 * 8) == cudaSuccess ? 0 : 1;
}
int sten_debug_timeline(void* host_out, int which) {
    return cudaMemcpyFromSymbol(host_out, which ? g_sten_tl2 : g_sten_tl, sizeof(long long) * 256 * 8) == cudaSuccess ? 0 : 1;
}
int sten_debug_waits(void* host_out, int max_ctas, int reset) {
    if (reset) {
        static unsigned long long zeros[16384][8];
        return cudaMemcpyToSymbol(g_sten_wait, zeros, sizeof(zeros)) == cudaSuccess ? 0 : 1;
    }
    return cudaMemcpyFromSymbol(host_out, g_sten_wait, size_t(max_ctas) * 8 * 8) == cudaSuccess ? 0 : 1;
}
#endif

}  // extern "C"
