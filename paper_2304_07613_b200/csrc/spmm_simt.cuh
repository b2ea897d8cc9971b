// spmm_simt.cuh -- K3: grouped n:m x dense SpMM on the CUDA cores (fp32 accumulate).
//
// Computes C = densify(values, idx) x B  (the sparse-dense GEMM of STen,
// PAPER.md:527-538, Fig. 5), redesigned for sm_100a:
//   (1) the paper's "load sparse values, broadcast into vector registers"
//       becomes a shared-memory broadcast: the g values of one kept k of a
//       group are stored contiguously ([k'][g]) so one LDS.128 feeds a warp;
//   (2) "indirect loads from specific rows of B" become indirect reads of a
//       B K-slab staged in shared memory by cp.async (16-byte LDGSTS,
//       double-buffered); the row offset of every kept k is precomputed per
//       slab, so the inner loop has no index arithmetic;
//   (3) "FMA" is FFMA into an RG x TN register tile per lane: RG rows of one
//       group (which share every kept k) x TN columns.  Each staged B element
//       read from shared memory feeds RG FMAs.
//
// CTA = 8 warps; warp w owns SUB sub-blocks of RG rows (each inside one group
// since RG | g; sub-blocks of different groups gather different B rows) and all
// BN = 32*TN columns of the tile, i.e. SUB*RG*TN fp32 accumulators per lane.
// BM = 8*SUB*RG rows per CTA sets the reuse of every staged B element across
// the CTA (BM*n/m rows use it), which keeps L2->SM traffic at 4/(BM*n/m) bytes
// per FMA for fp32.  Lane l owns the columns
// {j*32*EV + l*EV + e}, EV = 16/sizeof(T), so every shared/global vector access
// of a warp covers 512 contiguous bytes (conflict-free, coalesced).
//
// Split-K: the kept-k range of every row is cut into `split` contiguous parts
// (fixed by the plan, never by N); part p is computed by blockIdx.z == p into a
// private fp32 workspace slice and a second kernel adds the parts in order
// 0..split-1 -- so the summation order of a column is independent of N tiling.
#pragma once
#include "common.cuh"

namespace sten {

template <typename TAB, int RG, int TN, int SUB>
struct SimtCfg {
    static constexpr int kWarps = 8;
    static constexpr int kThreads = kWarps * 32;
    static constexpr int kEV = 16 / int(sizeof(TAB));    // elements per 16-byte vector
    static constexpr int kChunks = TN / kEV;               // 16-byte chunks per lane
    static constexpr int kBN = 32 * TN;                    // CTA columns
    static constexpr int kSubs = kWarps * SUB;             // RG-row sub-blocks per CTA
    static constexpr int kBM = kSubs * RG;                 // CTA rows
    static constexpr int kRGP = RG <= 1 ? 1 : RG <= 2 ? 2 : RG <= 4 ? 4 : 8;   // padded
    static constexpr int kSlabRows = sizeof(TAB) == 4 ? 32 : 64;   // target BK
    static constexpr int kMaxKS = kSlabRows;               // kept k per slab <= BK
    static_assert(TN % kEV == 0, "TN must be a multiple of the vector width");
};

// Number of m-blocks per slab for a given m.
template <typename TAB>
__host__ __device__ constexpr int simt_blocks_per_slab(int m) {
    return (sizeof(TAB) == 4 ? 32 : 64) / m > 0 ? (sizeof(TAB) == 4 ? 32 : 64) / m : 1;
}

template <typename TAB, int RG, int TN, int SUB>
__host__ __device__ constexpr size_t simt_smem_bytes(int m) {
    using Cfg = SimtCfg<TAB, RG, TN, SUB>;
    const int bk = simt_blocks_per_slab<TAB>(m) * m;
    return 2 * (size_t(bk) * Cfg::kBN * sizeof(TAB)                       // B slabs
                + size_t(Cfg::kSubs) * Cfg::kMaxKS * Cfg::kRGP * 4        // values (fp32)
                + size_t(Cfg::kSubs) * Cfg::kMaxKS * 4);                  // row offsets
}

template <int EV>
STEN_DEVICE_INLINE void unpack(const float4& raw, float (&b)[EV]) {
    if constexpr (EV == 4) {
        b[0] = raw.x; b[1] = raw.y; b[2] = raw.z; b[3] = raw.w;
    } else {   // 8 x bf16
        const uint32_t w[4] = {__float_as_uint(raw.x), __float_as_uint(raw.y),
                               __float_as_uint(raw.z), __float_as_uint(raw.w)};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            b[2 * q] = __uint_as_float(w[q] << 16);
            b[2 * q + 1] = __uint_as_float(w[q] & 0xffff0000u);
        }
    }
}

template <typename TC>
STEN_DEVICE_INLINE void store_out(TC* __restrict__ C, int64_t ldc, int64_t row, int64_t col,
                                  int64_t N, const float* v, int cnt, bool vec_ok) {
    TC* p = C + row * ldc + col;
    if (vec_ok && col + cnt <= N) {
        if constexpr (sizeof(TC) == 4) {
            if (cnt == 4) { *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]); return; }
            if (cnt == 8) {
                reinterpret_cast<float4*>(p)[0] = make_float4(v[0], v[1], v[2], v[3]);
                reinterpret_cast<float4*>(p)[1] = make_float4(v[4], v[5], v[6], v[7]);
                return;
            }
        } else {
            if (cnt == 4) {
                uint2 u;
                u.x = uint32_t(f32_to_bf16_rne(v[0])) | (uint32_t(f32_to_bf16_rne(v[1])) << 16);
                u.y = uint32_t(f32_to_bf16_rne(v[2])) | (uint32_t(f32_to_bf16_rne(v[3])) << 16);
                *reinterpret_cast<uint2*>(p) = u;
                return;
            }
            if (cnt == 8) {
                uint4 u;
                u.x = uint32_t(f32_to_bf16_rne(v[0])) | (uint32_t(f32_to_bf16_rne(v[1])) << 16);
                u.y = uint32_t(f32_to_bf16_rne(v[2])) | (uint32_t(f32_to_bf16_rne(v[3])) << 16);
                u.z = uint32_t(f32_to_bf16_rne(v[4])) | (uint32_t(f32_to_bf16_rne(v[5])) << 16);
                u.w = uint32_t(f32_to_bf16_rne(v[6])) | (uint32_t(f32_to_bf16_rne(v[7])) << 16);
                *reinterpret_cast<uint4*>(p) = u;
                return;
            }
        }
    }
    for (int e = 0; e < cnt; ++e)
        if (col + e < N) p[e] = from_f32<TC>(v[e]);
}

// Arguments common to the SpMM kernels.
struct SpmmArgs {
    const void* values;
    const uint8_t* idx;
    const void* B;
    void* C;            // final output (split == 1) or fp32 workspace [split][M][N]
    int64_t M, K, N, ldb, ldc;
    int n, m, g;
    int64_t Kp;         // kept per row
    int64_t KB;         // m-blocks per row
    int64_t kb_per_split;   // m-blocks per split-K part
    bool c_vec;         // C base/ldc allow vector stores
};

template <typename TAB, typename TC, int RG, int TN, int SUB>
__global__ void __launch_bounds__(256, 1)
spmm_simt_kernel(const SpmmArgs a) {
    using Cfg = SimtCfg<TAB, RG, TN, SUB>;
    constexpr int EV = Cfg::kEV;
    constexpr int RGP = Cfg::kRGP;
    constexpr int BN = Cfg::kBN;
    constexpr int BM = Cfg::kBM;
    constexpr int NSUB = Cfg::kSubs;
    constexpr int MAXKS = Cfg::kMaxKS;

    extern __shared__ __align__(128) unsigned char smem[];
    const int kbs = simt_blocks_per_slab<TAB>(a.m);             // m-blocks per slab
    const int bk = kbs * a.m;                                    // B rows per slab
    const size_t b_stage = size_t(bk) * BN * sizeof(TAB);
    unsigned char* sB[2] = {smem, smem + b_stage};
    float* sV[2];
    int* sO[2];
    {
        unsigned char* p = smem + 2 * b_stage;
        sV[0] = reinterpret_cast<float*>(p); p += NSUB * MAXKS * RGP * 4;
        sV[1] = reinterpret_cast<float*>(p); p += NSUB * MAXKS * RGP * 4;
        sO[0] = reinterpret_cast<int*>(p);   p += NSUB * MAXKS * 4;
        sO[1] = reinterpret_cast<int*>(p);
    }

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int64_t n0 = int64_t(blockIdx.x) * BN;
    const int64_t m0 = int64_t(blockIdx.y) * BM;
    const int part = blockIdx.z;
    const int64_t kb_begin = int64_t(part) * a.kb_per_split;
    const int64_t kb_end = min(a.KB, kb_begin + a.kb_per_split);
    const int64_t nslabs = kb_end > kb_begin ? (kb_end - kb_begin + kbs - 1) / kbs : 0;

    const TAB* __restrict__ V = static_cast<const TAB*>(a.values);
    const TAB* __restrict__ Bm = static_cast<const TAB*>(a.B);
    const int n = a.n;

    auto stage = [&](int64_t slab, int buf) {
        const int64_t kb0 = kb_begin + slab * kbs;
        const int nkb = int(min64(kbs, kb_end - kb0));
        const int rows = nkb * a.m;
        // B slab rows [kb0*m, kb0*m + rows) x columns [n0, n0 + BN): 16-byte cp.async
        constexpr int CPR = BN / EV;    // chunks per slab row
        for (int c = tid; c < rows * CPR; c += Cfg::kThreads) {
            const int kr = c / CPR, cc = c - kr * CPR;
            const int64_t col = n0 + int64_t(cc) * EV;
            const int64_t krow = kb0 * a.m + kr;
            const int bytes = int(max64(0, min64(EV, a.N - col))) * int(sizeof(TAB));
            const TAB* src = bytes > 0 ? Bm + krow * a.ldb + col : Bm;
            cp_async16(sB[buf] + (size_t(kr) * BN + cc * EV) * sizeof(TAB), src, bytes);
        }
        cp_async_commit();
        // values (transposed to [sub][k'][RGP], widened to fp32) and row byte offsets
        const int ks = nkb * n;
        for (int e = tid; e < BM * ks; e += Cfg::kThreads) {
            const int wr = e / ks, kk = e - wr * ks;
            const int64_t row = m0 + wr;
            float v = 0.0f;
            if (row < a.M) v = to_f32(V[row * a.Kp + kb0 * n + kk]);
            sV[buf][((wr / RG) * MAXKS + kk) * RGP + (wr % RG)] = v;
        }
        for (int e = tid; e < NSUB * ks; e += Cfg::kThreads) {
            const int sb = e / ks, kk = e - sb * ks;
            const int64_t row = m0 + int64_t(sb) * RG;
            int off = 0;
            if (row < a.M) {
                const int64_t grp = row / a.g;
                const int j = a.idx[(grp * a.KB + kb0) * n + kk];   // block kb0 + kk/n, slot kk%n
                off = ((kk / n) * a.m + j) * BN * int(sizeof(TAB));
            }
            sO[buf][sb * MAXKS + kk] = off;
        }
    };

    float acc[SUB][RG][TN];
#pragma unroll
    for (int q = 0; q < SUB; ++q)
#pragma unroll
        for (int r = 0; r < RG; ++r)
#pragma unroll
            for (int c = 0; c < TN; ++c) acc[q][r][c] = 0.0f;

    // warp w owns sub-blocks [w*SUB, (w+1)*SUB); sub-blocks past M are skipped
    const int sub0 = warp * SUB;
    const bool warp_active = (m0 + int64_t(sub0) * RG) < a.M;
    if (nslabs > 0) stage(0, 0);
    for (int64_t s = 0; s < nslabs; ++s) {
        const int buf = int(s & 1);
        if (s + 1 < nslabs) {
            stage(s + 1, buf ^ 1);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        if (warp_active) {
            const int64_t kb0 = kb_begin + s * kbs;
            const int ks = int(min64(kbs, kb_end - kb0)) * n;
            const unsigned char* bs = sB[buf] + size_t(lane) * EV * sizeof(TAB);
            const float* vs = sV[buf] + size_t(sub0) * MAXKS * RGP;
            const int* os = sO[buf] + sub0 * MAXKS;
#pragma unroll 2
            for (int kk = 0; kk < ks; ++kk) {
#pragma unroll
                for (int q = 0; q < SUB; ++q) {
                    const int off = os[q * MAXKS + kk];
                    float v[RGP];
                    const float* vp = vs + (q * MAXKS + kk) * RGP;
                    if constexpr (RGP >= 4) {
#pragma unroll
                        for (int u = 0; u < RGP / 4; ++u) {
                            const float4 t = lds128(vp + 4 * u);
                            v[4 * u] = t.x; v[4 * u + 1] = t.y; v[4 * u + 2] = t.z; v[4 * u + 3] = t.w;
                        }
                    } else {
#pragma unroll
                        for (int u = 0; u < RGP; ++u) v[u] = vp[u];
                    }
#pragma unroll
                    for (int j = 0; j < Cfg::kChunks; ++j) {
                        float b[EV];
                        unpack<EV>(lds128(bs + off + size_t(j) * 32 * EV * sizeof(TAB)), b);
#pragma unroll
                        for (int r = 0; r < RG; ++r)
#pragma unroll
                            for (int e = 0; e < EV; ++e)
                                acc[q][r][j * EV + e] = fmaf(v[r], b[e], acc[q][r][j * EV + e]);
                    }
                }
            }
        }
        __syncthreads();
    }

    if (!warp_active) return;
    const bool final_out = gridDim.z == 1;
#pragma unroll
    for (int q = 0; q < SUB; ++q) {
#pragma unroll
        for (int r = 0; r < RG; ++r) {
            const int64_t row = m0 + int64_t(sub0 + q) * RG + r;
            if (row >= a.M) continue;
#pragma unroll
            for (int j = 0; j < Cfg::kChunks; ++j) {
                const int64_t col = n0 + int64_t(j) * 32 * EV + lane * EV;
                if (final_out)
                    store_out<TC>(static_cast<TC*>(a.C), a.ldc, row, col, a.N, &acc[q][r][j * EV], EV, a.c_vec);
                else
                    store_out<float>(static_cast<float*>(a.C) + int64_t(part) * a.M * a.N, a.N, row, col, a.N,
                                     &acc[q][r][j * EV], EV, (a.N % 4) == 0);
            }
        }
    }
}

// Ordered reduction of split-K partials: C = ((p0 + p1) + p2) + ...
template <typename TC>
__global__ void __launch_bounds__(256)
splitk_reduce_kernel(const float* __restrict__ parts, int split, int64_t M, int64_t N,
                     TC* __restrict__ C, int64_t ldc) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= M * N) return;
    const int64_t r = i / N, c = i - r * N;
    float s = parts[i];
    for (int p = 1; p < split; ++p) s = __fadd_rn(s, parts[int64_t(p) * M * N + i]);
    C[r * ldc + c] = from_f32<TC>(s);
}

}  // namespace sten
