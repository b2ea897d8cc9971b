// spmm_mma.cuh -- K4: bf16 grouped n:m SpMM on the warp-level tensor-core path
// (mma.sync.m16n8k16, fp32 accumulate), for g a multiple of 8.
//
// The grouped layout makes the product of one group a DENSE contraction over
// its gathered rows (the g rows of a group share every kept k):
//     C_G[g x T] = V_G[g x K'] . B[S_G, T],   S_G = {kb*m + idx[G][kb][t]}
// We compute it transposed, C_G^T = B[S_G, T]^T . V_G^T, so the 16-wide MMA
// M-dimension runs over tokens and the 8-wide N-dimension over the group's
// rows.  The gather is free: `ldmatrix.x4.trans` takes one shared-memory row
// address PER LANE, so each lane simply points at the staged B row of the
// kept k it is responsible for -- no data is copied to build the gathered
// sub-tile.  Each gathered element then feeds 8*NR MACs (NR n8-blocks of the
// same group), i.e. arithmetic intensity on the gathered operand = g rows.
//
// CTA = 8 warps along rows; warp w owns SUB row-blocks of 8*NR rows (each in
// one group) x 64 tokens (MR = 4 m16 tiles).  Staging per K-slab (KBS m-blocks
// with KBS*n a multiple of 16): B slab [BK][64 tokens] via 16-byte cp.async into
// an XOR-swizzled layout (16-byte chunk ^ f(row), f chosen so the 8 rows an
// ldmatrix phase gathers mostly hit distinct bank groups), values tile
// [BM][KS] (row stride padded by 16 B: conflict-free ldmatrix), and per
// (row-block, kept k) the swizzled row descriptor.
#pragma once
#include "common.cuh"
#include "spmm_simt.cuh"   // SpmmArgs, store_out

namespace sten {

inline bool mma_supported(int g) { return g % 8 == 0; }

STEN_DEVICE_INLINE void ldsm_x4_trans(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
STEN_DEVICE_INLINE void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
STEN_DEVICE_INLINE void ldsm_x2(uint32_t addr, uint32_t& r0, uint32_t& r1) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0,%1}, [%2];\n"
                 : "=r"(r0), "=r"(r1)
                 : "r"(addr));
}
STEN_DEVICE_INLINE void mma_bf16_16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

template <int NR, int SUB>
struct MmaCfg {
    static constexpr int kWarps = 8;
    static constexpr int kThreads = 256;
    static constexpr int kMR = 4;                  // m16 token tiles per warp
    static constexpr int kBN = 16 * kMR;           // 64 tokens per CTA
    static constexpr int kRB = 8 * NR;             // rows per row-block
    static constexpr int kNRB = kWarps * SUB;      // row-blocks per CTA
    static constexpr int kBM = kNRB * kRB;
    static constexpr int kRowBytes = kBN * 2;      // 128 B per staged B row
};

// m-blocks per slab: the smallest count whose kept entries are a multiple of 16,
// scaled up so the slab has >= 32 B rows.
__host__ __device__ inline int mma_blocks_per_slab(int n, int m) {
    int a = n, b = 16;
    while (b) { int t = a % b; a = b; b = t; }
    int kbs = 16 / a;
    while (kbs * m < 32) kbs *= 2;
    return kbs;
}

template <int NR, int SUB>
__host__ __device__ inline size_t mma_smem_bytes(int n, int m) {
    using Cfg = MmaCfg<NR, SUB>;
    const int kbs = mma_blocks_per_slab(n, m);
    const int bk = kbs * m, ks = kbs * n;
    const size_t b = size_t(bk) * Cfg::kRowBytes;
    const size_t v = size_t(Cfg::kBM) * (ks * 2 + 16);
    const size_t o = size_t(Cfg::kNRB) * ks * 4;
    return 2 * (b + v + o);
}

// swizzle of a staged B row: f(row) from its (block, slot) so that the 8 rows
// one ldmatrix phase gathers (consecutive kept k) tend to differ in f.
STEN_DEVICE_INLINE int mma_swz(int kr, int n, int m) { return ((kr / m) * n + (kr % m) % n) & 7; }

template <typename TC, int NR, int SUB>
__global__ void __launch_bounds__(256, 1)
spmm_mma_kernel(const SpmmArgs a) {
    using Cfg = MmaCfg<NR, SUB>;
    constexpr int MR = Cfg::kMR;
    constexpr int BN = Cfg::kBN;
    constexpr int BM = Cfg::kBM;
    constexpr int RB = Cfg::kRB;
    constexpr int NRB = Cfg::kNRB;
    constexpr int ROWB = Cfg::kRowBytes;

    extern __shared__ __align__(128) unsigned char smem[];
    const int n = a.n, m = a.m;
    const int kbs = mma_blocks_per_slab(n, m);
    const int bk = kbs * m, ksmax = kbs * n;
    const int vstride = ksmax * 2 + 16;            // bytes per staged values row
    unsigned char* sB[2];
    unsigned char* sV[2];
    int* sO[2];
    {
        unsigned char* p = smem;
        sB[0] = p; p += size_t(bk) * ROWB;
        sB[1] = p; p += size_t(bk) * ROWB;
        sV[0] = p; p += size_t(BM) * vstride;
        sV[1] = p; p += size_t(BM) * vstride;
        sO[0] = reinterpret_cast<int*>(p); p += size_t(NRB) * ksmax * 4;
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

    const bf16_t* __restrict__ V = static_cast<const bf16_t*>(a.values);
    const bf16_t* __restrict__ Bm = static_cast<const bf16_t*>(a.B);

    auto stage = [&](int64_t slab, int buf) {
        const int64_t kb0 = kb_begin + slab * kbs;
        const int nkb = int(min64(kbs, kb_end - kb0));
        const int rows = nkb * m;
        constexpr int CPR = BN / 8;       // 16-byte chunks per staged row
        for (int c = tid; c < rows * CPR; c += Cfg::kThreads) {
            const int kr = c / CPR, cc = c - kr * CPR;
            const int64_t col = n0 + int64_t(cc) * 8;
            const int64_t krow = kb0 * m + kr;
            const int bytes = int(max64(0, min64(8, a.N - col))) * 2;
            const bf16_t* src = bytes > 0 ? Bm + krow * a.ldb + col : Bm;
            cp_async16(sB[buf] + size_t(kr) * ROWB + ((cc ^ mma_swz(kr, n, m)) * 16), src, bytes);
        }
        cp_async_commit();
        const int ks = nkb * n;
        // values tile [BM][ksmax] (zero beyond ks: padded MMA K-steps contribute 0)
        for (int e = tid; e < BM * ksmax; e += Cfg::kThreads) {
            const int r = e / ksmax, kk = e - r * ksmax;
            const int64_t row = m0 + r;
            bf16_t v = 0;
            if (row < a.M && kk < ks) v = V[row * a.Kp + kb0 * n + kk];
            *reinterpret_cast<bf16_t*>(sV[buf] + size_t(r) * vstride + kk * 2) = v;
        }
        // row descriptors: byte offset of the staged row | swizzle in the low 3 bits
        for (int e = tid; e < NRB * ksmax; e += Cfg::kThreads) {
            const int rb = e / ksmax, kk = e - rb * ksmax;
            const int64_t row = m0 + int64_t(rb) * RB;
            int kr = 0;
            if (row < a.M && kk < ks) {
                const int64_t grp = row / a.g;
                kr = (kk / n) * m + a.idx[(grp * a.KB + kb0) * n + kk];
            }
            sO[buf][rb * ksmax + kk] = kr * ROWB | mma_swz(kr, n, m);
        }
    };

    float acc[SUB][MR][NR][4];
#pragma unroll
    for (int q = 0; q < SUB; ++q)
#pragma unroll
        for (int i = 0; i < MR; ++i)
#pragma unroll
            for (int j = 0; j < NR; ++j)
#pragma unroll
                for (int e = 0; e < 4; ++e) acc[q][i][j][e] = 0.0f;

    const int rb0 = warp * SUB;
    const bool warp_active = (m0 + int64_t(rb0) * RB) < a.M;
    // per-lane ldmatrix roles
    const int a_k = (lane & 7) + ((lane >> 4) << 3);     // kept-k row this lane addresses (A)
    const int a_half = (lane >> 3) & 1;                   // token half (0-7 / 8-15)
    const int b_row = (lane & 7) + ((lane >> 4) << 3);   // values row within 16 (B)
    const int b_k8 = (lane >> 3) & 1;                     // k half (0-7 / 8-15)

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
            const int ksteps = (ks + 15) / 16;
            const uint32_t bbase = smem_u32(sB[buf]);
            const uint32_t vbase = smem_u32(sV[buf]);
            for (int kt = 0; kt < ksteps; ++kt) {
#pragma unroll
                for (int q = 0; q < SUB; ++q) {
                    const int rb = rb0 + q;
                    const int desc = sO[buf][rb * ksmax + kt * 16 + a_k];
                    const uint32_t rowaddr = bbase + uint32_t(desc & ~7);
                    const int swz = desc & 7;
                    uint32_t bf[NR][2];
                    if constexpr (NR == 2) {
                        const uint32_t va = vbase + uint32_t((rb * RB + b_row) * vstride + (kt * 16 + b_k8 * 8) * 2);
                        ldsm_x4(va, bf[0][0], bf[0][1], bf[1][0], bf[1][1]);
                    } else {
                        const uint32_t va = vbase + uint32_t((rb * RB + (lane & 7)) * vstride + (kt * 16 + b_k8 * 8) * 2);
                        ldsm_x2(va, bf[0][0], bf[0][1]);
                    }
#pragma unroll
                    for (int i = 0; i < MR; ++i) {
                        uint32_t af[4];
                        const int chunk = i * 2 + a_half;
                        ldsm_x4_trans(rowaddr + uint32_t((chunk ^ swz) * 16), af[0], af[1], af[2], af[3]);
#pragma unroll
                        for (int j = 0; j < NR; ++j) mma_bf16_16816(acc[q][i][j], af, bf[j][0], bf[j][1]);
                    }
                }
            }
        }
        __syncthreads();
    }

    if (!warp_active) return;
    // D fragment: d0,d1 -> (token = lane/4, rows 2*(lane%4)+{0,1}); d2,d3 -> token + 8
    const bool final_out = gridDim.z == 1;
    const int tq = lane >> 2, rq = (lane & 3) * 2;
#pragma unroll
    for (int q = 0; q < SUB; ++q)
#pragma unroll
        for (int j = 0; j < NR; ++j)
#pragma unroll
            for (int rr = 0; rr < 2; ++rr) {
                const int64_t row = m0 + int64_t(rb0 + q) * RB + j * 8 + rq + rr;
                if (row >= a.M) continue;
#pragma unroll
                for (int i = 0; i < MR; ++i)
#pragma unroll
                    for (int hh = 0; hh < 2; ++hh) {
                        const int64_t col = n0 + i * 16 + hh * 8 + tq;
                        if (col >= a.N) continue;
                        const float v = acc[q][i][j][hh * 2 + rr];
                        if (final_out) static_cast<TC*>(a.C)[row * a.ldc + col] = from_f32<TC>(v);
                        else static_cast<float*>(a.C)[int64_t(part) * a.M * a.N + row * a.N + col] = v;
                    }
            }
}

template <typename TC, int NR, int SUB>
inline cudaError_t launch_mma_cfg(const SpmmArgs& a, int split, cudaStream_t st) {
    using Cfg = MmaCfg<NR, SUB>;
    const size_t smem = mma_smem_bytes<NR, SUB>(a.n, a.m);
    auto kern = spmm_mma_kernel<TC, NR, SUB>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    dim3 grid(unsigned((a.N + Cfg::kBN - 1) / Cfg::kBN), unsigned((a.M + Cfg::kBM - 1) / Cfg::kBM),
              unsigned(split));
    kern<<<grid, Cfg::kThreads, smem, st>>>(a);
    return cudaGetLastError();
}

// mma tile variants (plan.tile): 1 = NR1/SUB4 (g % 8 == 0), 2 = NR2/SUB2 (g % 16 == 0);
// both give BM = 256 rows x 64 tokens per CTA.
template <typename TC>
inline sten_status launch_mma(const SpmmArgs& a, int tile, int split, cudaStream_t st) {
    cudaError_t e;
    if (tile == 2) e = launch_mma_cfg<TC, 2, 2>(a, split, st);
    else e = launch_mma_cfg<TC, 1, 4>(a, split, st);
    return e == cudaSuccess ? STEN_OK : STEN_ERR_CUDA;
}

}  // namespace sten
