// masked.cuh -- NEXT-2: the weight gradient of the grouped n:m linear in its own format (SDDMM).
//
// For C = densify(values, idx) . B and a loss gradient G = dL/dC [M][N], the
// gradient w.r.t. the stored values is the dense G B^T SAMPLED at the kept positions:
//     dV[r][kb n + t] = sum_c G[r][c] B[kb m + idx[r/g][kb][t]][c]
// -- the "(KeepAll, FixedMaskTensor)" weight gradient of STen's masked linear:
// the weight keeps its fixed mask, its gradient comes out in the same (values) layout, and an
// optimizer step updates the values in place (no re-sparsification: the fixed-mask fast path).
//
// Mapping: CTA = 8 warps, tile = 8 RR rows x 16 kept slots; lane l owns RR rows (one group:
// RR | g) x 4 kept slots, so every 16-byte vector of a G row feeds 4 kept slots and every gathered
// B vector feeds RR rows.  The 8 warps take interleaved token vectors; each lane sums its tokens
// in ascending order in blocks of 64 tokens (two-level summation: the rounding error grows with
// 64 + N / 512 terms, not N / 8) and the warps' partials are added in the fixed order w = 0..7 --
// deterministic, independent of timing.
#pragma once
#include "common.cuh"

namespace sten {

struct SddmmArgs {
    const void* G;          // [M][ldg]
    const void* B;          // [K][ldb]
    const uint8_t* idx;     // [M/g][K/m][n]
    void* dV;               // [M][Kp] (c dtype)
    int64_t M, K, N, ldg, ldb, KB, Kp;
    int n, m, g;
};

template <typename T>
STEN_DEVICE_INLINE void load_vec(const T* p, float (&x)[16 / sizeof(T)]) {
    const uint4 u = __ldg(reinterpret_cast<const uint4*>(p));
    if constexpr (sizeof(T) == 4) {
        x[0] = __uint_as_float(u.x); x[1] = __uint_as_float(u.y); x[2] = __uint_as_float(u.z); x[3] = __uint_as_float(u.w);
    } else {
        const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            x[2 * q] = __uint_as_float(w[q] << 16);
            x[2 * q + 1] = __uint_as_float(w[q] & 0xffff0000u);
        }
    }
}

template <typename T, typename TC, int RR>
__global__ void __launch_bounds__(256)
sddmm_grouped_nm_kernel(const SddmmArgs a) {
    constexpr int EV = 16 / int(sizeof(T));       // tokens per vector
    constexpr int KK = 4;                         // kept slots per lane
    constexpr int NW = 8;
    __shared__ float red[NW][32 * RR * KK];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t r0 = (int64_t(blockIdx.y) * 8 + (lane >> 2)) * RR;
    const int64_t kk0 = int64_t(blockIdx.x) * 16 + (lane & 3) * KK;
    const T* Gm = static_cast<const T*>(a.G);
    const T* Bm = static_cast<const T*>(a.B);
    // the B rows of this lane's kept slots (rows of one group share them); invalid slots -> row 0, unused
    int64_t brow[KK];
    bool kv[KK];
    const bool rv = r0 < a.M;
#pragma unroll
    for (int q = 0; q < KK; ++q) {
        const int64_t kk = kk0 + q;
        kv[q] = rv && kk < a.Kp;
        brow[q] = 0;
        if (kv[q]) {
            const int64_t kb = kk / a.n;
            const int t = int(kk - kb * a.n);
            brow[q] = kb * a.m + a.idx[((r0 / a.g) * a.KB + kb) * a.n + t];
        }
    }
    float acc[RR][KK], blk[RR][KK];
#pragma unroll
    for (int i = 0; i < RR; ++i)
#pragma unroll
        for (int q = 0; q < KK; ++q) acc[i][q] = blk[i][q] = 0.0f;
    int inblk = 0;
    const int64_t nvec = a.N / EV;                 // full vectors; the tail is done below
    if (rv) {
        for (int64_t v = warp; v < nvec; v += NW) {
            const int64_t c = v * EV;
            float gx[RR][EV], bx[KK][EV];
#pragma unroll
            for (int i = 0; i < RR; ++i) {
                if (r0 + i < a.M) load_vec<T>(Gm + (r0 + i) * a.ldg + c, gx[i]);
                else {
#pragma unroll
                    for (int e = 0; e < EV; ++e) gx[i][e] = 0.0f;
                }
            }
#pragma unroll
            for (int q = 0; q < KK; ++q) load_vec<T>(Bm + brow[q] * a.ldb + c, bx[q]);
#pragma unroll
            for (int e = 0; e < EV; ++e)
#pragma unroll
                for (int i = 0; i < RR; ++i)
#pragma unroll
                    for (int q = 0; q < KK; ++q) blk[i][q] = __fmaf_rn(gx[i][e], bx[q][e], blk[i][q]);
            if (++inblk == 64 / EV) {
#pragma unroll
                for (int i = 0; i < RR; ++i)
#pragma unroll
                    for (int q = 0; q < KK; ++q) { acc[i][q] = __fadd_rn(acc[i][q], blk[i][q]); blk[i][q] = 0.0f; }
                inblk = 0;
            }
        }
        // ragged tail (N % EV tokens): warp 0, scalar loads
        if (warp == 0) {
            for (int64_t c = nvec * EV; c < a.N; ++c)
#pragma unroll
                for (int i = 0; i < RR; ++i) {
                    const float gv = r0 + i < a.M ? to_f32(Gm[(r0 + i) * a.ldg + c]) : 0.0f;
#pragma unroll
                    for (int q = 0; q < KK; ++q) blk[i][q] = __fmaf_rn(gv, to_f32(Bm[brow[q] * a.ldb + c]), blk[i][q]);
                }
        }
#pragma unroll
        for (int i = 0; i < RR; ++i)
#pragma unroll
            for (int q = 0; q < KK; ++q) acc[i][q] = __fadd_rn(acc[i][q], blk[i][q]);
    }
#pragma unroll
    for (int i = 0; i < RR; ++i)
#pragma unroll
        for (int q = 0; q < KK; ++q) red[warp][(lane * RR + i) * KK + q] = acc[i][q];
    __syncthreads();
    // fixed-order reduction over the warps, one output per thread
    TC* dV = static_cast<TC*>(a.dV);
    for (int o = threadIdx.x; o < 32 * RR * KK; o += blockDim.x) {
        float s = red[0][o];
#pragma unroll
        for (int w = 1; w < NW; ++w) s = __fadd_rn(s, red[w][o]);
        const int l = o / (RR * KK), i = (o / KK) % RR, q = o % KK;
        const int64_t r = (int64_t(blockIdx.y) * 8 + (l >> 2)) * RR + i;
        const int64_t kk = int64_t(blockIdx.x) * 16 + (l & 3) * KK + q;
        if (r < a.M && kk < a.Kp) dV[r * a.Kp + kk] = from_f32<TC>(s);
    }
}

}  // namespace sten
