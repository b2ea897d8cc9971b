// masked.cuh -- NEXT-2: the weight gradient of the grouped n:m linear in its own format (SDDMM).
//
// For C = densify(values, idx) . B and a loss gradient G = dL/dC [M][N], the
// gradient w.r.t. the stored values is the dense G B^T SAMPLED at the kept positions:
//     dV[r][kb n + t] = sum_c G[r][c] B[kb m + idx[r/g][kb][t]][c]
// -- the "(KeepAll, FixedMaskTensor)" weight gradient of STen's masked linear:
// the weight keeps its fixed mask, its gradient comes out in the same (values) layout, and an
// optimizer step updates the values in place (no re-sparsification: the fixed-mask fast path).
//
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

// Mapping: CTA = 8 warps on 8 RR rows (8 groups when RR = 4) x 128 kept slots; warp w owns kept
// slots [16 w, 16 w + 16) of the CTA, lane l owns RR rows (one group: RR | g) x 4 kept slots
// (interleaved with the group's other 3 lanes).  Per
// chunk of TCH tokens the CTA stages in shared memory (cp.async, double buffered, rows padded by 16
// bytes so a warp's gathered row loads hit distinct banks) its G rows AND the dense range of B rows
// its kept slots can point at (128 / n m-blocks = 128 m / n rows), so every G element is reused by
// 128 kept slots and every B element by the tile's groups; TCH adapts to the format so both tiles
// fit (2:4 fp32: 32 tokens).  Per lane the tokens are summed in ascending order, one partial per
// chunk added to the accumulator (two-level summation) -- deterministic.
struct SddmmGeom {
    int wk, wr;                   // warps along the kept slots / along the rows (wk * wr = 8)
    int kpc, rows;                // kept slots and G rows of the CTA tile
    int tch, brows, rbg, rbb;     // tokens per chunk, staged B rows, padded row bytes of G and B
    size_t smem;
};
// The staged B range holds kpc m / n rows: sparser formats put fewer warps along the kept slots and
// more along the rows, so both tiles stay ~256 rows and the chunk stays >= 16 tokens.
__host__ __device__ inline SddmmGeom sddmm_geom(int n, int m, int rr, int esz) {
    SddmmGeom g{};
    g.wk = m <= 2 * n ? 8 : m <= 4 * n ? 4 : m <= 8 * n ? 2 : 1;
    g.wr = 8 / g.wk;
    g.kpc = 16 * g.wk;
    g.rows = g.wr * 8 * rr;
    g.brows = (g.kpc / n + 1) * m;                     // +1 block: a kept range may start mid-block
    const int ev = 16 / esz;
    int tch = 64;
    while (tch > ev && size_t(2) * (g.rows + g.brows) * (size_t(tch) * esz + 16) > 98304) tch >>= 1;
    g.tch = tch;
    g.rbg = tch * esz + 16;
    g.rbb = tch * esz + 16;
    g.smem = size_t(2) * (size_t(g.rows) * g.rbg + size_t(g.brows) * g.rbb);
    return g;
}

template <typename T, typename TC, int RR>
__global__ void __launch_bounds__(256)
sddmm_grouped_nm_kernel(const SddmmArgs a) {
    constexpr int EV = 16 / int(sizeof(T));       // tokens per vector
    constexpr int KK = 4;                         // kept slots per lane
    extern __shared__ __align__(16) unsigned char sm[];
    const SddmmGeom geo = sddmm_geom(a.n, a.m, RR, int(sizeof(T)));
    const int TCH = geo.tch, RBG = geo.rbg, RBB = geo.rbb, BROWS = geo.brows, ROWS = geo.rows;
    unsigned char* sg[2] = {sm, sm + size_t(ROWS) * RBG};
    unsigned char* sb[2] = {sm + size_t(2) * ROWS * RBG, sm + size_t(2) * ROWS * RBG + size_t(BROWS) * RBB};
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int wkk = warp % geo.wk, wrr = warp / geo.wk;           // this warp's kept block / row block
    const int64_t rt0 = int64_t(blockIdx.y) * ROWS;
    const int64_t r0 = rt0 + (int64_t(wrr) * 8 + (lane >> 2)) * RR;
    const int64_t kc0 = int64_t(blockIdx.x) * geo.kpc;             // first kept slot of the CTA
    const int64_t kbase = (kc0 / a.n) * a.m;                        // first staged B row
    // kept slot q of this lane: kc0 + 16 wkk + 4 q + (lane & 3) (the 4 lanes of a group take adjacent
    // slots, so their staged B rows spread over the bank slots)
    const int64_t kk0 = kc0 + wkk * 16 + (lane & 3);
    const T* Gm = static_cast<const T*>(a.G);
    const T* Bm = static_cast<const T*>(a.B);
    int boff[KK];                                                   // staged row of each kept slot
    const bool rv = r0 < a.M;
#pragma unroll
    for (int q = 0; q < KK; ++q) {
        const int64_t kk = kk0 + 4 * q;
        boff[q] = 0;
        if (rv && kk < a.Kp) {
            const int64_t kb = kk / a.n;
            const int t = int(kk - kb * a.n);
            boff[q] = int(kb * a.m + a.idx[((r0 / a.g) * a.KB + kb) * a.n + t] - kbase);
        }
    }
    const int64_t nch = (a.N + TCH - 1) / TCH;
    const int vpr = TCH / EV;                                       // vectors per staged row
    auto stage = [&](int64_t ch, int buf) {
        const int64_t c0 = ch * TCH;
        for (int e = threadIdx.x; e < (ROWS + BROWS) * vpr; e += blockDim.x) {
            const int r = e / vpr, v = e - r * vpr;
            const int64_t c = c0 + int64_t(v) * EV;
            int bytes = 0;
            const T* src = Gm;
            unsigned char* dst;
            if (r < ROWS) {
                const int64_t row = rt0 + r;
                // staged position of tile row r = (row block rb, group gi, row i): rb 8 RR + i 8 + gi -- the
                // 8 groups' i-th rows are adjacent, so a warp's reads of row i fall in distinct bank slots
                const int rb = r / (8 * RR), rl = r % (8 * RR);
                dst = sg[buf] + (rb * 8 * RR + (rl % RR) * 8 + rl / RR) * RBG + v * 16;
                if (row < a.M && c < a.N) { bytes = int(min64(EV, a.N - c)) * int(sizeof(T)); src = Gm + row * a.ldg + c; }
            } else {
                const int64_t row = kbase + (r - ROWS);
                dst = sb[buf] + (r - ROWS) * RBB + v * 16;
                if (row < a.K && c < a.N) { bytes = int(min64(EV, a.N - c)) * int(sizeof(T)); src = Bm + row * a.ldb + c; }
            }
            cp_async16(dst, src, bytes);
        }
        cp_async_commit();
    };
    auto unpack16 = [](const unsigned char* p, float (&x)[EV]) {
        const uint4 u = *reinterpret_cast<const uint4*>(p);
        if constexpr (sizeof(T) == 4) {
            x[0] = __uint_as_float(u.x); x[1] = __uint_as_float(u.y); x[2] = __uint_as_float(u.z); x[3] = __uint_as_float(u.w);
        } else {
            const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
            for (int qq = 0; qq < 4; ++qq) {
                x[2 * qq] = __uint_as_float(w[qq] << 16);
                x[2 * qq + 1] = __uint_as_float(w[qq] & 0xffff0000u);
            }
        }
    };
    float acc[RR][KK];
#pragma unroll
    for (int i = 0; i < RR; ++i)
#pragma unroll
        for (int q = 0; q < KK; ++q) acc[i][q] = 0.0f;
    stage(0, 0);
    for (int64_t ch = 0; ch < nch; ++ch) {
        if (ch + 1 < nch) stage(ch + 1, int((ch + 1) & 1));
        else cp_async_commit();
        cp_async_wait<1>();
        __syncthreads();
        if (rv) {
            const unsigned char* gb = sg[ch & 1] + (wrr * 8 * RR + (lane >> 2)) * RBG;   // + i 8 RBG for row i
            const unsigned char* bb = sb[ch & 1];
            float blk[RR][KK];
#pragma unroll
            for (int i = 0; i < RR; ++i)
#pragma unroll
                for (int q = 0; q < KK; ++q) blk[i][q] = 0.0f;
            // tokens beyond N are zero in the staged G and B: no per-vector bound check needed
#pragma unroll 2
            for (int v = 0; v < vpr; ++v) {
                float gx[RR][EV], bx[KK][EV];
#pragma unroll
                for (int i = 0; i < RR; ++i) unpack16(gb + i * 8 * RBG + v * 16, gx[i]);
#pragma unroll
                for (int q = 0; q < KK; ++q) unpack16(bb + boff[q] * RBB + v * 16, bx[q]);
#pragma unroll
                for (int e = 0; e < EV; ++e)
#pragma unroll
                    for (int i = 0; i < RR; ++i)
#pragma unroll
                        for (int q = 0; q < KK; ++q) blk[i][q] = __fmaf_rn(gx[i][e], bx[q][e], blk[i][q]);
            }
#pragma unroll
            for (int i = 0; i < RR; ++i)
#pragma unroll
                for (int q = 0; q < KK; ++q) acc[i][q] = __fadd_rn(acc[i][q], blk[i][q]);
        }
        __syncthreads();                                           // the buffer is refilled next iteration
    }
    TC* dV = static_cast<TC*>(a.dV);
    if (rv) {
#pragma unroll
        for (int i = 0; i < RR; ++i)
#pragma unroll
            for (int q = 0; q < KK; ++q)
                if (kk0 + 4 * q < a.Kp) dV[(r0 + i) * a.Kp + kk0 + 4 * q] = from_f32<TC>(acc[i][q]);
    }
}

}  // namespace sten
