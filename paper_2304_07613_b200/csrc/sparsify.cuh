// sparsify.cuh -- K1 (a1-a3: score, select, compact) and K2 (a4: densify) for sm_100a.
//
// K1 follows the grouped n:m construction of STen (arXiv 2304.07613):
//   group of g rows sharing one n-of-m pattern        PAPER.md:518 (Sec. 5)
//   kept set = argmax of the L1 norm of kept entries  PAPER.md:548-549 (Sec. 5.2)
// For reading (A) (R1) the argmax decomposes exactly per
// (group, m-block): keep the n positions with the largest summed |w|.
//
// Mapping: one thread per (group, m-block); consecutive threads take
// consecutive m-blocks of the same rows, so every warp reads g row segments of
// 32*m contiguous elements (16-byte vector loads when m*sizeof(T) allows).
// The first min(8, 32/m) rows of the group stay in registers between the score
// pass and the compaction pass; later rows are re-read (L1/L2 hits).  HBM roofline:
// M*K*s (read W) + M*K'*s (values) + (M/g)*(K/m)*n (idx) bytes.
#pragma once
#include "common.cuh"

namespace sten {

template <typename T, int MB>
STEN_DEVICE_INLINE void load_block(const T* __restrict__ p, T (&row)[MB], bool aligned) {
    constexpr int BYTES = MB * int(sizeof(T));
    if (aligned) {
        if constexpr (BYTES % 16 == 0) {
            uint4 tmp[BYTES / 16];
#pragma unroll
            for (int q = 0; q < BYTES / 16; ++q) tmp[q] = __ldg(reinterpret_cast<const uint4*>(p) + q);
            memcpy(row, tmp, BYTES);
            return;
        } else if constexpr (BYTES % 8 == 0) {
            uint2 tmp[BYTES / 8];
#pragma unroll
            for (int q = 0; q < BYTES / 8; ++q) tmp[q] = __ldg(reinterpret_cast<const uint2*>(p) + q);
            memcpy(row, tmp, BYTES);
            return;
        } else if constexpr (BYTES % 4 == 0) {
            uint32_t tmp[BYTES / 4];
#pragma unroll
            for (int q = 0; q < BYTES / 4; ++q) tmp[q] = __ldg(reinterpret_cast<const uint32_t*>(p) + q);
            memcpy(row, tmp, BYTES);
            return;
        }
    }
#pragma unroll
    for (int j = 0; j < MB; ++j) row[j] = p[j];
}

template <typename T, int MB>
STEN_DEVICE_INLINE void store_block(T* __restrict__ p, const T (&row)[MB], bool aligned) {
    constexpr int BYTES = MB * int(sizeof(T));
    if (aligned) {
        if constexpr (BYTES % 16 == 0) {
            uint4 tmp[BYTES / 16];
            memcpy(tmp, row, BYTES);
#pragma unroll
            for (int q = 0; q < BYTES / 16; ++q) reinterpret_cast<uint4*>(p)[q] = tmp[q];
            return;
        } else if constexpr (BYTES % 8 == 0) {
            uint2 tmp[BYTES / 8];
            memcpy(tmp, row, BYTES);
#pragma unroll
            for (int q = 0; q < BYTES / 8; ++q) reinterpret_cast<uint2*>(p)[q] = tmp[q];
            return;
        } else if constexpr (BYTES % 4 == 0) {
            uint32_t tmp[BYTES / 4];
            memcpy(tmp, row, BYTES);
#pragma unroll
            for (int q = 0; q < BYTES / 4; ++q) reinterpret_cast<uint32_t*>(p)[q] = tmp[q];
            return;
        }
    }
#pragma unroll
    for (int j = 0; j < MB; ++j) p[j] = row[j];
}

// rows of a group kept in registers between the two passes (<= 32 elements per thread)
template <int MB>
constexpr int sparsify_reg_rows() { return 32 / MB < 1 ? 1 : (32 / MB > 8 ? 8 : 32 / MB); }

template <typename T, int MB>
__global__ void __launch_bounds__(256)
sparsify_grouped_nm_kernel(const T* __restrict__ W, int64_t ldw, int64_t G, int64_t KB, int n,
                           int g, T* __restrict__ values, int64_t Kp, uint8_t* __restrict__ idx,
                           bool aligned) {
    const int64_t tid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (tid >= G * KB) return;
    const int64_t grp = tid / KB;
    const int64_t kb = tid - grp * KB;
    const T* w0 = W + grp * g * ldw + kb * MB;
    constexpr int kSparsifyRegRows = sparsify_reg_rows<MB>();

    // a1 score: s[j] = fl32(...fl32(|w_0j| + |w_1j|) ... + |w_(g-1)j|), ascending rows, RNE.
    float s[MB];
#pragma unroll
    for (int j = 0; j < MB; ++j) s[j] = 0.0f;
    T x[kSparsifyRegRows][MB];
#pragma unroll
    for (int i = 0; i < kSparsifyRegRows; ++i) {
        if (i < g) {
            load_block<T, MB>(w0 + i * ldw, x[i], aligned);
#pragma unroll
            for (int j = 0; j < MB; ++j) s[j] = __fadd_rn(s[j], fabsf(to_f32(x[i][j])));
        }
    }
    for (int i = kSparsifyRegRows; i < g; ++i) {
        T row[MB];
        load_block<T, MB>(w0 + i * ldw, row, aligned);
#pragma unroll
        for (int j = 0; j < MB; ++j) s[j] = __fadd_rn(s[j], fabsf(to_f32(row[j])));
    }

    // a2 select: rank[j] = #{i : s_i > s_j or (s_i == s_j and i < j)}; keep iff rank < n.
    uint32_t keep = 0;
#pragma unroll
    for (int j = 0; j < MB; ++j) {
        int rank = 0;
#pragma unroll
        for (int i = 0; i < MB; ++i) rank += (s[i] > s[j]) || (s[i] == s[j] && i < j);
        keep |= uint32_t(rank < n) << j;
    }

    // idx: kept positions ascending
    uint8_t* ip = idx + (grp * KB + kb) * n;
    {
        int t = 0;
#pragma unroll
        for (int j = 0; j < MB; ++j)
            if (keep >> j & 1u) ip[t++] = uint8_t(j);
    }

    // a3 compact: bit copy of the kept entries of every row of the group
#pragma unroll
    for (int i = 0; i < kSparsifyRegRows; ++i) {
        if (i < g) {
            T* vp = values + (grp * g + i) * Kp + kb * n;
            int t = 0;
#pragma unroll
            for (int j = 0; j < MB; ++j)
                if (keep >> j & 1u) vp[t++] = x[i][j];
        }
    }
    for (int i = kSparsifyRegRows; i < g; ++i) {
        T row[MB];
        load_block<T, MB>(w0 + i * ldw, row, aligned);
        T* vp = values + (grp * g + i) * Kp + kb * n;
        int t = 0;
#pragma unroll
        for (int j = 0; j < MB; ++j)
            if (keep >> j & 1u) vp[t++] = row[j];
    }
}

// K2 densify: one thread per (row, m-block); writes the full m-element block
// (zeros at pruned positions) with one vector store when aligned.
template <typename T, int MB>
__global__ void __launch_bounds__(256)
densify_grouped_nm_kernel(const T* __restrict__ values, const uint8_t* __restrict__ idx, int64_t M,
                          int64_t KB, int n, int g, int64_t Kp, T* __restrict__ W, int64_t ldw,
                          bool aligned) {
    const int64_t tid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (tid >= M * KB) return;
    const int64_t r = tid / KB;
    const int64_t kb = tid - r * KB;
    const uint8_t* ip = idx + ((r / g) * KB + kb) * n;
    const T* vp = values + r * Kp + kb * n;
    T row[MB];
#pragma unroll
    for (int j = 0; j < MB; ++j) row[j] = T(0);
    for (int t = 0; t < n; ++t) {
        const int pos = ip[t];
        const T v = vp[t];
#pragma unroll
        for (int j = 0; j < MB; ++j)
            if (j == pos) row[j] = v;
    }
    store_block<T, MB>(W + r * ldw + kb * MB, row, aligned);
}

}  // namespace sten
