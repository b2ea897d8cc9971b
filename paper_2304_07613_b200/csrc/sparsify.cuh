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
// The first min(4, 32/m) rows of the group stay in registers between the score
// pass and the compaction pass; later rows are re-read (L1/L2 hits).  HBM roofline:
// M*K*s (read W) + M*K'*s (values) + (M/g)*(K/m)*n (idx) bytes.
#pragma once
#include "common.cuh"

namespace sten {

// 256-bit global load (sm_100: LDG.E.ENL2.256): one request per lane for a 32-byte block, so a
// warp's instruction covers 1 KB contiguous instead of two half-used 512-byte passes.
STEN_DEVICE_INLINE void ldg256(const void* p, uint32_t (&v)[8]) {
    asm volatile("ld.global.nc.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "l"(p));
}

// aligned: 0 = element alignment only, 1 = 16-byte, 2 = 32-byte aligned block starts
template <typename T, int MB>
STEN_DEVICE_INLINE void load_block(const T* __restrict__ p, T (&row)[MB], int aligned) {
    constexpr int BYTES = MB * int(sizeof(T));
    if constexpr (BYTES % 32 == 0) {
        if (aligned == 2) {
            uint32_t tmp[BYTES / 4];
#pragma unroll
            for (int q = 0; q < BYTES / 32; ++q) {
                uint32_t v[8];
                ldg256(reinterpret_cast<const unsigned char*>(p) + 32 * q, v);
#pragma unroll
                for (int e = 0; e < 8; ++e) tmp[8 * q + e] = v[e];
            }
            memcpy(row, tmp, BYTES);
            return;
        }
    }
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

// rows of a group kept in registers between the two passes (<= 4 rows, <= 32 elements per thread:
// fewer registers, more resident warps, more loads in flight)
template <int MB>
constexpr int sparsify_reg_rows() { return 32 / MB < 1 ? 1 : (32 / MB > 4 ? 4 : 32 / MB); }

template <int BYTES> struct UintOf;
template <> struct UintOf<1> { using type = uint8_t; };
template <> struct UintOf<2> { using type = uint16_t; };
template <> struct UintOf<4> { using type = uint32_t; };
template <> struct UintOf<8> { using type = uint2; };
template <> struct UintOf<16> { using type = uint4; };

// number of kept-position slots a body carries: NK (vector stores) or MB - 1 (any n < MB)
template <int MB, int NK>
__host__ __device__ constexpr int kept_slots() { return NK > 0 ? NK : MB - 1; }

// a2 select: rank[j] = #{i : s_i > s_j or (s_i == s_j and i < j)}; keep iff rank < n.
// The rank rule is the total order (score descending, position ascending), so its n smallest
// ranks are found by n passes of an argmax that scans j ascending with a strict '>' (the first
// of equal scores wins) over the positions not taken yet: n*MB compares instead of MB*MB.
// pos[t] = the t-th kept position, ascending (t < n).
template <int MB, int NK>
STEN_DEVICE_INLINE void select_kept(const float (&s)[MB], int n, int (&pos)[kept_slots<MB, NK>()]) {
    uint32_t keep = 0;
    const int nsel = NK > 0 ? NK : n;
#pragma unroll
    for (int t = 0; t < kept_slots<MB, NK>(); ++t) {
        if (t < nsel) {
            int bj = -1;
            float bv = 0.0f;
#pragma unroll
            for (int j = 0; j < MB; ++j) {
                const bool better = !(keep >> j & 1u) && (bj < 0 || s[j] > bv);
                bj = better ? j : bj;
                bv = better ? s[j] : bv;
            }
            keep |= 1u << bj;
        }
    }
    uint32_t rem = keep;
#pragma unroll
    for (int t = 0; t < kept_slots<MB, NK>(); ++t) {
        pos[t] = __ffs(rem) - 1;
        rem &= rem - 1u;
    }
}

// the n idx bytes of one (group, m-block): one store when NK > 0
template <int NK, int NP>
STEN_DEVICE_INLINE void store_idx(uint8_t* __restrict__ ip, const int (&pos)[NP], int n) {
    if constexpr (NK > 0) {
        using IW = typename UintOf<NK>::type;
        IW iw;
        uint8_t ib[NK];
#pragma unroll
        for (int t = 0; t < NK; ++t) ib[t] = uint8_t(pos[t]);
        memcpy(&iw, ib, NK);
        *reinterpret_cast<IW*>(ip) = iw;
    } else {
#pragma unroll
        for (int t = 0; t < NP; ++t)
            if (t < n) ip[t] = uint8_t(pos[t]);
    }
}

// a3 compact: bit copy of the kept entries of one row block (select network, then one vector
// store when NK > 0) to vp = &values[r][kb n]
template <typename T, int MB, int NK>
STEN_DEVICE_INLINE void store_kept(const T (&row)[MB], const int (&pos)[kept_slots<MB, NK>()], T* __restrict__ vp,
                                   int n) {
    constexpr int NP = kept_slots<MB, NK>();
    // the select network on the 32-bit containers of the elements, one selp per position: written
    // as C++ selects, nvcc turns the chain into an indexed load from a stack copy of the row
    // (STL + LDL per kept entry), which made K1 local-memory-latency bound
    uint32_t rb[MB];
#pragma unroll
    for (int j = 0; j < MB; ++j) {
        if constexpr (sizeof(T) == 4) rb[j] = __float_as_uint(reinterpret_cast<const float&>(row[j]));
        else rb[j] = uint32_t(reinterpret_cast<const uint16_t&>(row[j]));
    }
    T out[NP];
#pragma unroll
    for (int t = 0; t < NP; ++t) {
        uint32_t v = rb[0];
#pragma unroll
        for (int j = 1; j < MB; ++j)
            asm("{\n\t.reg .pred q;\n\tsetp.eq.s32 q, %2, %3;\n\tselp.b32 %0, %1, %0, q;\n\t}"
                : "+r"(v) : "r"(rb[j]), "r"(pos[t]), "r"(j));
        if constexpr (sizeof(T) == 4) reinterpret_cast<float&>(out[t]) = __uint_as_float(v);
        else reinterpret_cast<uint16_t&>(out[t]) = uint16_t(v);
    }
    if constexpr (NK > 0) {
        using VW = typename UintOf<NK * int(sizeof(T))>::type;
        VW w;
        memcpy(&w, out, sizeof(VW));
        *reinterpret_cast<VW*>(vp) = w;
    } else {
#pragma unroll
        for (int t = 0; t < NP; ++t)
            if (t < n) vp[t] = out[t];
    }
}

// Loads of R rows of a group issued back to back (rows >= g are clamped to row 0 and their
// values ignored), so a thread has R*MB*s bytes in flight instead of one row per DRAM round trip.
template <typename T, int MB, int R, int ALIGNED>
STEN_DEVICE_INLINE void load_rows(const T* __restrict__ w0, int64_t ldw, int i0, int g, T (&x)[R][MB]) {
#pragma unroll
    for (int i = 0; i < R; ++i) {
        const int r = i0 + i < g ? i0 + i : 0;
        load_block<T, MB>(w0 + r * ldw, x[i], ALIGNED);
    }
}

template <typename T, int MB, int NK, int ALIGNED>
STEN_DEVICE_INLINE void sparsify_finish(const T* __restrict__ w0, int64_t ldw, int64_t grp, int64_t kb, int64_t KB,
                                        int n, int g, T* __restrict__ values, int64_t Kp, uint8_t* __restrict__ idx,
                                        const T (&x)[sparsify_reg_rows<MB>()][MB]);

// NK = n when n in {1, 2, 4} and the values/idx bases allow NK-element vector stores (the
// kept entries of a row are selected into registers and written with ONE store per row; the
// n idx bytes with one store); NK = 0: any n, per-position stores.
template <typename T, int MB, int NK, int ALIGNED>
STEN_DEVICE_INLINE void sparsify_body(const T* __restrict__ W, int64_t ldw, int64_t grp, int64_t kb, int64_t KB,
                                      int n, int g, T* __restrict__ values, int64_t Kp,
                                      uint8_t* __restrict__ idx) {
    const T* w0 = W + grp * g * ldw + kb * MB;
    constexpr int R = sparsify_reg_rows<MB>();
    T x[R][MB];                                   // rows 0..R-1 stay in registers for a3
    load_rows<T, MB, R, ALIGNED>(w0, ldw, 0, g, x);
    sparsify_finish<T, MB, NK, ALIGNED>(w0, ldw, grp, kb, KB, n, g, values, Kp, idx, x);
}

// a1-a3 of one (group, m-block) after its first R rows x were loaded (sparsify_body)
template <typename T, int MB, int NK, int ALIGNED>
STEN_DEVICE_INLINE void sparsify_finish(const T* __restrict__ w0, int64_t ldw, int64_t grp, int64_t kb, int64_t KB,
                                        int n, int g, T* __restrict__ values, int64_t Kp, uint8_t* __restrict__ idx,
                                        const T (&x)[sparsify_reg_rows<MB>()][MB]) {
    constexpr int R = sparsify_reg_rows<MB>();
    // a1 score: s[j] = fl32(...fl32(|w_0j| + |w_1j|) ... + |w_(g-1)j|), ascending rows, RNE.
    float s[MB];
#pragma unroll
    for (int j = 0; j < MB; ++j) s[j] = 0.0f;
#pragma unroll
    for (int i = 0; i < R; ++i)
        if (i < g) {
#pragma unroll
            for (int j = 0; j < MB; ++j) s[j] = __fadd_rn(s[j], fabsf(to_f32(x[i][j])));
        }
    for (int i0 = R; i0 < g; i0 += R) {
        T y[R][MB];
        load_rows<T, MB, R, ALIGNED>(w0, ldw, i0, g, y);
#pragma unroll
        for (int i = 0; i < R; ++i)
            if (i0 + i < g) {
#pragma unroll
                for (int j = 0; j < MB; ++j) s[j] = __fadd_rn(s[j], fabsf(to_f32(y[i][j])));
            }
    }

    int pos[kept_slots<MB, NK>()];
    select_kept<MB, NK>(s, n, pos);
    store_idx<NK, kept_slots<MB, NK>()>(idx + (grp * KB + kb) * (NK > 0 ? NK : n), pos, n);
    auto select_store = [&](const T (&row)[MB], int64_t r) {
        store_kept<T, MB, NK>(row, pos, values + r * Kp + kb * (NK > 0 ? NK : n), n);
    };
#pragma unroll
    for (int i = 0; i < R; ++i)
        if (i < g) select_store(x[i], grp * g + i);
    for (int i0 = R; i0 < g; i0 += R) {
        T y[R][MB];
        load_rows<T, MB, R, ALIGNED>(w0, ldw, i0, g, y);
#pragma unroll
        for (int i = 0; i < R; ++i)
            if (i0 + i < g) select_store(y[i], grp * g + i0 + i);
    }
}

template <typename T, int MB, int NK>
__global__ void __launch_bounds__(256)
sparsify_grouped_nm_kernel(const T* __restrict__ W, int64_t ldw, int64_t G, int64_t KB, int n,
                           int g, T* __restrict__ values, int64_t Kp, uint8_t* __restrict__ idx,
                           int aligned) {
    // let a programmatically dependent SpMM launch now: its prologue overlaps this grid, its
    // reads of values / idx wait (griddepcontrol.wait) until this grid has completed
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    const int64_t tid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (tid >= G * KB) return;
    int64_t grp, kb;
    if (G * KB <= int64_t(0x7fffffff)) {          // 32-bit division (no 64-bit division routine)
        const uint32_t t32 = uint32_t(tid), kb32 = uint32_t(KB);
        const uint32_t q = t32 / kb32;
        grp = q;
        kb = int64_t(t32 - q * kb32);
    } else {
        grp = tid / KB;
        kb = tid - grp * KB;
    }
    // uniform branch: the vector-load body or the scalar one, each with straight-line loads
    if (aligned == 2) sparsify_body<T, MB, NK, 2>(W, ldw, grp, kb, KB, n, g, values, Kp, idx);
    else if (aligned == 1) sparsify_body<T, MB, NK, 1>(W, ldw, grp, kb, KB, n, g, values, Kp, idx);
    else sparsify_body<T, MB, NK, 0>(W, ldw, grp, kb, KB, n, g, values, Kp, idx);
}

// Problems of one grouped sparsify launch -- the weights of one step (sten_sparsify_grouped_nm_batched).
constexpr int kMaxSparsifyBatch = 12;
struct SparsifyBatch {
    const void* W[kMaxSparsifyBatch];
    void* values[kMaxSparsifyBatch];
    uint8_t* idx[kMaxSparsifyBatch];
    int64_t ldw[kMaxSparsifyBatch], G[kMaxSparsifyBatch], KB[kMaxSparsifyBatch], Kp[kMaxSparsifyBatch];
    int n[kMaxSparsifyBatch], g[kMaxSparsifyBatch], aligned[kMaxSparsifyBatch];
    int m[kMaxSparsifyBatch], nk[kMaxSparsifyBatch];   // the body variant of each problem
    int block0[kMaxSparsifyBatch + 1];                  // first CTA of each problem; block0[count] = grid                   // first tile of each problem; tile0[count] = total
    int count;
};

// ---- grouped launch (sten_sparsify_grouped_nm_batched) ----------------------------------------
// EVERY weight of a step in ONE launch, whatever its (n, m, g): CTA b works on problem p
// (block0[p] <= b < block0[p+1]), one (group, m-block) item per thread with the body of the
// problem's (m, NK, alignment) -- exactly sparsify_grouped_nm_kernel's, so the same bits.  The
// registers of a launch are those of its largest body, and they set the resident warps (the bytes
// in flight of this latency-bound pass), so there are two instantiations: LEAN = the vector-store
// bodies (NK in {1, 2}) on 16/32-byte aligned rows for m in {2, 4, 8, 10} (every bench format:
// 64 registers fp32, 4 CTAs / SM), and the full set for anything else.
__host__ __device__ inline bool sparsify_lean_ok(int m, int nk, int aligned) {
    return nk > 0 && aligned > 0 && (m == 2 || m == 4 || m == 8 || m == 10);
}

template <typename T, int MB, int LEAN>
STEN_DEVICE_INLINE void sparsify_grouped_item(const SparsifyBatch& bt, int p, int64_t grp, int64_t kb) {
    const T* W = static_cast<const T*>(bt.W[p]);
    T* values = static_cast<T*>(bt.values[p]);
    const int nk = bt.nk[p], al = bt.aligned[p];
#define STEN_SP_BODY(NK_, AL_) \
    sparsify_body<T, MB, NK_, AL_>(W, bt.ldw[p], grp, kb, bt.KB[p], bt.n[p], bt.g[p], values, bt.Kp[p], bt.idx[p])
    if constexpr (LEAN) {
        if (nk == 2) {
            if (al == 2) STEN_SP_BODY(2, 2); else STEN_SP_BODY(2, 1);
        } else {
            if (al == 2) STEN_SP_BODY(1, 2); else STEN_SP_BODY(1, 1);
        }
    } else {
        if (nk == 2) {
            if (al == 2) STEN_SP_BODY(2, 2); else if (al == 1) STEN_SP_BODY(2, 1); else STEN_SP_BODY(2, 0);
        } else if (nk == 1) {
            if (al == 2) STEN_SP_BODY(1, 2); else if (al == 1) STEN_SP_BODY(1, 1); else STEN_SP_BODY(1, 0);
        } else {
            if (al == 2) STEN_SP_BODY(0, 2); else if (al == 1) STEN_SP_BODY(0, 1); else STEN_SP_BODY(0, 0);
        }
    }
#undef STEN_SP_BODY
}

#ifndef STEN_SP_BATCH_THREADS
#define STEN_SP_BATCH_THREADS 128
#endif
constexpr int kSpBatchThreads = STEN_SP_BATCH_THREADS;     // threads per CTA of the grouped launch
template <typename T, int LEAN>
__global__ void __launch_bounds__(kSpBatchThreads)
sparsify_grouped_nm_batched_kernel(const __grid_constant__ SparsifyBatch bt) {
    // let a programmatically dependent SpMM launch now: its prologue overlaps this grid
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    const int b = int(blockIdx.x);
    int p = 0;
    while (p + 1 < bt.count && b >= bt.block0[p + 1]) ++p;
    const int64_t tid = int64_t(b - bt.block0[p]) * blockDim.x + threadIdx.x;
    const int64_t KB = bt.KB[p];
    if (tid >= bt.G[p] * KB) return;
    const uint32_t t32 = uint32_t(tid), kb32 = uint32_t(KB);       // G*KB < 2^31 (checked on the host)
    const uint32_t q = t32 / kb32;
    const int64_t grp = q, kb = int64_t(t32 - q * kb32);
    if constexpr (LEAN) {
        switch (bt.m[p]) {
            case 2: sparsify_grouped_item<T, 2, 1>(bt, p, grp, kb); break;
            case 4: sparsify_grouped_item<T, 4, 1>(bt, p, grp, kb); break;
            case 8: sparsify_grouped_item<T, 8, 1>(bt, p, grp, kb); break;
            default: sparsify_grouped_item<T, 10, 1>(bt, p, grp, kb); break;
        }
    } else {
        switch (bt.m[p]) {
            case 2: sparsify_grouped_item<T, 2, 0>(bt, p, grp, kb); break;
            case 4: sparsify_grouped_item<T, 4, 0>(bt, p, grp, kb); break;
            case 6: sparsify_grouped_item<T, 6, 0>(bt, p, grp, kb); break;
            case 8: sparsify_grouped_item<T, 8, 0>(bt, p, grp, kb); break;
            case 10: sparsify_grouped_item<T, 10, 0>(bt, p, grp, kb); break;
            case 12: sparsify_grouped_item<T, 12, 0>(bt, p, grp, kb); break;
            default: sparsify_grouped_item<T, 16, 0>(bt, p, grp, kb); break;
        }
    }
}

// NEXT-2 SameFormat re-sparsification: re-pack a new dense W' with an EXISTING pattern
// ("the new tensor is sparsified using the SameFormatSparsifier to maintain the same format",
// PAPER.md:398): values[r][kb n + t] = W'[r][kb m + idx[r/g][kb][t]].  One thread per
// (row, m-block): one vector load of the block, n selects, n stores.  HBM-bound like K1.
template <typename T, int MB>
__global__ void __launch_bounds__(256)
same_format_grouped_nm_kernel(const T* __restrict__ W, int64_t ldw, int64_t M, int64_t KB, int n, int g,
                              const uint8_t* __restrict__ idx, T* __restrict__ values, int64_t Kp, int aligned,
                              unsigned long long* __restrict__ outside) {
    const int64_t tid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    uint32_t out_cnt = 0;
    if (tid < M * KB) {
        const int64_t r = tid / KB, kb = tid - r * KB;
        T row[MB];
        if (aligned == 2) load_block<T, MB>(W + r * ldw + kb * MB, row, 2);
        else if (aligned == 1) load_block<T, MB>(W + r * ldw + kb * MB, row, 1);
        else load_block<T, MB>(W + r * ldw + kb * MB, row, 0);
        const uint8_t* ip = idx + ((r / g) * KB + kb) * n;
        T* vp = values + r * Kp + kb * n;
        uint32_t kept = 0;
        for (int t = 0; t < n; ++t) {
            const int j = ip[t];
            kept |= 1u << j;
            T v = row[0];
#pragma unroll
            for (int q = 1; q < MB; ++q) v = j == q ? row[q] : v;
            vp[t] = v;
        }
        if (outside) {
            // fixed-mask check: nonzero entries of W' at pruned positions
#pragma unroll
            for (int q = 0; q < MB; ++q) out_cnt += (!(kept >> q & 1u) && to_f32(row[q]) != 0.0f) ? 1u : 0u;
        }
    }
    if (outside) {
        const uint32_t w = __reduce_add_sync(0xffffffffu, out_cnt);
        if ((threadIdx.x & 31) == 0 && w) atomicAdd(outside, (unsigned long long)w);
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
