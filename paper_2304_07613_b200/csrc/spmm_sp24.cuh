// spmm_sp24.cuh -- K6: grouped n:m x dense SpMM on the 2:4 structured-sparse tensor cores
// (tcgen05.mma.sp.kind::f16, bf16 in, fp32 accumulate in TMEM).  NEXT-4 of SURVEY.md 8(f).
//
// The grouped n:m mask of every row (the group shares it) is, for n = 1 (any m)
// and for n = 2 with 4 | m, also a 2:4 mask on the aligned 4-windows of K: a 4-window meets at
// most two m-blocks when n = 1, and lies inside one block when 4 | m.  So the product
// C = densify(values, idx) . B is a sparse-A GEMM the hardware runs natively:
// A = the weight, compressed to 2 stored values per 4-window (explicit zeros where a window
// holds fewer than 2 kept entries), plus 2-bit positions ("metadata") per stored value.
//
//   sp24_pack_kernel  -- (values, idx) -> the packed operand: v24 [M128][Kc] bf16 (Kc = K128/2,
//                        K128 = K rounded up to 128, rows padded to a multiple of 128 with zeros)
//                        and the metadata image meta [M128/128][K128/128][128 lanes][4] u32,
//                        laid out exactly as TMEM wants it (one 32-bit column per 32 logical k,
//                        measured with tools/sp_probe.cu: row r, 4-group j of a column ->
//                        lane r%8 + 16 (r/16) + 8 (j/4), nibble j%4 + 4 ((r/8)%2), nibble =
//                        pos0 | pos1 << 2 with pos0 < pos1).
//   spmm_sp24_kernel  -- CTA tile MB*128 rows x BN tokens, K-tiles of 128 logical k:
//                        warp 0 = TMA producer (A boxes [128 rows][64 stored k] SWIZZLE_128B,
//                        B boxes [128 k][64 tokens] SWIZZLE_128B = the MN-major operand, metadata
//                        2 KB bulk copies), warp 1 = MMA issuer (tcgen05.cp 128x128b of the
//                        metadata into TMEM, then 4 sparse MMAs M128 x N=BN x K32 per row block,
//                        tcgen05.commit frees the stage), warp 2 = TMEM allocator, warps 4..7 =
//                        epilogue (tcgen05.ld 32x32b: lane = row, columns = tokens).
#pragma once
#include "common.cuh"
#include "spmm_simt.cuh"   // store_out
#include "spmm_tc.cuh"     // tcgen05 / TMEM helpers
#include "tma_host.h"

namespace sten {

// formats whose every pattern is 2:4 on aligned 4-windows of K
__host__ __device__ inline bool sp24_compatible(int n, int m) { return n == 1 || (n == 2 && m % 4 == 0); }

__host__ __device__ inline int64_t sp24_k128(int64_t K) { return (K + 127) / 128 * 128; }
__host__ __device__ inline int64_t sp24_m128(int64_t M) { return (M + 127) / 128 * 128; }

// ---- pack: one thread per metadata word (128-row block, K-tile, lane, 32-k chunk) ------------------
// The word holds 8 (row, 4-window) nibbles; the same thread writes those 8 windows' 2 stored values.
template <int N_>
__global__ void __launch_bounds__(256)
sp24_pack_kernel(const bf16_t* __restrict__ values, const uint8_t* __restrict__ idx, int64_t M, int64_t K, int n_rt,
                 int m, int g, bf16_t* __restrict__ v24, uint32_t* __restrict__ meta) {
    const int n = N_ > 0 ? N_ : n_rt;
    const int64_t KT = sp24_k128(K) / 128, Kc = sp24_k128(K) / 2, KB = K / m, Kp = KB * n;
    const int64_t words = sp24_m128(M) / 128 * KT * 512;
    const int64_t wid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (wid >= words) return;
    const int c = int(wid & 3), L = int((wid >> 2) & 127);
    const int64_t kt = (wid >> 9) % KT, mb = (wid >> 9) / KT;
    uint32_t word = 0;
#pragma unroll
    for (int b = 0; b < 8; ++b) {
        const int rr = L % 8 + 16 * (L / 16) + 8 * (b / 4);
        const int j = 4 * ((L / 8) % 2) + b % 4;
        const int64_t r = mb * 128 + rr;
        const int64_t w = kt * 32 + c * 8 + j;               // 4-window index along K
        const int64_t k0 = 4 * w;
        int pos[2] = {0, 1};
        bf16_t val[2] = {0, 0};
        int cnt = 0;
        if (r < M && k0 < K) {
            const int64_t G = r / g;
            const int64_t kb_lo = k0 / m, kb_hi = min64(KB - 1, (k0 + 3) / m);
            for (int64_t kb = kb_lo; kb <= kb_hi; ++kb)
                for (int t = 0; t < n; ++t) {
                    const int64_t k = kb * m + idx[(G * KB + kb) * n + t];
                    if (k >= k0 && k < k0 + 4 && cnt < 2) {
                        pos[cnt] = int(k - k0);
                        val[cnt] = values[r * Kp + kb * n + t];
                        ++cnt;
                    }
                }
            if (cnt == 1) {                                   // second slot: an explicit zero elsewhere
                const int q = pos[0] == 3 ? 2 : 3;
                if (q < pos[0]) { pos[1] = pos[0]; val[1] = val[0]; pos[0] = q; val[0] = 0; }
                else { pos[1] = q; val[1] = 0; }
            }
        }
        word |= uint32_t(pos[0] | (pos[1] << 2)) << (4 * b);
        if (r < sp24_m128(M)) {
            bf16_t* dst = v24 + r * Kc + 2 * w;
            *reinterpret_cast<uint32_t*>(dst) = uint32_t(val[0]) | (uint32_t(val[1]) << 16);
        }
    }
    meta[wid] = word;
}

// ---- SpMM ------------------------------------------------------------------------------------------
struct Sp24Args {
    const void* v24;
    const uint32_t* meta;
    const void* B;
    void* C;
    int64_t M, K, N, ldb, ldc;
    int64_t KT;            // K-tiles of 128 logical k (metadata image blocks)
    int64_t Kc;            // stored k per row (K128 / 2)
    int nkt;               // K-steps of 64 logical k per tile (stages)
    int row_tiles, col_tiles;
    bool c_vec;
    // fused epilogue (NEXT-3 on the tensor-core path): C = act(A.B + bias[row]) + residual[row][col]
    const float* bias;     // [M] fp32 or NULL
    int act;               // 0 none, 1 GELU (erf form), 2 ReLU
    const void* residual;  // [M][ldr] of the C dtype or NULL
    int64_t ldr;
    int exp;               // debug experiments (STEN_SP24_EXP, timing only): 1 no MMA, 2 no B loads,
                           // 4 no A loads, 8 no metadata, 16 no epilogue stores, 32 no TMEM
                           // drain, 64 no metadata TMEM stores
};

// the fused epilogue on 32 consecutive tokens [col, col + 32) of one row (fp32 accumulators as bits)
template <typename TC>
STEN_DEVICE_INLINE void sp24_epilogue(const Sp24Args& a, int64_t row, int64_t col, uint32_t (&r)[32]) {
    if (!a.bias && !a.act && !a.residual) return;
    if (row >= a.M) return;
    const float b = a.bias ? a.bias[row] : 0.0f;
    const TC* R = a.residual ? static_cast<const TC*>(a.residual) + row * a.ldr : nullptr;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
        float x = __uint_as_float(r[j]) + b;
        if (a.act == 1) x = 0.5f * x * (1.0f + erff(x * 0.70710678118654752f));
        else if (a.act == 2) x = fmaxf(x, 0.0f);
        if (R && col + j < a.N) x = __fadd_rn(x, to_f32(R[col + j]));
        r[j] = __float_as_uint(x);
    }
}

STEN_DEVICE_INLINE void tc_mma_sp_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t e_tmem,
                                     uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %5, 0;\n\t"
        "tcgen05.mma.sp.cta_group::1.kind::f16 [%0], %1, %2, [%3], %4, p;\n\t}\n" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(e_tmem), "r"(idesc), "r"(acc)
        : "memory");
}
// shared -> TMEM copy of 128 lanes x 128 bits (4 columns); source = 128 rows of 16 bytes, described
// by a no-swizzle matrix descriptor (8-row core matrices of 128 bytes, SBO = 128 bytes)
STEN_DEVICE_INLINE void tc_cp_128x128b(uint32_t taddr, uint64_t sdesc) {
    asm volatile("tcgen05.cp.cta_group::1.128x128b [%0], %1;\n" ::"r"(taddr), "l"(sdesc) : "memory");
}
STEN_DEVICE_INLINE void tmem_st_32x32b_x2(uint32_t taddr, uint32_t r0, uint32_t r1) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};\n" ::"r"(taddr), "r"(r0), "r"(r1) : "memory");
}
STEN_DEVICE_INLINE void tmem_ld_32x32b_x32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr)
        : "memory");
}
STEN_DEVICE_INLINE uint2 ldg_nc_u2(const void* p) {
    uint2 v;
    asm volatile("ld.global.nc.v2.u32 {%0, %1}, [%2];\n" : "=r"(v.x), "=r"(v.y) : "l"(p));
    return v;
}

// MN-major SWIZZLE_128B operand descriptor (B = [64-token chunks][k rows of 128 bytes]):
// LBO = byte stride between 64-token chunks, SBO = 1024 (8 k rows), layout type 2, version 1.
STEN_DEVICE_INLINE uint64_t tc_sdesc_mn_sw128(uint32_t saddr, uint32_t lbo) {
    return uint64_t((saddr >> 4) & 0x3FFFu) | (uint64_t((lbo >> 4) & 0x3FFFu) << 16) |
           (uint64_t(1024 >> 4) << 32) | (uint64_t(1) << 46) | (uint64_t(2) << 61);
}

// Persistent CTA (one per SM), 16 warps:
//   warp 0       TMA producer: per 64-k stage one A box [MB*128 rows][32 stored k] (SWIZZLE_64B, the
//                K-major operand) and BN/64 B boxes [64 k][64 tokens] (SWIZZLE_128B, MN-major)
//   warp 1       MMA issuer: 2 sparse MMAs (K32) per row block per stage, M128 x N=BN
//   warp 2       TMEM allocator
//   warps 4..7   metadata: each lane loads its TMEM lane's 2 words per row block and stage from
//                the metadata image (L2) and writes them with tcgen05.st (lane quadrant = warp % 4)
//   warps 8..15  epilogue: two warps per lane quadrant split the BN columns; TMEM -> registers ->
//                C; D is released to the MMA warp as soon as it is read, so a tile's stores overlap
//                the next tile's loads and MMAs
// Tiles are walked row-tile fastest, so the CTAs running together share their B columns in L2.
template <int MB, int BN, int ST>
struct Sp24Cfg {
    static constexpr int kBM = 128 * MB;
    static constexpr int kAStage = MB * 128 * 64;           // [MB*128 rows][32 stored k] bf16, 64-byte rows
    static constexpr int kABoxRows = MB % 2 == 0 ? 256 : 128;   // TMA boxes of <= 256 rows
    static constexpr int kABoxes = MB * 128 / kABoxRows;
    static constexpr int kBStage = 64 * BN * 2;             // [BN/64 chunks][64 k][64 tokens] bf16
    static constexpr int kStage = kAStage + kBStage;        // multiple of 1024
    static constexpr int kHdr = 1024;
    static constexpr int kStageOut = 8 * 32 * 32 * 4;       // epilogue staging: 8 warps x [32 rows][32 tokens] fp32
    static constexpr size_t kSmem = size_t(kHdr) + size_t(ST) * kStage + kStageOut + 1024;   // + alignment slack
    static constexpr int kDCols = MB * BN;
    static constexpr int kECols = ST * MB * 2;
    static constexpr int kTmemCols = (kDCols + kECols) <= 256 ? 256 : 512;
    static constexpr int kThreads = 512;
    static_assert(kDCols + kECols <= 512, "TMEM budget");
    static_assert(BN % 64 == 0 && BN <= 256, "BN");
    static_assert(kSmem <= 232448, "smem");
};

template <typename TC, int MB, int BN, int ST>
__global__ void __launch_bounds__(512, 1)
spmm_sp24_kernel(const Sp24Args a, const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                 const __grid_constant__ CUtensorMap tmC) {
    using Cfg = Sp24Cfg<MB, BN, ST>;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);       // [ST] A+B landed (tx) + 4 metadata warps
    uint64_t* empty = full + ST;                               // [ST] MMA commit
    uint64_t* dfull = empty + ST;                              // MMA commit: tile accumulated
    uint64_t* dempty = dfull + 1;                              // 8 epilogue warps: D read out
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(dempty + 1);
    auto sA = [&](int s) { return smem + Cfg::kHdr + size_t(s) * Cfg::kStage; };
    auto sB = [&](int s) { return smem + Cfg::kHdr + size_t(s) * Cfg::kStage + Cfg::kAStage; };

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nkt = a.nkt;
    const int ntiles = a.row_tiles * a.col_tiles;

    if (threadIdx.x == 0) {
        for (int s = 0; s < ST; ++s) { mbar_init(&full[s], 5); mbar_init(&empty[s], 1); }
        mbar_init(dfull, 1);
        mbar_init(dempty, 8);
        fence_mbar_init();
    }
    if (warp == 2) tmem_alloc(tmem_slot, Cfg::kTmemCols);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t tD = tmem, tE = tmem + Cfg::kDCols;

    if (warp == 0) {
        // ======================= TMA producer =======================
        if (lane == 0) {
            asm volatile("griddepcontrol.wait;\n" ::: "memory");
            const uint32_t tx = uint32_t((a.exp & 4) ? 0 : Cfg::kAStage) + uint32_t((a.exp & 2) ? 0 : Cfg::kBStage);
            int g = 0;
            for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
                const int64_t m0 = int64_t(t % a.row_tiles) * Cfg::kBM, n0 = int64_t(t / a.row_tiles) * BN;
                for (int kt = 0; kt < nkt; ++kt, ++g) {
                    const int s = g % ST;
                    if (g >= ST) mbar_wait(&empty[s], uint32_t(((g / ST) - 1) & 1));
                    mbar_arrive_expect_tx(&full[s], tx);
                    if (!(a.exp & 4)) {
#pragma unroll
                        for (int h = 0; h < Cfg::kABoxes; ++h)
                            tma_load_2d(sA(s) + h * Cfg::kABoxRows * 64, &tmA, &full[s], kt * 32,
                                        int(m0 + Cfg::kABoxRows * h));
                    }
                    if (!(a.exp & 2)) {
#pragma unroll
                        for (int c = 0; c < BN / 64; ++c)
                            tma_load_2d(sB(s) + c * 8192, &tmB, &full[s], int(n0 + 64 * c), kt * 64);
                    }
                }
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        // ======================= MMA issuer =======================
        const uint32_t idesc = tc_idesc(BN) | (1u << 2) | (1u << 16);    // sparse A, B MN-major
        int g = 0, it = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
            if (it > 0) mbar_wait(dempty, uint32_t((it - 1) & 1));      // epilogue has read the last D
            tc_fence_after();
            for (int kt = 0; kt < nkt; ++kt, ++g) {
                const int s = g % ST;
                mbar_wait(&full[s], uint32_t((g / ST) & 1));
                tc_fence_after();
                if (elect_one()) {
                    const uint32_t a_base = smem_u32(sA(s)), b_base = smem_u32(sB(s));
#pragma unroll
                    for (int mb = 0; mb < MB; ++mb) {
                        if (a.exp & 1) continue;
                        const uint32_t ecol = tE + uint32_t((s * MB + mb) * 2);
#pragma unroll
                        for (int kk = 0; kk < 2; ++kk)
                            // A: K-major SWIZZLE_64B (64-byte rows, 512-byte atoms), row block mb at mb*8 KB,
                            // K32 step = 32 bytes; B: 32 k rows per step (4 KB); metadata column pair ecol,
                            // member kk in the descriptor's sparse-id2 field
                            tc_mma_sp_ss(tD + uint32_t(mb * BN), tc_sdesc_sw(a_base + mb * 8192 + kk * 32, 64),
                                         tc_sdesc_mn_sw128(b_base + kk * 4096, 8192), ecol, idesc | uint32_t(kk),
                                         (kt > 0 || kk > 0) ? 1u : 0u);
                    }
                    tc_commit(&empty[s]);
                }
                __syncwarp();
            }
            if (elect_one()) tc_commit(dfull);
            __syncwarp();
        }
    } else if (warp >= 4 && warp < 8) {
        // ======================= metadata writers =======================
        const int q = warp & 3;
        const int tl = 32 * q + lane;                                  // TMEM lane
        int g = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
            const int64_t mb0 = int64_t(t % a.row_tiles) * MB;
            for (int kt = 0; kt < nkt; ++kt, ++g) {
                const int s = g % ST;
                uint2 w[MB];
#pragma unroll
                for (int mb = 0; mb < MB; ++mb) {
                    const int64_t blk = (mb0 + mb) * a.KT + (kt >> 1);
                    const bool in = (mb0 + mb) * 128 < sp24_m128(a.M) && !(a.exp & 8);
                    w[mb] = in ? ldg_nc_u2(a.meta + (blk * 128 + tl) * 4 + 2 * (kt & 1)) : make_uint2(0x44444444u, 0x44444444u);
                }
                if (g >= ST) mbar_wait(&empty[s], uint32_t(((g / ST) - 1) & 1));
                tc_fence_after();
                if (!(a.exp & 64)) {
#pragma unroll
                    for (int mb = 0; mb < MB; ++mb)
                        tmem_st_32x32b_x2(tE + uint32_t((s * MB + mb) * 2) + (uint32_t(32 * q) << 16), w[mb].x, w[mb].y);
                    tmem_wait_st();
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&full[s]);
            }
        }
    } else if (warp >= 8) {
        // ======================= epilogue =======================
        // TMEM -> registers (tcgen05.ld 32x32b: lane = row, 32 consecutive tokens) -> a per-warp staging
        // tile [32 rows][32 tokens] in shared memory -> TMA store (cp.async.bulk.tensor, clipped at M / N)
        const int q = warp & 3, h = (warp - 8) >> 2;                  // lane quadrant, column half
        constexpr int HC = BN / 2;                                     // columns per warp and row block
        constexpr int ES = int(sizeof(TC));
        unsigned char* stage_out = smem + Cfg::kHdr + size_t(ST) * Cfg::kStage + size_t(warp - 8) * 32 * 32 * 4;
        int it = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
            const int64_t m0 = int64_t(t % a.row_tiles) * Cfg::kBM, n0 = int64_t(t / a.row_tiles) * BN;
            mbar_wait(dfull, uint32_t(it & 1));
            tc_fence_after();
#pragma unroll 1
            for (int mb = 0; mb < MB; ++mb) {
                const int64_t row0 = m0 + 128 * mb + 32 * q;
#pragma unroll 1
                for (int c0 = 0; c0 < HC; c0 += 32) {
                    uint32_t r[32];
                    if (!(a.exp & 32)) {
                        tmem_ld_32x32b_x32(tD + (uint32_t(32 * q) << 16) + uint32_t(mb * BN + h * HC + c0), r);
                        tmem_wait_ld();
                    }
                    if (mb == MB - 1 && c0 + 32 >= HC) {
                        // all of this warp's D columns are in registers: release D to the MMA warp
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) mbar_arrive(dempty);
                    }
                    const int64_t col0 = n0 + h * HC + c0;
                    if (row0 >= a.M || col0 >= a.N || (a.exp & 16)) continue;
                    sp24_epilogue<TC>(a, row0 + lane, col0, r);
                    // the previous TMA store of this warp has finished reading the staging tile
                    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
                    __syncwarp();
                    // row `lane` of the staging tile: 32 tokens, 16-byte chunks rotated by the lane so a
                    // warp's st.shared spread over the banks
                    unsigned char* srow = stage_out + size_t(lane) * 32 * ES;
                    constexpr int CH = 32 * ES / 16;                      // 16-byte chunks per row
#pragma unroll
                    for (int cc = 0; cc < CH; ++cc) {
                        const int c = (cc + lane) % CH;
                        uint4 u;
                        if constexpr (ES == 4) {
                            u = make_uint4(r[4 * c], r[4 * c + 1], r[4 * c + 2], r[4 * c + 3]);
                        } else {
                            uint32_t p[4];
#pragma unroll
                            for (int e = 0; e < 4; ++e)
                                p[e] = uint32_t(f32_to_bf16_rne(__uint_as_float(r[8 * c + 2 * e]))) |
                                       (uint32_t(f32_to_bf16_rne(__uint_as_float(r[8 * c + 2 * e + 1]))) << 16);
                            u = make_uint4(p[0], p[1], p[2], p[3]);
                        }
                        *reinterpret_cast<uint4*>(srow + c * 16) = u;
                    }
                    fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) {
                        asm volatile(
                            "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];\n" ::"l"(&tmC),
                            "r"(int(col0)), "r"(int(row0)), "r"(smem_u32(stage_out))
                            : "memory");
                        asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
                    }
                }
            }
        }
        if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
        __syncwarp();
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(tmem, Cfg::kTmemCols);
    }
}

// ---- 2-SM variant: cta_group::2 (a CTA pair on two SMs shares every MMA) -------------------------
// The pair computes 256 rows x 256 tokens per tile with tcgen05.mma.sp.cta_group::2 (M = 256,
// N = 256): each SM stages only ITS 128 rows of A and ITS 128 tokens of B (the MMA reads the two
// halves of B from both SMs), so the per-SM shared-memory traffic per MMA drops from 4 KB + 16 KB to
// 4 KB + 8 KB -- the sparse MMA is shared-memory bound in the 1-SM form.
// Stages of 128 logical k: per CTA one A box [128 rows][64 stored k] (SWIZZLE_128B), two B boxes
// [128 k][64 tokens] (SWIZZLE_128B) and the stage's metadata (128 lanes x 16 bytes, a 3-D TMA box of
// the metadata image), all completing on the LEADER's (cluster rank 0) stage barrier; the leader's
// MMA lane copies both CTAs' metadata into their TMEM (tcgen05.cp.cta_group::2 128x128b) and issues
// 4 sparse MMAs; its commits arrive on both CTAs' empty / D-full barriers (multicast); both CTAs'
// epilogue warps drain their own rows and arrive on the leader's D-empty barrier remotely.
template <int ST>
struct Sp24Cfg2 {
    static constexpr int kBM = 256;                          // pair rows (128 per CTA)
    static constexpr int kBN = 256;                          // pair tokens (128 per CTA's B half)
    static constexpr int kAStage = 128 * 128;                // [128 rows][64 stored k] bf16 (SWIZZLE_128B)
    static constexpr int kBStage = 128 * 128 * 2;            // [2 chunks][128 k][64 tokens] bf16 (SWIZZLE_128B)
    static constexpr int kEStage = 2048;                     // [128 lanes][4 u32]
    static constexpr int kStage = kAStage + kBStage + kEStage;
    static constexpr int kHdr = 1024;
    static constexpr int kStageOut = 8 * 32 * 32 * 4;
    static constexpr size_t kSmem = size_t(kHdr) + size_t(ST) * kStage + kStageOut + 1024;
    static constexpr int kDCols = 256;
    static constexpr int kECols = ST * 4;
    static constexpr int kThreads = 512;
    static_assert(kDCols + kECols <= 512, "TMEM budget");
    static_assert(kSmem <= 232448, "smem");
};

STEN_DEVICE_INLINE void tc_mma_sp_ss_2sm(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t e_tmem,
                                         uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %5, 0;\n\t"
        "tcgen05.mma.sp.cta_group::2.kind::f16 [%0], %1, %2, [%3], %4, p;\n\t}\n" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(e_tmem), "r"(idesc), "r"(acc)
        : "memory");
}
STEN_DEVICE_INLINE void tc_cp_128x128b_2sm(uint32_t taddr, uint64_t sdesc) {
    asm volatile("tcgen05.cp.cta_group::2.128x128b [%0], %1;\n" ::"r"(taddr), "l"(sdesc) : "memory");
}
STEN_DEVICE_INLINE void tc_commit_2sm_mc(uint64_t* bar, uint16_t mask) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(
            smem_u32(bar)),
        "h"(mask)
        : "memory");
}
STEN_DEVICE_INLINE void tma_load_2d_2sm(void* smem_dst, const void* tmap, uint32_t bar_leader, int x, int y) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], "
        "[%2];\n" ::"r"(smem_u32(smem_dst)),
        "l"(tmap), "r"(bar_leader), "r"(x), "r"(y)
        : "memory");
}
STEN_DEVICE_INLINE void tma_load_3d_2sm(void* smem_dst, const void* tmap, uint32_t bar_leader, int x, int y, int z) {
    asm volatile(
        "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, "
        "%5}], [%2];\n" ::"r"(smem_u32(smem_dst)),
        "l"(tmap), "r"(bar_leader), "r"(x), "r"(y), "r"(z)
        : "memory");
}
STEN_DEVICE_INLINE void mbar_arrive_remote(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(cluster_addr) : "memory");
}
STEN_DEVICE_INLINE void mbar_wait_cluster(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "WAITC_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAITC_%=;\n\t}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}

template <typename TC, int ST>
__global__ void __launch_bounds__(512, 1)
spmm_sp24_2sm_kernel(const Sp24Args a, const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmE) {
    using Cfg = Sp24Cfg2<ST>;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);       // [ST] (leader) A + B + E of both CTAs
    uint64_t* empty = full + ST;                               // [ST] (each) leader's MMA commit
    uint64_t* dfull = empty + ST;                              // (each) leader's commit: tile accumulated
    uint64_t* dempty = dfull + 1;                              // (leader) 16 epilogue warps: D read out
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(dempty + 1);
    auto sA = [&](int s) { return smem + Cfg::kHdr + size_t(s) * Cfg::kStage; };
    auto sB = [&](int s) { return smem + Cfg::kHdr + size_t(s) * Cfg::kStage + Cfg::kAStage; };
    auto sE = [&](int s) { return smem + Cfg::kHdr + size_t(s) * Cfg::kStage + Cfg::kAStage + Cfg::kBStage; };

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();                   // 0 = leader
    const int pair = int(blockIdx.x >> 1), npairs = int(gridDim.x >> 1);
    const int nkt = int(a.KT);                                 // stages of 128 logical k
    const int ntiles = a.row_tiles * a.col_tiles;

    if (threadIdx.x == 0) {
        for (int s = 0; s < ST; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        mbar_init(dfull, 1);
        mbar_init(dempty, 16);
        fence_mbar_init();
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                     "r"(512)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n" ::: "memory");
    }
    tc_fence_before();
    cluster_sync_all();                                        // barriers of both CTAs initialised
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t tD = tmem, tE = tmem + Cfg::kDCols;
    const uint32_t full0 = map_cluster(smem_u32(full), 0);     // the leader's stage barriers
    const uint32_t dempty0 = map_cluster(smem_u32(dempty), 0);

    if (warp == 0) {
        // ======================= TMA producer (both CTAs) =======================
        if (lane == 0) {
            asm volatile("griddepcontrol.wait;\n" ::: "memory");
            int g = 0;
            const int mrows = int(sp24_m128(a.M) / 128);
            for (int t = pair; t < ntiles; t += npairs) {
                const int64_t mblk = int64_t(t % a.row_tiles) * 2 + rank;        // this CTA's 128-row block
                const int64_t n0 = int64_t(t / a.row_tiles) * Cfg::kBN + 128 * rank;
                for (int kt = 0; kt < nkt; ++kt, ++g) {
                    const int s = g % ST;
                    if (g >= ST) mbar_wait(&empty[s], uint32_t(((g / ST) - 1) & 1));
                    if (rank == 0) mbar_arrive_expect_tx(&full[s], (a.exp & 6) ? 0u : uint32_t(2 * Cfg::kStage));
                    const uint32_t bar = full0 + uint32_t(s) * 8u;
                    if (!(a.exp & 6)) {
                        tma_load_2d_2sm(sA(s), &tmA, bar, kt * 64, int(mblk * 128));
#pragma unroll
                        for (int c = 0; c < 2; ++c)
                            tma_load_2d_2sm(sB(s) + c * 16384, &tmB, bar, int(n0 + 64 * c), kt * 128);
                        // metadata image block (mblk, kt); a block past M128 is clamped (its rows are padding)
                        tma_load_3d_2sm(sE(s), &tmE, bar, 0, 0, int((mblk < mrows ? mblk : mrows - 1) * a.KT + kt));
                    }
                }
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        // ======================= MMA issuer (leader only) =======================
        if (rank == 0) {
            const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(256 >> 3) << 17) |
                                   (uint32_t(256 >> 4) << 24) | (1u << 2) | (1u << 16);   // M 256, N 256, sparse, B MN-major
            int g = 0, it = 0;
            for (int t = pair; t < ntiles; t += npairs, ++it) {
                if (it > 0) mbar_wait_cluster(dempty, uint32_t((it - 1) & 1));
                tc_fence_after();
                for (int kt = 0; kt < nkt; ++kt, ++g) {
                    const int s = g % ST;
                    mbar_wait_cluster(&full[s], uint32_t((g / ST) & 1));
                    tc_fence_after();
                    if (elect_one()) {
                        const uint32_t a_base = smem_u32(sA(s)), b_base = smem_u32(sB(s));
                        const uint32_t ecol = tE + uint32_t(s * 4);
                        if (!(a.exp & 1)) {
                            tc_cp_128x128b_2sm(ecol, tc_sdesc(smem_u32(sE(s)), 16, 128));
                            const uint64_t adesc = tc_sdesc_sw128(a_base);
#pragma unroll
                            for (int kk = 0; kk < 4; ++kk)
                                tc_mma_sp_ss_2sm(tD, adesc + uint64_t(kk * 2), tc_sdesc_mn_sw128(b_base + kk * 4096, 16384),
                                                 ecol + uint32_t(kk & 2), idesc | uint32_t(kk & 1),
                                                 (kt > 0 || kk > 0) ? 1u : 0u);
                        }
                        tc_commit_2sm_mc(&empty[s], uint16_t(0x3));
                    }
                    __syncwarp();
                }
                if (elect_one()) tc_commit_2sm_mc(dfull, uint16_t(0x3));
                __syncwarp();
            }
        }
    } else if (warp >= 8) {
        // ======================= epilogue (both CTAs, own rows) =======================
        const int q = warp & 3, h = (warp - 8) >> 2;
        constexpr int HC = 128;                                        // columns per warp (of 256)
        constexpr int ES = int(sizeof(TC));
        unsigned char* stage_out = smem + Cfg::kHdr + size_t(ST) * Cfg::kStage + size_t(warp - 8) * 32 * 32 * 4;
        int it = 0;
        for (int t = pair; t < ntiles; t += npairs, ++it) {
            const int64_t m0 = int64_t(t % a.row_tiles) * Cfg::kBM + 128 * rank;
            const int64_t n0 = int64_t(t / a.row_tiles) * Cfg::kBN;
            mbar_wait_cluster(dfull, uint32_t(it & 1));
            tc_fence_after();
            const int64_t row0 = m0 + 32 * q;
#pragma unroll 1
            for (int c0 = 0; c0 < HC; c0 += 32) {
                uint32_t r[32];
                if (!(a.exp & 32)) {
                    tmem_ld_32x32b_x32(tD + (uint32_t(32 * q) << 16) + uint32_t(h * HC + c0), r);
                    tmem_wait_ld();
                }
                if (c0 + 32 >= HC) {
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive_remote(dempty0);
                }
                const int64_t col0 = n0 + h * HC + c0;
                if (row0 >= a.M || col0 >= a.N || (a.exp & 16)) continue;
                sp24_epilogue<TC>(a, row0 + lane, col0, r);
                if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
                __syncwarp();
                unsigned char* srow = stage_out + size_t(lane) * 32 * ES;
                constexpr int CH = 32 * ES / 16;
#pragma unroll
                for (int cc = 0; cc < CH; ++cc) {
                    const int c = (cc + lane) % CH;
                    uint4 u;
                    if constexpr (ES == 4) {
                        u = make_uint4(r[4 * c], r[4 * c + 1], r[4 * c + 2], r[4 * c + 3]);
                    } else {
                        uint32_t pk[4];
#pragma unroll
                        for (int e = 0; e < 4; ++e)
                            pk[e] = uint32_t(f32_to_bf16_rne(__uint_as_float(r[8 * c + 2 * e]))) |
                                    (uint32_t(f32_to_bf16_rne(__uint_as_float(r[8 * c + 2 * e + 1]))) << 16);
                        u = make_uint4(pk[0], pk[1], pk[2], pk[3]);
                    }
                    *reinterpret_cast<uint4*>(srow + c * 16) = u;
                }
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
                    asm volatile(
                        "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];\n" ::"l"(&tmC),
                        "r"(int(col0)), "r"(int(row0)), "r"(smem_u32(stage_out))
                        : "memory");
                    asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
                }
            }
        }
        if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
        __syncwarp();
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();                                        // the peer's TMEM / smem stay alive until the pair is done
    if (warp == 2) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(512) : "memory");
    }
}

}  // namespace sten
