// spmm_tc.cuh -- K5: bf16 grouped n:m SpMM on the 5th-generation tensor cores
// (tcgen05.mma, accumulators in TMEM), for g a multiple of 16.
//
// As in K4, the product of one group is a dense contraction over its gathered
// rows:  C_G^T[T x RB] = B[S_G, T]^T . V_G^T  (tokens are
// the MMA M dimension, RB <= g rows of one group the N dimension).  A shared-
// memory matrix descriptor cannot gather rows, so the gathered operand is built
// in TENSOR MEMORY:
//   * gather warps (teams of 4, one per TMEM lane quadrant) read the staged dense
//     B slab with `ldmatrix.x4.trans`, one row address per lane = the staged row of
//     the kept k that lane feeds, and write the 16-token x 16-k fragment straight
//     into TMEM with `tcgen05.st.16x256b` (the fragment layout of ldmatrix.trans
//     matches the 16x256b lane/column pattern once the 16 k of a step are
//     assigned to the 4 matrices as {0,1,4,5,..} / {2,3,6,7,..});
//   * one thread issues `tcgen05.mma.cta_group::1.kind::f16` with A in TMEM
//     ([128 tokens x 16 k], 8 columns), B = the group's values from shared memory
//     (canonical K-major layout, no swizzle) and D = the group's fp32
//     accumulators in TMEM (RB columns per row block);
//   * `tcgen05.commit` arrives on mbarriers that free the A buffer (gather ring),
//     the shared-memory stage (producer ring) and finally hand D to the epilogue,
//     which reads it with `tcgen05.ld.32x32b` (lane = token, column = row) and
//     stores 32 consecutive tokens per row per instruction.
// CTA = 512 threads: warp 0 producer (cp.async of the swizzled B slab, the values
// tile and the idx words), warp 1 MMA issuer, warp 2 TMEM allocator, warps 4..15
// three gather teams; warps 0..3 run the epilogue.  Tile: 256 rows x 128 tokens.
#pragma once
#include "common.cuh"
#include "spmm_simt.cuh"   // SpmmArgs, store_out
#include "spmm_mma.cuh"    // ldsm_x4_trans
#include "tma_host.h"

namespace sten {

inline bool tc_supported(int g) { return g % 16 == 0; }

// ---- tcgen05 / TMEM helpers ---------------------------------------------------------------------
STEN_DEVICE_INLINE void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(dst_smem)),
                 "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
}
STEN_DEVICE_INLINE void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(taddr), "r"(ncols) : "memory");
}
STEN_DEVICE_INLINE void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
STEN_DEVICE_INLINE void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
STEN_DEVICE_INLINE void tc_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(bar))
                 : "memory");
}
STEN_DEVICE_INLINE void tmem_st_16x256b(uint32_t taddr, uint32_t r0, uint32_t r1, uint32_t r2, uint32_t r3) {
    asm volatile("tcgen05.st.sync.aligned.16x256b.x1.b32 [%0], {%1, %2, %3, %4};\n" ::"r"(taddr), "r"(r0), "r"(r1),
                 "r"(r2), "r"(r3)
                 : "memory");
}
STEN_DEVICE_INLINE void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }
STEN_DEVICE_INLINE void tmem_ld_32x32b_x16(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr)
        : "memory");
}
STEN_DEVICE_INLINE void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }

// D[tmem] (+)= A[tmem] . B[smem desc]; kind::f16 (bf16 in, fp32 accumulate), cta_group::1
STEN_DEVICE_INLINE void tc_mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(acc)
        : "memory");
}

// Instruction descriptor, kind::f16: D fp32, A/B bf16, both K-major, M = 128, N = n.
__host__ __device__ constexpr uint32_t tc_idesc(int n) {
    return (1u << 4)                        // c_format = F32
           | (1u << 7)                      // a_format = BF16
           | (1u << 10)                     // b_format = BF16
           | (uint32_t(n >> 3) << 17)       // n_dim
           | (uint32_t(128 >> 4) << 24);    // m_dim
}

// Shared-memory matrix descriptor, SWIZZLE_NONE (canonical core matrices of 8 rows x 16 B):
// lbo = byte stride between core matrices along K, sbo = along M/N; version 1 (sm_100).
STEN_DEVICE_INLINE uint64_t tc_sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    return uint64_t((saddr >> 4) & 0x3FFFu) | (uint64_t((lbo >> 4) & 0x3FFFu) << 16) |
           (uint64_t((sbo >> 4) & 0x3FFFu) << 32) | (uint64_t(1) << 46);
}

template <int RB>
struct TcCfg {
    static constexpr int kBM = 256;              // rows per CTA (D: 256 TMEM columns)
    static constexpr int kBN = 128;              // tokens per CTA (TMEM lanes)
    static constexpr int kNRB = kBM / RB;        // row blocks (one MMA N = RB each)
    static constexpr int kRowBytes = kBN * 2;
    static constexpr int kStages = 3;
    static constexpr int kNA = 8;                // A units in TMEM: 4 k16 steps x 8 columns = 32 columns each
    static constexpr int kTeams = 3;
    static constexpr int kThreads = 512;
};

struct TcLayout {
    size_t hdr, b_stage, v_stage, i_stage, stage, stages, total;
    int bk, ksp, iwords;
    __host__ __device__ TcLayout(int bm, int bn, int nrb, int nstages, int kbs, int n, int m) {
        bk = kbs * m;
        ksp = kbs * n;                                      // multiple of 16
        iwords = ksp / 4 + 1;
        hdr = 1024;                                         // mbarriers, TMEM base, idx bases
        b_stage = (size_t(bk) * bn * 2 + 1023) & ~size_t(1023);   // 2 x [bk][64 tokens], SWIZZLE_128B
        v_stage = align128(size_t(bm) * ksp * 2);           // [ksp/16][bm/8][2][8][8] bf16
        i_stage = align128(size_t(nrb) * iwords * 4);
        stage = (b_stage + v_stage + i_stage + 1023) & ~size_t(1023);
        stages = hdr;
        total = hdr + size_t(nstages) * stage;
    }
};

template <typename TC, int RB>
__global__ void __launch_bounds__(512, 1)
spmm_tc_kernel(const SpmmArgs a, const __grid_constant__ CUtensorMap tmB, const __grid_constant__ CUtensorMap tmV) {
    using Cfg = TcCfg<RB>;
    constexpr int BM = Cfg::kBM, BN = Cfg::kBN, NRB = Cfg::kNRB, ST = Cfg::kStages, NA = Cfg::kNA;
    constexpr int ROWB = Cfg::kRowBytes;
    constexpr int TEAMS = Cfg::kTeams;
    constexpr int CPR = BN / 8;                          // 16-byte chunks per staged B row

    extern __shared__ __align__(1024) unsigned char smem[];
    const int n = a.n, m = a.m, kbs = a.kbs;
    const TcLayout L(BM, BN, NRB, ST, kbs, n, m);
    const int ksp = L.ksp, iwords = L.iwords;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);          // [ST] producer -> everyone
    uint64_t* empty = full + ST;                                   // [ST] MMA commit -> producer
    uint64_t* aready = empty + ST;                                 // [NA] gather team -> MMA
    uint64_t* afree = aready + NA;                                 // [NA] MMA commit -> gather team
    uint64_t* dready = afree + NA;                                 // [1] MMA commit -> epilogue
    uint32_t* tmem_base_slot = reinterpret_cast<uint32_t*>(dready + 1);
    int64_t* gbase = reinterpret_cast<int64_t*>(smem + 512);      // [NRB] idx base of each row block

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int64_t n0 = int64_t(blockIdx.x) * BN;
    const int64_t m0 = int64_t(blockIdx.y) * BM;
    const int64_t kb_begin = 0, kb_end = a.KB;
    (void)CPR;
    const int nslabs = int((kb_end - kb_begin + kbs - 1) / kbs);

    auto sB = [&](int buf) { return smem + L.stages + size_t(buf) * L.stage; };
    auto sV = [&](int buf) { return smem + L.stages + size_t(buf) * L.stage + L.b_stage; };
    auto sI = [&](int buf) { return smem + L.stages + size_t(buf) * L.stage + L.b_stage + L.v_stage; };

    if (tid == 0) {
        for (int s = 0; s < ST; ++s) {
            mbar_init(&full[s], 32);          // idx cp.async arrivals (one per producer lane) + TMA bytes
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < NA; ++b) {
            mbar_init(&aready[b], 4);
            mbar_init(&afree[b], 1);
        }
        mbar_init(dready, 1);
        fence_mbar_init();
    }
    if (warp == 2) tmem_alloc(tmem_base_slot, 512);
    for (int rb = tid; rb < NRB; rb += 512) {
        const int64_t row = m0 + int64_t(rb) * RB;
        gbase[rb] = row < a.M ? (row / a.g) * a.KB * n : int64_t(-1);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_base_slot;
    const uint32_t tmem_d = tmem_base;                     // columns [0, 256): row r -> column r
    const uint32_t tmem_a = tmem_base + 256;               // A ring: buffer b -> columns [256 + 8b, +8)
    const int ksteps_full = ksp / 16;

    if (warp == 0) {
        // ======================= producer =======================
        // B slab: two TMA boxes [bk rows][64 tokens] with 128-byte swizzle (chunk c of row r at
        // c ^ (r & 7)); values: one 5-D TMA box that lands in the canonical K-major layout
        // [ksp/16][BM/8][2][8 rows][8 k]; idx words: cp.async (arrive.noinc, one per lane).
        const uint32_t tx_bytes = uint32_t(L.bk) * ROWB + uint32_t(BM * ksp * 2);
        for (int s = 0; s < nslabs; ++s) {
            const int buf = s % ST;
            if (s >= ST) mbar_wait(&empty[buf], uint32_t(((s / ST) - 1) & 1));
            const int64_t kb0 = kb_begin + int64_t(s) * kbs;
            const int nkb = int(min64(kbs, kb_end - kb0));
            const int ks = nkb * n;
            if (lane == 0) {
                mbar_expect_tx(&full[buf], tx_bytes);
                tma_load_2d(sB(buf), &tmB, &full[buf], int(n0), int(kb0 * m));
                tma_load_2d(sB(buf) + size_t(L.bk) * 128, &tmB, &full[buf], int(n0) + 64, int(kb0 * m));
                tma_load_5d(sV(buf), &tmV, &full[buf], 0, 0, 0, int(m0 / 8), int(kb0 * n / 16));
            }
            for (int e = lane; e < NRB * iwords; e += 32) {
                const int rb = e / iwords, w = e - rb * iwords;
                const int64_t gb = gbase[rb];
                const int64_t start = gb + kb0 * n;
                const int64_t woff = (start & ~int64_t(3)) + 4 * w;
                const int bytes = gb >= 0 ? int(max64(0, min64(4, min64(a.idx_bytes, start + ks) - woff))) : 0;
                cp_async4(sI(buf) + size_t(e) * 4, bytes ? a.idx + woff : a.idx, bytes);
            }
            cp_async_mbar_arrive_noinc(&full[buf]);
        }
    } else if (warp == 1) {
        // ======================= MMA issuer (one thread) =======================
        // work unit u = (slab, row block): all k16 steps of the slab for that row block; its
        // gathered A occupies TMEM columns [256 + 32 (u % NA), +8 * ksteps)
        if (lane == 0) {
            const uint32_t idesc = tc_idesc(RB);
            int u = 0;
            for (int s = 0; s < nslabs; ++s) {
                const int buf = s % ST;
                mbar_wait(&full[buf], uint32_t((s / ST) & 1));
                tc_fence_after();
                const int64_t kb0 = kb_begin + int64_t(s) * kbs;
                const int ks = int(min64(kbs, kb_end - kb0)) * n;
                const int ksteps = (ks + 15) / 16;
                const uint32_t vbase = smem_u32(sV(buf));
                for (int rb = 0; rb < NRB; ++rb, ++u) {
                    const int ab = u % NA;
                    mbar_wait(&aready[ab], uint32_t((u / NA) & 1));
                    tc_fence_after();
                    for (int kt = 0; kt < ksteps; ++kt) {
                        const uint32_t bsa = vbase + uint32_t(((kt * (BM / 8) + rb * (RB / 8)) * 2) * 128);
                        tc_mma_ts(tmem_d + uint32_t(rb * RB), tmem_a + uint32_t(ab * 32 + kt * 8), tc_sdesc(bsa, 128, 256),
                                  idesc, (s > 0 || kt > 0) ? 1u : 0u);
                    }
                    tc_commit(&afree[ab]);
                }
                (void)ksteps_full;
                tc_commit(&empty[buf]);
            }
            tc_commit(dready);
        }
    } else if (warp >= 4) {
        // ======================= gather teams =======================
        const int team = (warp - 4) / 4, q = warp % 4;           // TMEM lane quadrant q
        // ldmatrix.x4.trans roles: matrix mi = lane/8, row = lane%8; the 16 kept k of a step are
        // assigned so that the fragment lands in TMEM columns in natural k-pair order
        const int mi = lane >> 3, rr = lane & 7;
        const int slot = (rr >> 1) * 4 + (mi & 1) * 2 + (rr & 1);     // k slot 0..15 this lane addresses
        const int tok8 = (mi >> 1);                                     // +8 tokens for matrices 2, 3
        int u = 0;
        for (int s = 0; s < nslabs; ++s) {
            const int buf = s % ST;
            const int64_t kb0 = kb_begin + int64_t(s) * kbs;
            const int ks = int(min64(kbs, kb_end - kb0)) * n;
            const int ksteps = (ks + 15) / 16;
            bool waited = false;
            for (int rb = 0; rb < NRB; ++rb, ++u) {
                if (u % TEAMS != team) continue;
                if (!waited) {
                    mbar_wait(&full[buf], uint32_t((s / ST) & 1));
                    waited = true;
                }
                const int ab = u % NA;
                if (u >= NA) mbar_wait(&afree[ab], uint32_t(((u / NA) - 1) & 1));
                tc_fence_after();
                const int64_t start = gbase[rb] + kb0 * n;
                const uint8_t* ib = sI(buf) + size_t(rb) * iwords * 4 + int(start & 3);
                for (int kt = 0; kt < ksteps; ++kt) {
                    // staged row of the kept k this lane addresses (padded slots: row 0, values 0)
                    const int kk = kt * 16 + slot;
                    const int kr = kk < ks ? (kk / n) * m + ib[kk] : 0;
                    const uint32_t rowaddr = smem_u32(sB(buf)) + uint32_t(kr * 128);
                    const int swz = kr & 7;
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int tok = 32 * q + 16 * h;                   // first token of the 16
                        const int chunk = tok / 8 + tok8;                  // 16-byte token chunk 0..15
                        const uint32_t half = uint32_t(chunk >> 3) * uint32_t(L.bk) * 128u;
                        uint32_t r0, r1, r2, r3;
                        ldsm_x4_trans(rowaddr + half + uint32_t(((chunk & 7) ^ swz) * 16), r0, r1, r2, r3);
                        // 16x256b: (lane t/4, col 2(t%4)), (.., +1), (lane t/4+8, ..), (.., +1)
                        tmem_st_16x256b(tmem_a + uint32_t(ab * 32 + kt * 8) + (uint32_t(tok) << 16), r0, r1, r2, r3);
                    }
                }
                tmem_wait_st();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&aready[ab]);
            }
        }
    }

    // ======================= epilogue (warps 0..3: TMEM lane quadrants) =======================
    if (warp < 4) {
        mbar_wait(dready, 0);
        tc_fence_after();
        const int64_t col = n0 + 32 * warp + lane;                 // this thread's token
        TC* C = static_cast<TC*>(a.C);
        for (int c0 = 0; c0 < BM; c0 += 16) {
            uint32_t r[16];
            tmem_ld_32x32b_x16(tmem_d + (uint32_t(32 * warp) << 16) + uint32_t(c0), r);
            tmem_wait_ld();
            if (col < a.N) {
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    const int64_t row = m0 + c0 + j;
                    if (row < a.M) C[row * a.ldc + col] = from_f32<TC>(__uint_as_float(r[j]));
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(tmem_base, 512);
    }
}

template <int RB>
inline size_t tc_smem(int kbs, int n, int m) {
    using Cfg = TcCfg<RB>;
    return TcLayout(Cfg::kBM, Cfg::kBN, Cfg::kNRB, Cfg::kStages, kbs, n, m).total;
}

template <int RB>
inline int tc_slab_blocks(int n, int m) {
    int x = n, y = 16;
    while (y) { int t = x % y; x = y; y = t; }
    const int q = 16 / x;
    int best = q;
    for (int kbs = q; kbs * n <= 64 && kbs * m <= 512; kbs += q) {
        if (tc_smem<RB>(kbs, n, m) > 232448) break;
        best = kbs;
    }
    return best;
}

template <typename TC, int RB>
inline cudaError_t launch_tc_cfg(SpmmArgs a, cudaStream_t st) {
    using Cfg = TcCfg<RB>;
    a.kbs = tc_slab_blocks<RB>(a.n, a.m);
    a.split = 1;
    a.kb_per_split = a.KB;
    const size_t smem = tc_smem<RB>(a.kbs, a.n, a.m);
    if (smem > 232448) return cudaErrorInvalidValue;
    const TcLayout L(Cfg::kBM, Cfg::kBN, Cfg::kNRB, Cfg::kStages, a.kbs, a.n, a.m);
    CUtensorMap tmB, tmV;
    memset(&tmB, 0, sizeof(tmB));
    memset(&tmV, 0, sizeof(tmV));
    {   // B [K][ldb] bf16: box {64 tokens, bk rows}, 128-byte swizzle
        const uint64_t dims[2] = {uint64_t(a.N), uint64_t(a.K)};
        const uint64_t strides[1] = {uint64_t(a.ldb) * 2};
        const uint32_t box[2] = {64u, uint32_t(L.bk)};
        if (!make_tmap_nd(&tmB, a.B, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dims, strides, box,
                          CU_TENSOR_MAP_SWIZZLE_128B))
            return cudaErrorInvalidValue;
    }
    {   // values [M][Kp] bf16 viewed as {8 k, 8 rows, 2 halves, M/8 row groups, Kp/16 steps}
        const uint64_t dims[5] = {8, 8, 2, uint64_t((a.M + 7) / 8), uint64_t(a.Kp / 16)};
        const uint64_t strides[4] = {uint64_t(a.Kp) * 2, 16, uint64_t(a.Kp) * 16, 32};
        const uint32_t box[5] = {8, 8, 2, uint32_t(Cfg::kBM / 8), uint32_t(L.ksp / 16)};
        if (!make_tmap_nd(&tmV, a.values, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, dims, strides, box,
                          CU_TENSOR_MAP_SWIZZLE_NONE))
            return cudaErrorInvalidValue;
    }
    auto kern = spmm_tc_kernel<TC, RB>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    dim3 grid(unsigned((a.N + Cfg::kBN - 1) / Cfg::kBN), unsigned((a.M + Cfg::kBM - 1) / Cfg::kBM));
    kern<<<grid, Cfg::kThreads, smem, st>>>(a, tmB, tmV);
    return cudaGetLastError();
}

// tcgen05 tile variants (plan.tile): 1 = RB 16, 2 = RB 32, 3 = RB 64 (RB | g); no split-K.
template <typename TC>
inline sten_status launch_tc(const SpmmArgs& a, int tile, cudaStream_t st) {
    cudaError_t e;
    if (tile == 3) e = launch_tc_cfg<TC, 64>(a, st);
    else if (tile == 2) e = launch_tc_cfg<TC, 32>(a, st);
    else e = launch_tc_cfg<TC, 16>(a, st);
    return e == cudaSuccess ? STEN_OK : STEN_ERR_CUDA;
}

}  // namespace sten
