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
// CTA = 768 threads: warp 0 B + idx producer (TMA of the swizzled B slab, cp.async of the idx
// words), warp 3 values producer (TMA), warp 1 MMA issuer, warp 2 TMEM allocator, warps 4..23
// five gather teams of four warps; warps 0..3 run the epilogue.  Tile: 256 rows x 128 tokens.
#pragma once
#include "common.cuh"
#include "spmm_simt.cuh"   // SpmmArgs, store_out
#include "spmm_mma.cuh"    // ldsm_x4_trans
#include "tma_host.h"

// debug experiments (timing builds only): bit 0 skips the TMEM stores, bit 1 the MMAs, bit 2 the ldmatrix
#ifndef STEN_TC_EXP
#define STEN_TC_EXP 0
#endif

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

// one lane of a converged warp (tcgen05.mma / commit are issued by a single thread; issuing from
// a converged warp through elect.sync keeps the issue path short -- a lone divergent lane costs
// ~58 cycles per MMA on this part against a 32-cycle N = 64 floor, tools/tc_microbench.cu)
STEN_DEVICE_INLINE bool elect_one() {
    uint32_t pred = 0;
    asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}\n" : "=r"(pred));
    return pred != 0;
}

// Instruction descriptor, kind::f16: D fp32, A/B bf16, both K-major, M = 128, N = n.
__host__ __device__ constexpr uint32_t tc_idesc(int n) {
    return (1u << 4)                        // c_format = F32
           | (1u << 7)                      // a_format = BF16
           | (1u << 10)                     // b_format = BF16
           | (uint32_t(n >> 3) << 17)       // n_dim
           | (uint32_t(128 >> 4) << 24);    // m_dim
}

// Shared-memory matrix descriptor, K-major SWIZZLE_128B: rows of 128 bytes (64 bf16 k), 8-row
// atoms of 1024 bytes (SBO), LBO unused (1); version 1 (sm_100), layout type 2 at bit 61.  A k16
// step inside the atom advances the start address by 32 bytes (the swizzle acts on address bits).
STEN_DEVICE_INLINE uint64_t tc_sdesc_sw128(uint32_t saddr) {
    return uint64_t((saddr >> 4) & 0x3FFFu) | (uint64_t(1) << 16) | (uint64_t(1024 >> 4) << 32) |
           (uint64_t(1) << 46) | (uint64_t(2) << 61);
}
// Same for rows of `rowb` = 128 / 64 / 32 bytes (SWIZZLE_128B / 64B / 32B: layout types 2 / 4 / 6,
// 8-row atoms of 8 rowb bytes).
STEN_DEVICE_INLINE uint64_t tc_sdesc_sw(uint32_t saddr, int rowb) {
    const uint64_t lt = rowb == 128 ? 2 : rowb == 64 ? 4 : 6;
    return uint64_t((saddr >> 4) & 0x3FFFu) | (uint64_t(1) << 16) | (uint64_t((8 * rowb) >> 4) << 32) |
           (uint64_t(1) << 46) | (lt << 61);
}
// values row bytes staged per slab: the smallest swizzle span holding ksp bf16
__host__ __device__ constexpr int tc_vrow(int ksp) { return ksp <= 16 ? 32 : ksp <= 32 ? 64 : 128; }

// Shared-memory matrix descriptor, SWIZZLE_NONE (canonical core matrices of 8 rows x 16 B):
// lbo = byte stride between core matrices along K, sbo = along M/N; version 1 (sm_100).
STEN_DEVICE_INLINE uint64_t tc_sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    return uint64_t((saddr >> 4) & 0x3FFFu) | (uint64_t((lbo >> 4) & 0x3FFFu) << 16) |
           (uint64_t((sbo >> 4) & 0x3FFFu) << 32) | (uint64_t(1) << 46);
}

// Staged-row permutation of the B slab (see launch_tc_cfg): the slab of kbs m-blocks lands in
// shared memory with row R(b, j) for block b (slab-local) and slot j, chosen so that the 8 rows
// one ldmatrix phase gathers fall in distinct 128-byte swizzle rows (R % 8) whenever possible.
//   mode 1 (n = 1): R = (b&1) + 2*(b>>2) + (kbs/2)*((b>>1)&1) + kbs*j  ->  R%8 = b0 + 2*b2 + 4*b3
//   mode 2 (n = 2): R = (j&1) + 2*(b>>1) + kbs*(b&1) + 2*kbs*(j>>1)    ->  R%8 = (j&1) + 2*((b>>1)&3)
//   mode 0:         R = b*m + j (natural)
STEN_DEVICE_INLINE int tc_staged_row(int b, int j, int mode, int kbs, int m) {
    if (mode == 1) return (b & 1) + 2 * (b >> 2) + (kbs >> 1) * ((b >> 1) & 1) + kbs * j;
    if (mode == 2) return (j & 1) + 2 * (b >> 1) + kbs * (b & 1) + 2 * kbs * (j >> 1);
    return b * m + j;
}

template <int RB>
struct TcCfg {
    static constexpr int kBM = 256;              // rows per CTA (D: 256 TMEM columns)
    static constexpr int kBN = 128;              // tokens per CTA (TMEM lanes)
    static constexpr int kNRB = kBM / RB;        // row blocks (one MMA N = RB each)
    static constexpr int kRowBytes = kBN * 2;
    static constexpr int kNA = 8;                // A units in TMEM: 4 k16 steps x 8 columns = 32 columns each
    static constexpr int kTeams = 5;
    static constexpr int kThreads = 32 * (4 + 4 * kTeams);     // 768
};

// Shared memory: header (mbarriers, TMEM base, idx bases) | B ring [STB] (B slab + idx words) |
// values ring [STV].  The two rings advance slab by slab but are released by different consumers:
// B + idx by the gather teams (after their ldmatrix), values by the MMA commits.
struct TcLayout {
    size_t hdr, b_stage, i_off, v_stage, b_ring, total;
    int bk, ksp, iwords, vrow;
    __host__ __device__ TcLayout(int bm, int bn, int nrb, int stb, int stv, int kbs, int n, int m) {
        bk = kbs * m;
        ksp = kbs * n;                                      // multiple of 16, <= 64
        iwords = ksp / 4 + 1;
        hdr = 1024;
        i_off = size_t(bk) * bn * 2;                        // 2 x [bk][64 tokens], SWIZZLE_128B
        b_stage = (i_off + size_t(nrb) * iwords * 4 + 1023) & ~size_t(1023);
        vrow = tc_vrow(ksp);
        v_stage = size_t(bm) * vrow;                        // [bm][vrow / 2 k] bf16, swizzled rows
        b_ring = hdr + size_t(stb) * b_stage;
        total = b_ring + size_t(stv) * v_stage;
    }
};

template <typename TC, int RB, int STB, int STV>
__global__ void __launch_bounds__(768, 1)
spmm_tc_kernel(const SpmmArgs a, const __grid_constant__ CUtensorMap tmB, const __grid_constant__ CUtensorMap tmV) {
    using Cfg = TcCfg<RB>;
    constexpr int BM = Cfg::kBM, BN = Cfg::kBN, NRB = Cfg::kNRB, NA = Cfg::kNA;
    constexpr int ROWB = Cfg::kRowBytes;
    constexpr int TEAMS = Cfg::kTeams;

    extern __shared__ __align__(1024) unsigned char smem[];
    const int n = a.n, m = a.m, kbs = a.kbs;
    const TcLayout L(BM, BN, NRB, STB, STV, kbs, n, m);
    const int iwords = L.iwords;
    uint64_t* bfull = reinterpret_cast<uint64_t*>(smem);          // [STB] B + idx landed
    uint64_t* bempty = bfull + STB;                                 // [STB] gathers done with the B slab
    uint64_t* vfull = bempty + STB;                                 // [STV] values landed
    uint64_t* vempty = vfull + STV;                                 // [STV] MMAs done with the values
    uint64_t* aready = vempty + STV;                                // [NA] gather team -> MMA
    uint64_t* afree = aready + NA;                                  // [NA] MMA commit -> gather team
    uint64_t* dready = afree + NA;                                  // [1] MMA commit -> epilogue
    uint32_t* tmem_base_slot = reinterpret_cast<uint32_t*>(dready + 1);
    int64_t* gbase = reinterpret_cast<int64_t*>(smem + 512);       // [NRB] idx base of each row block
    int* ioff = reinterpret_cast<int*>(smem + 512 + 8 * NRB);      // [NRB] byte offset of its idx in a stage

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    // row tiles fastest: the CTAs that share a token tile (and its B slabs) run together
    const int64_t m0 = int64_t(blockIdx.x) * BM;
    const int64_t n0 = int64_t(blockIdx.y) * BN;
    const int64_t kb_begin = 0, kb_end = a.KB;
    const int nslabs = int((kb_end - kb_begin + kbs - 1) / kbs);

    auto sB = [&](int buf) { return smem + L.hdr + size_t(buf) * L.b_stage; };
    auto sI = [&](int buf) { return smem + L.hdr + size_t(buf) * L.b_stage + L.i_off; };
    auto sV = [&](int buf) { return smem + L.b_ring + size_t(buf) * L.v_stage; };

    STEN_TSTAMP(0);
    if (tid == 0) {
        for (int s = 0; s < STB; ++s) {
            mbar_init(&bfull[s], 33);         // warp 0: lane 0 arrive.expect_tx (B) + 32 idx cp.async arrivals
            mbar_init(&bempty[s], 4 * NRB);   // every gather warp of every unit of the slab
        }
        for (int s = 0; s < STV; ++s) {
            mbar_init(&vfull[s], 1);          // warp 3 lane 0 arrive.expect_tx (values)
            mbar_init(&vempty[s], 1);         // MMA commit
        }
        for (int b = 0; b < NA; ++b) {
            mbar_init(&aready[b], 4);
            mbar_init(&afree[b], 1);
        }
        mbar_init(dready, 1);
        fence_mbar_init();
    }
    if (warp == 2) tmem_alloc(tmem_base_slot, 512);
    for (int rb = tid; rb < NRB; rb += Cfg::kThreads) {
        const int64_t row = m0 + int64_t(rb) * RB;
        gbase[rb] = row < a.M ? (row / a.g) * a.KB * n : int64_t(-1);
        ioff[rb] = rb * iwords * 4 + (row < a.M ? int(((row / a.g) * a.KB * n) & 3) : 0);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    STEN_TSTAMP(1);
    const uint32_t tmem_base = *tmem_base_slot;
    const uint32_t tmem_d = tmem_base;                     // columns [0, 256): row r -> column r
    const uint32_t tmem_a = tmem_base + 256;               // A ring: buffer b -> columns [256 + 32b, +32)

    if (warp == 0) {
        // ======================= B + idx producer (warp 0) =======================
        // B slab: two TMA boxes [bk rows][64 tokens] with 128-byte swizzle (chunk c of row r at
        // c ^ (r & 7)), rows in the staged order of tc_staged_row; idx words of the NRB row blocks:
        // cp.async (arrive.noinc, one per lane).  Per-lane idx word addressing is fixed across
        // slabs: the slab start advances by ksp (a multiple of 16), so only kb0 n changes.
        constexpr int kMaxE = (NRB * 17 + 31) / 32;              // iwords <= 64 / 4 + 1
        int64_t ebase[kMaxE];
        int ec[kMaxE];
#pragma unroll
        for (int j = 0; j < kMaxE; ++j) {
            const int e = lane + 32 * j;
            ebase[j] = -1;
            ec[j] = 0;
            if (e < NRB * iwords) {
                const int rb = e / iwords, w = e - rb * iwords;
                const int64_t gb = gbase[rb];
                if (gb >= 0) {
                    ebase[j] = (gb & ~int64_t(3)) + 4 * w;
                    ec[j] = int(gb & 3) - 4 * w;
                }
            }
        }
        const uint32_t tx_bytes = uint32_t(L.bk) * ROWB;
        for (int s = 0; s < nslabs; ++s) {
            const int buf = s % STB;
            STEN_CLK(tw0);
            if (s >= STB) mbar_wait(&bempty[buf], uint32_t(((s / STB) - 1) & 1));
            STEN_WACC(0, tw0);
            STEN_TL(s, 0);
            const int64_t kb0 = kb_begin + int64_t(s) * kbs;
            const int ks = int(min64(kbs, kb_end - kb0)) * n;
            if (lane == 0) {
                mbar_arrive_expect_tx(&bfull[buf], tx_bytes);
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    unsigned char* dst = sB(buf) + size_t(h) * L.bk * 128;
                    const int x = int(n0) + 64 * h;
                    if (a.bperm == 1) tma_load_5d(dst, &tmB, &bfull[buf], x, 0, int(kb0 / 4), 0, 0);
                    else if (a.bperm == 2) tma_load_5d(dst, &tmB, &bfull[buf], x, 0, int(kb0 / 2), 0, 0);
                    else tma_load_2d(dst, &tmB, &bfull[buf], x, int(kb0 * m));
                }
                STEN_TL(s, 6);
            }
            uint32_t* dsti = reinterpret_cast<uint32_t*>(sI(buf));
#pragma unroll
            for (int j = 0; j < kMaxE; ++j) {
                const int e = lane + 32 * j;
                if (e < NRB * iwords) {
                    const int64_t woff = ebase[j] + kb0 * n;
                    const int bytes =
                        ebase[j] >= 0 ? int(max64(0, min64(4, min64(a.idx_bytes - woff, int64_t(ec[j] + ks))))) : 0;
                    cp_async4(dsti + e, bytes ? a.idx + woff : a.idx, bytes);
                }
            }
            STEN_TL(s, 7);
            cp_async_mbar_arrive_noinc(&bfull[buf]);
            STEN_TL(s, 1);
            if (s == STB - 1) STEN_TSTAMP(2);
        }
    } else if (warp == 3) {
        // ======================= values producer (warp 3, lane 0) =======================
        // one TMA box [BM rows][vrow / 2 k] per slab = the K-major swizzled MMA B operand
        if (lane == 0) {
            const uint32_t vbytes = uint32_t(BM * L.vrow);
            for (int s = 0; s < nslabs; ++s) {
                const int buf = s % STV;
                if (s >= STV) mbar_wait(&vempty[buf], uint32_t(((s / STV) - 1) & 1));
                const int64_t kb0 = kb_begin + int64_t(s) * kbs;
                mbar_arrive_expect_tx(&vfull[buf], vbytes);
                tma_load_2d(sV(buf), &tmV, &vfull[buf], int(kb0 * n), int(m0));
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        // ======================= MMA issuer (warp 1, one elected lane issues) =======================
        // work unit u = (slab, row block): all k16 steps of the slab for that row block; its
        // gathered A occupies TMEM columns [256 + 32 (u % NA), +8 * ksteps).  The B descriptor of
        // (rb, kt) is the slab's base descriptor + (rb RB vrow + kt 32) / 16 in the address field.
        const uint32_t idesc = tc_idesc(RB);
        int u = 0;
        STEN_CLK(tm0);
        for (int s = 0; s < nslabs; ++s) {
            const int buf = s % STV;
            STEN_CLK(tw1);
            mbar_wait(&vfull[buf], uint32_t((s / STV) & 1));
            STEN_WACC(1, tw1);
            STEN_TL(s, 2);
            tc_fence_after();
            const int64_t kb0 = kb_begin + int64_t(s) * kbs;
            const int ks = int(min64(kbs, kb_end - kb0)) * n;
            const int ksteps = (ks + 15) / 16;
            const uint64_t vdesc = tc_sdesc_sw(smem_u32(sV(buf)), L.vrow);
            for (int rb = 0; rb < NRB; ++rb, ++u) {
                const int ab = u % NA;
                STEN_CLK(tw2);
                mbar_wait(&aready[ab], uint32_t((u / NA) & 1));
                STEN_WACC(2, tw2);
                tc_fence_after();
                if (elect_one()) {
                    const uint32_t dcol = tmem_d + uint32_t(rb * RB);
                    const uint32_t acol = tmem_a + uint32_t(ab * 32);
                    const uint64_t bdesc = vdesc + uint64_t((rb * RB * L.vrow) >> 4);
#pragma unroll
                    for (int kt = 0; kt < 4; ++kt)
                        if (kt < ksteps && !(STEN_TC_EXP & 2))
                            tc_mma_ts(dcol, acol + uint32_t(kt * 8), bdesc + uint64_t(kt * 2), idesc,
                                      (s > 0 || kt > 0) ? 1u : 0u);
                    tc_commit(&afree[ab]);
                }
                __syncwarp();
            }
            if (elect_one()) tc_commit(&vempty[buf]);
            __syncwarp();
            STEN_TL(s, 3);
        }
        STEN_WACC(6, tm0);
        if (elect_one()) tc_commit(dready);
        __syncwarp();
    } else if (warp >= 4) {
        // ======================= gather teams =======================
        const int team = (warp - 4) / 4, q = warp % 4;           // TMEM lane quadrant q
        // ldmatrix.x4.trans roles: matrix mi = lane/8, row = lane%8; the 16 kept k of a step are
        // assigned so that the fragment lands in TMEM columns in natural k-pair order
        const int mi = lane >> 3, rr = lane & 7;
        const int slot = (rr >> 1) * 4 + (mi & 1) * 2 + (rr & 1);     // k slot 0..15 this lane addresses
        const int tok8 = (mi >> 1);                                     // +8 tokens for matrices 2, 3
        const int cbase = 4 * (q & 1) + tok8;
        // staged row of slot kk (block b = kk / n, position j = idx byte) per tc_staged_row, split
        // into a per-lane part fixed across units and a part linear in j's two lowest pieces:
        //   R = rbase[kt] + (j & 1) c1 + (j >> 1) c2
        int rbase[4];
#pragma unroll
        for (int kt = 0; kt < 4; ++kt) rbase[kt] = tc_staged_row((kt * 16 + slot) / n, 0, a.bperm, kbs, m);
        const int c1 = a.bperm == 1 ? kbs : 1;
        const int c2 = a.bperm == 0 ? 2 : 2 * kbs;
        int u = 0;
        STEN_CLK(tg0);
        for (int s = 0; s < nslabs; ++s) {
            const int buf = s % STB;
            const int64_t kb0 = kb_begin + int64_t(s) * kbs;
            const int ks = int(min64(kbs, kb_end - kb0)) * n;
            const int ksteps = (ks + 15) / 16;
            bool waited = false;
            for (int rb = 0; rb < NRB; ++rb, ++u) {
                if (u % TEAMS != team) continue;
                STEN_CLK(tw3);
                if (!waited) {
                    mbar_wait(&bfull[buf], uint32_t((s / STB) & 1));
                    waited = true;
                    if (warp == 4) STEN_TL(s, 4);
                }
                STEN_WACC(3, tw3);
                STEN_CLK(tw5);
                if (warp == 4) STEN_TL2(u, 0);
                const uint8_t* ib = sI(buf) + ioff[rb];
                // staged rows of the kept k this lane addresses in each k16 step (padded slots:
                // row 0, their values are 0); 16-byte token chunk of (q, h, tok8) = 4 q + 2 h + tok8:
                // B half q / 2, swizzled chunk ((4 (q & 1) + 2 h + tok8) ^ (row & 7)) of the row
                const uint32_t sBbase = smem_u32(sB(buf)) + uint32_t(q >> 1) * uint32_t(L.bk) * 128u;
                uint32_t rowaddr[4];
                int rsw[4];
#pragma unroll
                for (int kt = 0; kt < 4; ++kt) {
                    const int kk = kt * 16 + slot;
                    int kr = 0;
                    if (kk < ks) {
                        const int j = ib[kk];
                        kr = rbase[kt] + (j & 1) * c1 + (j >> 1) * c2;
                    }
                    rowaddr[kt] = sBbase + uint32_t(kr * 128);
                    rsw[kt] = kr & 7;
                }
                uint32_t r[4][2][4];
#pragma unroll
                for (int kt = 0; kt < 4; ++kt)
                    if (kt < ksteps && !(STEN_TC_EXP & 4))
#pragma unroll
                        for (int h = 0; h < 2; ++h)
                            ldsm_x4_trans(rowaddr[kt] + uint32_t(((cbase + 2 * h) ^ rsw[kt]) * 16), r[kt][h][0],
                                          r[kt][h][1], r[kt][h][2], r[kt][h][3]);
                if (warp == 4) STEN_TL2(u, 1);
                const int ab = u % NA;
                STEN_CLK(tw4);
                if (u >= NA) mbar_wait(&afree[ab], uint32_t(((u / NA) - 1) & 1));
                STEN_WACC(4, tw4);
                tc_fence_after();
#pragma unroll
                for (int kt = 0; kt < 4; ++kt)
                    if (kt < ksteps && !(STEN_TC_EXP & 1))
#pragma unroll
                        for (int h = 0; h < 2; ++h)
                            // 16x256b: (lane t/4, col 2(t%4)), (.., +1), (lane t/4+8, ..), (.., +1)
                            tmem_st_16x256b(tmem_a + uint32_t(ab * 32 + kt * 8) + (uint32_t(32 * q + 16 * h) << 16),
                                            r[kt][h][0], r[kt][h][1], r[kt][h][2], r[kt][h][3]);
                // the fragments are in registers (consumed by the stores): this warp is done with
                // the B slab and the idx words of the slab
                __syncwarp();
                if (lane == 0) mbar_arrive(&bempty[buf]);
                if (warp == 4) STEN_TL2(u, 2);
                tmem_wait_st();
                if (warp == 4) STEN_TL2(u, 3);
                tc_fence_before();
                __syncwarp();
                STEN_WACC(5, tw5);
                if (warp == 4 && rb == 0) STEN_TL(s, 5);
                if (lane == 0) mbar_arrive(&aready[ab]);
            }
        }
        STEN_WACC(7, tg0);
    }

    // ======================= epilogue (warps 0..3: TMEM lane quadrants) =======================
    if (warp < 4) {
        mbar_wait(dready, 0);
        tc_fence_after();
        STEN_TSTAMP(3);
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
    STEN_TSTAMP(4);
    tc_fence_before();
    __syncthreads();
    STEN_TSTAMP(5);
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(tmem_base, 512);
    }
}

// slab geometry: kbs m-blocks per slab (kept per slab ksp = kbs n a multiple of 16 and <= 64,
// kbs a multiple of 8 for the B views) and the ring depths, largest slab first that fits with
// the deepest rings (STB, STV) in {(3, 3), (2, 3), (2, 2)}
struct TcPlan {
    int kbs, stb, stv;
    size_t smem;
};
template <int RB>
inline TcPlan tc_plan(int n, int m) {
    using Cfg = TcCfg<RB>;
    int x = n, y = 16;
    while (y) { int t = x % y; x = y; y = t; }
    const int q = (16 / x) % 8 == 0 ? 16 / x : 8;
    static const int depths[3][2] = {{3, 3}, {2, 3}, {2, 2}};
    TcPlan best{q, 2, 2, TcLayout(Cfg::kBM, Cfg::kBN, Cfg::kNRB, 2, 2, q, n, m).total};
    int kmax = q;
    for (int kbs = q; kbs * n <= 64 && kbs * m <= 512; kbs += q) kmax = kbs;
    for (int kbs = kmax; kbs >= q; kbs -= q) {
        for (auto& d : depths) {
            const size_t sm = TcLayout(Cfg::kBM, Cfg::kBN, Cfg::kNRB, d[0], d[1], kbs, n, m).total;
            if (sm <= 232448) return TcPlan{kbs, d[0], d[1], sm};
        }
    }
    return best;
}

template <typename TC, int RB, int STB, int STV>
inline cudaError_t launch_tc_kernel(const SpmmArgs& a, const CUtensorMap& tmB, const CUtensorMap& tmV, size_t smem,
                                    cudaStream_t st) {
    using Cfg = TcCfg<RB>;
    auto kern = spmm_tc_kernel<TC, RB, STB, STV>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    dim3 grid(unsigned((a.M + Cfg::kBM - 1) / Cfg::kBM), unsigned((a.N + Cfg::kBN - 1) / Cfg::kBN));
    kern<<<grid, Cfg::kThreads, smem, st>>>(a, tmB, tmV);
    return cudaGetLastError();
}

template <typename TC, int RB>
inline cudaError_t launch_tc_cfg(SpmmArgs a, cudaStream_t st) {
    using Cfg = TcCfg<RB>;
    TcPlan P = tc_plan<RB>(a.n, a.m);
#ifdef STEN_TC_KBS
    P.kbs = STEN_TC_KBS;
#endif
#ifdef STEN_TC_STB
    P.stb = STEN_TC_STB;
    P.stv = STEN_TC_STV;
#endif
    a.kbs = P.kbs;
    a.split = 1;
    a.bperm = (a.n == 1 && a.kbs >= 16) ? 1 : (a.n == 2 && a.m % 2 == 0 && a.kbs >= 8) ? 2 : 0;
#ifdef STEN_TC_NOPERM
    a.bperm = 0;
#endif
    a.kb_per_split = a.KB;
    const TcLayout L(Cfg::kBM, Cfg::kBN, Cfg::kNRB, P.stb, P.stv, a.kbs, a.n, a.m);
    if (L.total > 232448) return cudaErrorInvalidValue;
    CUtensorMap tmB, tmV;
    memset(&tmB, 0, sizeof(tmB));
    memset(&tmV, 0, sizeof(tmV));
    {   // B [K][ldb] bf16 with the staged-row permutation of tc_staged_row (128-byte swizzle):
        //   mode 1: {tokens, b0 (2, m rows), b>>2 (KB/4, 4m rows), b1 (2, 2m rows), j (m, 1 row)}
        //   mode 2: {tokens, j0 (2, 1 row), b>>1 (KB/2, 2m rows), b0 (2, m rows), j>>1 (m/2, 2 rows)}
        const uint64_t rs = uint64_t(a.ldb) * 2, M_ = uint64_t(a.m), KB_ = uint64_t(a.KB);
        const uint32_t kbs = uint32_t(a.kbs);
        bool ok;
        if (a.bperm == 1) {
            const uint64_t dims[5] = {uint64_t(a.N), 2, KB_ / 4, 2, M_};
            const uint64_t strides[4] = {M_ * rs, 4 * M_ * rs, 2 * M_ * rs, rs};
            const uint32_t box[5] = {64u, 2u, kbs / 4, 2u, uint32_t(a.m)};
            ok = make_tmap_nd(&tmB, a.B, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B);
        } else if (a.bperm == 2) {
            const uint64_t dims[5] = {uint64_t(a.N), 2, KB_ / 2, 2, M_ / 2};
            const uint64_t strides[4] = {rs, 2 * M_ * rs, M_ * rs, 2 * rs};
            const uint32_t box[5] = {64u, 2u, kbs / 2, 2u, uint32_t(a.m / 2)};
            ok = make_tmap_nd(&tmB, a.B, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B);
        } else {
            const uint64_t dims[2] = {uint64_t(a.N), uint64_t(a.K)};
            const uint64_t strides[1] = {rs};
            const uint32_t box[2] = {64u, uint32_t(L.bk)};
            ok = make_tmap_nd(&tmB, a.B, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B);
        }
        if (!ok) return cudaErrorInvalidValue;
    }
    {   // values [M][K'] bf16 (row stride Kp): box [BM rows][vrow / 2 k] with the matching swizzle =
        // the K-major SWIZZLE_{128,64,32}B operand layout; k >= K' (ragged last slab) is zero-filled
        const uint64_t dims[2] = {uint64_t(a.KB) * uint64_t(a.n), uint64_t(a.M)};
        const uint64_t strides[1] = {uint64_t(a.Kp) * 2};
        const uint32_t box[2] = {uint32_t(L.vrow / 2), uint32_t(Cfg::kBM)};
        const CUtensorMapSwizzle sw = L.vrow == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                      : L.vrow == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B;
        if (!make_tmap_nd(&tmV, a.values, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dims, strides, box, sw))
            return cudaErrorInvalidValue;
    }
    if (P.stb == 3 && P.stv == 3) return launch_tc_kernel<TC, RB, 3, 3>(a, tmB, tmV, L.total, st);
    if (P.stb == 2 && P.stv == 3) return launch_tc_kernel<TC, RB, 2, 3>(a, tmB, tmV, L.total, st);
    if (P.stb == 2 && P.stv == 2) return launch_tc_kernel<TC, RB, 2, 2>(a, tmB, tmV, L.total, st);
    return cudaErrorInvalidValue;
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
