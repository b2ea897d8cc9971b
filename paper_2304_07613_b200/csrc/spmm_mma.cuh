// spmm_mma.cuh -- K4: bf16 grouped n:m SpMM on the warp-level tensor-core path
// (mma.sync.m16n8k16, fp32 accumulate), for g a multiple of 8.
//
// The grouped layout makes the product of one group a DENSE contraction over
// its gathered rows (the g rows of a group share every kept k):
//     C_G[g x T] = V_G[g x K'] . B[S_G, T],   S_G = {kb*m + idx[G][kb][t]}
// computed transposed, C_G^T = B[S_G, T]^T . V_G^T, so the 16-wide MMA M
// dimension runs over tokens and the 8-wide N dimension over the group's rows.
// The gather is free: `ldmatrix.x4.trans` takes one shared-memory row address
// PER LANE, so each lane points at the staged B row of the kept k it feeds --
// the paper's "indirect loads from specific rows of B" at the
// granularity of a tensor-core fragment.  Each gathered 16x16 A fragment feeds
// NR = RB/8 MMAs (RB rows of one group), i.e. the operand intensity is the group.
//
// Cooperative staging with a STAGES-deep ring and full/empty mbarriers: every warp
// computes, and after finishing slab s each warp waits until all warps released
// slab s-1's buffer (empty mbarrier) and then issues its share of the loads of
// slab s+STAGES-1 into it.  A slab consists of:
//   * the dense B slab [kbs*m rows][BN tokens] with 16-byte cp.async into an
//     XOR-swizzled layout (16-byte chunk c of row r goes to c ^ f(r), f(r) =
//     (r/m*n + r%m%n) & 7) so the 8 gathered rows one ldmatrix phase reads
//     mostly hit distinct bank groups (1:m is conflict-free);
//   * the values tile [BM][KSP] (row stride padded by 16 B: conflict-free
//     ldmatrix for the B fragments);
//   * the raw idx words of every sub-block's group;
// every thread hands its copies' completion to the full barrier with
// cp.async.mbarrier.arrive.noinc.  A warp turns its idx bytes into swizzled
// row descriptors (warp-private), then
// per 16 kept k: per sub-block one ldmatrix(.x4/.x2) of values, per 16 tokens one
// ldmatrix.x4.trans gather and NR MMAs.  The tile is parked in shared memory and
// stored coalesced (split-K partials are reduced over the cluster, fixed order).
#pragma once
#include "common.cuh"
#include "spmm_simt.cuh"   // SpmmArgs, store_out, cluster_reduce_store, STEN_TSTAMP

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

// RB rows per sub-block (8 or 16, RB | g), MR m16 token tiles per warp, SUB sub-blocks per
// warp, WARPS warps per CTA (all compute and all stage).
template <int RB, int MR, int SUB, int WARPS>
struct MmaCfg {
    static constexpr int kCW = WARPS;
    static constexpr int kNR = RB / 8;
    static constexpr int kBN = 16 * MR;            // tokens per CTA
    static constexpr int kSubs = kCW * SUB;
    static constexpr int kBM = kSubs * RB;
    static constexpr int kRowBytes = kBN * 2;      // staged B row
    static constexpr int kStages = 3;
};

struct MmaLayout {
    size_t hdr, b_stage, v_stage, i_stage, stage, stages, offs, total;
    int bk, ksp, iwords, vstride;
    __host__ __device__ MmaLayout(int bm, int bn, int nsub, int nstages, int kbs, int n, int m) {
        bk = kbs * m;
        ksp = kbs * n;                                   // multiple of 16
        iwords = ksp / 4 + 1;
        vstride = ksp * 2 + 16;
        hdr = align128(size_t(nstages) * 16 + size_t(nsub) * 8);
        b_stage = align128(size_t(bk) * bn * 2);
        v_stage = align128(size_t(bm) * vstride);
        i_stage = align128(size_t(nsub) * iwords * 4);
        stage = b_stage + v_stage + i_stage;
        stages = hdr;
        offs = hdr + size_t(nstages) * stage;
        const size_t pipe = offs + size_t(nsub) * ksp * 4;
        const size_t tile = hdr + size_t(bm) * bn * 4;
        total = pipe > tile ? pipe : tile;
    }
};

// swizzle of a staged B row: f(row) from its (block, slot) so that the 8 consecutive
// kept rows one ldmatrix phase gathers differ in f whenever they come from distinct slots
STEN_DEVICE_INLINE int mma_swz(int kb_local, int j, int n) { return (kb_local * n + j % n) & 7; }

template <typename TC, int RB, int MR, int SUB, int WARPS>
__global__ void __launch_bounds__(WARPS * 32, 1)
spmm_mma_kernel(const SpmmArgs a) {
    using Cfg = MmaCfg<RB, MR, SUB, WARPS>;
    constexpr int CW = Cfg::kCW;
    constexpr int NR = Cfg::kNR;
    constexpr int BN = Cfg::kBN;
    constexpr int BM = Cfg::kBM;
    constexpr int NSUB = Cfg::kSubs;
    constexpr int ST = Cfg::kStages;
    constexpr int ROWB = Cfg::kRowBytes;
    constexpr int NT = WARPS * 32;
    constexpr int CPR = BN / 8;                   // 16-byte chunks per staged B row

    extern __shared__ __align__(128) unsigned char smem[];
    const int n = a.n, m = a.m, kbs = a.kbs;
    const MmaLayout L(BM, BN, NSUB, ST, kbs, n, m);
    const int ksp = L.ksp, iwords = L.iwords, vstride = L.vstride;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);
    uint64_t* empty = full + ST;
    int64_t* gbase = reinterpret_cast<int64_t*>(smem + ST * 16);

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int64_t n0 = int64_t(blockIdx.x) * BN;
    const int64_t m0 = int64_t(blockIdx.y) * BM;
    // split-K part z = blockIdx.z owns slabs [z T / S, (z+1) T / S) of the T slabs (balanced: the
    // parts differ by at most one slab, so no CTA of the cluster idles at the reduction barrier)
    const int64_t tot_slabs = (a.KB + kbs - 1) / kbs;
    const int64_t kb_begin = (tot_slabs * int64_t(blockIdx.z) / a.split) * kbs;
    const int64_t kb_end = min64(a.KB, (tot_slabs * int64_t(blockIdx.z + 1) / a.split) * kbs);
    const int nslabs = kb_end > kb_begin ? int((kb_end - kb_begin + kbs - 1) / kbs) : 0;

    auto sB = [&](int buf) { return smem + L.stages + size_t(buf) * L.stage; };
    auto sV = [&](int buf) { return smem + L.stages + size_t(buf) * L.stage + L.b_stage; };
    auto sI = [&](int buf) { return smem + L.stages + size_t(buf) * L.stage + L.b_stage + L.v_stage; };

    if (tid == 0) {
        for (int s = 0; s < ST; ++s) {
            mbar_init(&full[s], NT);          // one cp.async-completion arrive per thread
            mbar_init(&empty[s], CW);
        }
        fence_mbar_init();
    }
    for (int sb = tid; sb < NSUB; sb += NT) {
        const int64_t row = m0 + int64_t(sb) * RB;
        gbase[sb] = row < a.M ? (row / a.g) * a.KB * n : int64_t(-1);
    }
    __syncthreads();

    const bf16_t* __restrict__ V = static_cast<const bf16_t*>(a.values);
    const bf16_t* __restrict__ Bm = static_cast<const bf16_t*>(a.B);
    // Division-free per-thread staging state.  B slab: this thread copies 16-byte chunk
    // column cc of rows kr0, kr0 + RST, ...; the (block, slot) of each row is stepped.
    constexpr int RST = NT / CPR;                          // rows per step (NT, CPR powers of two)
    const int cc = tid % CPR, kr0 = tid / CPR;
    const int dq = RST / m, dr = RST - (RST / m) * m;      // block / slot increments per step
    const int kbl0 = kr0 / m, j0 = kr0 - kbl0 * m;
    const int64_t colB = n0 + int64_t(cc) * 8;
    const int bytesB = int(max64(0, min64(8, a.N - colB))) * 2;
    // values: chunk c8 (8 values) of rows vr0, vr0 + VST, ...
    const int cpv = ksp / 8;
    const int VST = NT / cpv, vr0 = tid / cpv, c8 = tid - (tid / cpv) * cpv;
    // This thread's share of the loads of slab `s` into buffer `buf` (always ends with the
    // arrive(s) on full[buf] that account for this thread, even when it had nothing to copy).
    auto stage = [&](int s, int buf) {
        if (s < nslabs) {
            const int64_t kb0 = kb_begin + int64_t(s) * kbs;
            const int nkb = int(min64(kbs, kb_end - kb0));
            const int rows = nkb * m, ks = nkb * n;
            // dense B slab rows [kb0*m, +rows) x tokens [n0, n0+BN), swizzled 16-byte chunks
            {
                const bf16_t* src = Bm + (kb0 * m + kr0) * a.ldb + colB;
                const int64_t src_step = int64_t(RST) * a.ldb;
                unsigned char* dst = sB(buf) + size_t(kr0) * ROWB;
                int kbl = kbl0, j = j0;
                for (int kr = kr0; kr < rows; kr += RST) {
                    cp_async16(dst + ((cc ^ mma_swz(kbl, j, n)) * 16), bytesB ? src : Bm, bytesB);
                    src += src_step;
                    dst += RST * ROWB;
                    kbl += dq;
                    j += dr;
                    if (j >= m) { j -= m; ++kbl; }
                }
            }
            // values tile [BM][ksp] (row stride vstride), zero beyond ks / M
            if (a.v_async) {
                const int k0 = c8 * 8;
                const int kbytes = max(0, min(8, ks - k0)) * 2;
                const bf16_t* src = V + (m0 + vr0) * a.Kp + kb0 * n + k0;
                for (int r = vr0; r < BM; r += VST) {
                    const int bytes = (m0 + r < a.M) ? kbytes : 0;
                    cp_async16(sV(buf) + size_t(r) * vstride + k0 * 2, bytes ? src : V, bytes);
                    src += int64_t(VST) * a.Kp;
                }
            } else {
                for (int e = tid; e < BM * ksp; e += NT) {
                    const int r = e / ksp, kk = e - r * ksp;
                    const int64_t row = m0 + r;
                    *reinterpret_cast<bf16_t*>(sV(buf) + size_t(r) * vstride + kk * 2) =
                        (row < a.M && kk < ks) ? V[row * a.Kp + kb0 * n + kk] : bf16_t(0);
                }
            }
            // raw idx words of every sub-block's group
            for (int e = tid; e < NSUB * iwords; e += NT) {
                const int sb = e / iwords, w = e - sb * iwords;
                const int64_t gb = gbase[sb];
                const int64_t start = gb + kb0 * n;
                const int64_t woff = (start & ~int64_t(3)) + 4 * w;
                const int bytes = gb >= 0 ? int(max64(0, min64(4, min64(a.idx_bytes, start + ks) - woff))) : 0;
                cp_async4(sI(buf) + size_t(e) * 4, bytes ? a.idx + woff : a.idx, bytes);
            }
        }
        if (a.v_async || s >= nslabs) {
            cp_async_mbar_arrive_noinc(&full[buf]);     // the arrive fires when this thread's copies land
        } else {
            // plain stores were used for the values: a release arrive publishes them, and the
            // pending-count-neutral async arrive still waits for this thread's copies
            cp_async_mbar_arrive(&full[buf]);
            mbar_arrive(&full[buf]);
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
    const int sub0 = warp * SUB;

#pragma unroll
    for (int s = 0; s < ST - 1; ++s) stage(s, s);

    const bool warp_active = (m0 + int64_t(sub0) * RB) < a.M;
    int* wo = reinterpret_cast<int*>(smem + L.offs) + sub0 * ksp;     // [SUB][ksp] descriptors
    const int a_k = (lane & 7) + ((lane >> 4) << 3);     // kept-k row this lane addresses (A)
    const int a_half = (lane >> 3) & 1;                   // token half (0-7 / 8-15)
    const int b_row = (lane & 7) + ((lane >> 4) << 3);   // values row within 16 (B fragment)
    const int b_k8 = (lane >> 3) & 1;                     // k half (0-7 / 8-15)
    const int kbl_lo = lane / n, kbl_hi = (lane + 32) / n; // slab-local m-block of slots lane, lane+32
    for (int s = 0; s < nslabs; ++s) {
        const int buf = s % ST;
        mbar_wait(&full[buf], uint32_t((s / ST) & 1));
        if (warp_active) {
            const int64_t kb0 = kb_begin + int64_t(s) * kbs;
            const int ks = int(min64(kbs, kb_end - kb0)) * n;
#pragma unroll
            for (int q = 0; q < SUB; ++q) {
                const int64_t start = gbase[sub0 + q] + kb0 * n;
                const uint8_t* ib = sI(buf) + size_t(sub0 + q) * iwords * 4 + int(start & 3);
#pragma unroll
                for (int h = 0; h < 2; ++h) {                     // ksp <= 64: slots lane, lane + 32
                    const int kk = lane + 32 * h;
                    if (kk >= ksp) break;
                    int d = 0;                                    // padded slots: row 0 (values are 0)
                    if (kk < ks) {
                        const int kbl = h ? kbl_hi : kbl_lo, j = ib[kk];
                        d = (kbl * m + j) * ROWB | mma_swz(kbl, j, n);
                    }
                    wo[q * ksp + kk] = d;
                }
            }
            __syncwarp();
            const uint32_t bbase = smem_u32(sB(buf));
            const uint32_t vbase = smem_u32(sV(buf));
            const int ksteps = (ks + 15) / 16;
            for (int kt = 0; kt < ksteps; ++kt) {
#pragma unroll
                for (int q = 0; q < SUB; ++q) {
                    const int desc = wo[q * ksp + kt * 16 + a_k];
                    const uint32_t rowaddr = bbase + uint32_t(desc & ~7);
                    const int swz = desc & 7;
                    uint32_t bf[NR][2];
                    if constexpr (NR == 2) {
                        ldsm_x4(vbase + uint32_t(((sub0 + q) * RB + b_row) * vstride + (kt * 16 + b_k8 * 8) * 2),
                                bf[0][0], bf[0][1], bf[1][0], bf[1][1]);
                    } else {
                        ldsm_x2(vbase + uint32_t(((sub0 + q) * RB + (lane & 7)) * vstride + (kt * 16 + b_k8 * 8) * 2),
                                bf[0][0], bf[0][1]);
                    }
#pragma unroll
                    for (int i = 0; i < MR; ++i) {
                        uint32_t af[4];
                        ldsm_x4_trans(rowaddr + uint32_t(((i * 2 + a_half) ^ swz) * 16), af[0], af[1], af[2], af[3]);
#pragma unroll
                        for (int jn = 0; jn < NR; ++jn) mma_bf16_16816(acc[q][i][jn], af, bf[jn][0], bf[jn][1]);
                    }
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[buf]);
        // refill the buffer of slab s-1 with slab s+ST-1 once every warp has released it
        const int sn = s + ST - 1;
        if (sn < nslabs) {
            if (s >= 1) mbar_wait(&empty[(s - 1) % ST], uint32_t(((s - 1) / ST) & 1));
            stage(sn, sn % ST);
        }
    }
    // ---- epilogue: park the fp32 tile [BM][BN] in shared memory, then store / cluster-reduce ----
    __syncthreads();
    float* tile = reinterpret_cast<float*>(smem + L.hdr);
    {
        // D fragment: d0,d1 -> (token = lane/4, rows 2*(lane%4)+{0,1}); d2,d3 -> token + 8
        const int tq = lane >> 2, rq = (lane & 3) * 2;
#pragma unroll
        for (int q = 0; q < SUB; ++q)
#pragma unroll
            for (int jn = 0; jn < NR; ++jn)
#pragma unroll
                for (int i = 0; i < MR; ++i)
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const int row = (sub0 + q) * RB + jn * 8 + rq + (e & 1);
                        const int col = i * 16 + tq + (e >> 1) * 8;
                        tile[size_t(row) * BN + col] = acc[q][i][jn][e];
                    }
    }
    cluster_reduce_store<TC, BM, BN, NT>(smem + L.hdr, a, m0, n0);
}

// mma tile variants (plan.tile), 16 warps, 1 CTA / SM:
//   1: RB = 8  (8 | g),  MR = 8, SUB = 2 -> BM = 256, BN = 128
//   2: RB = 16 (16 | g), MR = 8, SUB = 1 -> BM = 256, BN = 128
template <int RB, int MR, int SUB, int WARPS>
inline size_t mma_smem(int kbs, int n, int m) {
    using Cfg = MmaCfg<RB, MR, SUB, WARPS>;
    return MmaLayout(Cfg::kBM, Cfg::kBN, Cfg::kSubs, Cfg::kStages, kbs, n, m).total;
}

// m-blocks per slab: a multiple of 16/gcd(n,16) (kept per slab a multiple of 16), the
// largest whose ring fits 227 KB.
template <int RB, int MR, int SUB, int WARPS>
inline int mma_slab_blocks(int n, int m) {
    int a = n, b = 16;
    while (b) { int t = a % b; a = b; b = t; }
    const int q = 16 / a;
    int best = q;
    for (int kbs = q; kbs * n <= 64 && kbs * m <= 512; kbs += q) {
        if (mma_smem<RB, MR, SUB, WARPS>(kbs, n, m) > 232448) break;
        best = kbs;
    }
    return best;
}

template <typename TC, int RB, int MR, int SUB, int WARPS>
inline cudaError_t launch_mma_cfg(SpmmArgs a, int split, cudaStream_t st) {
    using Cfg = MmaCfg<RB, MR, SUB, WARPS>;
    a.kbs = mma_slab_blocks<RB, MR, SUB, WARPS>(a.n, a.m);
    const int64_t slabs = (a.KB + a.kbs - 1) / a.kbs;
    a.split = int(slabs < split ? slabs : split);                 // balanced whole-slab parts
    a.kb_per_split = ((slabs + a.split - 1) / a.split) * a.kbs;  // largest part (informational)
    const size_t smem = mma_smem<RB, MR, SUB, WARPS>(a.kbs, a.n, a.m);
    if (smem > 232448) return cudaErrorInvalidValue;
    auto kern = spmm_mma_kernel<TC, RB, MR, SUB, WARPS>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned((a.N + Cfg::kBN - 1) / Cfg::kBN), unsigned((a.M + Cfg::kBM - 1) / Cfg::kBM),
                       unsigned(a.split));
    cfg.blockDim = dim3(WARPS * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 1;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = unsigned(a.split);
    cfg.attrs = attr;
    cfg.numAttrs = a.split > 1 ? 1 : 0;
    e = cudaLaunchKernelEx(&cfg, kern, a);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

template <typename TC>
inline sten_status launch_mma(const SpmmArgs& a, int tile, int split, cudaStream_t st) {
    cudaError_t e;
    if (tile == 2) e = launch_mma_cfg<TC, 16, 8, 1, 16>(a, split, st);
    else e = launch_mma_cfg<TC, 8, 8, 2, 16>(a, split, st);
    return e == cudaSuccess ? STEN_OK : STEN_ERR_CUDA;
}

}  // namespace sten
