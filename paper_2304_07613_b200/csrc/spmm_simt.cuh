// spmm_simt.cuh -- K3: grouped n:m x dense SpMM on the CUDA cores (fp32 accumulate).
//
// Computes C = densify(values, idx) x B  (the sparse-dense GEMM of STen,
// PAPER.md:527-538, Fig. 5), redesigned for sm_100a:
//   (1) "load sparse values, broadcast into vector registers" -> the values
//       tile of a K-slab is staged in shared memory ([row][k'], cp.async) and a
//       warp reads 4 consecutive k' of one row with one broadcast LDS.128, so
//       the RG rows of a sub-block cost RG wavefronts per 4 kept k;
//   (2) "indirect loads from specific rows of B" -> indirect LDS.128 reads of
//       a B K-slab staged in shared memory by a STAGES-deep cp.async ring; the
//       byte offset of every kept k of the warp's sub-blocks is rebuilt
//       warp-privately once per slab, so the inner loop is LDS + FFMA only;
//   (3) "FMA" -> FFMA into an RG x TN register tile per lane and sub-block
//       (RG rows of one group share every kept k, so each B element read from
//       shared memory feeds RG FMAs).
//
// CTA = WARPS warps; warp w owns SUB sub-blocks of RG rows (RG | g) and all
// BN = 32*TN columns of the tile.  Lane l owns columns {j*32*EV + l*EV + e},
// EV = 16/sizeof(T): every vector access of a warp covers 512 contiguous bytes.
// BM = WARPS*SUB*RG rows per CTA sets the reuse of every staged B element
// (BM*n/m rows use it): L2->SM traffic is sizeof(T)/(BM*n/m) bytes per FMA.
//
// Split-K (plan.split_k = S > 1): the S CTAs of one output tile form a thread-
// block cluster (1,1,S); CTA z computes the partial sum of the z-th contiguous
// range of m-blocks, parks it in its shared memory, and after a cluster
// barrier every CTA reduces 1/S of the tile by reading the S partials over
// DSMEM in the fixed order z = 0..S-1.  No workspace, no second launch, and
// the per-column summation order depends only on (K, n, m, plan) -- never on N.
#pragma once
#include <cuda.h>
#include <type_traits>
#include "common.cuh"

namespace sten {

// Optional per-CTA phase timestamps (debug builds with -DSTEN_TIMING only; tools/phase_timing.py).
#ifdef STEN_TIMING
__device__ unsigned long long g_sten_timing[16384][8];
#define STEN_TSTAMP(i)                                                                                    \
    do {                                                                                                  \
        if (threadIdx.x == 0) {                                                                           \
            unsigned long long t_;                                                                        \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                     \
            const unsigned cta_ = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);          \
            if (cta_ < 16384) g_sten_timing[cta_][i] = t_;                                               \
            if (cta_ < 16384 && (i) == 0) {                                                               \
                unsigned sm_;                                                                             \
                asm volatile("mov.u32 %0, %%smid;" : "=r"(sm_));                                          \
                g_sten_timing[cta_][7] = sm_ + 1;                                                         \
            }                                                                                             \
        }                                                                                                 \
    } while (0)
// per-CTA accumulated cycles of named waits / phases (lane 0 of the warps that time them)
__device__ unsigned long long g_sten_wait[16384][8];
// per-slab event timeline of CTA 0 (slab < 256, event < 8): clock64 at the event
__device__ long long g_sten_tl[256][8];
#define STEN_TL(slab, ev)                                                                                 \
    do {                                                                                                  \
        if (blockIdx.x == 0 && blockIdx.y == 0 && (threadIdx.x & 31) == 0 && (slab) < 256)                \
            g_sten_tl[(slab)][(ev)] = clock64();                                                          \
    } while (0)
__device__ long long g_sten_tl2[256][8];
#define STEN_TL2(u, ev)                                                                                   \
    do {                                                                                                  \
        if (blockIdx.x == 0 && blockIdx.y == 0 && (threadIdx.x & 31) == 0 && (u) < 256)                   \
            g_sten_tl2[(u)][(ev)] = clock64();                                                            \
    } while (0)
#define STEN_CLK(v) const long long v = clock64()
#define STEN_WACC(i, t0_)                                                                                 \
    do {                                                                                                  \
        if ((threadIdx.x & 31) == 0) {                                                                    \
            const unsigned cta_ = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);          \
            if (cta_ < 16384) atomicAdd(&g_sten_wait[cta_][i], (unsigned long long)(clock64() - (t0_)));  \
        }                                                                                                 \
    } while (0)
#else
#define STEN_TSTAMP(i) do { } while (0)
#define STEN_CLK(v) do { } while (0)
#define STEN_TL(slab, ev) do { } while (0)
#define STEN_TL2(u, ev) do { } while (0)
#define STEN_WACC(i, t0_) do { } while (0)
#endif

constexpr int kMaxPeers = 8;    // NVLink domain of one 8-GPU box

// Arguments common to the SpMM kernels.
struct SpmmArgs {
    const void* values;
    const uint8_t* idx;
    const void* B;
    void* C;
    int64_t M, K, N, ldb, ldc;
    int n, m, g;
    int64_t Kp;            // kept per row
    int64_t KB;            // m-blocks per row
    int64_t kb_per_split;  // m-blocks per split-K part (multiple of the slab)
    int split;             // S (cluster z extent)
    int kbs;               // m-blocks per K-slab
    bool c_vec;            // C base/ldc allow vector stores
    bool v_tma;            // values tile staged by a 3-D TMA box into [ksp/KU][BM][KU]
    bool v_async;          // else: values rows vector-aligned -> 16B (fp32) / 8B (bf16) cp.async
    int64_t idx_bytes;     // size of the idx array (bounds the aligned-down idx word loads)
    int bperm;             // tcgen05 path: staged-row permutation of the B slab (tc_staged_row)
    // fused all-gather epilogue (sten_spmm_grouped_nm_allgather): npeer > 0 -> the tile is stored to
    // every C_peer[p] (peer-mapped [M][ldc] buffers, already offset to this rank's first column)
    int npeer;
    void* C_peer[kMaxPeers];
    // fused epilogue (sten_spmm_grouped_nm_bias_act): C = act(C + bias[row]) before the store
    const float* bias;     // [M] or NULL
    int act;               // 0 none, 1 GELU (erf form), 2 ReLU
    const void* residual;  // [M][ldr] of the C dtype, added after the activation (NEXT-3: x + Linear(x)), or NULL
    int64_t ldr;
    // split-K through global memory (grouped launch, sten_spmm_grouped_nm_batched_ex): when ws != NULL
    // the S parts of a tile park their partials in ws [tile][S][BM][BN] (fp32) and the last part to
    // arrive (counter per tile, left at zero) reduces them in the fixed order z = 0..S-1 -- the same
    // order as the cluster reduction, so both give the same bits
    float* ws;
    unsigned* ctr;
};

// the fused epilogue on the fp32 accumulators of one output row (NEXT-3: "bias + GELU ...
// epilogue fusion into the SpMM"); GELU(x) = x/2 (1 + erf(x / sqrt 2))
STEN_DEVICE_INLINE void epilogue(const SpmmArgs& a, int64_t row, float* v, int cnt) {
    if (!a.bias && a.act == 0) return;
    const float b = a.bias ? a.bias[row] : 0.0f;
    for (int e = 0; e < cnt; ++e) {
        float x = v[e] + b;
        if (a.act == 1) x = 0.5f * x * (1.0f + erff(x * 0.70710678118654752f));
        else if (a.act == 2) x = fmaxf(x, 0.0f);
        v[e] = x;
    }
}

// residual add of the fused epilogue: v[e] += R[row][col + e] (R in the C dtype)
template <typename TC>
STEN_DEVICE_INLINE void add_residual(const SpmmArgs& a, int64_t row, int64_t col, float* v, int cnt) {
    if (!a.residual) return;
    const TC* R = static_cast<const TC*>(a.residual) + row * a.ldr;
    for (int e = 0; e < cnt; ++e)
        if (col + e < a.N) v[e] = __fadd_rn(v[e], to_f32(R[col + e]));
}

// destination p of the epilogue: C itself, or peer buffer p of the fused all-gather
template <typename TC>
STEN_DEVICE_INLINE TC* out_ptr(const SpmmArgs& a, int p) {
    return static_cast<TC*>(a.npeer ? a.C_peer[p] : a.C);
}

// WARPS = warps per CTA: WARPS-1 consumer warps + 1 producer warp.
template <typename TAB, int RG, int TN, int SUB, int WARPS>
struct SimtCfg {
    static constexpr int kWarps = WARPS - 1;                 // consumer warps
    static constexpr int kThreads = WARPS * 32;
    static constexpr int kEV = 16 / int(sizeof(TAB));      // elements per 16-byte vector
    static constexpr int kChunks = TN / kEV;                 // 16-byte chunks per lane and B row
    static constexpr int kBN = 32 * TN;                      // CTA columns
    static constexpr int kSubs = (WARPS - 1) * SUB;          // RG-row sub-blocks per CTA
    static constexpr int kBM = kSubs * RG;                   // CTA rows
    static constexpr int kStages = 3;
    static constexpr int kKU = RG <= 4 ? 4 : 2;             // kept k per inner-loop step
    static_assert(TN % kEV == 0, "TN must be a multiple of the vector width");
};

__host__ __device__ inline int gcd_int(int a, int b) {
    while (b) { int t = a % b; a = b; b = t; }
    return a;
}

// m-blocks per K-slab: a multiple of 4/gcd(n,4) (so kept-per-slab is a multiple
// of 4) with at most `target_rows` B rows (at least one such multiple).
__host__ __device__ inline int simt_kbs(int n, int m, int target_rows) {
    const int q = 4 / gcd_int(n, 4);
    int kbs = q;
    while ((kbs + q) * m <= target_rows) kbs += q;
    return kbs;
}

template <typename TAB>
__host__ __device__ constexpr int simt_target_rows() { return sizeof(TAB) == 4 ? 32 : 64; }

__host__ __device__ constexpr size_t align128(size_t x) { return (x + 127) & ~size_t(127); }

// Shared-memory layout (byte offsets from the dynamic smem base):
//   [0, hdr)            mbarriers full[ST] | per-sub idx base (int64) | block-row table [ksp]
//   stage s             B slab [bk][BN] | values [BM][ksp] | idx words [NSUB][iwords]
//   offs                warp-private row addresses [NSUB][ksp]
//   zero                one zero B row (target of padded kept slots)
//   split-K partial tile [BM][BN] fp32 parked at `hdr` after the main loop
struct SimtLayout {
    size_t hdr, b_stage, v_stage, i_stage, stage, stages, offs, zero, total;
    int bk, ksp, iwords;
    __host__ __device__ SimtLayout(int bm, int bn, int nsub, int esz, int nstages, int kbs, int n, int m) {
        bk = kbs * m;
        ksp = kbs * n;                                                   // multiple of 4
        iwords = ksp / 4 + 1;                                            // covers a 3-byte misalignment
        hdr = align128(size_t(nstages) * 16 + size_t(nsub) * 8);         // full/empty mbarriers, idx bases
        b_stage = align128(size_t(bk) * bn * esz);
        v_stage = align128(size_t(bm) * ksp * esz);
        i_stage = align128(size_t(nsub) * iwords * 4);
        stage = b_stage + v_stage + i_stage;
        stages = hdr;
        offs = hdr + size_t(nstages) * stage;                            // warp-private row addresses
        zero = align128(offs + size_t(nsub) * ksp * 4);
        const size_t pipe = zero + size_t(bn) * esz;
        const size_t tile = hdr + size_t(bm) * bn * 4;
        total = pipe > tile ? pipe : tile;
    }
};

template <typename TAB, int RG, int TN, int SUB, int WARPS>
struct SimtSmem : SimtLayout {
    using Cfg = SimtCfg<TAB, RG, TN, SUB, WARPS>;
    __host__ __device__ SimtSmem(int kbs, int n, int m)
        : SimtLayout(Cfg::kBM, Cfg::kBN, Cfg::kSubs, int(sizeof(TAB)), Cfg::kStages, kbs, n, m) {}
};

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

// ---- thread-block cluster helpers (split-K reduction over DSMEM) ------------------------------
STEN_DEVICE_INLINE void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
STEN_DEVICE_INLINE uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
    return r;
}
STEN_DEVICE_INLINE uint32_t map_cluster(uint32_t smem_addr, uint32_t rank) {
    uint32_t d;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(d) : "r"(smem_addr), "r"(rank));
    return d;
}
STEN_DEVICE_INLINE float4 ld_dsmem128(uint32_t addr) {
    float4 v;
    asm volatile("ld.shared::cluster.v4.f32 {%0,%1,%2,%3}, [%4];\n"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "r"(addr));
    return v;
}

// After every CTA of the cluster parked its fp32 partial tile [BM][BN] at the
// start of its shared memory: reduce 1/S of the tile over DSMEM in the fixed
// order z = 0..S-1 and store it to C.
template <typename TC, int BM, int BN, int NT>
STEN_DEVICE_INLINE void cluster_reduce_store(unsigned char* tile_smem, const SpmmArgs& a, int64_t m0, int64_t n0) {
    cluster_sync_all();
    const uint32_t S = uint32_t(a.split);
    const uint32_t me = cluster_ctarank();
    constexpr int E4 = BM * BN / 4;
    const int e_begin = int(uint64_t(E4) * me / S), e_end = int(uint64_t(E4) * (me + 1) / S);
    const uint32_t base = smem_u32(tile_smem);
    const int np = a.npeer ? a.npeer : 1;
    for (int e = e_begin + int(threadIdx.x); e < e_end; e += NT) {
        const uint32_t off = uint32_t(e) * 16u;
        float4 s = ld_dsmem128(map_cluster(base + off, 0));
        for (uint32_t z = 1; z < S; ++z) {
            const float4 t = ld_dsmem128(map_cluster(base + off, z));
            s.x = __fadd_rn(s.x, t.x); s.y = __fadd_rn(s.y, t.y);
            s.z = __fadd_rn(s.z, t.z); s.w = __fadd_rn(s.w, t.w);
        }
        const int row = (e * 4) / BN, col = (e * 4) % BN;
        const int64_t gr = m0 + row, gc = n0 + col;
        if (gr < a.M && gc < a.N) {
            float v[4] = {s.x, s.y, s.z, s.w};
            epilogue(a, gr, v, 4);
            add_residual<TC>(a, gr, gc, v, 4);
            for (int p = 0; p < np; ++p) store_out<TC>(out_ptr<TC>(a, p), a.ldc, gr, gc, a.N, v, 4, a.c_vec);
        }
    }
    cluster_sync_all();                     // keep every partial alive until all reads are done
}

// Warp-specialised pipeline: warps 0..WARPS-2 consume (LDS + FFMA2), warp WARPS-1 produces.
// Per stage the producer (1) waits until every consumer warp released the buffer
// (empty mbarrier), (2) arms the full mbarrier with the TMA byte count and issues the
// TMA loads of the B slab (and of the values tile when it is TMA-able), (3) issues
// cp.async for the raw idx words (and the values otherwise), and (4) hands their
// completion to the full mbarrier (cp.async.mbarrier.arrive.noinc, one per lane).
// A consumer waits on the full barrier, turns its sub-blocks' idx bytes into shared
// addresses of staged B rows (warp-private), runs the LDS/FFMA2 loop and arrives on
// the empty barrier.  No CTA-wide barrier per slab.
template <typename TAB, typename TC, int RG, int TN, int SUB, int WARPS, int MINB>
__device__ __forceinline__ void spmm_simt_body(const SpmmArgs& a, const CUtensorMap* tmB, const CUtensorMap* tmV,
                                               const int bx, const int by, const int bz) {
    using Cfg = SimtCfg<TAB, RG, TN, SUB, WARPS>;
    constexpr int EV = Cfg::kEV;
    constexpr int BN = Cfg::kBN;
    constexpr int BM = Cfg::kBM;
    constexpr int NSUB = Cfg::kSubs;
    constexpr int NT = WARPS * 32;
    constexpr int CW = WARPS - 1;                            // consumer warps
    constexpr int ST = Cfg::kStages;
    constexpr int ROWB = BN * int(sizeof(TAB));              // bytes per staged B row
    constexpr int KU = Cfg::kKU;                             // kept k per inner step

    extern __shared__ __align__(128) unsigned char smem[];
    const int n = a.n, m = a.m, kbs = a.kbs;
    const SimtSmem<TAB, RG, TN, SUB, WARPS> L(kbs, n, m);
    const int ksp = L.ksp, iwords = L.iwords;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);
    uint64_t* empty = full + ST;
    int64_t* gbase = reinterpret_cast<int64_t*>(smem + ST * 16);         // idx row base of each sub-block

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int64_t n0 = int64_t(bx) * BN;
    const int64_t m0 = int64_t(by) * BM;
    // split-K part z = blockIdx.z owns slabs [z T / S, (z+1) T / S) of the T slabs (balanced: the
    // parts differ by at most one slab, so no CTA of the cluster idles at the reduction barrier)
    const int64_t tot_slabs = (a.KB + kbs - 1) / kbs;
    const int64_t kb_begin = (tot_slabs * int64_t(bz) / a.split) * kbs;
    const int64_t kb_end = min64(a.KB, (tot_slabs * int64_t(bz + 1) / a.split) * kbs);
    const int nslabs = kb_end > kb_begin ? int((kb_end - kb_begin + kbs - 1) / kbs) : 0;

    auto sB = [&](int buf) { return smem + L.stages + size_t(buf) * L.stage; };
    auto sV = [&](int buf) { return smem + L.stages + size_t(buf) * L.stage + L.b_stage; };
    auto sI = [&](int buf) { return smem + L.stages + size_t(buf) * L.stage + L.b_stage + L.v_stage; };

    STEN_TSTAMP(0);
    if (tid == 0) {
        for (int s = 0; s < ST; ++s) {
            mbar_init(&full[s], 32);          // one cp.async-completion arrive per producer lane
            mbar_init(&empty[s], CW);
        }
        fence_mbar_init();
    }
    for (int sb = tid; sb < NSUB; sb += NT) {
        const int64_t row = m0 + int64_t(sb) * RG;
        gbase[sb] = row < a.M ? (row / a.g) * a.KB * n : int64_t(-1);
    }
    for (int e = tid; e < BN * int(sizeof(TAB)) / 4; e += NT) reinterpret_cast<uint32_t*>(smem + L.zero)[e] = 0u;
    __syncthreads();
    STEN_TSTAMP(1);

    float acc[SUB][RG][TN];
#pragma unroll
    for (int q = 0; q < SUB; ++q)
#pragma unroll
        for (int r = 0; r < RG; ++r)
#pragma unroll
            for (int c = 0; c < TN; ++c) acc[q][r][c] = 0.0f;
    const int sub0 = warp * SUB;

    if (warp == CW) {
        // ======================= producer warp =======================
        // programmatic dependent launch: the prologue above overlapped the tail of the kernel
        // that produced values / idx (the sparsifier); wait for it before the first read
        asm volatile("griddepcontrol.wait;\n" ::: "memory");
        const TAB* __restrict__ V = static_cast<const TAB*>(a.values);
        const uint32_t v_bytes = a.v_tma ? uint32_t(BM * ksp * sizeof(TAB)) : 0u;
        const uint32_t tx_bytes = uint32_t(L.bk) * ROWB + v_bytes;
        for (int s = 0; s < nslabs; ++s) {
            const int buf = s % ST;
            if (s >= ST) mbar_wait(&empty[buf], uint32_t(((s / ST) - 1) & 1));
            const int64_t kb0 = kb_begin + int64_t(s) * kbs;
            const int nkb = int(min64(kbs, kb_end - kb0));
            const int ks = nkb * n;
            if (lane == 0) {
                fence_proxy_async_smem();
                mbar_expect_tx(&full[buf], tx_bytes);
                tma_load_2d(sB(buf), tmB, &full[buf], int(n0), int(kb0 * m));
                if (a.v_tma) tma_load_3d(sV(buf), tmV, &full[buf], 0, int(m0), int(kb0 * n / KU));
            }
            if (!a.v_tma) {
                // values tile in k-group-major layout [ksp/KU][BM][KU] (zero beyond ks and beyond M)
                if (a.v_async) {
                    const int ngr = ksp / KU;
                    for (int e = lane; e < BM * ngr; e += 32) {
                        const int r = e / ngr, kg = e - r * ngr;
                        const int64_t row = m0 + r;
                        const int k0 = kg * KU;
                        const int bytes = (row < a.M) ? max(0, min(KU, ks - k0)) * int(sizeof(TAB)) : 0;
                        unsigned char* dst = sV(buf) + (size_t(kg) * BM + r) * KU * sizeof(TAB);
                        const TAB* src = bytes > 0 ? V + row * a.Kp + kb0 * n + k0 : V;
                        if constexpr (KU * sizeof(TAB) == 16) cp_async16(dst, src, bytes);
                        else if constexpr (KU * sizeof(TAB) == 8) cp_async8(dst, src, bytes);
                        else cp_async4(dst, src, bytes);
                    }
                } else if constexpr (sizeof(TAB) == 4) {
                    for (int e = lane; e < BM * ksp; e += 32) {
                        const int r = e / ksp, kk = e - r * ksp;
                        const int64_t row = m0 + r;
                        const int bytes = (row < a.M && kk < ks) ? 4 : 0;
                        cp_async4(sV(buf) + ((size_t(kk / KU) * BM + r) * KU + kk % KU) * 4,
                                  bytes ? V + row * a.Kp + kb0 * n + kk : V, bytes);
                    }
                } else {
                    for (int e = lane; e < BM * ksp; e += 32) {
                        const int r = e / ksp, kk = e - r * ksp;
                        const int64_t row = m0 + r;
                        reinterpret_cast<TAB*>(sV(buf))[(size_t(kk / KU) * BM + r) * KU + kk % KU] =
                            (row < a.M && kk < ks) ? V[row * a.Kp + kb0 * n + kk] : TAB(0);
                    }
                }
            }
            // raw idx: the aligned 4-byte words covering [start, start + ks) of each sub-block's group
            for (int e = lane; e < NSUB * iwords; e += 32) {
                const int sb = e / iwords, w = e - sb * iwords;
                const int64_t gb = gbase[sb];
                const int64_t start = gb + kb0 * n;
                const int64_t woff = (start & ~int64_t(3)) + 4 * w;
                const int bytes = gb >= 0 ? int(max64(0, min64(4, min64(a.idx_bytes, start + ks) - woff))) : 0;
                cp_async4(sI(buf) + size_t(e) * 4, bytes ? a.idx + woff : a.idx, bytes);
            }
            cp_async_mbar_arrive_noinc(&full[buf]);
        }
        if (a.split == 1) return;
    } else {
        // ======================= consumer warps =======================
        const bool warp_active = (m0 + int64_t(sub0) * RG) < a.M;
        const uint32_t lane_off = uint32_t(lane) * 16u;
        const uint32_t inv_n = (65536u + uint32_t(n) - 1) / uint32_t(n);   // kk / n = (kk inv_n) >> 16, kk < 64
        // fast row addressing when n | KU: slot t of k-step kg lies in block kg KU/n + t/n
        const bool n_divides_ku = KU % n == 0;
        const int kstep_bytes = n_divides_ku ? (KU / n) * m * ROWB : 0;
        int tb[KU];
#pragma unroll
        for (int t = 0; t < KU; ++t) tb[t] = n_divides_ku ? (t / n) * m * ROWB : 0;
        const uint32_t zero_row = smem_u32(smem + L.zero);
        for (int s = 0; s < nslabs; ++s) {
            const int buf = s % ST;
            mbar_wait(&full[buf], uint32_t((s / ST) & 1));
            if (s == 0) STEN_TSTAMP(2);
            if (warp_active) {
                const int64_t kb0 = kb_begin + int64_t(s) * kbs;
                const int ks = int(min64(kbs, kb_end - kb0)) * n;
                const int nkg = (ks + KU - 1) / KU;
                const uint32_t bbase = smem_u32(sB(buf));
                // idx bytes of sub q in this slab begin at byte (gbase & 3) of its first word (the
                // slab start advances by ksp, a multiple of 4, so the misalignment is fixed); the KU
                // row addresses of a step are computed in registers: two broadcast word loads, a
                // funnel shift, block b = kk / n by multiply-shift (kk < 64)
                uint32_t iaddr[SUB];
                int imis[SUB];
#pragma unroll
                for (int q = 0; q < SUB; ++q) {
                    iaddr[q] = smem_u32(sI(buf)) + uint32_t((sub0 + q) * iwords * 4);
                    imis[q] = int(gbase[sub0 + q] & 3);
                }
                const unsigned char* vbase = sV(buf) + size_t(sub0) * RG * KU * sizeof(TAB);
                // The k-loop, specialised on the addressing mode.  Every staged-row address already
                // includes this lane's byte offset.  FAST (n | KU, full slab): slot t of k-step kg lies
                // in block kg KU / n + t / n, so its row address is base_t[t] + idx_byte(t) ROWB with
                // base_t advanced by one k-step per iteration -- a byte permute and a shift-add per
                // kept k.  Otherwise: block b = kk / n by multiply-shift, padded slots read a zero row.
                auto kloop = [&](auto fast_tag, auto aligned_tag) {
                    constexpr bool FAST = decltype(fast_tag)::value;
                    // ALIGNED: every sub-block's idx bytes start on a word (gbase % 4 == 0, e.g. all C2
                    // shapes), so a k-step's KU = 4 bytes are ONE word: no second load, no funnel shift
                    constexpr bool ALIGNED = decltype(aligned_tag)::value && KU == 4;
                    uint32_t base_t[KU];
#pragma unroll
                    for (int t = 0; t < KU; ++t) base_t[t] = bbase + lane_off + uint32_t(tb[t]);
                    for (int kg = 0; kg < nkg; ++kg) {
                        const unsigned char* vg = vbase + size_t(kg) * BM * KU * sizeof(TAB);
#pragma unroll
                        for (int q = 0; q < SUB; ++q) {
                            uint32_t offs[KU];
                            {
                                uint32_t x;
                                if constexpr (ALIGNED) {
                                    x = lds32_addr(iaddr[q] + uint32_t(kg) * 4u);
                                } else {
                                    const int o = imis[q] + kg * KU;
                                    const uint32_t wa = iaddr[q] + uint32_t(o & ~3);
                                    x = __funnelshift_r(lds32_addr(wa), lds32_addr(wa + 4u), uint32_t(o & 3) * 8u);
                                }
                                if constexpr (FAST) {
#pragma unroll
                                    for (int t = 0; t < KU; ++t)
                                        offs[t] = base_t[t] + __byte_perm(x, 0u, 0x4440u + uint32_t(t)) * uint32_t(ROWB);
                                } else {
#pragma unroll
                                    for (int t = 0; t < KU; ++t) {
                                        const int kk = kg * KU + t;
                                        const int b = int((uint32_t(kk) * inv_n) >> 16);
                                        const int j = int((x >> (8 * t)) & 0xffu);
                                        offs[t] = (kk < ks ? bbase + uint32_t((b * m + j) * ROWB) : zero_row) + lane_off;
                                    }
                                }
                            }
                            float v[RG][KU];
#pragma unroll
                            for (int r = 0; r < RG; ++r) {
                                const unsigned char* vp = vg + size_t(q * RG + r) * KU * sizeof(TAB);
                                if constexpr (sizeof(TAB) == 4 && KU == 4) {
                                    const float4 t = *reinterpret_cast<const float4*>(vp);
                                    v[r][0] = t.x; v[r][1] = t.y; v[r][2] = t.z; v[r][3] = t.w;
                                } else if constexpr (sizeof(TAB) == 4) {
                                    const float2 t = *reinterpret_cast<const float2*>(vp);
                                    v[r][0] = t.x; v[r][1] = t.y;
                                } else if constexpr (KU == 4) {
                                    const uint2 t = *reinterpret_cast<const uint2*>(vp);
                                    v[r][0] = __uint_as_float(t.x << 16); v[r][1] = __uint_as_float(t.x & 0xffff0000u);
                                    v[r][2] = __uint_as_float(t.y << 16); v[r][3] = __uint_as_float(t.y & 0xffff0000u);
                                } else {
                                    const uint32_t t = *reinterpret_cast<const uint32_t*>(vp);
                                    v[r][0] = __uint_as_float(t << 16); v[r][1] = __uint_as_float(t & 0xffff0000u);
                                }
                            }
#pragma unroll
                            for (int t = 0; t < KU; ++t) {
#pragma unroll
                                for (int j = 0; j < Cfg::kChunks; ++j) {
                                    float b[EV];
                                    unpack<EV>(lds128_addr(offs[t] + uint32_t(j) * 512u), b);
                                    // b pair outer, rows inner: consecutive FFMA2 share the B operand
#pragma unroll
                                    for (int e = 0; e < EV; e += 2)
#pragma unroll
                                        for (int r = 0; r < RG; ++r) {
                                            float2& c2 = *reinterpret_cast<float2*>(&acc[q][r][j * EV + e]);
                                            c2 = __ffma2_rn(make_float2(v[r][t], v[r][t]), make_float2(b[e], b[e + 1]), c2);
                                        }
                                }
                            }
                        }
                        if constexpr (FAST) {
#pragma unroll
                            for (int t = 0; t < KU; ++t) base_t[t] += uint32_t(kstep_bytes);
                        }
                    }
                };
                bool idx_aligned = true;
#pragma unroll
                for (int q = 0; q < SUB; ++q) idx_aligned = idx_aligned && imis[q] == 0;
                if (n_divides_ku && ks % KU == 0) {
                    if (idx_aligned) kloop(std::true_type{}, std::true_type{});
                    else kloop(std::true_type{}, std::false_type{});
                } else {
                    kloop(std::false_type{}, std::false_type{});
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[buf]);
        }
        STEN_TSTAMP(3);
        if (a.split == 1) {
            if (!warp_active) return;
            if (a.bias || a.act) {
#pragma unroll
                for (int q = 0; q < SUB; ++q)
#pragma unroll
                    for (int r = 0; r < RG; ++r) {
                        const int64_t row = m0 + int64_t(sub0 + q) * RG + r;
                        if (row < a.M) epilogue(a, row, acc[q][r], TN);
                    }
            }
            const int np = a.npeer ? a.npeer : 1;
            for (int p = 0; p < np; ++p) {
                TC* C = out_ptr<TC>(a, p);
#pragma unroll
                for (int q = 0; q < SUB; ++q)
#pragma unroll
                    for (int r = 0; r < RG; ++r) {
                        const int64_t row = m0 + int64_t(sub0 + q) * RG + r;
                        if (row >= a.M) continue;
#pragma unroll
                        for (int j = 0; j < Cfg::kChunks; ++j) {
                            const int64_t col = n0 + int64_t(j) * 32 * EV + lane * EV;
                            if (p == 0) add_residual<TC>(a, row, col, &acc[q][r][j * EV], EV);
                            store_out<TC>(C, a.ldc, row, col, a.N, &acc[q][r][j * EV], EV, a.c_vec);
                        }
                    }
            }
            return;
        }
    }
    if (a.ws) {
        // split-K through global memory: this part's partial tile -> ws, then the last part reduces
        const int64_t ntx = (a.N + BN - 1) / BN;
        const int64_t tile_lin = int64_t(by) * ntx + bx;
        float* part = a.ws + (tile_lin * a.split + bz) * int64_t(BM) * BN;
        if (warp < CW) {
#pragma unroll
            for (int q = 0; q < SUB; ++q)
#pragma unroll
                for (int r = 0; r < RG; ++r) {
                    const int row = (sub0 + q) * RG + r;
#pragma unroll
                    for (int j = 0; j < Cfg::kChunks; ++j)
#pragma unroll
                        for (int e4 = 0; e4 < EV; e4 += 4) {
                            const int col = j * 32 * EV + lane * EV + e4;
                            __stcg(reinterpret_cast<float4*>(part + size_t(row) * BN + col),
                                   make_float4(acc[q][r][j * EV + e4], acc[q][r][j * EV + e4 + 1],
                                               acc[q][r][j * EV + e4 + 2], acc[q][r][j * EV + e4 + 3]));
                        }
                }
        }
        __threadfence();
        __syncthreads();
        __shared__ unsigned last_flag;
        if (tid == 0) last_flag = atomicAdd(a.ctr + tile_lin, 1u) == unsigned(a.split - 1) ? 1u : 0u;
        __syncthreads();
        STEN_TSTAMP(4);
        if (!last_flag) return;
        __threadfence();
        const float* tile0 = a.ws + tile_lin * a.split * int64_t(BM) * BN;
        constexpr int E4 = BM * BN / 4;
        const int np = a.npeer ? a.npeer : 1;
        for (int e = tid; e < E4; e += NT) {
            float4 sum = __ldcg(reinterpret_cast<const float4*>(tile0) + e);
            for (int z = 1; z < a.split; ++z) {
                const float4 t = __ldcg(reinterpret_cast<const float4*>(tile0 + size_t(z) * BM * BN) + e);
                sum.x = __fadd_rn(sum.x, t.x); sum.y = __fadd_rn(sum.y, t.y);
                sum.z = __fadd_rn(sum.z, t.z); sum.w = __fadd_rn(sum.w, t.w);
            }
            const int row = (e * 4) / BN, col = (e * 4) % BN;
            const int64_t gr = m0 + row, gc = n0 + col;
            if (gr < a.M && gc < a.N) {
                float v[4] = {sum.x, sum.y, sum.z, sum.w};
                epilogue(a, gr, v, 4);
                add_residual<TC>(a, gr, gc, v, 4);
                for (int p = 0; p < np; ++p) store_out<TC>(out_ptr<TC>(a, p), a.ldc, gr, gc, a.N, v, 4, a.c_vec);
            }
        }
        if (tid == 0) a.ctr[tile_lin] = 0u;                       // leave the counter at zero for the next call
        STEN_TSTAMP(5);
        return;
    }
    // split-K: park the partial tile [BM][BN] (fp32) after the header, reduce over the cluster
    __syncthreads();
    float* tile = reinterpret_cast<float*>(smem + L.hdr);
    if (warp < CW) {
#pragma unroll
        for (int q = 0; q < SUB; ++q)
#pragma unroll
            for (int r = 0; r < RG; ++r) {
                const int row = (sub0 + q) * RG + r;
#pragma unroll
                for (int j = 0; j < Cfg::kChunks; ++j)
#pragma unroll
                    for (int e4 = 0; e4 < EV; e4 += 4) {
                        const int col = j * 32 * EV + lane * EV + e4;
                        *reinterpret_cast<float4*>(tile + size_t(row) * BN + col) =
                            make_float4(acc[q][r][j * EV + e4], acc[q][r][j * EV + e4 + 1],
                                        acc[q][r][j * EV + e4 + 2], acc[q][r][j * EV + e4 + 3]);
                    }
            }
    }
    STEN_TSTAMP(4);
    cluster_reduce_store<TC, BM, BN, NT>(smem + L.hdr, a, m0, n0);
    STEN_TSTAMP(5);
}

// one problem per launch: grid (N tiles, M tiles, split-K parts)
template <typename TAB, typename TC, int RG, int TN, int SUB, int WARPS, int MINB>
__global__ void __launch_bounds__(WARPS * 32, MINB)
spmm_simt_kernel(const SpmmArgs a, const __grid_constant__ CUtensorMap tmB, const __grid_constant__ CUtensorMap tmV) {
    spmm_simt_body<TAB, TC, RG, TN, SUB, WARPS, MINB>(a, &tmB, &tmV, int(blockIdx.x), int(blockIdx.y),
                                                       int(blockIdx.z));
}

// Grouped launch of independent problems (the cases of a step; cuBLAS-grouped-GEMM style): CTA b
// runs tile (b - tile0[p]) of problem p, row-tile-major, whole K (no split-K, no cluster).  The
// problems share the kernel variant (dtypes, RG, tile); the list is ordered longest-K first on
// the host so the block scheduler fills the tail with short tiles.
constexpr int kMaxBatch = 12;
struct SpmmBatch {
    SpmmArgs a[kMaxBatch];
    CUtensorMap tmB[kMaxBatch];
    CUtensorMap tmV[kMaxBatch];
    int tile0[kMaxBatch + 1];    // first CTA of each problem; tile0[count] = grid size
    int ntx[kMaxBatch];          // N tiles of each problem
    int var[kMaxBatch];          // mixed launch: which of the two tile variants serves the problem
    int count;
};
// CTA b -> problem p, part z = unit % S (the S parts of a tile are adjacent CTAs), tile = unit / S

template <typename TAB, typename TC, int RG, int TN, int SUB, int WARPS, int MINB>
__global__ void __launch_bounds__(WARPS * 32, MINB)
spmm_simt_batched_kernel(const __grid_constant__ SpmmBatch bt) {
    const int b = int(blockIdx.x);
    int p = 0;
    while (p + 1 < bt.count && b >= bt.tile0[p + 1]) ++p;
    const int u = b - bt.tile0[p];
    const int S = bt.a[p].split;
    const int t = u / S;
    spmm_simt_body<TAB, TC, RG, TN, SUB, WARPS, MINB>(bt.a[p], &bt.tmB[p], &bt.tmV[p], t % bt.ntx[p],
                                                       t / bt.ntx[p], u - t * S);
}

// Mixed grouped launch: two tile variants with the same warp count in ONE launch (e.g. the 256-token
// tile for 2:4 / 1:4 and the 240-row tile, with 3x longer K-slabs, for 1:10); bt.var[p] selects the
// body of problem p.  Shared memory = the larger layout; registers = the larger variant.
template <typename TAB, typename TC, int RG, int TNA, int SUBA, int TNB, int SUBB, int WARPS>
__global__ void __launch_bounds__(WARPS * 32, 1)
spmm_simt_batched2_kernel(const __grid_constant__ SpmmBatch bt) {
    const int b = int(blockIdx.x);
    int p = 0;
    while (p + 1 < bt.count && b >= bt.tile0[p + 1]) ++p;
    const int u = b - bt.tile0[p];
    const int S = bt.a[p].split;
    const int t = u / S;
    if (bt.var[p] == 0)
        spmm_simt_body<TAB, TC, RG, TNA, SUBA, WARPS, 1>(bt.a[p], &bt.tmB[p], &bt.tmV[p], t % bt.ntx[p], t / bt.ntx[p],
                                                         u - t * S);
    else
        spmm_simt_body<TAB, TC, RG, TNB, SUBB, WARPS, 1>(bt.a[p], &bt.tmB[p], &bt.tmV[p], t % bt.ntx[p], t / bt.ntx[p],
                                                         u - t * S);
}

}  // namespace sten
