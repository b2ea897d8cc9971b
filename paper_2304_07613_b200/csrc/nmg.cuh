// nmg.cuh -- the paper's own chunked n:m:g format on sm_100a:
// conversion (greedy), densify and the sparse x dense
// product of Fig. 5.  Layout and readings: include/sten.h, R17-R21.
//
//   column  = m consecutive rows of W at one input column k (m-blocks along M)
//   chunk   = L = C(m,n) g consecutive columns of one row block; each of the C(m,n)
//             patterns (revolving-door order) is used by exactly g columns
//   values  [M/m][K/L][L][n], idx [M/m][K/L][L] uint16 (original column in the chunk)
#pragma once
#include "common.cuh"
#include "spmm_simt.cuh"   // SpmmArgs, cluster_reduce_store (split-K over DSMEM)

namespace sten {

// ---- pattern order ---------------------------------------------------------------------------
// Revolving-door list of the n-subsets of {0..m-1} as bitmasks: RD(m, n) = RD(m-1, n) followed
// by reverse(RD(m-1, n-1)) with bit m-1 set; adjacent entries differ in one position
// ("the nonzero pattern between adjacent groups differs in only one location").
constexpr int kNmgMaxPatterns = 64;
struct NmgPatterns {
    uint32_t mask[kNmgMaxPatterns];
    int count;
};

__host__ __device__ constexpr NmgPatterns nmg_revolving_door(int m, int n) {
    NmgPatterns r{};
    if (n == 0) { r.mask[0] = 0u; r.count = 1; return r; }
    if (n == m) { r.mask[0] = (1u << m) - 1u; r.count = 1; return r; }
    const NmgPatterns a = nmg_revolving_door(m - 1, n);
    const NmgPatterns b = nmg_revolving_door(m - 1, n - 1);
    int k = 0;
    for (int i = 0; i < a.count && k < kNmgMaxPatterns; ++i) r.mask[k++] = a.mask[i];
    for (int i = b.count - 1; i >= 0 && k < kNmgMaxPatterns; --i) r.mask[k++] = b.mask[i] | (1u << (m - 1));
    r.count = a.count + b.count;
    return r;
}

// position of the t-th set bit of mask (t-th kept row of the pattern, ascending)
__host__ __device__ constexpr int nmg_pos(uint32_t mask, int t) {
    int c = 0;
    for (int j = 0; j < 32; ++j)
        if (mask >> j & 1u) {
            if (c == t) return j;
            ++c;
        }
    return -1;
}

__host__ __device__ constexpr int nmg_binom(int m, int n) {
    long long r = 1;
    for (int i = 1; i <= n; ++i) r = r * (m - n + i) / i;
    return int(r);
}

struct NmgArgs {
    const void* W;          // sparsify: dense input; densify: output
    int64_t ldw;
    const void* values_in;  // densify input
    void* values;           // sparsify output
    const uint16_t* idx_in; // densify input
    uint16_t* idx;          // sparsify output
    int64_t M, K, NC, RB;   // NC = K / L chunks per row block, RB = M / m row blocks
    int n, m, g, C, L;
    NmgPatterns pat;
    int method;             // sparsify: 0 greedy, 1 exchange from pattern b / g, 2 greedy + exchange
};

// ---- conversion: one warp per chunk ------------------------------------------------------------
// Keys of the C(m,n)^2 g (column b, pattern p) items: fp32 magnitude bits (>= +0, so the bit
// pattern orders like the value) above (0xFFFF - b) above (0xFFFF - p): the largest key is the
// highest magnitude, then the lower column, then the lower pattern id -- the sorted order of
// PAPER.md:555 with DESIGN.md R19's tie-break.  Processing the sorted list and accepting an item
// when its column is free and its pattern has < g columns equals repeatedly accepting the
// largest still-acceptable item (acceptability only ever turns false), which is what each
// step's warp-wide max does.
constexpr int kNmgWarpsPerCta = 4;
constexpr int kNmgRegKeys = 8;          // keys per lane held in registers when L C <= 256

__host__ __device__ inline size_t nmg_warp_smem(int L, int C, int m, int esz) {
    const size_t keys = size_t(L) * C * 8;
    const size_t w = (size_t(m) * L * esz + 15) & ~size_t(15);
    return keys + w + ((size_t(C) * 4 + size_t(L) * 2 + 15) & ~size_t(15));
}

// KPL = keys per lane held in registers (2, 4, 6 or 8: the smallest with 32 KPL >= L C); for
// L C > 256 the keys live in shared memory (KPL unused)
template <typename T, int KPL>
__global__ void __launch_bounds__(kNmgWarpsPerCta * 32)
nmg_sparsify_kernel(const NmgArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    // kept row t of pattern p, tabulated once per CTA (the bit scan is not in the per-key path)
    __shared__ int8_t spos[kNmgMaxPatterns * 16];
    for (int e = threadIdx.x; e < a.C * a.n; e += blockDim.x)
        spos[e] = int8_t(nmg_pos(a.pat.mask[e / a.n], e % a.n));
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t chunk = int64_t(blockIdx.x) * kNmgWarpsPerCta + warp;
    if (chunk >= a.RB * a.NC) return;
    const int64_t rb = chunk / a.NC, c = chunk - rb * a.NC;
    const int L = a.L, C = a.C, n = a.n, g = a.g, m = a.m;
    unsigned char* ws = smem + size_t(warp) * nmg_warp_smem(L, C, m, int(sizeof(T)));
    unsigned long long* key = reinterpret_cast<unsigned long long*>(ws);
    T* sw = reinterpret_cast<T*>(ws + size_t(L) * C * 8);                       // the m x L block of W
    unsigned char* tail = ws + size_t(L) * C * 8 + ((size_t(m) * L * sizeof(T) + 15) & ~size_t(15));
    int* cnt = reinterpret_cast<int*>(tail);                                     // 4-byte aligned
    int16_t* pat_of = reinterpret_cast<int16_t*>(tail + size_t(C) * 4);
    const T* W = static_cast<const T*>(a.W);
    const T* w0 = W + rb * a.m * a.ldw + c * L;   // column b, row r: w0[r * ldw + b]

    // the chunk's m x L block, row by row (coalesced), into shared memory
    for (int e = lane; e < m * L; e += 32) {
        const int r = e / L, b = e - r * L;
        sw[e] = w0[int64_t(r) * a.ldw + b];
    }
    for (int b = lane; b < L; b += 32) pat_of[b] = -1;
    for (int p = lane; p < C; p += 32) cnt[p] = 0;
    __syncwarp();
    const int NI = L * C;
    auto make_key = [&](int i) -> unsigned long long {
        const int b = i / C, p = i - b * C;
        float s = 0.0f;
        for (int t = 0; t < n; ++t) s = __fadd_rn(s, fabsf(to_f32(sw[spos[p * n + t] * L + b])));
        return (static_cast<unsigned long long>(__float_as_uint(s)) << 32) |
               (static_cast<unsigned long long>(0xFFFFu - uint32_t(b)) << 16) | (0xFFFFu - uint32_t(p));
    };
    // warp max of a 64-bit key with two redux.sync: max of the high words, then max of the low
    // words among the lanes holding that high word
    auto warp_max = [&](unsigned long long k) {
        const uint32_t hi = uint32_t(k >> 32), lo = uint32_t(k);
        const uint32_t mh = __reduce_max_sync(0xffffffffu, hi);
        const uint32_t ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
        return (static_cast<unsigned long long>(mh) << 32) | ml;
    };
    auto kb = [](unsigned long long k) { return int(0xFFFFu - uint32_t((k >> 16) & 0xFFFFu)); };
    auto kp = [](unsigned long long k) { return int(0xFFFFu - uint32_t(k & 0xFFFFu)); };

    if (a.method == 1) {
        // the paper's GPU variant starts from an arbitrary assignment: column b gets pattern b / g
        for (int b = lane; b < L; b += 32) pat_of[b] = int16_t(b / g);
    } else if (L <= 32 && C <= 8 && NI > 96) {      // (small chunks: the L-step loop below is cheaper)
        // Round-based exact greedy (L <= 32: lane b owns column b).  The largest acceptable item
        // is always the largest "proposal" (each free column's best not-full pattern), so in a
        // round the warp sorts the proposals (bitonic, descending) and accepts the longest prefix
        // in which no pattern exceeds its capacity g; a proposal to a pattern that fills inside
        // the round ends it.  Identical to the sequential greedy, <= C + 1 rounds instead of L.
        unsigned long long kc[8];
#pragma unroll
        for (int p = 0; p < 8; ++p) kc[p] = (lane < L && p < C) ? make_key(lane * C + p) : 0ull;
        int cntr[8];
#pragma unroll
        for (int p = 0; p < 8; ++p) cntr[p] = 0;
        bool assigned = lane >= L;
        int mypat = -1;
        __shared__ uint32_t acc_scratch[kNmgWarpsPerCta][32];      // per-warp column -> accepted pattern + 1
        uint32_t* accf = acc_scratch[warp];
        accf[lane] = 0u;
        __syncwarp();
        for (int round = 0; round <= C; ++round) {
            unsigned long long prop = 0ull;
            if (!assigned) {
#pragma unroll
                for (int p = 0; p < 8; ++p)
                    if (p < C && cntr[p] < g && kc[p] > prop) prop = kc[p];
            }
            if (!__any_sync(0xffffffffu, prop != 0ull)) break;
            // bitonic sort of the 32 proposals, descending across lanes
            unsigned long long v = prop;
#pragma unroll
            for (int k = 2; k <= 32; k <<= 1)
#pragma unroll
                for (int j = k >> 1; j > 0; j >>= 1) {
                    const unsigned long long o = __shfl_xor_sync(0xffffffffu, v, j);
                    const bool up = (lane & k) == 0, lower = (lane & j) == 0;
                    const unsigned long long mn = o < v ? o : v, mx = o < v ? v : o;
                    v = (lower == up) ? mx : mn;
                }
            // sorted position `lane` holds v; its pattern, and how many earlier positions share it
            const bool real = v != 0ull;
            const int vp = real ? kp(v) : -1;
            const unsigned same = __match_any_sync(0xffffffffu, vp);
            const int before = __popc(same & ((1u << lane) - 1u));            // earlier, same pattern
            int cp = 0;
#pragma unroll
            for (int p = 0; p < 8; ++p) cp = (p == vp) ? cntr[p] : cp;
            const bool ok = real && cp + before + 1 <= g;
            const unsigned bad = __ballot_sync(0xffffffffu, real && !ok);
            const int stop = bad ? __ffs(bad) - 1 : 32;
            const bool acc = real && lane < stop;
            // tell each column lane whether its proposal was accepted (inverse permutation via smem)
            if (acc) accf[kb(v)] = uint32_t(vp) + 1u;
            __syncwarp();
            if (!assigned && lane < L) {
                const uint32_t f = accf[lane];
                if (f) { assigned = true; mypat = int(f) - 1; }
            }
            __syncwarp();
            if (acc) accf[kb(v)] = 0u;
            // capacity update, identical in every lane
#pragma unroll
            for (int p = 0; p < 8; ++p) cntr[p] += __popc(__ballot_sync(0xffffffffu, acc && vp == p));
            __syncwarp();
        }
        if (lane < L) pat_of[lane] = int16_t(mypat);
    } else if (NI <= 32 * KPL) {
        // keys in registers; a key is zeroed when its column is taken or its pattern is full
        unsigned long long kr[KPL];
        int kcol[KPL], kpat[KPL];                // each key's column and pattern, decoded once
#pragma unroll
        for (int j = 0; j < KPL; ++j) {
            const int i = lane + 32 * j;
            kr[j] = i < NI ? make_key(i) : 0ull;
            kcol[j] = i < NI ? i / C : -1;
            kpat[j] = i < NI ? i - (i / C) * C : -1;
        }
        for (int step = 0; step < L; ++step) {
            unsigned long long best = 0ull;
#pragma unroll
            for (int j = 0; j < KPL; ++j) best = kr[j] > best ? kr[j] : best;
            best = warp_max(best);
            const int b = kb(best), p = kp(best);
            const int c_old = cnt[p];
            __syncwarp();
            if (lane == 0) { pat_of[b] = int16_t(p); cnt[p] = c_old + 1; }
            __syncwarp();
            const bool full = c_old + 1 >= g;
#pragma unroll
            for (int j = 0; j < KPL; ++j)
                kr[j] = (kcol[j] == b || (full && kpat[j] == p)) ? 0ull : kr[j];
        }
    } else {
        for (int i = lane; i < NI; i += 32) key[i] = make_key(i);
        __syncwarp();
        for (int step = 0; step < L; ++step) {
            unsigned long long best = 0ull;
            for (int i = lane; i < NI; i += 32) {
                const unsigned long long k = key[i];
                if (k > best && pat_of[kb(k)] < 0 && cnt[kp(k)] < g) best = k;
            }
            best = warp_max(best);
            if (lane == 0) { pat_of[kb(best)] = int16_t(kp(best)); cnt[kp(best)] += 1; }
            __syncwarp();
        }
    }
    __syncwarp();
    if (a.method != 0) {
        // Exchange refinement, the paper's GPU conversion: swap the patterns of two
        // columns when that raises the pair's magnitude, until no swap is made.  Sequential order of
        // DESIGN.md R22 (pairs (i, j), i < j ascending, the first improving j taken, then the scan
        // continues with i's new pattern), computed warp-parallel: the 32 lanes test j0..j0+31 against
        // i's current pattern and a ballot finds the first improving one -- the same swaps, in the same
        // order, as the oracle.  Magnitudes: a table [L][C] in the (now unused) key space.
        float* mag = reinterpret_cast<float*>(key);
        for (int i = lane; i < NI; i += 32) {
            const int b = i / C, p = i - b * C;
            float s = 0.0f;
            for (int t = 0; t < n; ++t) s = __fadd_rn(s, fabsf(to_f32(sw[spos[p * n + t] * L + b])));
            mag[i] = s;
        }
        __syncwarp();
        bool changed = true;
        while (changed) {
            changed = false;
            for (int i = 0; i < L; ++i) {
                int j0 = i + 1;
                while (j0 < L) {
                    const int pi = pat_of[i];
                    const int j = j0 + lane;
                    bool imp = false;
                    if (j < L) {
                        const int pj = pat_of[j];
                        if (pj != pi) {
                            const double now = double(mag[i * C + pi]) + double(mag[j * C + pj]);
                            const double swp = double(mag[i * C + pj]) + double(mag[j * C + pi]);
                            imp = swp > now;
                        }
                    }
                    const unsigned bal = __ballot_sync(0xffffffffu, imp);
                    if (!bal) { j0 += 32; continue; }
                    const int jj = j0 + __ffs(bal) - 1;
                    __syncwarp();
                    if (lane == 0) { const int16_t pj = pat_of[jj]; pat_of[jj] = int16_t(pi); pat_of[i] = pj; }
                    __syncwarp();
                    changed = true;
                    j0 = jj + 1;
                }
            }
        }
    }
    // store: slot = p g + (number of lower columns with the same pattern)
    T* V = static_cast<T*>(a.values);
    const int64_t base = chunk * L;
    for (int b = lane; b < L; b += 32) {
        const int p = pat_of[b];
        int rank = 0;
        for (int b2 = 0; b2 < b; ++b2) rank += pat_of[b2] == p;
        const int64_t slot = base + int64_t(p) * g + rank;
        a.idx[slot] = uint16_t(b);
        for (int t = 0; t < n; ++t) V[slot * n + t] = sw[spos[p * n + t] * L + b];
    }
}

// ---- densify: one thread per (chunk, slot); writes the whole m-row column once -----------------
template <typename T>
__global__ void __launch_bounds__(256) nmg_densify_kernel(const NmgArgs a, T* __restrict__ Wout) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= a.RB * a.NC * a.L) return;
    const int64_t chunk = i / a.L;
    const int s = int(i - chunk * a.L);
    const int64_t rb = chunk / a.NC, c = chunk - rb * a.NC;
    const int b = a.idx_in[i];
    const uint32_t mk = a.pat.mask[s / a.g];
    const T* V = static_cast<const T*>(a.values_in) + i * a.n;
    T* col = Wout + rb * a.m * a.ldw + c * a.L + b;
    int t = 0;
    for (int r = 0; r < a.m; ++r) {
        const bool kept = (mk >> r) & 1u;
        col[int64_t(r) * a.ldw] = kept ? V[t] : T(0);
        t += kept;
    }
}

// ---- product (Fig. 5) ----------------------------------------------------------------------------
// CTA = 8 warps x BN = 256 tokens (lane: 8 tokens, two 16-byte vectors 512 B apart for fp32, so a
// warp's gathered row read is two conflict-free 512-byte passes); warp w owns row block rbc + w
// (m rows; accumulators acc[m][8] in registers with static row indices, because the pattern order
// is a compile-time table -- "chunks, which fix the order of sparsity permutations, allow kernels
// to avoid branches based on the sparsity structure").  A K-stage of CPS whole chunks
// is staged by cp.async in a 3-stage ring: the CPS L rows of B (shared by the CTA's 8 row blocks)
// and, per row block, its CPS L idx entries and CPS L n values.  Per slot a warp reads the idx
// (broadcast), gathers its B row, reads the n values (broadcast) and does 4n FFMA2 per lane --
// "loaded from sparse values, then broadcast into vector registers ... indirect loads from
// specific rows of B ... FMA".  Split-K over whole chunks: the S CTAs of a tile
// form a thread-block cluster (1,1,S) and reduce their fp32 partial tiles over DSMEM in the fixed
// order z = 0..S-1 (the (A) kernel's cluster_reduce_store), so the result is deterministic.
// Each gathered B element feeds n FMAs (the (A) layout's feeds g), so for fp32 the shared-memory
// datapath caps this kernel near n/4 of the FFMA peak.
struct NmgSpmmArgs {
    const void* values;
    const uint16_t* idx;
    const void* B;
    void* C;
    int64_t M, K, N, ldb, ldc, NC, RB;
    int g, L, cps;          // cps = chunks per K-stage
    int split;              // S: split-K parts (cluster z extent)
    bool c_vec;
};

constexpr int kNmgSpmmWarps = 8;
constexpr int kNmgStages = 3;
constexpr int kNmgBN = 256;

// per-stage shared memory: B [cps L][BN] | idx [8][cps L] u16 | values [8][cps L n]
template <typename TAB>
__host__ __device__ inline size_t nmg_spmm_stage_bytes(int rows, int n) {
    const size_t b = size_t(rows) * kNmgBN * sizeof(TAB);
    const size_t i = (size_t(kNmgSpmmWarps) * rows * 2 + 15) & ~size_t(15);
    const size_t v = (size_t(kNmgSpmmWarps) * rows * n * sizeof(TAB) + 15) & ~size_t(15);
    return b + i + v;
}

template <typename TAB, typename TC, int NN, int MM>
__global__ void __launch_bounds__(kNmgSpmmWarps * 32, 2)
nmg_spmm_kernel(const NmgSpmmArgs a) {
    constexpr NmgPatterns P = nmg_revolving_door(MM, NN);
    constexpr int CP = nmg_binom(MM, NN);
    static_assert(CP <= kNmgMaxPatterns, "too many patterns");
    constexpr int EV = 8;                                   // tokens per lane
    constexpr int NT = kNmgSpmmWarps * 32;
    constexpr int ROWB = kNmgBN * int(sizeof(TAB));         // bytes per staged B row
    extern __shared__ __align__(16) unsigned char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t n0 = int64_t(blockIdx.x) * kNmgBN;
    const int64_t rbc = int64_t(blockIdx.y) * kNmgSpmmWarps;          // first row block of the CTA
    const int L = a.L, g = a.g;
    const int rows = a.cps * L;                                        // B rows per stage
    const size_t b_bytes = size_t(rows) * ROWB;
    const size_t i_bytes = (size_t(kNmgSpmmWarps) * rows * 2 + 15) & ~size_t(15);
    const size_t stage_bytes = nmg_spmm_stage_bytes<TAB>(rows, NN);
    const TAB* B = static_cast<const TAB*>(a.B);
    const TAB* V = static_cast<const TAB*>(a.values);
    // split-K part z: chunks [z NC / S, (z+1) NC / S), staged cps at a time
    const int64_t c_lo = a.NC * int64_t(blockIdx.z) / a.split, c_hi = a.NC * int64_t(blockIdx.z + 1) / a.split;
    const int64_t nstages = (c_hi - c_lo + a.cps - 1) / a.cps;

    auto load_stage = [&](int64_t st, int buf) {
        unsigned char* dst = smem + size_t(buf) * stage_bytes;
        const int64_t c0 = c_lo + st * a.cps;
        const int nch = int(min64(a.cps, c_hi - c0));
        const int64_t k0 = c0 * L;
        constexpr int CH = ROWB / 16;                                  // 16-byte chunks per B row
        for (int e = threadIdx.x; e < rows * CH; e += NT) {
            const int r = e / CH, ch = e - r * CH;
            const int64_t k = k0 + r;
            const int64_t col = n0 + int64_t(ch) * (16 / int(sizeof(TAB)));
            int bytes = 0;
            if (r < nch * L && col < a.N) bytes = int(min64(16, (a.N - col) * int64_t(sizeof(TAB))));
            cp_async16(dst + size_t(r) * ROWB + size_t(ch) * 16, bytes ? B + k * a.ldb + col : B, bytes);
        }
        // idx and values of the CTA's row blocks: contiguous runs (4-byte words; L is even for
        // every compiled format, so runs start and end on 4-byte boundaries)
        const int iw = nch * L / 2, vw = nch * L * NN * int(sizeof(TAB)) / 4;
        for (int e = threadIdx.x; e < kNmgSpmmWarps * (iw + vw); e += NT) {
            const int w = e / (iw + vw), o = e - w * (iw + vw);
            const int64_t rb = rbc + w;
            const bool ok = rb < a.RB;
            const int64_t chunk = ok ? rb * a.NC + c0 : 0;
            if (o < iw) {
                cp_async4(dst + b_bytes + (size_t(w) * rows) * 2 + size_t(o) * 4,
                          reinterpret_cast<const unsigned char*>(a.idx + chunk * L) + size_t(o) * 4, ok ? 4 : 0);
            } else {
                const int ov = o - iw;
                cp_async4(dst + b_bytes + i_bytes + size_t(w) * rows * NN * sizeof(TAB) + size_t(ov) * 4,
                          reinterpret_cast<const unsigned char*>(V + chunk * L * NN) + size_t(ov) * 4, ok ? 4 : 0);
            }
        }
        cp_async_commit();
    };

    float acc[MM][EV];
#pragma unroll
    for (int r = 0; r < MM; ++r)
#pragma unroll
        for (int e = 0; e < EV; ++e) acc[r][e] = 0.0f;

    const int64_t rb = rbc + warp;
    // kNmgStages-deep ring: stages st+1 .. st+kNmgStages-1 are in flight while st is consumed
    for (int64_t st = 0; st < kNmgStages - 1; ++st) {
        if (st < nstages) load_stage(st, int(st));
        else cp_async_commit();                                        // keep the group count uniform
    }
    for (int64_t st = 0; st < nstages; ++st) {
        const int buf = int(st % kNmgStages);
        asm volatile("cp.async.wait_group %0;\n" ::"n"(kNmgStages - 2) : "memory");
        __syncthreads();                                               // stage st visible; st-1 consumed
        if (st + kNmgStages - 1 < nstages) load_stage(st + kNmgStages - 1, int((st + kNmgStages - 1) % kNmgStages));
        else cp_async_commit();
        if (rb < a.RB) {
            const unsigned char* sb = smem + size_t(buf) * stage_bytes;
            const uint32_t sB = smem_u32(sb) + uint32_t(lane) * 16u;
            const uint16_t* sI = reinterpret_cast<const uint16_t*>(sb + b_bytes) + size_t(warp) * rows;
            const TAB* sV = reinterpret_cast<const TAB*>(sb + b_bytes + i_bytes) + size_t(warp) * rows * NN;
            const int nch = int(min64(a.cps, c_hi - (c_lo + st * a.cps)));
            for (int cl = 0; cl < nch; ++cl) {
                const uint32_t sBc = sB + uint32_t(cl * L) * uint32_t(ROWB);
                const uint16_t* ip = sI + cl * L;
                const TAB* vp = sV + size_t(cl) * L * NN;
#pragma unroll
                for (int p = 0; p < CP; ++p) {
#pragma unroll 4
                    for (int j = 0; j < g; ++j) {
                        const int s = p * g + j;
                        const uint32_t addr = sBc + uint32_t(ip[s]) * uint32_t(ROWB);
                        float2 b[4];
                        if constexpr (sizeof(TAB) == 4) {
                            const float4 x0 = lds128_addr(addr), x1 = lds128_addr(addr + 512u);
                            b[0] = make_float2(x0.x, x0.y); b[1] = make_float2(x0.z, x0.w);
                            b[2] = make_float2(x1.x, x1.y); b[3] = make_float2(x1.z, x1.w);
                        } else {
                            const float4 x = lds128_addr(addr);
                            const uint32_t w[4] = {__float_as_uint(x.x), __float_as_uint(x.y),
                                                   __float_as_uint(x.z), __float_as_uint(x.w)};
#pragma unroll
                            for (int q = 0; q < 4; ++q)
                                b[q] = make_float2(__uint_as_float(w[q] << 16), __uint_as_float(w[q] & 0xffff0000u));
                        }
#pragma unroll
                        for (int t = 0; t < NN; ++t) {
                            const float v = to_f32(vp[s * NN + t]);
                            const int r = nmg_pos(P.mask[p], t);
#pragma unroll
                            for (int q = 0; q < 4; ++q) {
                                float2& c2 = *reinterpret_cast<float2*>(&acc[r][2 * q]);
                                c2 = __ffma2_rn(make_float2(v, v), b[q], c2);
                            }
                        }
                    }
                }
            }
        }
    }
    // token of accumulator e: fp32 -> n0 + 4 lane + (e & 3) + 128 (e >> 2); bf16 -> n0 + 8 lane + e
    auto col_of = [&](int e) -> int {
        return sizeof(TAB) == 4 ? 4 * lane + (e & 3) + 128 * (e >> 2) : 8 * lane + e;
    };
    if (a.split == 1) {
        if (rb >= a.RB) return;
        TC* Cp = static_cast<TC*>(a.C);
#pragma unroll
        for (int r = 0; r < MM; ++r) {
            TC* row = Cp + (rb * MM + r) * a.ldc;
#pragma unroll
            for (int e = 0; e < EV; ++e) {
                const int64_t col = n0 + col_of(e);
                if (col < a.N) row[col] = from_f32<TC>(acc[r][e]);
            }
        }
        return;
    }
    // split-K: park the fp32 partial tile [8 MM][BN] at the start of shared memory, reduce over the
    // cluster in the fixed order z = 0..S-1
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    __syncthreads();
    float* tile = reinterpret_cast<float*>(smem);
#pragma unroll
    for (int r = 0; r < MM; ++r)
#pragma unroll
        for (int e = 0; e < EV; ++e) tile[(warp * MM + r) * kNmgBN + col_of(e)] = acc[r][e];
    SpmmArgs ra;
    memset(&ra, 0, sizeof(ra));
    ra.C = a.C; ra.M = a.M; ra.N = a.N; ra.ldc = a.ldc; ra.split = a.split; ra.c_vec = a.c_vec;
    cluster_reduce_store<TC, kNmgSpmmWarps * MM, kNmgBN, NT>(smem, ra, rbc * MM, n0);
}

}  // namespace sten
