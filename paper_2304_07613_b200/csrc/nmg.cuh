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

__host__ __device__ inline size_t nmg_warp_smem(int L, int C) {
    return (size_t(L) * C * 8 + size_t(L) * 2 + size_t(C) * 4 + 15) & ~size_t(15);
}

template <typename T>
__global__ void __launch_bounds__(kNmgWarpsPerCta * 32)
nmg_sparsify_kernel(const NmgArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t chunk = int64_t(blockIdx.x) * kNmgWarpsPerCta + warp;
    if (chunk >= a.RB * a.NC) return;
    const int64_t rb = chunk / a.NC, c = chunk - rb * a.NC;
    const int L = a.L, C = a.C, n = a.n, g = a.g;
    unsigned char* ws = smem + size_t(warp) * nmg_warp_smem(L, C);
    unsigned long long* key = reinterpret_cast<unsigned long long*>(ws);
    int* cnt = reinterpret_cast<int*>(ws + size_t(L) * C * 8);                       // 4-byte aligned
    int16_t* pat_of = reinterpret_cast<int16_t*>(ws + size_t(L) * C * 8 + size_t(C) * 4);
    const T* W = static_cast<const T*>(a.W);
    const T* w0 = W + rb * a.m * a.ldw + c * L;   // column b, row r: w0[r * ldw + b]

    const int NI = L * C;
    for (int i = lane; i < NI; i += 32) {
        const int b = i / C, p = i - b * C;
        const uint32_t mk = a.pat.mask[p];
        float s = 0.0f;
        for (int t = 0; t < n; ++t) s = __fadd_rn(s, fabsf(to_f32(w0[int64_t(nmg_pos(mk, t)) * a.ldw + b])));
        key[i] = (static_cast<unsigned long long>(__float_as_uint(s)) << 32) |
                 (static_cast<unsigned long long>(0xFFFFu - uint32_t(b)) << 16) | (0xFFFFu - uint32_t(p));
    }
    for (int b = lane; b < L; b += 32) pat_of[b] = -1;
    for (int p = lane; p < C; p += 32) cnt[p] = 0;
    __syncwarp();
    for (int step = 0; step < L; ++step) {
        unsigned long long best = 0ull;
        for (int i = lane; i < NI; i += 32) {
            const unsigned long long k = key[i];
            const int b = int(0xFFFFu - uint32_t((k >> 16) & 0xFFFFu));
            const int p = int(0xFFFFu - uint32_t(k & 0xFFFFu));
            if (k > best && pat_of[b] < 0 && cnt[p] < g) best = k;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long other = __shfl_xor_sync(0xffffffffu, best, o);
            best = other > best ? other : best;
        }
        if (lane == 0) {
            const int b = int(0xFFFFu - uint32_t((best >> 16) & 0xFFFFu));
            const int p = int(0xFFFFu - uint32_t(best & 0xFFFFu));
            pat_of[b] = int16_t(p);
            cnt[p] += 1;
        }
        __syncwarp();
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
        const uint32_t mk = a.pat.mask[p];
        for (int t = 0; t < n; ++t) V[slot * n + t] = w0[int64_t(nmg_pos(mk, t)) * a.ldw + b];
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
// CTA = 8 warps x BN = 128 tokens (lane: 4 consecutive tokens); warp w owns RBW row blocks (m
// rows each; accumulators acc[RBW][m][4] in registers, static row indices because the pattern
// order is a compile-time table -- the paper's "chunks, which fix the order of sparsity
// permutations, allow kernels to avoid branches based on the sparsity structure").
// A K-stage of CPS whole chunks (CPS L rows of B) is staged in shared memory by cp.async (double
// buffered) and shared by every row block of the CTA; per slot a warp reads the idx and the n
// values (uniform loads, L1 broadcast), gathers its B row from shared memory (LDS.128 for fp32)
// and does 4 n FMAs per lane -- "broadcast into vector registers ... indirect loads from specific
// rows of B ... FMA".
struct NmgSpmmArgs {
    const void* values;
    const uint16_t* idx;
    const void* B;
    void* C;
    int64_t M, K, N, ldb, ldc, NC, RB;
    int g, L, cps;          // cps = chunks per K-stage
};

constexpr int kNmgSpmmWarps = 8;
constexpr int kNmgBN = 128;

template <typename TAB>
__host__ __device__ inline size_t nmg_spmm_stage_bytes(int rows) {
    return size_t(rows) * kNmgBN * sizeof(TAB);
}

template <typename TAB, typename TC, int NN, int MM, int RBW>
__global__ void __launch_bounds__(kNmgSpmmWarps * 32)
nmg_spmm_kernel(const NmgSpmmArgs a) {
    constexpr NmgPatterns P = nmg_revolving_door(MM, NN);
    constexpr int CP = nmg_binom(MM, NN);
    static_assert(CP <= kNmgMaxPatterns, "too many patterns");
    constexpr int EV = 4;                                   // tokens per lane
    extern __shared__ __align__(16) unsigned char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t n0 = int64_t(blockIdx.x) * kNmgBN;
    const int64_t rb0 = (int64_t(blockIdx.y) * kNmgSpmmWarps + warp) * RBW;
    const int L = a.L, g = a.g;
    const int rows = a.cps * L;                             // B rows per stage
    const size_t stage_bytes = nmg_spmm_stage_bytes<TAB>(rows);
    const TAB* B = static_cast<const TAB*>(a.B);
    const int64_t nstages = (a.NC + a.cps - 1) / a.cps;

    // cooperative cp.async of one stage: rows [c0 L, (c0 + cps) L) x tokens [n0, n0 + BN)
    constexpr int CH = kNmgBN * int(sizeof(TAB)) / 16;      // 16-byte chunks per staged row
    auto load_stage = [&](int64_t st, int buf) {
        unsigned char* dst = smem + size_t(buf) * stage_bytes;
        const int64_t k0 = st * a.cps * L;
        for (int e = threadIdx.x; e < rows * CH; e += kNmgSpmmWarps * 32) {
            const int r = e / CH, ch = e - r * CH;
            const int64_t k = k0 + r;
            const int64_t col = n0 + int64_t(ch) * (16 / int(sizeof(TAB)));
            int bytes = 0;
            if (k < a.K && col < a.N) bytes = int(min64(16, (a.N - col) * int64_t(sizeof(TAB))));
            cp_async16(dst + size_t(r) * kNmgBN * sizeof(TAB) + size_t(ch) * 16, bytes ? B + k * a.ldb + col : B,
                       bytes);
        }
        cp_async_commit();
    };

    float acc[RBW][MM][EV];
#pragma unroll
    for (int q = 0; q < RBW; ++q)
#pragma unroll
        for (int r = 0; r < MM; ++r)
#pragma unroll
            for (int e = 0; e < EV; ++e) acc[q][r][e] = 0.0f;

    const TAB* V = static_cast<const TAB*>(a.values);
    if (nstages > 0) load_stage(0, 0);
    for (int64_t st = 0; st < nstages; ++st) {
        const int buf = int(st & 1);
        if (st + 1 < nstages) {
            load_stage(st + 1, buf ^ 1);
            asm volatile("cp.async.wait_group 1;\n" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        }
        __syncthreads();
        const unsigned char* sB = smem + size_t(buf) * stage_bytes + size_t(lane) * EV * sizeof(TAB);
        const int64_t c_begin = st * a.cps;
        const int nch = int(min64(a.cps, a.NC - c_begin));
#pragma unroll
        for (int q = 0; q < RBW; ++q) {
            const int64_t rb = rb0 + q;
            if (rb >= a.RB) break;
            for (int cl = 0; cl < nch; ++cl) {
                const int64_t chunk = rb * a.NC + c_begin + cl;
                const uint16_t* ip = a.idx + chunk * L;
                const TAB* vp = V + chunk * L * NN;
                const unsigned char* sc = sB + size_t(cl) * L * kNmgBN * sizeof(TAB);
#pragma unroll
                for (int p = 0; p < CP; ++p) {
                    for (int j = 0; j < g; ++j) {
                        const int s = p * g + j;
                        const int b = __ldg(ip + s);
                        float bv[EV];
                        if constexpr (sizeof(TAB) == 4) {
                            const float4 t4 = *reinterpret_cast<const float4*>(sc + size_t(b) * kNmgBN * 4);
                            bv[0] = t4.x; bv[1] = t4.y; bv[2] = t4.z; bv[3] = t4.w;
                        } else {
                            const uint2 t2 = *reinterpret_cast<const uint2*>(sc + size_t(b) * kNmgBN * 2);
                            bv[0] = __uint_as_float(t2.x << 16); bv[1] = __uint_as_float(t2.x & 0xffff0000u);
                            bv[2] = __uint_as_float(t2.y << 16); bv[3] = __uint_as_float(t2.y & 0xffff0000u);
                        }
#pragma unroll
                        for (int t = 0; t < NN; ++t) {
                            const float v = to_f32(vp[s * NN + t]);
                            const int r = nmg_pos(P.mask[p], t);
#pragma unroll
                            for (int e = 0; e < EV; ++e) acc[q][r][e] = fmaf(v, bv[e], acc[q][r][e]);
                        }
                    }
                }
            }
        }
        __syncthreads();                                    // buffer buf is refilled next stage
    }
    // epilogue: rows rb m + r, tokens n0 + 4 lane + e
    TC* Cp = static_cast<TC*>(a.C);
#pragma unroll
    for (int q = 0; q < RBW; ++q) {
        const int64_t rb = rb0 + q;
        if (rb >= a.RB) break;
#pragma unroll
        for (int r = 0; r < MM; ++r) {
            TC* row = Cp + (rb * MM + r) * a.ldc;
#pragma unroll
            for (int e = 0; e < EV; ++e) {
                const int64_t col = n0 + int64_t(lane) * EV + e;
                if (col < a.N) row[col] = from_f32<TC>(acc[q][r][e]);
            }
        }
    }
}

}  // namespace sten
