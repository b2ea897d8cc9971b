/*
 * sten_oracle.c -- plain, slow, obviously-correct CPU ORACLE for the grouped
 * n:m layout of STen (arXiv 2304.07613).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header, table or helper with the CUDA path
 * (paper_2304_07613_b200/csrc); neither side includes the other.
 *
 * Reading of the paper followed here:
 *   - n:m: "each group of m elements has n nonzeros"
 *   - group: "each nonzero pattern is repeated g times,
 *     forming a group"
 *     -> reading (A) free grouping: g consecutive rows share one n-of-m pattern
 *        per m-block along K (the contraction axis).
 *   - objective: argmax ||X^|| with the L1 norm
 *     -> for (A) the argmax decomposes per (group, m-block): keep the n
 *        positions with the largest summed |w| over the group's g rows.
 *   - densify: "a single iteration over the values, reordering their
 *     location according to the stored index"
 *   - product: the sparse-dense GEMM C = A_sparse * B
 *
 * Arithmetic readings (paper silent; readings R4, R5, R10):
 *   - score s[j] = fl32(...fl32(|w[r0][j]| + |w[r0+1][j]|) ... + |w[r0+g-1][j]|),
 *     fp32, rows in ascending order, round-to-nearest-even, adds only.
 *     (built with -ffp-contract=off; there are no multiplies anyway)
 *   - rank[j] = #{ i : s[i] > s[j]  or  (s[i] == s[j] and i < j) };
 *     keep j iff rank[j] < n; idx lists kept j ascending.
 *   - SpMM reference in fp64, ascending k; Bound = sum |v|*|b| in fp64.
 *
 * Element types: dtype 0 = fp32, dtype 1 = bf16 stored as uint16 bit
 * patterns; bf16 is widened to fp32 exactly (bits << 16).
 *
 * Layouts (same logical layout as include/sten.h, written out independently):
 *   W      [M][ldw]            row-major, K <= ldw
 *   values [M][K/m*n]          row-major; values[r][kb*n+t]
 *   idx    [M/g][K/m][n]       uint8, ascending within each (group, block)
 *   B      [K][ldb]            row-major, N <= ldb
 *   C, Bound [M][N] (double)   row-major, only columns [c0, c1) written
 *
 * Parity status: every function here is pinned by tests/test_oracle_pins.py
 * (brute force over all C(m,n) subsets, textbook per-block top-n at g=1,
 * SPEC.md examples, closed forms B = I, integer-exact masked dense product,
 * energy inequalities).  No function is "parity unpinned".
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

#ifdef _OPENMP
#include <omp.h>
#endif

static float widen(int dtype, const void* base, int64_t i)
{
    if (dtype == 0) return ((const float*)base)[i];
    uint32_t bits = (uint32_t)((const uint16_t*)base)[i] << 16;
    float f;
    memcpy(&f, &bits, sizeof f);
    return f;
}

static void copy_elem(int dtype, void* dst, int64_t di, const void* src, int64_t si)
{
    if (dtype == 0) ((float*)dst)[di] = ((const float*)src)[si];
    else ((uint16_t*)dst)[di] = ((const uint16_t*)src)[si];
}

static void zero_elem(int dtype, void* dst, int64_t di)
{
    if (dtype == 0) ((float*)dst)[di] = 0.0f;
    else ((uint16_t*)dst)[di] = 0;
}

static int check_args(int n, int m, int g, int dtype, int64_t M, int64_t K)
{
    if (n < 1 || m > 16 || n >= m || g < 1) return 1;
    if (dtype != 0 && dtype != 1) return 1;
    if (M < 0 || K < 0) return 1;
    if (M % g != 0 || K % m != 0) return 2;
    return 0;
}

/* a1-a3: magnitude sparsifier to grouped n:m (reading A). */
int oracle_sparsify(int n, int m, int g, int dtype,
                    const void* W, int64_t M, int64_t K, int64_t ldw,
                    void* values, uint8_t* idx)
{
    int rc = check_args(n, m, g, dtype, M, K);
    if (rc) return rc;
    if (ldw < K) return 2;
    int64_t KB = K / m, Kp = KB * n, G = M / g;
    for (int64_t grp = 0; grp < G; ++grp) {
        for (int64_t kb = 0; kb < KB; ++kb) {
            float s[16];
            /* score: L1 magnitude of each in-block position over the group's rows */
            for (int j = 0; j < m; ++j) {
                float acc = 0.0f;
                for (int i = 0; i < g; ++i) {
                    int64_t r = grp * g + i;
                    acc = acc + fabsf(widen(dtype, W, r * ldw + kb * m + j));
                }
                s[j] = acc;
            }
            /* select: rank rule (larger score first, lower position on ties) */
            int t = 0;
            for (int j = 0; j < m; ++j) {
                int rank = 0;
                for (int i = 0; i < m; ++i)
                    if (s[i] > s[j] || (s[i] == s[j] && i < j)) rank++;
                if (rank < n) {
                    idx[(grp * KB + kb) * n + t] = (uint8_t)j;
                    t++;
                }
            }
            /* compact: bit copy of the kept weights of every row of the group */
            for (int i = 0; i < g; ++i) {
                int64_t r = grp * g + i;
                for (int u = 0; u < n; ++u) {
                    int j = idx[(grp * KB + kb) * n + u];
                    copy_elem(dtype, values, r * Kp + kb * n + u, W, r * ldw + kb * m + j);
                }
            }
        }
    }
    return 0;
}

/* a4: densify -- zero-fill, then scatter each stored value to its position. */
int oracle_densify(int n, int m, int g, int dtype,
                   const void* values, const uint8_t* idx, int64_t M, int64_t K,
                   void* W_out, int64_t ldw)
{
    int rc = check_args(n, m, g, dtype, M, K);
    if (rc) return rc;
    if (ldw < K) return 2;
    int64_t KB = K / m, Kp = KB * n;
    for (int64_t r = 0; r < M; ++r)
        for (int64_t k = 0; k < K; ++k)
            zero_elem(dtype, W_out, r * ldw + k);
    for (int64_t r = 0; r < M; ++r) {
        int64_t grp = r / g;
        for (int64_t kb = 0; kb < KB; ++kb)
            for (int u = 0; u < n; ++u) {
                int j = idx[(grp * KB + kb) * n + u];
                copy_elem(dtype, W_out, r * ldw + kb * m + j, values, r * Kp + kb * n + u);
            }
    }
    return 0;
}

/* a5-a7: C[r][c] = sum_{kb,t} values[r][kb*n+t] * B[kb*m + idx][c]   (fp64,
 * ascending k), and Bound[r][c] = sum |values| * |B|.  Columns [c0, c1). */
int oracle_spmm(int n, int m, int g, int dtype,
                const void* values, const uint8_t* idx, int64_t M, int64_t K,
                const void* B, int64_t ldb, int64_t N, int64_t c0, int64_t c1,
                double* C, double* Bound, int nthreads)
{
    int rc = check_args(n, m, g, dtype, M, K);
    if (rc) return rc;
    if (ldb < N || c0 < 0 || c1 > N || c0 > c1) return 2;
    int64_t KB = K / m, Kp = KB * n;
#ifdef _OPENMP
    if (nthreads < 1) nthreads = 1;
#pragma omp parallel for num_threads(nthreads) schedule(dynamic, 1)
#endif
    for (int64_t r = 0; r < M; ++r) {
        int64_t grp = r / g;
        for (int64_t c = c0; c < c1; ++c) {
            double acc = 0.0, bound = 0.0;
            for (int64_t kb = 0; kb < KB; ++kb)
                for (int u = 0; u < n; ++u) {
                    int64_t k = kb * m + idx[(grp * KB + kb) * n + u];
                    double v = (double)widen(dtype, values, r * Kp + kb * n + u);
                    double b = (double)widen(dtype, B, k * ldb + c);
                    acc += v * b;
                    bound += fabs(v) * fabs(b);
                }
            C[r * N + c] = acc;
            if (Bound) Bound[r * N + c] = bound;
        }
    }
    return 0;
}

/* Independent second path for the product: naive fp64 triple loop over a
 * dense (already masked) A[M][lda] times B[K][ldb]. */
int oracle_dense_matmul(int dtype, const void* A, int64_t M, int64_t K, int64_t lda,
                        const void* B, int64_t ldb, int64_t N, double* C, int nthreads)
{
    if (lda < K || ldb < N) return 2;
#ifdef _OPENMP
    if (nthreads < 1) nthreads = 1;
#pragma omp parallel for num_threads(nthreads) schedule(dynamic, 1)
#endif
    for (int64_t r = 0; r < M; ++r)
        for (int64_t c = 0; c < N; ++c) {
            double acc = 0.0;
            for (int64_t k = 0; k < K; ++k)
                acc += (double)widen(dtype, A, r * lda + k) * (double)widen(dtype, B, k * ldb + c);
            C[r * N + c] = acc;
        }
    return 0;
}

/* energy = ||X^||_1 / ||X||_1, fp64. */
double oracle_energy(int dtype, const void* Xhat, const void* X, int64_t M, int64_t K, int64_t ld)
{
    double num = 0.0, den = 0.0;
    for (int64_t r = 0; r < M; ++r)
        for (int64_t k = 0; k < K; ++k) {
            num += fabs((double)widen(dtype, Xhat, r * ld + k));
            den += fabs((double)widen(dtype, X, r * ld + k));
        }
    return den > 0.0 ? num / den : 0.0;
}

int oracle_max_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* ==========================================================================
 * Chunked n:m:g -- the paper's own format (DESIGN.md
 * readings R17-R21).  Test infrastructure, like everything in this file.
 *
 *   "each nonzero pattern is repeated g times, forming a group ... we combine
 *    groups into chunks with all C(m,n) combinations of nonzeros in fixed
 *    order ... we permit reordering the blocks of m elements within each
 *    chunk, and so store an index encoding the original location of each
 *    block"
 *   "The permutation order in chunks is selected so the nonzero pattern
 *    between adjacent groups differs in only one location"
 *   CPU conversion: "compute the total magnitude of the preserved elements for
 *    each column of a chunk with all permutations of nonzero patterns ...
 *    C(m,n)^2 g such columnwise magnitudes.  This list is then sorted and
 *    processed from highest to lowest.  We use a specific nonzero pattern for a
 *    column ... only if this column was not yet selected and the group
 *    corresponding to the pattern is not yet full."
 *   densify: "a single iteration over the values, reordering their location
 *    according to the stored index"
 *
 * Readings (paper silent): R17 a block ("column" of a chunk) is m consecutive
 * rows of W at one input column k -- the m-blocks run along the output rows M
 * and the chunks along K, L = C(m,n) g consecutive columns per chunk; R18 the
 * fixed pattern order is the revolving-door order R(m,n) = R(m-1,n) followed by
 * reverse(R(m-1,n-1)) each with m-1 added (adjacent patterns differ in one
 * element in, one out); R19 magnitude of (column b, pattern p) = fp32 sum of
 * |w| over p's positions ascending; ties in the sorted list by column
 * ascending, then pattern id ascending; R20 within a group (pattern) the g
 * columns are stored in ascending original column order; R21 idx is uint16.
 *
 * Layouts:  W [M][ldw]; values [M/m][K/L][L][n]; idx [M/m][K/L][L] (uint16,
 * original column offset in the chunk); slot s of a chunk has pattern s / g.
 * ========================================================================== */

static int nmg_binom(int m, int n)
{
    if (n < 0 || n > m) return 0;
    long r = 1;
    for (int i = 1; i <= n; ++i) r = r * (m - n + i) / i;
    return (int)r;
}

/* Revolving-door list R(m, n) of n-subsets of {0..m-1}, written as bitmasks
 * into out[0 .. C(m,n)-1]; returns the count.  Recursive definition (R18). */
static int nmg_revolving_door(int m, int n, uint32_t* out)
{
    if (n == 0) { out[0] = 0u; return 1; }
    if (n == m) { out[0] = (m >= 32) ? 0xffffffffu : ((1u << m) - 1u); return 1; }
    int a = nmg_revolving_door(m - 1, n, out);
    uint32_t* tmp = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)nmg_binom(m - 1, n - 1));
    int b = nmg_revolving_door(m - 1, n - 1, tmp);
    for (int i = 0; i < b; ++i) out[a + i] = tmp[b - 1 - i] | (1u << (m - 1));
    free(tmp);
    return a + b;
}

/* Patterns as ascending position lists: pos[p*n + t]. */
int oracle_nmg_patterns(int n, int m, int32_t* pos)
{
    if (n < 1 || n >= m || m > 16) return 1;
    int C = nmg_binom(m, n);
    uint32_t* mask = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)C);
    nmg_revolving_door(m, n, mask);
    for (int p = 0; p < C; ++p) {
        int t = 0;
        for (int j = 0; j < m; ++j)
            if (mask[p] >> j & 1u) pos[p * n + t++] = j;
    }
    free(mask);
    return 0;
}

static int nmg_check(int n, int m, int g, int dtype, int64_t M, int64_t K)
{
    if (n < 1 || n >= m || m > 16 || g < 1 || (dtype != 0 && dtype != 1) || M < 0 || K < 0) return 1;
    int64_t L = (int64_t)nmg_binom(m, n) * g;
    if (L > 65535) return 1;
    if (M % m != 0 || K % L != 0) return 2;
    return 0;
}

/* Greedy conversion of one chunk, sorted list processed in
 * order (magnitude desc, column asc, pattern asc). */
int oracle_nmg_sparsify(int n, int m, int g, int dtype,
                        const void* W, int64_t M, int64_t K, int64_t ldw,
                        void* values, uint16_t* idx)
{
    int rc = nmg_check(n, m, g, dtype, M, K);
    if (rc) return rc;
    if (ldw < K) return 2;
    const int C = nmg_binom(m, n);
    const int64_t L = (int64_t)C * g, NC = K / L, RB = M / m;
    int32_t* pos = (int32_t*)malloc(sizeof(int32_t) * (size_t)C * n);
    oracle_nmg_patterns(n, m, pos);
    const int64_t NI = L * C;
    float* mag = (float*)malloc(sizeof(float) * (size_t)NI);
    int64_t* order = (int64_t*)malloc(sizeof(int64_t) * (size_t)NI);
    int* pat_of = (int*)malloc(sizeof(int) * (size_t)L);
    int* cnt = (int*)malloc(sizeof(int) * (size_t)C);
    for (int64_t rb = 0; rb < RB; ++rb)
        for (int64_t c = 0; c < NC; ++c) {
            /* item i = b*C + p: magnitude of column b under pattern p */
            for (int64_t b = 0; b < L; ++b)
                for (int p = 0; p < C; ++p) {
                    float s = 0.0f;
                    for (int t = 0; t < n; ++t)
                        s = s + fabsf(widen(dtype, W, (rb * m + pos[p * n + t]) * ldw + c * L + b));
                    mag[b * C + p] = s;
                }
            /* sort: insertion sort by (mag desc, b asc, p asc) -- plain and obviously correct */
            for (int64_t i = 0; i < NI; ++i) order[i] = i;
            for (int64_t i = 1; i < NI; ++i) {
                int64_t x = order[i], j = i - 1;
                while (j >= 0 && (mag[order[j]] < mag[x] ||
                                  (mag[order[j]] == mag[x] && order[j] > x))) {
                    order[j + 1] = order[j];
                    --j;
                }
                order[j + 1] = x;
            }
            /* process from highest to lowest */
            for (int64_t b = 0; b < L; ++b) pat_of[b] = -1;
            for (int p = 0; p < C; ++p) cnt[p] = 0;
            for (int64_t i = 0; i < NI; ++i) {
                int64_t b = order[i] / C;
                int p = (int)(order[i] % C);
                if (pat_of[b] < 0 && cnt[p] < g) { pat_of[b] = p; cnt[p]++; }
            }
            /* store: slot s = p*g + (rank of b among the columns of pattern p, ascending b) */
            for (int p = 0; p < C; ++p) {
                int64_t s = (int64_t)p * g;
                for (int64_t b = 0; b < L; ++b)
                    if (pat_of[b] == p) {
                        int64_t slot = (rb * NC + c) * L + s;
                        idx[slot] = (uint16_t)b;
                        for (int t = 0; t < n; ++t)
                            copy_elem(dtype, values, slot * n + t, W, (rb * m + pos[p * n + t]) * ldw + c * L + b);
                        ++s;
                    }
            }
        }
    free(pos); free(mag); free(order); free(pat_of); free(cnt);
    return 0;
}

/* The paper's GPU conversion: "Initially, columns are arbitrarily assigned to
 * groups.  Each thread iterates over the columns in the other sparsity groups and attempts to
 * exchange the nonzero pattern it is assigned with an alternative nonzero pattern.  If such a swap
 * improves the overall magnitude for the pair of columns, it is performed atomically.  This
 * continues until no changes are made."  Written out sequentially (R22): passes over the
 * pairs (i, j), i < j ascending, of columns holding different patterns; swap when
 * mag[i][p_j] + mag[j][p_i] > mag[i][p_i] + mag[j][p_j] (the two-term sums in fp64, exact for
 * fp32 magnitudes); stop after a pass without a swap.  init 0: column b starts with pattern b / g
 * (the "arbitrary" start); init 1: the greedy assignment of oracle_nmg_sparsify.  Magnitudes and
 * storage order as the greedy. */
int oracle_nmg_sparsify_exchange(int n, int m, int g, int dtype,
                                 const void* W, int64_t M, int64_t K, int64_t ldw, int init,
                                 void* values, uint16_t* idx)
{
    int rc = nmg_check(n, m, g, dtype, M, K);
    if (rc) return rc;
    if (ldw < K || (init != 0 && init != 1)) return 2;
    if (init == 1) {
        /* start from the greedy result: run it, then read each column's pattern back */
        rc = oracle_nmg_sparsify(n, m, g, dtype, W, M, K, ldw, values, idx);
        if (rc) return rc;
    }
    const int C = nmg_binom(m, n);
    const int64_t L = (int64_t)C * g, NC = K / L, RB = M / m;
    int32_t* pos = (int32_t*)malloc(sizeof(int32_t) * (size_t)C * n);
    oracle_nmg_patterns(n, m, pos);
    float* mag = (float*)malloc(sizeof(float) * (size_t)(L * C));
    int* pat_of = (int*)malloc(sizeof(int) * (size_t)L);
    for (int64_t rb = 0; rb < RB; ++rb)
        for (int64_t c = 0; c < NC; ++c) {
            for (int64_t b = 0; b < L; ++b)
                for (int p = 0; p < C; ++p) {
                    float s = 0.0f;
                    for (int t = 0; t < n; ++t)
                        s = s + fabsf(widen(dtype, W, (rb * m + pos[p * n + t]) * ldw + c * L + b));
                    mag[b * C + p] = s;
                }
            if (init == 0) {
                for (int64_t b = 0; b < L; ++b) pat_of[b] = (int)(b / g);
            } else {
                for (int64_t s = 0; s < L; ++s) pat_of[idx[(rb * NC + c) * L + s]] = (int)(s / g);
            }
            int changed = 1;
            while (changed) {
                changed = 0;
                for (int64_t i = 0; i < L; ++i)
                    for (int64_t j = i + 1; j < L; ++j) {
                        int pi = pat_of[i], pj = pat_of[j];
                        if (pi == pj) continue;
                        double now = (double)mag[i * C + pi] + (double)mag[j * C + pj];
                        double swp = (double)mag[i * C + pj] + (double)mag[j * C + pi];
                        if (swp > now) { pat_of[i] = pj; pat_of[j] = pi; changed = 1; }
                    }
            }
            for (int p = 0; p < C; ++p) {
                int64_t s = (int64_t)p * g;
                for (int64_t b = 0; b < L; ++b)
                    if (pat_of[b] == p) {
                        int64_t slot = (rb * NC + c) * L + s;
                        idx[slot] = (uint16_t)b;
                        for (int t = 0; t < n; ++t)
                            copy_elem(dtype, values, slot * n + t, W, (rb * m + pos[p * n + t]) * ldw + c * L + b);
                        ++s;
                    }
            }
        }
    free(pos); free(mag); free(pat_of);
    return 0;
}

int oracle_nmg_densify(int n, int m, int g, int dtype, const void* values, const uint16_t* idx,
                       int64_t M, int64_t K, void* W_out, int64_t ldw)
{
    int rc = nmg_check(n, m, g, dtype, M, K);
    if (rc) return rc;
    if (ldw < K) return 2;
    const int C = nmg_binom(m, n);
    const int64_t L = (int64_t)C * g, NC = K / L, RB = M / m;
    int32_t* pos = (int32_t*)malloc(sizeof(int32_t) * (size_t)C * n);
    oracle_nmg_patterns(n, m, pos);
    for (int64_t r = 0; r < M; ++r)
        for (int64_t k = 0; k < K; ++k) zero_elem(dtype, W_out, r * ldw + k);
    for (int64_t rb = 0; rb < RB; ++rb)
        for (int64_t c = 0; c < NC; ++c)
            for (int64_t s = 0; s < L; ++s) {
                int64_t slot = (rb * NC + c) * L + s;
                int p = (int)(s / g);
                for (int t = 0; t < n; ++t)
                    copy_elem(dtype, W_out, (rb * m + pos[p * n + t]) * ldw + c * L + idx[slot], values, slot * n + t);
            }
    free(pos);
    return 0;
}

/* C[r][c] = sum over chunks, slots, kept t (fp64, storage order); Bound = sum |v||b|. */
int oracle_nmg_spmm(int n, int m, int g, int dtype, const void* values, const uint16_t* idx,
                    int64_t M, int64_t K, const void* B, int64_t ldb, int64_t N,
                    double* Cout, double* Bound, int nthreads)
{
    int rc = nmg_check(n, m, g, dtype, M, K);
    if (rc) return rc;
    if (ldb < N) return 2;
    const int C = nmg_binom(m, n);
    const int64_t L = (int64_t)C * g, NC = K / L, RB = M / m;
    int32_t* pos = (int32_t*)malloc(sizeof(int32_t) * (size_t)C * n);
    oracle_nmg_patterns(n, m, pos);
    for (int64_t i = 0; i < M * N; ++i) { Cout[i] = 0.0; if (Bound) Bound[i] = 0.0; }
#ifdef _OPENMP
    if (nthreads < 1) nthreads = 1;
#pragma omp parallel for num_threads(nthreads) schedule(dynamic, 1)
#endif
    for (int64_t rb = 0; rb < RB; ++rb)
        for (int64_t c = 0; c < NC; ++c)
            for (int64_t s = 0; s < L; ++s) {
                int64_t slot = (rb * NC + c) * L + s;
                int64_t k = c * L + idx[slot];
                int p = (int)(s / g);
                for (int t = 0; t < n; ++t) {
                    int64_t r = rb * m + pos[p * n + t];
                    double v = (double)widen(dtype, values, slot * n + t);
                    for (int64_t col = 0; col < N; ++col) {
                        double b = (double)widen(dtype, B, k * ldb + col);
                        Cout[r * N + col] += v * b;
                        if (Bound) Bound[r * N + col] += fabs(v) * fabs(b);
                    }
                }
            }
    free(pos);
    return 0;
}

/* SameFormat re-sparsification (NEXT-2): re-pack a new dense W' with an EXISTING grouped n:m
 * pattern -- "The new tensor is sparsified using the SameFormatSparsifier to maintain the same
 * format it had before" (the fixed-pattern fast path):
 *   values[r][kb*n+t] = W'[r][kb*m + idx[r/g][kb][t]]                                      */
int oracle_same_format(int n, int m, int g, int dtype, const void* W, int64_t M, int64_t K, int64_t ldw,
                       const uint8_t* idx, void* values)
{
    int rc = check_args(n, m, g, dtype, M, K);
    if (rc) return rc;
    if (ldw < K) return 2;
    int64_t KB = K / m, Kp = KB * n;
    for (int64_t r = 0; r < M; ++r)
        for (int64_t kb = 0; kb < KB; ++kb)
            for (int t = 0; t < n; ++t) {
                int j = idx[((r / g) * KB + kb) * n + t];
                copy_elem(dtype, values, r * Kp + kb * n + t, W, r * ldw + kb * m + j);
            }
    return 0;
}


/* NEXT-2 masked linear, weight gradient in the grouped n:m format (the "(KeepAll, FixedMaskTensor)"
 * gradient of PAPER.md:606-617; the masked-dense training path of PAPER.md:584-621): for the product
 * C = densify(values, idx) x B, the gradient of a loss with dL/dC = G [M][N] w.r.t. the stored values
 * is dV[r][kb*n+t] = sum_c G[r][c] * B[kb*m + idx[r/g][kb][t]][c] -- the dense G B^T sampled at the
 * kept positions (SDDMM).  Summed in fp64 in ascending c; Bound = sum |G| |B|. */
int oracle_sddmm(int n, int m, int g, int dtype, const void* Gm, int64_t M, int64_t N, const void* B,
                 int64_t K, const uint8_t* idx, double* dV, double* Bound, int nthreads)
{
    int rc = check_args(n, m, g, dtype, M, K);
    if (rc) return rc;
    if (N < 0) return 2;
    int64_t KB = K / m, Kp = KB * n;
#ifdef _OPENMP
    if (nthreads < 1) nthreads = 1;
#pragma omp parallel for num_threads(nthreads) schedule(dynamic, 1)
#endif
    for (int64_t r = 0; r < M; ++r)
        for (int64_t kb = 0; kb < KB; ++kb)
            for (int t = 0; t < n; ++t) {
                int64_t k = kb * m + idx[((r / g) * KB + kb) * n + t];
                double acc = 0.0, bound = 0.0;
                for (int64_t c = 0; c < N; ++c) {
                    double x = (double)widen(dtype, Gm, r * N + c), y = (double)widen(dtype, B, k * N + c);
                    acc += x * y;
                    bound += fabs(x) * fabs(y);
                }
                dV[r * Kp + kb * n + t] = acc;
                if (Bound) Bound[r * Kp + kb * n + t] = bound;
            }
    return 0;
}

/* NEXT-2 fixed-mask fast path ("we avoid unnecessary conversions when the nonzero
 * locations of the initial and replacement tensors match"): the SameFormat values of a new dense W
 * at the existing pattern idx, and the number of nonzero entries of W OUTSIDE that pattern (0 <=> the
 * nonzero locations match, so the re-pack is the whole conversion). */
int oracle_mask_check(int n, int m, int g, int dtype, const void* W, int64_t M, int64_t K, int64_t ldw,
                      const uint8_t* idx, void* values, int64_t* outside)
{
    int rc = oracle_same_format(n, m, g, dtype, W, M, K, ldw, idx, values);
    if (rc) return rc;
    int64_t KB = K / m, cnt = 0;
    for (int64_t r = 0; r < M; ++r)
        for (int64_t kb = 0; kb < KB; ++kb)
            for (int j = 0; j < m; ++j) {
                int kept = 0;
                for (int t = 0; t < n; ++t) kept |= idx[((r / g) * KB + kb) * n + t] == j;
                if (!kept && widen(dtype, W, r * ldw + kb * m + j) != 0.0f) ++cnt;
            }
    *outside = cnt;
    return 0;
}
