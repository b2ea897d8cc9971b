/*
 * sten.h -- C ABI of the B200-native grouped n:m hot path of STen
 * (arXiv 2304.07613, Sec. 5 "Grouped n:m Sparsity").
 *
 * The library (paper_2304_07613_b200/libsten.so) exports exactly the
 * functions declared here.  No torch / CUDA types appear in the signatures:
 * a stream is passed as an opaque `void*` holding a cudaStream_t (NULL = the
 * legacy default stream).
 *
 * ---------------------------------------------------------------------------
 * The layout (reading (A) "free grouping", R1/R2):
 *   W  is M x K (M = output features = group axis, K = input features =
 *      sparse / contraction axis).  K is cut into K/m blocks of m consecutive
 *      elements ("each group of m elements has n nonzeros").
 *   g consecutive rows form a group that shares ONE n-of-m pattern per block
 *   ("each nonzero pattern is repeated g times, forming a group",
 *   PAPER.md:518).  Kept positions maximise the L1 norm of the kept entries
 *   (PAPER.md:548-549): per (group, block) the n positions with the largest
 *   score s[j] = sum_{i<g} |w[group*g+i][block*m+j]| are kept.
 *
 *   values [M][K/m*n]       row-major, element type = the W dtype;
 *                           values[r][kb*n+t] = W[r][kb*m + idx[r/g][kb][t]]
 *   idx    [M/g][K/m][n]    uint8, in-block positions, strictly ascending
 *
 * Arithmetic contract (R4, R5, R10):
 *   - scores are fp32 sums of |w| over the group's rows in ascending row
 *     order, round-to-nearest-even, no contraction; bf16 inputs are widened
 *     exactly; ties go to the lower in-block position;
 *   - exactly n entries are stored per (row, block), even if some are zero;
 *   - SpMM accumulates in fp32; the per-column summation order depends only
 *     on (M, K, n, m, g) and the plan, never on N or on the column tiling, so
 *     a column-sharded product equals the unsharded one bit for bit when both
 *     use the same plan (sten_spmm_plan_query on the global shape).
 *
 * Conventions for every entry point:
 *   - Pointers are DEVICE pointers of the current device unless the name ends
 *     in _host.  The caller allocates every buffer; the library allocates no
 *     persistent memory, keeps no global state and is safe to call
 *     concurrently on different streams / devices.
 *   - Work is enqueued asynchronously on `stream` (except the _host calls,
 *     which return after the stream has drained).
 *   - Argument errors are detected synchronously BEFORE any launch, so an
 *     error return leaves every output untouched:
 *        NULL pointer, n/m/g out of range, unknown dtype  -> STEN_ERR_INVALID_ARG
 *        M % g != 0, K % m != 0, ld < extent, negative size -> STEN_ERR_SHAPE
 *        no compiled variant / misaligned vector pointer or ld
 *          (16-byte base alignment; fp32 ld % 4, bf16 ld % 8)  -> STEN_ERR_UNSUPPORTED
 *        a CUDA launch / copy error                        -> STEN_ERR_CUDA
 *     There is no CPU fallback: without a usable device the calls fail.
 *   - Outputs must not overlap inputs.
 *   - Supported formats: 1 <= n < m <= 16 with m in {2,4,6,8,10,12,16};
 *     any g >= 1 with g | M.  Empty problems (M, K or N == 0) are valid
 *     no-ops apart from zero-filling outputs whose value is defined
 *     (C = 0 when K == 0).
 */
#ifndef STEN_H_
#define STEN_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    STEN_OK = 0,
    STEN_ERR_INVALID_ARG = 1,
    STEN_ERR_SHAPE = 2,
    STEN_ERR_UNSUPPORTED = 3,
    STEN_ERR_CUDA = 4
} sten_status;

typedef enum { STEN_F32 = 0, STEN_BF16 = 1 } sten_dtype;

/* n kept of every m consecutive K elements; g rows per group. */
typedef struct { int32_t n, m, g; } sten_nmg;

/* SpMM kernel families (sten_spmm_plan.algo). */
typedef enum {
    STEN_ALGO_AUTO = 0,       /* library chooses                                    */
    STEN_ALGO_SIMT = 1,       /* CUDA-core FFMA, fp32 accumulate (fp32 or bf16 in)  */
    STEN_ALGO_MMA_SYNC = 2,   /* bf16 warp-level mma.sync on gathered rows          */
    STEN_ALGO_TCGEN05 = 3     /* bf16 tcgen05 / TMEM on gathered dense sub-tiles    */
} sten_algo;

/* Execution plan of one SpMM.  split_k = number of K partitions reduced in a
 * fixed order (1 = none); tile = kernel tile variant of the algorithm (0 =
 * library choice; see DESIGN.md for the table).  Fields are filled by
 * sten_spmm_plan_query; a caller may override them (a value out of range or a
 * variant not compiled for this g -> STEN_ERR_UNSUPPORTED). */
typedef struct {
    int32_t algo;
    int32_t split_k;
    int32_t tile;
    int32_t reserved[5];
} sten_spmm_plan;

/* a1-a3: magnitude sparsifier dense -> grouped n:m.
 *   W      [M][ldw] dtype dt, K <= ldw                      (input)
 *   values [M][K/m*n] dtype dt                              (output, overwritten)
 *   idx    [M/g][K/m][n] uint8                              (output, overwritten) */
sten_status sten_sparsify_grouped_nm(sten_nmg f, sten_dtype dt,
                                     const void* W, int64_t M, int64_t K, int64_t ldw,
                                     void* values, uint8_t* idx, void* stream);

/* Grouped sparsify: the weights of one step in ONE launch whatever their (n, m, g) (e.g. the 9 C2
 * weights of three sparsity classes), each CTA working on one problem exactly as
 * sten_sparsify_grouped_nm does (same bits).  All problems share dt.
 * count in [1, 12]; every problem is validated before any launch (errors as the single call). */
typedef struct {
    sten_nmg f;
    int32_t reserved;
    const void* W;          /* [M][ldw]          */
    int64_t M, K, ldw;
    void* values;           /* [M][K/m*n]        */
    uint8_t* idx;           /* [M/g][K/m][n]     */
} sten_sparsify_problem;
sten_status sten_sparsify_grouped_nm_batched(int32_t count, const sten_sparsify_problem* problems,
                                             sten_dtype dt, void* stream);

/* NEXT-2 SameFormat re-sparsification: re-pack a new dense W
 * [M][ldw] (e.g. the weights after an optimizer step) with an EXISTING pattern idx, so the
 * format stays fixed: values[r][kb*n+t] = W[r][kb*m + idx[r/g][kb][t]] (bit copies).
 *   idx    [M/g][K/m][n] uint8 (input, as produced by sten_sparsify_grouped_nm)
 *   values [M][K/m*n] dtype dt (output, overwritten)
 * idx entries must be < m (not checked on the device). */
sten_status sten_resparsify_same_format(sten_nmg f, sten_dtype dt,
                                        const void* W, int64_t M, int64_t K, int64_t ldw,
                                        const uint8_t* idx, void* values, void* stream);

/* NEXT-3 fused epilogue with a residual (a BERT encoder's x + Linear(x)):
 *   C = act(densify(values, idx) x B + bias[row]) + R[row][col]
 * bias [M] fp32 or NULL, act 0 none / 1 GELU (erf) / 2 ReLU, R [M][ldr] of c_dt or NULL (must not
 * alias C).  The SIMT kernel's epilogue (plan algo AUTO/SIMT); otherwise as
 * sten_spmm_grouped_nm_bias_act. */
sten_status sten_spmm_grouped_nm_epilogue(sten_nmg f, sten_dtype ab_dt,
                                          const void* values, const uint8_t* idx, int64_t M, int64_t K,
                                          const void* B, int64_t ldb, int64_t N,
                                          void* C, int64_t ldc, sten_dtype c_dt,
                                          const float* bias, int32_t act, const void* residual, int64_t ldr,
                                          const sten_spmm_plan* plan, void* stream);

/* NEXT-2 fixed-mask fast path ("we avoid unnecessary conversions when the
 * nonzero locations of the initial and replacement tensors match"): the SameFormat re-pack of a
 * new dense W at the existing pattern idx (values as sten_resparsify_same_format) AND, in the same
 * pass, *outside = the number of nonzero entries of W at pruned positions (device int64, 8-byte
 * aligned; set by the call).  *outside == 0 <=> the nonzero locations match and the re-pack is the
 * whole conversion; otherwise the caller re-sparsifies.  outside may be NULL (plain SameFormat). */
sten_status sten_mask_check_repack(sten_nmg f, sten_dtype dt,
                                   const void* W, int64_t M, int64_t K, int64_t ldw,
                                   const uint8_t* idx, void* values, int64_t* outside, void* stream);

/* NEXT-2 masked linear, weight gradient in the grouped n:m format (SDDMM; the
 * "(KeepAll, FixedMaskTensor)" gradient of PAPER.md:606-617): for C = densify(values, idx) x B
 * and G = dL/dC,
 *     dV[r][kb*n+t] = sum_c G[r][c] * B[kb*m + idx[r/g][kb][t]][c]
 *   G [M][ldg] ab_dt, B [K][ldb] ab_dt (N columns each), idx [M/g][K/m][n],
 *   dV [M][K/m*n] c_dt (overwritten; the values layout).
 * fp32 accumulation, deterministic order; G, B bases and rows 16-byte
 * aligned (else STEN_ERR_UNSUPPORTED).  Other errors as the SpMM. */
sten_status sten_sddmm_grouped_nm(sten_nmg f, sten_dtype ab_dt,
                                  const void* G, int64_t M, int64_t N, int64_t ldg,
                                  const void* B, int64_t K, int64_t ldb, const uint8_t* idx,
                                  void* dV, sten_dtype c_dt, void* stream);

/* a4: grouped n:m -> dense.  W_out [M][ldw] receives zeros at
 * pruned positions and the stored values at kept ones (columns >= K untouched). */
sten_status sten_densify(sten_nmg f, sten_dtype dt,
                         const void* values, const uint8_t* idx, int64_t M, int64_t K,
                         void* W_out, int64_t ldw, void* stream);

/* a5-a7 (Fig. 5): C = densify(values, idx) x B.
 *   values/idx as produced by sten_sparsify_grouped_nm, element type ab_dt
 *   B [K][ldb] ab_dt, N <= ldb       C [M][ldc] c_dt, N <= ldc, overwritten (beta = 0) */
sten_status sten_spmm_grouped_nm(sten_nmg f, sten_dtype ab_dt,
                                 const void* values, const uint8_t* idx, int64_t M, int64_t K,
                                 const void* B, int64_t ldb, int64_t N,
                                 void* C, int64_t ldc, sten_dtype c_dt, void* stream);

/* SpMM with the all-gather of C fused into the epilogue (token sharding):
 * this rank computes C_loc = densify(values, idx) x B for its N token columns and the kernel's
 * epilogue stores every C tile straight into each of the `npeers` gathered output buffers
 * C_peers[p] ([M][ldc], c_dt; peer-mapped device pointers -- CUDA IPC / symmetric memory over
 * NVLink, or local buffers) at columns [col0, col0 + N): one kernel does the product and the
 * exchange, the transfer overlapping the math tile by tile.  C_peers is a HOST array of
 * 1..8 device pointers.  Completion on the other ranks needs a cross-rank barrier after the
 * kernel (the caller's).  The fused epilogue is the SIMT kernel's (plan NULL / AUTO -> SIMT;
 * another algo -> STEN_ERR_UNSUPPORTED); the column order of the sum does not depend on N, so
 * the gathered buffer equals the single-GPU product bit for bit with the global plan. */
sten_status sten_spmm_grouped_nm_allgather(sten_nmg f, sten_dtype ab_dt,
                                           const void* values, const uint8_t* idx, int64_t M, int64_t K,
                                           const void* B, int64_t ldb, int64_t N,
                                           void* const* C_peers, int32_t npeers, int64_t col0, int64_t ldc,
                                           sten_dtype c_dt, const sten_spmm_plan* plan, void* stream);

/* NEXT-3 epilogue fusion (the BERT FFN1 pattern): C = act(densify(values, idx) x B
 * + bias) computed in the SpMM's fp32 epilogue (after the split-K reduction) before the store.
 *   bias [M] fp32 device pointer or NULL (bias of output feature r, added to row r of C)
 *   act  0 = none, 1 = GELU x/2 (1 + erf(x / sqrt 2)), 2 = ReLU; other -> STEN_ERR_INVALID_ARG
 * The fused epilogue is the SIMT kernel's (plan NULL / AUTO -> SIMT; another algo ->
 * STEN_ERR_UNSUPPORTED); arguments otherwise as sten_spmm_grouped_nm_ex. */
sten_status sten_spmm_grouped_nm_bias_act(sten_nmg f, sten_dtype ab_dt,
                                          const void* values, const uint8_t* idx, int64_t M, int64_t K,
                                          const void* B, int64_t ldb, int64_t N,
                                          void* C, int64_t ldc, sten_dtype c_dt,
                                          const float* bias, int32_t act,
                                          const sten_spmm_plan* plan, void* stream);

/* Grouped launch of independent fp32 problems (e.g. the linears of a step): ONE kernel launch
 * whose CTAs each run one whole-K output tile of one problem (cuBLAS-grouped-GEMM style; no
 * split-K, no cluster), the problems ordered longest-K first.  Every problem: fp32 values / B /
 * C, arguments and layout as sten_spmm_grouped_nm; all problems must map to the same SIMT
 * variant (the same row-group class: g % 8 == 0, g % 4 == 0, g % 2 == 0 or odd) else
 * STEN_ERR_UNSUPPORTED.  count in 1..12; tile 0/1 (8 warps, 56 x 256) or 2 (16 warps,
 * 120 x 256).  Results equal sten_spmm_grouped_nm_ex with the same tile and split_k = 1. */
typedef struct {
    sten_nmg f;
    int32_t reserved;
    const void* values;
    const uint8_t* idx;
    int64_t M, K;
    const void* B;
    int64_t ldb, N;
    void* C;
    int64_t ldc;
} sten_spmm_problem;
sten_status sten_spmm_grouped_nm_batched(int32_t count, const sten_spmm_problem* problems, int32_t tile,
                                         void* stream);

/* Grouped launch WITH per-problem split-K (the whole step of independent SpMMs in one launch).
 * splits[p] (NULL or 0 = automatic: every problem's K is cut so that the units of all problems
 * carry about the same work, ~3 units per resident CTA) splits problem p's m-blocks into S_p
 * balanced parts of whole slabs; the S_p parts of an output tile park fp32 partials in the
 * workspace and the last part to arrive adds them in the fixed order z = 0..S_p-1 (the cluster
 * reduction's order: the same bits as sten_spmm_grouped_nm_ex with plan {SIMT, S_p, tile}).
 * workspace: caller-allocated, >= sten_spmm_batched_workspace_size bytes, 16-byte aligned; it
 * starts with one counter per split tile that MUST be zero before the first call (memset the
 * buffer once after allocating it); every call leaves them at zero.  Calls sharing a workspace
 * must be stream-ordered.  tile: 1 / 2 / 3 = that SIMT tile for every problem; 0 = per problem (the
 * 240-row x 128-token tile 3, whose K-slabs are 3x longer, for m >= 8 n; the 120 x 256 tile 2
 * otherwise -- both in ONE launch).  Other arguments and errors as sten_spmm_grouped_nm_batched; a
 * workspace smaller than needed -> STEN_ERR_SHAPE, NULL while needed -> STEN_ERR_INVALID_ARG. */
sten_status sten_spmm_grouped_nm_batched_ex(int32_t count, const sten_spmm_problem* problems,
                                            const int32_t* splits, int32_t tile,
                                            void* workspace, int64_t workspace_bytes, void* stream);
sten_status sten_spmm_batched_workspace_size(int32_t count, const sten_spmm_problem* problems,
                                             const int32_t* splits, int32_t tile, int64_t* bytes);

/* The plan sten_spmm_grouped_nm would use for this problem. */
sten_status sten_spmm_plan_query(sten_nmg f, sten_dtype ab_dt, int64_t M, int64_t K, int64_t N,
                                 sten_dtype c_dt, sten_spmm_plan* plan);

/* sten_spmm_grouped_nm with an explicit plan (NULL = AUTO). */
sten_status sten_spmm_grouped_nm_ex(sten_nmg f, sten_dtype ab_dt,
                                    const void* values, const uint8_t* idx, int64_t M, int64_t K,
                                    const void* B, int64_t ldb, int64_t N,
                                    void* C, int64_t ldc, sten_dtype c_dt,
                                    const sten_spmm_plan* plan, void* stream);

/* Measured plan choice for one SpMM shape (the on-device analogue of a GEMM
 * library's heuristic + benchmark mode).  Runs every compiled variant that
 * accepts the arguments -- SIMT tiles x split-K, and for bf16 the mma.sync
 * tiles x split-K and the tcgen05 row blocks -- `reps` timed times each on
 * `stream` (CUDA events; one untimed launch first) and writes the fastest
 * (minimum time) to *best (the AUTO plan is always a candidate, so the result
 * is never slower than AUTO on the measured launches).  Arguments are those of
 * sten_spmm_grouped_nm_ex; C is scratch while tuning (its final contents are
 * the product computed with the last candidate).  Synchronises `stream`.
 * reps < 1 -> STEN_ERR_INVALID_ARG; argument errors as for the SpMM. */
sten_status sten_spmm_autotune(sten_nmg f, sten_dtype ab_dt,
                               const void* values, const uint8_t* idx, int64_t M, int64_t K,
                               const void* B, int64_t ldb, int64_t N,
                               void* C, int64_t ldc, sten_dtype c_dt,
                               int32_t reps, void* stream, sten_spmm_plan* best);

/* End-to-end sparse linear layer with HOST input/output buffers: copies
 * W_host [M][ldw] and B_host [K][ldb] to the device, sparsifies W, multiplies,
 * copies C back to C_host [M][ldc] and waits for the stream.  Host buffers
 * should be pinned (cudaHostAlloc / torch pin_memory) for asynchronous copies.
 * `workspace` is a device buffer of at least
 * sten_sparse_linear_host_workspace_size(...) bytes (16-byte aligned). */
int64_t sten_sparse_linear_host_workspace_size(sten_nmg f, sten_dtype ab_dt, int64_t M,
                                               int64_t K, int64_t N, sten_dtype c_dt);
sten_status sten_sparse_linear_host(sten_nmg f, sten_dtype ab_dt,
                                    const void* W_host, int64_t M, int64_t K, int64_t ldw,
                                    const void* B_host, int64_t ldb, int64_t N,
                                    void* C_host, int64_t ldc, sten_dtype c_dt,
                                    void* workspace, int64_t workspace_bytes, void* stream);

/* ---------------------------------------------------------------------------
 * Chunked n:m:g -- the paper's own format (
 * DESIGN.md readings R17-R21).
 *
 *   A "column" is one block of m consecutive ROWS of W at one input column k
 *   (the m-blocks run along the output rows M); a chunk is L = C(m,n) g
 *   consecutive columns k of one row block.  Every one of the C(m,n) nonzero
 *   patterns is used by exactly g columns of a chunk ("each nonzero pattern is
 *   repeated g times, forming a group ... chunks with all C(m,n) combinations
 *   of nonzeros in fixed order").  The fixed order is the
 *   revolving-door order (adjacent patterns differ in one position).
 *   Columns are reordered inside the chunk: slot s holds a column of pattern
 *   s / g, the g columns of a pattern in ascending original position, and idx
 *   stores each slot's original column offset in the chunk.
 *
 *   values [M/m][K/L][L][n]  dtype dt; values[rb][c][s][t] = W[rb m + pos_t(s/g)][c L + idx[rb][c][s]]
 *   idx    [M/m][K/L][L]     uint16
 *
 *   Conversion = the paper's CPU greedy, computed exactly on
 *   the GPU: the C(m,n)^2 g (column, pattern) magnitudes of a chunk (fp32 sums of
 *   |w| over the pattern's positions, ascending) processed from highest to lowest
 *   (ties: lower column, then lower pattern id), a column taking a pattern if
 *   it is unassigned and the pattern has < g columns.
 *
 *   Shapes: M % m == 0 and K % L == 0 (else STEN_ERR_SHAPE; the caller pads);
 *   1 <= n < m <= 16, C(m,n) <= 64 and L * C(m,n) <= 2048 (else
 *   STEN_ERR_UNSUPPORTED).  The SpMM is compiled for (n, m) in {1:2, 1:4, 2:4,
 *   1:8, 3:6, 2:8, 1:10} and fp32 / bf16 inputs (fp32 accumulate); other formats
 *   convert and densify but their product returns STEN_ERR_UNSUPPORTED.  Pointers, streams,
 *   ownership and error behaviour as for the grouped n:m calls above.
 * --------------------------------------------------------------------------- */
sten_status sten_nmg_sparsify(sten_nmg f, sten_dtype dt,
                              const void* W, int64_t M, int64_t K, int64_t ldw,
                              void* values, uint16_t* idx, void* stream);

/* sten_nmg_sparsify with a choice of conversion algorithm:
 *   method 0  the CPU greedy above (= sten_nmg_sparsify);
 *   method 1  the paper's GPU conversion: columns start with an arbitrary
 *             assignment (column b -> pattern b / g), then pairs of columns holding different
 *             patterns swap them whenever that raises the pair's magnitude, until a pass makes
 *             no swap; the swaps follow the sequential order of DESIGN.md R22 (pairs (i, j),
 *             i < j ascending; the two-term sums compared in fp64), so the result is deterministic
 *             and equals the oracle's;
 *   method 2  the greedy, refined by the same exchange passes (never lower L1 than the greedy).
 * Layout, shapes and errors as sten_nmg_sparsify; method out of range -> STEN_ERR_INVALID_ARG. */
sten_status sten_nmg_sparsify_ex(sten_nmg f, sten_dtype dt,
                                 const void* W, int64_t M, int64_t K, int64_t ldw,
                                 void* values, uint16_t* idx, int32_t method, void* stream);

/* to dense: W_out [M][ldw], zeros at pruned positions. */
sten_status sten_nmg_densify(sten_nmg f, sten_dtype dt,
                             const void* values, const uint16_t* idx, int64_t M, int64_t K,
                             void* W_out, int64_t ldw, void* stream);

/* C = densify(values, idx) x B (Fig. 5): B [K][ldb] ab_dt,
 * C [M][ldc] c_dt, overwritten.  B base and ldb 16-byte aligned. */
sten_status sten_nmg_spmm(sten_nmg f, sten_dtype ab_dt,
                          const void* values, const uint16_t* idx, int64_t M, int64_t K,
                          const void* B, int64_t ldb, int64_t N,
                          void* C, int64_t ldc, sten_dtype c_dt, void* stream);

/* sten_sparse_linear_host without the final wait: the copies and kernels are only enqueued
 * on `stream` (host buffers must be pinned and stay valid, and C_host is written, when the
 * stream reaches the D2H copy); the caller synchronises.  Calls on different streams overlap
 * their PCIe copies with each other's kernels. */
sten_status sten_sparse_linear_host_async(sten_nmg f, sten_dtype ab_dt,
                                          const void* W_host, int64_t M, int64_t K, int64_t ldw,
                                          const void* B_host, int64_t ldb, int64_t N,
                                          void* C_host, int64_t ldc, sten_dtype c_dt,
                                          void* workspace, int64_t workspace_bytes, void* stream);

/* Several independent linears from host memory, pipelined over three caller streams: every
 * problem's H2D copies (W, B) are issued back to back on `copy_in`, its sparsify + SpMM on
 * `compute` as soon as its inputs have landed, and its D2H copy of C on `copy_out` as soon as C is
 * ready -- so the host link carries H2D and D2H at the same time and the kernels hide under the
 * copies (the step costs ~ the H2D bytes at the link's rate plus the LAST problem's kernels and D2H;
 * put a small problem last).  Per problem: host buffers pinned and valid until copy_out drains,
 * its own `workspace` (sten_sparse_linear_host_workspace_size bytes), the same arithmetic and
 * bits as sten_sparse_linear_host_async.  The three streams start after whatever the caller
 * ordered before them; the caller joins copy_out (and compute) before reading C_host.  The call
 * creates one event per problem and stage and releases it before returning (no state kept).
 * count in [1, 64]; every problem is validated before anything is enqueued. */
typedef struct {
    sten_nmg f;
    int32_t reserved;
    const void* W_host;     /* [M][ldw] ab_dt */
    int64_t M, K, ldw;
    const void* B_host;     /* [K][ldb] ab_dt */
    int64_t ldb, N;
    void* C_host;           /* [M][ldc] c_dt */
    int64_t ldc;
    void* workspace;        /* device */
    int64_t workspace_bytes;
} sten_host_linear_problem;
sten_status sten_sparse_linear_host_pipelined_async(int32_t count, const sten_host_linear_problem* problems,
                                                    sten_dtype ab_dt, sten_dtype c_dt, void* copy_in,
                                                    void* compute, void* copy_out);

/* ---------------------------------------------------------------------------
 * K6: the 2:4 structured-sparse tensor-core path (NEXT-4; bf16 in, fp32 accumulate).
 *
 * Every grouped n:m mask with n == 1 (any m) or n == 2 and 4 | m is also a 2:4
 * mask on the aligned 4-windows of K (a 4-window meets at most two m-blocks for
 * n = 1 and lies inside one block when 4 | m), so C = densify(values, idx) x B
 * runs on tcgen05.mma.sp with the weight as the compressed
 * A operand.  The group structure is carried by idx; any g | M.
 *
 * Packed operand (caller-allocated, sizes from sten_sp24_packed_size):
 *   v24  [M128][K128/2] bf16: per row, 2 stored values per 4-window of K in
 *        ascending position (an explicit 0 where the window keeps < 2 entries);
 *        M128 / K128 = M / K rounded up to 128, padding rows/windows are 0.
 *   meta [M128/128][K128/128][128][4] uint32: the 2-bit in-window positions,
 *        one 32-bit word per (128-row block, 32 logical k, TMEM lane) in the
 *        tensor-memory lane layout of the sparse MMA:
 *        row r, 4-window j of the 32 -> lane r%8 + 16(r/16) + 8(j/4),
 *        nibble j%4 + 4((r/8)%2); nibble = pos0 | pos1 << 2, pos0 < pos1.
 * Formats: n == 1, or n == 2 with m % 4 == 0 (else STEN_ERR_UNSUPPORTED).
 * --------------------------------------------------------------------------- */
sten_status sten_sp24_packed_size(sten_nmg f, int64_t M, int64_t K,
                                  int64_t* v24_bytes, int64_t* meta_bytes);

/* (values, idx) of sten_sparsify_grouped_nm (bf16) -> (v24, meta).  A layout
 * conversion (bit copies of the kept values), HBM-bound; v24 / meta 4-byte aligned. */
sten_status sten_sp24_pack(sten_nmg f, sten_dtype dt, const void* values, const uint8_t* idx,
                           int64_t M, int64_t K, void* v24, uint32_t* meta, void* stream);

/* C [M][ldc] (c_dt, overwritten) = densify(values, idx) x B, B [K][ldb] bf16
 * (B base, v24 and meta 16-byte aligned, ldb % 8 == 0).  tile: 0 = default
 * (6 when K >= 2048, else 1), 1 = 256 rows x 192 tokens, 2 = 256 x 128,
 * 3 = 384 x 128, 4 = 128 x 256, 5 = 128 x 128 (one CTA per SM, persistent),
 * 6 = a CTA pair on two SMs (tcgen05 cta_group::2, 256 x 256 per pair).  fp32 accumulation in TMEM over
 * K in ascending 32-k steps (independent of N and the token tiling). */
sten_status sten_spmm_sp24(const void* v24, const uint32_t* meta, int64_t M, int64_t K,
                           const void* B, int64_t ldb, int64_t N,
                           void* C, int64_t ldc, sten_dtype c_dt, int32_t tile, void* stream);

/* sten_spmm_sp24 with the fused epilogue of NEXT-3 (a transformer linear on the tensor cores):
 *   C = act(densify(values, idx) x B + bias[row]) + R[row][col]
 * bias [M] fp32 or NULL, act 0 none / 1 GELU (erf) / 2 ReLU, R [M][ldr] of c_dt or NULL (must not
 * alias C; ldr >= N).  Applied to the fp32 accumulators after the TMEM read, before the store. */
sten_status sten_spmm_sp24_epilogue(const void* v24, const uint32_t* meta, int64_t M, int64_t K,
                                    const void* B, int64_t ldb, int64_t N,
                                    void* C, int64_t ldc, sten_dtype c_dt,
                                    const float* bias, int32_t act, const void* residual, int64_t ldr,
                                    int32_t tile, void* stream);

const char* sten_status_string(sten_status s);
const char* sten_algo_name(int32_t algo);
/* Number of kernel launches the last call of each entry point enqueues is
 * deterministic; this returns the count for one sten_spmm_grouped_nm_ex call
 * with `plan` (used by bench.py's gpu_launches accounting). */
int32_t sten_spmm_launch_count(const sten_spmm_plan* plan);
int32_t sten_version(void);

#ifdef __cplusplus
}
#endif

#endif /* STEN_H_ */
