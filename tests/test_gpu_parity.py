"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle (-m gpu).

Bars (BASELINE.json north_star):
  * idx and values: bit-exact;  densify: bit-exact;
  * C (fp32 in, fp32 out): max_{r,c} |C - C_ref| / Bound[r,c] <= 1e-5,
    Bound = sum |v| |b| (fp64, from the oracle);
  * C (bf16 in):          same metric <= 2e-2;
  * integer-valued inputs (P7) and B = I (P8): bit-exact on every path;
  * column-sharded == unsharded (P11): bit-exact with the same plan.
"""
import numpy as np
import pytest
import torch

import oracle
import synthetic
from paper_2304_07613_b200 import sten

pytestmark = pytest.mark.gpu

NM_SET = [(1, 2), (2, 4), (1, 4), (2, 8), (1, 8), (1, 10), (1, 12), (3, 6), (4, 16)]
TOL = {"f32": 1e-5, "bf16": 2e-2}


def dev(x: np.ndarray, dtype: str, ld_multiple: int = 8) -> torch.Tensor:
    """Device copy of a 2-D host array whose leading dimension is padded to a
    multiple of `ld_multiple` elements (the ABI wants 16-byte aligned rows);
    returns the [rows][cols] view."""
    x = np.ascontiguousarray(x)
    rows, cols = x.shape
    ld = -(-cols // ld_multiple) * ld_multiple if cols else ld_multiple
    if dtype == "bf16":
        t = torch.zeros((rows, ld), dtype=torch.bfloat16)
        t[:, :cols] = torch.from_numpy(x.view(np.int16)).view(torch.bfloat16)
    else:
        t = torch.zeros((rows, ld), dtype=torch.float32)
        t[:, :cols] = torch.from_numpy(x)
    return t.cuda()[:, :cols]


def host(t: torch.Tensor) -> np.ndarray:
    t = t.cpu()
    if t.dtype == torch.bfloat16:
        return t.view(torch.int16).numpy().view(np.uint16)
    return t.numpy()


def rel_err(C: torch.Tensor, C_ref: np.ndarray, Bound: np.ndarray) -> float:
    c = C.float().cpu().numpy().astype(np.float64)
    return float(np.max(np.abs(c - C_ref) / np.maximum(Bound, 1e-30))) if c.size else 0.0


def gpu_sparsify(W, n, m, g, dtype):
    v, i = sten.sparsify_grouped_nm(dev(W, dtype), n, m, g)
    torch.cuda.synchronize()
    return v, i


# ----------------------------------------------------------------------------------------
# K1 sparsify / K2 densify: bit-exact
# ----------------------------------------------------------------------------------------
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("n,m", NM_SET)
@pytest.mark.parametrize("g", [1, 3, 4, 16])
def test_sparsify_densify_bit_exact(dtype, n, m, g):
    M, K = 8 * g, 37 * m            # ragged: 37 blocks spans >1 warp, odd counts
    W = synthetic.weights(M, K, seed=n * 100 + m * 10 + g, dtype=dtype)
    if dtype == "f32":
        W[:g, :m] = 0.25                       # a tied block
    v_ref, i_ref = oracle.sparsify(W, n, m, g)
    v, i = gpu_sparsify(W, n, m, g, dtype)
    assert np.array_equal(host(i), i_ref)
    assert np.array_equal(host(v).view(np.uint8), v_ref.view(np.uint8))
    Wd = sten.densify(v, i, n, m, g, K)
    assert np.array_equal(host(Wd).view(np.uint8), oracle.densify(v_ref, i_ref, n, m, g, K).view(np.uint8))


def test_sparsify_unaligned_ld_and_integer_ties():
    n, m, g = 2, 4, 4
    W = synthetic.integer_matrix(16, 44, seed=3, lo=-2, hi=2)
    Wt = torch.from_numpy(np.pad(W, ((0, 0), (0, 1)))).cuda()[:, :44]   # ldw = 45: scalar path
    v, i = sten.sparsify_grouped_nm(Wt, n, m, g)
    v_ref, i_ref = oracle.sparsify(W, n, m, g)
    assert np.array_equal(host(i), i_ref) and np.array_equal(host(v), v_ref)
    assert np.array_equal(host(i), oracle.brute_select(W, n, m, g))


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("n,m", [(1, 8), (2, 8), (4, 8), (2, 4), (1, 16), (3, 6)])
@pytest.mark.parametrize("ld_multiple", [1, 4, 8, 16])
@pytest.mark.parametrize("out_offset", [0, 1])
def test_sparsify_load_and_store_paths(dtype, n, m, ld_multiple, out_offset):
    """Every load width (scalar / 16-byte / 256-bit, chosen by the W base and ldw) and both
    store forms (one vector store per row when values/idx bases allow n-element vectors, else
    per-position stores: out_offset = 1 misaligns both outputs) give the oracle's bytes."""
    g, M, K = 4, 24, 41 * m
    W = synthetic.weights(M, K, seed=7 * n + m + ld_multiple, dtype=dtype)
    Wt = dev(W, dtype, ld_multiple=ld_multiple)
    tdt = torch.float32 if dtype == "f32" else torch.bfloat16
    kept = K // m * n
    vbuf = torch.empty(M * kept + 1, dtype=tdt, device="cuda")
    ibuf = torch.empty((M // g) * (K // m) * n + 1, dtype=torch.uint8, device="cuda")
    v = vbuf[out_offset:out_offset + M * kept].view(M, kept)
    i = ibuf[out_offset:out_offset + (M // g) * (K // m) * n].view(M // g, K // m, n)
    sten.sparsify_grouped_nm(Wt, n, m, g, values=v, idx=i)
    torch.cuda.synchronize()
    v_ref, i_ref = oracle.sparsify(W, n, m, g)
    assert np.array_equal(host(i), i_ref)
    assert np.array_equal(host(v).view(np.uint8), v_ref.view(np.uint8))


def test_sparsify_large_group_and_fp32_near_ties():
    n, m, g = 1, 2, 3
    e = np.float32(2.0 ** -24)
    W = np.array([[1.0, 1.0 + 2.0 ** -23], [e, 0.0], [e, 0.0]], np.float32)
    _, i = gpu_sparsify(W, n, m, g, "f32")
    assert host(i).tolist() == [[[1]]]                  # fp32 score rule (reading R4)
    W = synthetic.weights(128, 64, seed=1)
    for g in (32, 64, 128):
        v_ref, i_ref = oracle.sparsify(W, 2, 4, g)
        v, i = gpu_sparsify(W, 2, 4, g, "f32")
        assert np.array_equal(host(i), i_ref) and np.array_equal(host(v), v_ref)


def test_p0_worked_example_on_gpu(golden_dir):
    import json, os
    ex = json.load(open(os.path.join(golden_dir, "p0_worked_example.json")))
    W = np.array(ex["W"], np.float32)
    v, i = gpu_sparsify(W, ex["n"], ex["m"], ex["g"], "f32")
    assert host(i).tolist() == ex["idx"] and host(v).tolist() == ex["values"]
    B = torch.tensor([[k + 1, 1] + [0, 0] for k in range(8)], dtype=torch.float32).cuda()  # ldb = 4
    C = sten.spmm_grouped_nm(v, i, B[:, :2], ex["n"], ex["m"], ex["g"])
    assert C.cpu().tolist() == ex["C"]


# ----------------------------------------------------------------------------------------
# SpMM parity on every algorithm / tile / split
# ----------------------------------------------------------------------------------------
SIMT_TILES = [1, 2, 3, 4, 5, 6, 7]


def _spmm_case(M, K, N, n, m, g, dtype, plan=None, out_dtype=None, seed=0):
    W = synthetic.weights(M, K, seed=seed + 1, dtype=dtype)
    B = synthetic.activations(K, N, seed=seed + 2, dtype=dtype)
    v_ref, i_ref = oracle.sparsify(W, n, m, g)
    C_ref, Bound = oracle.spmm(v_ref, i_ref, B, n, m, g, nthreads=oracle.max_threads())
    v, i = gpu_sparsify(W, n, m, g, dtype)
    C = sten.spmm_grouped_nm(v, i, dev(B, dtype), n, m, g, plan=plan, out_dtype=out_dtype)
    torch.cuda.synchronize()
    return C, C_ref, Bound


@pytest.mark.parametrize("tile", SIMT_TILES)
@pytest.mark.parametrize("g", [1, 2, 4, 8])
@pytest.mark.parametrize("split", [1, 3, 8])
@pytest.mark.parametrize("n,m", [(2, 4), (1, 10)])
def test_spmm_simt_f32(tile, g, split, n, m):
    plan = sten.make_plan(sten.ALGO_SIMT, split_k=split, tile=tile)
    # M not a multiple of the CTA rows, N ragged (not a multiple of 4*32), several K slabs;
    # 1:10 with K = 50 m-blocks gives K' = 50 (rows not 16-byte aligned: 4-byte staging path)
    C, C_ref, Bound = _spmm_case(M=40 * g if g < 8 else 24 * g, K=50 * m, N=301, n=n, m=m, g=g, dtype="f32",
                                 plan=plan, seed=tile * 10 + g)
    assert rel_err(C, C_ref, Bound) <= TOL["f32"]


@pytest.mark.parametrize("tile", [1, 2])
@pytest.mark.parametrize("split", [1, 4])
@pytest.mark.parametrize("n,m,K", [(2, 4, 256), (1, 10, 500), (1, 10, 520)])
def test_spmm_simt_bf16(tile, split, n, m, K):
    plan = sten.make_plan(sten.ALGO_SIMT, split_k=split, tile=tile)
    C, C_ref, Bound = _spmm_case(M=96, K=K, N=200, n=n, m=m, g=4, dtype="bf16", plan=plan,
                                 out_dtype=torch.float32, seed=tile + split)
    assert rel_err(C, C_ref, Bound) <= 1e-5


@pytest.mark.parametrize("n,m", NM_SET)
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_spmm_auto_all_formats(n, m, dtype):
    g = 4
    C, C_ref, Bound = _spmm_case(M=96, K=24 * m, N=160, n=n, m=m, g=g, dtype=dtype, seed=n + m,
                                 out_dtype=torch.float32)
    assert rel_err(C, C_ref, Bound) <= 1e-5     # fp32 output: only fp32 accumulation error


@pytest.mark.parametrize("g", [8, 16, 64])
@pytest.mark.parametrize("n,m", [(2, 4), (1, 4), (1, 10), (3, 6)])
@pytest.mark.parametrize("split", [1, 2])
def test_spmm_mma_bf16(g, n, m, split):
    tile = 2 if g % 16 == 0 else 1
    plan = sten.make_plan(sten.ALGO_MMA_SYNC, split_k=split, tile=tile)
    C, C_ref, Bound = _spmm_case(M=max(2 * g, 320), K=40 * m, N=200, n=n, m=m, g=g, dtype="bf16", plan=plan,
                                 out_dtype=torch.float32, seed=g + n + m)
    assert rel_err(C, C_ref, Bound) <= 1e-5     # fp32 output: only fp32 accumulation error
    plan1 = sten.make_plan(sten.ALGO_MMA_SYNC, split_k=split, tile=1)
    C1, _, _ = _spmm_case(M=max(2 * g, 320), K=40 * m, N=200, n=n, m=m, g=g, dtype="bf16", plan=plan1,
                          out_dtype=torch.bfloat16, seed=g + n + m)
    assert rel_err(C1, C_ref, Bound) <= TOL["bf16"]


@pytest.mark.parametrize("algo,dtype,g", [(sten.ALGO_SIMT, "f32", 4), (sten.ALGO_SIMT, "bf16", 4),
                                          (sten.ALGO_MMA_SYNC, "bf16", 16)])
def test_p7_integer_exact(algo, dtype, g):
    n, m = 2, 4
    M, K, N = 4 * g * 8, 64, 136
    W = synthetic.integer_matrix(M, K, seed=1, dtype=dtype)
    B = synthetic.integer_matrix(K, N, seed=2, dtype=dtype)
    v_ref, i_ref = oracle.sparsify(W, n, m, g)
    C_ref, _ = oracle.spmm(v_ref, i_ref, B, n, m, g)
    v, i = gpu_sparsify(W, n, m, g, dtype)
    C = sten.spmm_grouped_nm(v, i, dev(B, dtype), n, m, g, plan=sten.make_plan(algo, split_k=2),
                             out_dtype=torch.float32)
    assert np.array_equal(C.cpu().numpy().astype(np.float64), C_ref)


@pytest.mark.parametrize("dtype,g", [("f32", 4), ("bf16", 8)])
def test_p8_identity_gives_densify(dtype, g):
    n, m, K = 1, 4, 64
    W = synthetic.weights(2 * g, K, seed=4, dtype=dtype)
    v, i = gpu_sparsify(W, n, m, g, dtype)
    I = torch.eye(K, dtype=torch.float32 if dtype == "f32" else torch.bfloat16).cuda()
    C = sten.spmm_grouped_nm(v, i, I, n, m, g)
    D = sten.densify(v, i, n, m, g, K)
    assert torch.equal(C, D)


def test_p9_spec_example():
    v, i = gpu_sparsify(np.array([[2, 0], [0, 3]], np.float32), 1, 2, 1, "f32")
    B = torch.ones((2, 4), dtype=torch.float32).cuda()
    assert sten.spmm_grouped_nm(v, i, B[:, :2], 1, 2, 1).cpu().tolist() == [[2, 2], [3, 3]]


# ----------------------------------------------------------------------------------------
# P11: column shards == unsharded (same plan), edge cases, errors
# ----------------------------------------------------------------------------------------
@pytest.mark.parametrize("dtype,g", [("f32", 4), ("bf16", 16)])
def test_p11_column_shards_bit_exact(dtype, g):
    n, m, M, K, N, P = 1, 4, 256, 512, 1024, 4
    W = synthetic.weights(M, K, seed=8, dtype=dtype)
    B = dev(synthetic.activations(K, N, seed=8, dtype=dtype), dtype)
    v, i = gpu_sparsify(W, n, m, g, dtype)
    plan = sten.spmm_plan(n, m, g, M, K, N, ab_dtype=B.dtype, c_dtype=torch.float32)
    full = sten.spmm_grouped_nm(v, i, B, n, m, g, plan=plan, out_dtype=torch.float32)
    for p in range(P):
        cols = slice(p * N // P, (p + 1) * N // P)
        shard = sten.spmm_grouped_nm(v, i, B[:, cols], n, m, g, plan=plan, out_dtype=torch.float32)
        assert torch.equal(shard, full[:, cols])


def test_empty_and_k_zero():
    v = torch.empty((8, 0), dtype=torch.float32, device="cuda")
    i = torch.empty((2, 0, 2), dtype=torch.uint8, device="cuda")
    B = torch.empty((0, 16), dtype=torch.float32, device="cuda")
    C = torch.full((8, 16), 7.0, device="cuda")
    sten.spmm_grouped_nm(v, i, B, 2, 4, 4, out=C)
    assert torch.count_nonzero(C).item() == 0
    B2 = torch.empty((16, 0), dtype=torch.float32, device="cuda")
    v2, i2 = sten.sparsify_grouped_nm(torch.randn(8, 16, device="cuda"), 2, 4, 4)
    assert sten.spmm_grouped_nm(v2, i2, B2, 2, 4, 4).shape == (8, 0)


def test_error_leaves_outputs_untouched():
    W = torch.randn(12, 16, device="cuda")
    v = torch.full((12, 8), 5.0, device="cuda")
    i = torch.full((3, 4, 2), 9, dtype=torch.uint8, device="cuda")
    with pytest.raises(sten.StenError):
        sten.sparsify_grouped_nm(W, 2, 4, 5, values=v, idx=i)      # 12 % 5 != 0
    assert torch.all(v == 5.0) and torch.all(i == 9)


def test_host_e2e_entry_point():
    n, m, g, M, K, N = 2, 4, 4, 64, 128, 96
    W = synthetic.weights(M, K, seed=5)
    B = synthetic.activations(K, N, seed=5)
    Wh = torch.from_numpy(W).pin_memory()
    Bh = torch.from_numpy(B).pin_memory()
    Ch = torch.empty((M, N), dtype=torch.float32).pin_memory()
    ws = torch.empty(sten.sparse_linear_host_workspace_size(n, m, g, M, K, N), dtype=torch.uint8, device="cuda")
    sten.sparse_linear_host(Wh, Bh, n, m, g, Ch, ws)
    v_ref, i_ref = oracle.sparsify(W, n, m, g)
    C_ref, Bound = oracle.spmm(v_ref, i_ref, B, n, m, g)
    assert rel_err(Ch, C_ref, Bound) <= 1e-5
    # async variant on two side streams (the bench's e2e path): same bytes once the streams drain
    Ch2 = torch.zeros((M, N), dtype=torch.float32).pin_memory()
    Ch3 = torch.zeros((M, N), dtype=torch.float32).pin_memory()
    ws2 = torch.empty_like(ws)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    sten.sparse_linear_host_async(Wh, Bh, n, m, g, Ch2, ws, stream=s1)
    sten.sparse_linear_host_async(Wh, Bh, n, m, g, Ch3, ws2, stream=s2)
    torch.cuda.synchronize()
    assert torch.equal(Ch2, Ch) and torch.equal(Ch3, Ch)


def test_host_pipelined_entry_point():
    """The pipelined host call (H2D / kernels / D2H on three streams handed over by events, the bench's
    e2e path) over mixed problems: every C equals the single-stream call's bytes and the oracle; run
    twice back to back on the same buffers (the events order reuse of each workspace)."""
    g = 4
    specs = [(256, 768, 300, 2, 4), (120, 800, 129, 1, 10), (64, 256, 256, 1, 4), (40, 96, 33, 2, 4)]
    probs, singles, refs = [], [], []
    for k, (M, K, N, n, m) in enumerate(specs):
        W = synthetic.weights(M, K, seed=300 + k)
        B = synthetic.activations(K, N, seed=310 + k)
        Wh, Bh = torch.from_numpy(W).pin_memory(), torch.from_numpy(B).pin_memory()
        Ch = torch.full((M, N), float("nan")).pin_memory()
        ws = torch.empty(sten.sparse_linear_host_workspace_size(n, m, g, M, K, N), dtype=torch.uint8, device="cuda")
        probs.append((Wh, Bh, n, m, g, Ch, ws))
        C1 = torch.empty((M, N)).pin_memory()
        sten.sparse_linear_host(Wh, Bh, n, m, g, C1, torch.empty_like(ws))
        singles.append(C1)
        v_ref, i_ref = oracle.sparsify(W, n, m, g)
        refs.append(oracle.spmm(v_ref, i_ref, B, n, m, g))
    s_in, s_c, s_out = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    for rep in range(2):
        sten.sparse_linear_host_pipelined_async(probs, s_in, s_c, s_out)
        torch.cuda.synchronize()
        for (Wh, Bh, n, m, g_, Ch, ws), C1, (C_ref, Bound) in zip(probs, singles, refs):
            assert torch.equal(Ch, C1)
            assert rel_err(Ch, C_ref, Bound) <= 1e-5


# ----------------------------------------------------------------------------------------
# BASELINE.json sizes, in the launch configuration bench.py uses: sampled outputs
# ----------------------------------------------------------------------------------------
def _plan_cache(cfg, dtype, g):
    import json, os
    path = os.path.join(os.path.dirname(sten.__file__), "plans", "c%d_%s_g%d_step.json" % (cfg + 1, dtype, g))
    if not os.path.exists(path):
        return {}
    with open(path) as f:
        return json.load(f)


@pytest.mark.parametrize("cfg", [1, 2])
def test_baseline_configs_sampled(cfg):
    """Every case of C2 (all 9) and C3 at full size, with the plans bench.py times (the step-tuned
    plan cache where it has the case, else AUTO): sparsify bit-exact on the whole weight, the
    product on sampled token columns against the oracle."""
    rng = np.random.default_rng(cfg)
    g = 4 if cfg == 1 else 16
    cases = synthetic.config_cases(cfg, g=g)
    cache = _plan_cache(cfg, cases[0].dtype, g)
    for ci, case in enumerate(cases):
        W = synthetic.weights(case.M, case.K, seed=1234 + ci, dtype=case.dtype, k_pad=case.k_pad)
        B = synthetic.activations(case.K, case.N, seed=1234 + ci, dtype=case.dtype, k_pad=case.k_pad)
        v_ref, i_ref = oracle.sparsify(W, case.n, case.m, case.g)
        v, i = gpu_sparsify(W, case.n, case.m, case.g, case.dtype)
        assert np.array_equal(host(i), i_ref)
        assert np.array_equal(host(v).view(np.uint8), v_ref.view(np.uint8))
        pd = cache.get(case.label())
        plan = sten.make_plan(pd["algo"], pd["split_k"], pd["tile"]) if pd else None
        C = sten.spmm_grouped_nm(v, i, dev(B, case.dtype), case.n, case.m, case.g, out_dtype=torch.float32,
                                 plan=plan)
        cols = np.sort(rng.choice(case.N, size=24, replace=False))
        Cs = C.cpu().numpy()[:, cols].astype(np.float64)
        C_ref, Bound = oracle.spmm(v_ref, i_ref, np.ascontiguousarray(B[:, cols]), case.n, case.m, case.g,
                                   nthreads=oracle.max_threads())
        assert float(np.max(np.abs(Cs - C_ref) / np.maximum(Bound, 1e-30))) <= TOL[case.dtype] * (
            1 if case.dtype == "f32" else 0.05), case.label()


@pytest.mark.parametrize("cfg,dtype,g,shard", [(3, "f32", 4, 1), (3, "bf16", 16, 1), (4, "bf16", 64, 8),
                                                 (4, "f32", 4, 8)])
def test_baseline_configs_c4_c5_sampled(cfg, dtype, g, shard):
    """C4 (BERT-base encoder linears, 32768 tokens) and C5 (8192x8192 1:8) at their full sizes,
    or at the per-GPU token shard of an 8-GPU run (N / 8), in the AUTO launch configuration;
    sampled columns against the oracle."""
    rng = np.random.default_rng(cfg + shard)
    for case in synthetic.config_cases(cfg, g=g, dtype=dtype):
        N = case.N // shard
        W = synthetic.weights(case.M, case.K, seed=1234 + cfg, dtype=dtype, k_pad=case.k_pad)
        v_ref, i_ref = oracle.sparsify(W, case.n, case.m, case.g)
        v, i = gpu_sparsify(W, case.n, case.m, case.g, dtype)
        assert np.array_equal(host(i), i_ref)
        cols = np.sort(rng.choice(N, size=16, replace=False))
        B = synthetic.activations(case.K, N, seed=1234 + cfg, dtype=dtype, k_pad=case.k_pad)
        Bd = dev(B, dtype)
        C = sten.spmm_grouped_nm(v, i, Bd, case.n, case.m, case.g, out_dtype=torch.float32)
        C_ref, Bound = oracle.spmm(v_ref, i_ref, np.ascontiguousarray(B[:, cols]), case.n, case.m, case.g,
                                   nthreads=oracle.max_threads())
        Cs = C.cpu().numpy()[:, cols].astype(np.float64)
        assert float(np.max(np.abs(Cs - C_ref) / np.maximum(Bound, 1e-30))) <= 1e-5, case.label()
        del C, Bd


@pytest.mark.parametrize("g", [8, 16])
@pytest.mark.parametrize("split", [1, 3])
def test_spmm_mma_unaligned_values(g, split):
    """1:10 with K' = 41 per row: values rows are not 16-byte aligned (synchronous staging)."""
    plan = sten.make_plan(sten.ALGO_MMA_SYNC, split_k=split, tile=2 if g % 16 == 0 else 1)
    C, C_ref, Bound = _spmm_case(M=16 * g, K=410, N=136, n=1, m=10, g=g, dtype="bf16", plan=plan,
                                 out_dtype=torch.float32, seed=g + split)
    assert rel_err(C, C_ref, Bound) <= 1e-5


# ----------------------------------------------------------------------------------------
# K5 tcgen05 (A gathered into TMEM, accumulators in TMEM), 16 | g
# ----------------------------------------------------------------------------------------
@pytest.mark.parametrize("g,tile", [(16, 1), (32, 2), (64, 3), (64, 1), (128, 3)])
@pytest.mark.parametrize("n,m", [(2, 4), (1, 4), (1, 10), (3, 6)])
def test_spmm_tcgen05(g, tile, n, m):
    plan = sten.make_plan(sten.ALGO_TCGEN05, split_k=1, tile=tile)
    # M and N ragged vs the 256 x 128 CTA tile, several K slabs
    # K' = 64 n per row (the tcgen05 path stages values in 16-k steps); 64 m-blocks = several slabs
    C, C_ref, Bound = _spmm_case(M=max(g, 320 // g * g), K=64 * m, N=200, n=n, m=m, g=g, dtype="bf16", plan=plan,
                                 out_dtype=torch.float32, seed=g + n + m + tile)
    assert rel_err(C, C_ref, Bound) <= 1e-5


@pytest.mark.parametrize("n,m,kb", [(1, 4, 72), (2, 4, 72), (3, 6, 40)])
def test_spmm_tcgen05_ragged_last_slab(n, m, kb):
    """K' not a multiple of the 64-k slab (nor of 16): the last slab's k16 steps are part padding."""
    plan = sten.make_plan(sten.ALGO_TCGEN05, split_k=1, tile=1)
    C, C_ref, Bound = _spmm_case(M=272, K=kb * m, N=136, n=n, m=m, g=16, dtype="bf16", plan=plan,
                                 out_dtype=torch.float32, seed=kb + n)
    assert rel_err(C, C_ref, Bound) <= 1e-5


def test_spmm_tcgen05_rejects_unaligned_blocks():
    v = torch.zeros((32, 36), dtype=torch.bfloat16, device="cuda")      # K/m = 36 blocks: not a multiple of 8
    i = torch.zeros((2, 36, 1), dtype=torch.uint8, device="cuda")
    B = torch.zeros((144, 64), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(sten.StenError):
        sten.spmm_grouped_nm(v, i, B, 1, 4, 16, plan=sten.make_plan(sten.ALGO_TCGEN05, 1, 1))


@pytest.mark.parametrize("out", ["f32", "bf16"])
def test_spmm_tcgen05_integer_exact_and_bf16_out(out):
    n, m, g = 2, 4, 16
    M, K, N = 512, 256, 384
    W = synthetic.integer_matrix(M, K, seed=11, dtype="bf16")
    B = synthetic.integer_matrix(K, N, seed=12, dtype="bf16")
    v_ref, i_ref = oracle.sparsify(W, n, m, g)
    C_ref, Bound = oracle.spmm(v_ref, i_ref, B, n, m, g)
    v, i = gpu_sparsify(W, n, m, g, "bf16")
    od = torch.float32 if out == "f32" else torch.bfloat16
    C = sten.spmm_grouped_nm(v, i, dev(B, "bf16"), n, m, g, plan=sten.make_plan(sten.ALGO_TCGEN05, 1, 1),
                             out_dtype=od)
    if out == "f32":
        assert np.array_equal(C.cpu().numpy().astype(np.float64), C_ref)
    else:
        assert rel_err(C, C_ref, Bound) <= TOL["bf16"]


# ----------------------------------------------------------------------------------------
# measured plan choice: the tuned plan is a valid plan and reproduces the oracle
# ----------------------------------------------------------------------------------------
@pytest.mark.parametrize("dtype,g", [("f32", 4), ("bf16", 16)])
def test_spmm_autotune(dtype, g):
    n, m = 2, 4
    M, K, N = 16 * g, 512, 384
    W = synthetic.weights(M, K, seed=31, dtype=dtype)
    B = synthetic.activations(K, N, seed=31, dtype=dtype)
    v_ref, i_ref = oracle.sparsify(W, n, m, g)
    C_ref, Bound = oracle.spmm(v_ref, i_ref, B, n, m, g)
    v, i = gpu_sparsify(W, n, m, g, dtype)
    Bd = dev(B, dtype)
    scratch = torch.empty((M, N), dtype=torch.float32, device="cuda")
    plan = sten.spmm_autotune(v, i, Bd, n, m, g, out=scratch, reps=2)
    assert plan.algo in (sten.ALGO_SIMT, sten.ALGO_MMA_SYNC, sten.ALGO_TCGEN05)
    C = sten.spmm_grouped_nm(v, i, Bd, n, m, g, out_dtype=torch.float32, plan=plan)
    assert rel_err(C, C_ref, Bound) <= 1e-5


# ----------------------------------------------------------------------------------------
# NEXT-2: SameFormat re-sparsification -- bit-exact vs the oracle
# ----------------------------------------------------------------------------------------
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("n,m,g", [(2, 4, 4), (1, 4, 1), (1, 10, 2), (3, 6, 3), (2, 8, 4), (4, 16, 1)])
@pytest.mark.parametrize("ld_multiple", [1, 8])
def test_resparsify_same_format_bit_exact(dtype, n, m, g, ld_multiple):
    M, K = 10 * g, 23 * m
    W = synthetic.weights(M, K, seed=n + m + g, dtype=dtype)
    W2 = synthetic.weights(M, K, seed=1000 + n + m + g, dtype=dtype)     # "after an optimizer step"
    _, i = gpu_sparsify(W, n, m, g, dtype)
    v2 = sten.resparsify_same_format(dev(W2, dtype, ld_multiple=ld_multiple), i, n, m, g)
    torch.cuda.synchronize()
    _, i_ref = oracle.sparsify(W, n, m, g)
    v2_ref = oracle.same_format(W2, i_ref, n, m, g)
    assert np.array_equal(host(v2).view(np.uint8), v2_ref.view(np.uint8))


# ----------------------------------------------------------------------------------------
# 8(e): SpMM with the all-gather fused into the epilogue (peer buffers; local stand-ins here)
# ----------------------------------------------------------------------------------------
@pytest.mark.parametrize("split", [1, 3])
@pytest.mark.parametrize("P", [2, 4])
def test_spmm_fused_allgather_equals_unsharded(split, P):
    """P simulated ranks each compute their token shard and push it into all P gathered buffers;
    every buffer then equals the unsharded product bit for bit (global plan, pin P11)."""
    n, m, g, M, K, N = 2, 4, 4, 96, 256, 4 * 136
    W = synthetic.weights(M, K, seed=21)
    B = synthetic.activations(K, N, seed=22)
    v, i = gpu_sparsify(W, n, m, g, "f32")
    Bd = dev(B, "f32")
    plan = sten.make_plan(sten.ALGO_SIMT, split_k=split, tile=1)
    C_full = sten.spmm_grouped_nm(v, i, Bd, n, m, g, plan=plan)
    outs = [torch.full((M, N), float("nan"), device="cuda") for _ in range(P)]
    per = N // P
    for r in range(P):                                   # rank r's call
        sten.spmm_grouped_nm_allgather(v, i, Bd[:, r * per:(r + 1) * per], n, m, g, outs, r * per, plan=plan)
    torch.cuda.synchronize()
    for o in outs:
        assert torch.equal(o, C_full)
    v_ref, i_ref = oracle.sparsify(W, n, m, g)
    C_ref, Bound = oracle.spmm(v_ref, i_ref, B, n, m, g)
    assert rel_err(outs[0], C_ref, Bound) <= 1e-5
    with pytest.raises(sten.StenError):                   # the fused epilogue is the SIMT kernel's
        sten.spmm_grouped_nm_allgather(v, i, Bd[:, :per], n, m, g, outs, 0,
                                       plan=sten.make_plan(sten.ALGO_MMA_SYNC, 1, 1))


def test_partitions_nccl_world1_vs_oracle():
    """Every partition class of parallel.py (TokenShardedSpmm with the chunked NCCL all-gather on
    its side stream, RowShardedSpmm, FusedAllGatherSpmm on symmetric memory) on a one-rank NCCL
    group with the real CUDA compute, compared element by element with the oracle (fp32 1e-5,
    bf16 2e-2) and bit for bit with the unsharded product under the global plan (P11); fp32 and
    bf16 (g = 64 forces the fused path's SIMT plan coercion)."""
    import os, socket, subprocess, sys
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    out = subprocess.run([sys.executable, os.path.join(root, "tests", "_dist_world1.py")], cwd=root, env=env,
                         capture_output=True, text=True, timeout=600)
    assert "ALL OK" in out.stdout, out.stdout + out.stderr
    assert out.stdout.count("CASE ") == 4 * 6


# ----------------------------------------------------------------------------------------
# NEXT-3: bias + activation fused into the SpMM epilogue
# ----------------------------------------------------------------------------------------
@pytest.mark.parametrize("act", [0, 1, 2])
@pytest.mark.parametrize("split", [1, 4])
@pytest.mark.parametrize("with_bias", [True, False])
def test_spmm_bias_act_epilogue(act, split, with_bias):
    n, m, g, M, K, N = 2, 4, 4, 120, 384, 200
    W = synthetic.weights(M, K, seed=31)
    B = synthetic.activations(K, N, seed=32)
    bias = (np.random.default_rng(33).standard_normal(M) * 0.1).astype(np.float32)
    v, i = gpu_sparsify(W, n, m, g, "f32")
    plan = sten.make_plan(sten.ALGO_SIMT, split_k=split, tile=1)
    C = sten.spmm_grouped_nm_bias_act(v, i, dev(B, "f32"), n, m, g,
                                      bias=torch.from_numpy(bias).cuda() if with_bias else None, act=act, plan=plan)
    torch.cuda.synchronize()
    v_ref, i_ref = oracle.sparsify(W, n, m, g)
    C_ref, Bound = oracle.spmm(v_ref, i_ref, B, n, m, g)
    Y = oracle.bias_act(C_ref, bias if with_bias else None, act)
    # |act(c) - act(c_ref)| <= 1.13 |c - c_ref| (GELU' <= 1.13), plus fp32 rounding of the bias add
    # and erff (a few ulp of the result)
    tol = 1.13 * 1e-5 * Bound + 4e-7 * np.abs(Y) + 1e-7 * (np.abs(C_ref) + (np.abs(bias)[:, None] if with_bias else 0))
    assert (np.abs(C.cpu().numpy().astype(np.float64) - Y) <= tol + 1e-30).all()


# ----------------------------------------------------------------------------------------
# Grouped (batched) launch of independent problems
# ----------------------------------------------------------------------------------------
@pytest.mark.parametrize("tile", [1, 2])
def test_spmm_batched_equals_single_launches(tile):
    """One grouped launch over mixed shapes / sparsities / ragged sizes equals the per-problem
    launches (same tile, split_k = 1) bit for bit, and the oracle within 1e-5."""
    g = 4
    shapes = [(64, 96, 300, 2, 4), (120, 400, 129, 1, 10), (200, 64, 256, 1, 4), (56, 768, 40, 2, 4)]
    probs, singles, refs = [], [], []
    for k, (M, K, N, n, m) in enumerate(shapes):
        W = synthetic.weights(M, K, seed=40 + k)
        B = synthetic.activations(K, N, seed=50 + k)
        v, i = gpu_sparsify(W, n, m, g, "f32")
        Bd = dev(B, "f32")
        C = torch.full((M, N), float("nan"), device="cuda")
        probs.append((v, i, Bd, n, m, g, C))
        singles.append(sten.spmm_grouped_nm(v, i, Bd, n, m, g, plan=sten.make_plan(sten.ALGO_SIMT, 1, tile)))
        v_ref, i_ref = oracle.sparsify(W, n, m, g)
        refs.append(oracle.spmm(v_ref, i_ref, B, n, m, g))
    sten.spmm_grouped_nm_batched(probs, tile=tile)
    torch.cuda.synchronize()
    for (v, i, Bd, n, m, g_, C), S, (C_ref, Bound) in zip(probs, singles, refs):
        assert torch.equal(C, S)
        assert rel_err(C, C_ref, Bound) <= 1e-5


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("lean", [True, False])
def test_sparsify_batched_mixed_classes_equals_oracle(dtype, lean):
    """ONE grouped sparsify launch over mixed (n, m, g) equals the oracle bit for bit (idx and values)
    for every problem.  lean: every problem has a vector-store body on aligned rows (the lean
    instantiation: m in {2, 4, 8, 10}, n in {1, 2}); else the full one -- per-position stores
    (n = 3, 5), element-aligned rows, m = 6 / 12 / 16, g from 1 to 16, ragged sizes."""
    if lean:
        specs = [(96, 3072, 2, 4, 4), (64, 768, 1, 4, 4), (40, 800, 1, 10, 4), (33, 80, 1, 2, 1),
                 (36, 96, 2, 8, 3), (8, 40, 2, 4, 8), (24, 160, 1, 8, 8), (30, 120, 2, 10, 5)]
    else:
        specs = [(96, 3072, 2, 4, 4), (64, 768, 1, 4, 4), (40, 800, 1, 10, 4), (48, 96, 3, 6, 16),
                 (33, 80, 1, 2, 1), (24, 160, 5, 16, 8), (36, 96, 2, 8, 3), (16, 72, 1, 12, 2),
                 (8, 40, 2, 4, 8), (30, 66, 1, 6, 5)]
    probs, refs, keep = [], [], []
    for k, (M, K, n, m, g) in enumerate(specs):
        W = synthetic.weights(M, K, seed=90 + k, dtype=dtype)
        ld = K + (3 if (k % 3 == 2 and not lean) else 0)        # element-aligned rows for some problems
        Wp = np.zeros((M, ld), dtype=W.dtype)
        Wp[:, :K] = W
        Wd = dev(Wp, dtype, ld_multiple=1)[:, :K]
        Kp = K // m * n
        tdt = torch.float32 if dtype == "f32" else torch.bfloat16
        vals = torch.full((M, Kp), float("nan"), dtype=tdt, device="cuda")
        idx = torch.full((M // g, K // m, n), 255, dtype=torch.uint8, device="cuda")
        probs.append((Wd, n, m, g, vals, idx))
        refs.append(oracle.sparsify(W, n, m, g))
        keep.append(Wp)
    sten.sparsify_grouped_nm_batched(probs)
    torch.cuda.synchronize()
    for k, ((Wd, n, m, g, vals, idx), (v_ref, i_ref)) in enumerate(zip(probs, refs)):
        assert np.array_equal(idx.cpu().numpy().reshape(i_ref.shape), i_ref), k
        assert np.array_equal(host(vals), v_ref), k


@pytest.mark.parametrize("tile", [0, 1, 2, 3])
@pytest.mark.parametrize("splits", [None, [3, 2, 1, 5]])
def test_spmm_batched_split_k_equals_cluster_split(tile, splits):
    """The grouped launch with per-problem split-K through the workspace equals, bit for bit, the
    single launches with the same (tile, split) (cluster DSMEM reduction, same fixed z order), and
    the oracle within 1e-5; called twice on the same workspace (the counters are left at zero)."""
    g = 4
    shapes = [(64, 384, 300, 2, 4), (120, 800, 129, 1, 10), (200, 256, 256, 1, 4), (56, 768, 40, 2, 4)]
    probs, refs = [], []
    for k, (M, K, N, n, m) in enumerate(shapes):
        W = synthetic.weights(M, K, seed=70 + k)
        B = synthetic.activations(K, N, seed=80 + k)
        v, i = gpu_sparsify(W, n, m, g, "f32")
        probs.append((v, i, dev(B, "f32"), n, m, g, torch.full((M, N), float("nan"), device="cuda")))
        v_ref, i_ref = oracle.sparsify(W, n, m, g)
        refs.append(oracle.spmm(v_ref, i_ref, B, n, m, g))
    nb = sten.batched_workspace_size(probs, splits, tile)
    ws = torch.zeros(max(nb, 16) // 4 + 4, dtype=torch.float32, device="cuda")
    for rep in range(2):
        for p in probs:
            p[6].fill_(float("nan"))
        sten.spmm_grouped_nm_batched_ex(probs, ws, splits, tile)
        torch.cuda.synchronize()
        for k, ((v, i, Bd, n, m, g_, C), (C_ref, Bound)) in enumerate(zip(probs, refs)):
            assert rel_err(C, C_ref, Bound) <= 1e-5
            if splits is not None:
                t = tile if tile else (3 if m >= 8 * n else 2)
                S = sten.spmm_grouped_nm(v, i, Bd, n, m, g, plan=sten.make_plan(sten.ALGO_SIMT, splits[k], t))
                torch.cuda.synchronize()
                assert torch.equal(C, S), k
    nwords = 0
    assert torch.count_nonzero(ws[: 4].view(torch.int32)) == 0 or nb == 0


def test_grouped_c2_problem_set():
    """The C2 step's 9 problems through the grouped split-K launch with automatic splits (the bench's
    launch) vs the oracle on sampled columns of every case, twice on one workspace (the tile counters
    are left at zero), the same bits both times."""
    cases = synthetic.config_cases(1, g=4, dtype="f32")
    probs, host_in = [], []
    for k, c in enumerate(cases):
        W = synthetic.weights(c.M, c.K, seed=1234 + k, k_pad=c.k_pad)
        B = synthetic.activations(c.K, c.N, seed=1234 + k, k_pad=c.k_pad)
        v, i = gpu_sparsify(W, c.n, c.m, c.g, "f32")
        probs.append((v, i, dev(B, "f32"), c.n, c.m, c.g, torch.full((c.M, c.N), float("nan"), device="cuda")))
        host_in.append((W, B))
    nb = sten.batched_workspace_size(probs, None, 2)
    ws = torch.zeros(max(nb, 16) // 4 + 4, dtype=torch.float32, device="cuda")
    outs = []
    for rep in range(2):
        for p in probs:
            p[6].fill_(float("nan"))
        sten.spmm_grouped_nm_batched_ex(probs, ws, None, 2)
        torch.cuda.synchronize()
        outs.append([p[6].clone() for p in probs])
    assert all(torch.equal(a, b) for a, b in zip(outs[0], outs[1]))
    cols = np.array([0, 1, 255, 256, 511, 700, 1023])
    for k, (c, (W, B)) in enumerate(zip(cases, host_in)):
        v_ref, i_ref = oracle.sparsify(W, c.n, c.m, c.g)
        C_ref, Bound = oracle.spmm(v_ref, i_ref, np.ascontiguousarray(B[:, cols]), c.n, c.m, c.g,
                                   nthreads=oracle.max_threads())
        C = outs[0][k][:, torch.from_numpy(cols).cuda()]
        assert rel_err(C, C_ref, Bound) <= 1e-5, c.label()


def test_new_entry_points_reject_bad_arguments():
    """Argument errors of the fused / grouped entry points are returned before any launch."""
    n, m, g, M, K, N = 2, 4, 4, 32, 64, 40
    W = torch.from_numpy(synthetic.weights(M, K, seed=61)).cuda()
    B = torch.from_numpy(synthetic.activations(K, N, seed=62)).cuda()
    v, i = sten.sparsify_grouped_nm(W, n, m, g)
    C = torch.zeros((M, N), device="cuda")
    with pytest.raises(sten.StenError) as e:                                 # act out of range
        sten.spmm_grouped_nm_bias_act(v, i, B, n, m, g, act=7, out=C)
    assert e.value.status == 1
    with pytest.raises(sten.StenError) as e:                                 # fused epilogue is SIMT-only
        sten.spmm_grouped_nm_bias_act(v, i, B, n, m, g, act=1, out=C, plan=sten.make_plan(sten.ALGO_MMA_SYNC, 1, 1))
    assert e.value.status == 3
    with pytest.raises(sten.StenError) as e:                                 # gathered buffer too narrow
        sten.spmm_grouped_nm_allgather(v, i, B, n, m, g, [torch.zeros((M, N), device="cuda")], 8)
    assert e.value.status == 2
    with pytest.raises(sten.StenError) as e:                                 # mixed row-group classes
        v8, i8 = sten.sparsify_grouped_nm(W, n, m, 8)
        sten.spmm_grouped_nm_batched([(v, i, B, n, m, 4, C), (v8, i8, B, n, m, 8, torch.zeros_like(C))])
    assert e.value.status == 3
    with pytest.raises(sten.StenError) as e:                                 # unknown tile
        sten.spmm_grouped_nm_batched([(v, i, B, n, m, g, C)], tile=5)
    assert e.value.status == 3
    assert torch.count_nonzero(C) == 0                                       # nothing was written
