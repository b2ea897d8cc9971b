"""NEXT-3: the BERT-base encoder layer on the grouped n:m kernels against an
independent fp64 CPU reference of the same layer: the weights sparsified by the ORACLE, every op
(masked linear, bias, GELU, residual, attention, LayerNorm) in plain torch fp64 -- plus the fused
epilogue's residual path alone against the oracle product."""
import numpy as np
import pytest
import torch
import torch.nn.functional as F

import oracle
import synthetic
from paper_2304_07613_b200 import encoder, sten
from test_gpu_parity import dev

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("act", [0, 1])
@pytest.mark.parametrize("split", [1, 3])
def test_epilogue_residual(act, split):
    n, m, g, M, K, N = 2, 4, 4, 96, 256, 200
    W = synthetic.weights(M, K, seed=41)
    B = synthetic.activations(K, N, seed=42)
    R = synthetic.activations(M, N, seed=43)
    bias = (np.random.default_rng(44).standard_normal(M) * 0.1).astype(np.float32)
    v, i = sten.sparsify_grouped_nm(dev(W, "f32"), n, m, g)
    C = sten.spmm_grouped_nm_epilogue(v, i, dev(B, "f32"), n, m, g, bias=torch.from_numpy(bias).cuda(), act=act,
                                      residual=dev(R, "f32"), plan=sten.make_plan(sten.ALGO_SIMT, split, 1))
    torch.cuda.synchronize()
    v_ref, i_ref = oracle.sparsify(W, n, m, g)
    C_ref, Bound = oracle.spmm(v_ref, i_ref, B, n, m, g)
    ref = oracle.bias_act(C_ref, bias, act) + R.astype(np.float64)
    err = np.abs(C.cpu().numpy().astype(np.float64) - ref)
    # |act(c) - act(c_ref)| <= 1.13 |c - c_ref| (GELU slope bound) + the fp32 roundings of bias/act/residual
    assert (err <= 1.13 * 1e-5 * Bound + 1e-5 * (np.abs(ref) + 1)).all()


def _reference_layer(wts_np, x, batch, seq, n, m, g):
    """fp64 torch CPU reference; weights masked by the ORACLE sparsifier."""
    t = {k: torch.from_numpy(np.asarray(v, np.float64)) for k, v in wts_np.items()}

    def masked(name):
        W = wts_np[name].astype(np.float32)
        v, i = oracle.sparsify(W, n, m, g)
        return torch.from_numpy(oracle.densify(v, i, n, m, g, W.shape[1]).astype(np.float64))

    H, heads, d = 768, 12, 64
    xT = torch.from_numpy(x.astype(np.float64))
    qkv = masked("qkv") @ xT + t["bqkv"][:, None]
    q, k, v = qkv.view(3, heads, d, batch, seq).permute(0, 3, 1, 4, 2)
    a = torch.softmax(q @ k.transpose(-1, -2) / np.sqrt(d), dim=-1) @ v
    aT = a.permute(1, 3, 0, 2).reshape(H, batch * seq)

    def ln(h, gname, bname):
        mu = h.mean(0, keepdim=True)
        var = ((h - mu) ** 2).mean(0, keepdim=True)
        return (h - mu) / torch.sqrt(var + 1e-12) * t[gname][:, None] + t[bname][:, None]

    h = ln(masked("o") @ aT + t["bo"][:, None] + xT, "ln1_g", "ln1_b")
    f = F.gelu(masked("w1") @ h + t["b1"][:, None])
    y = ln(masked("w2") @ f + t["b2"][:, None] + h, "ln2_g", "ln2_b")
    return y.numpy()


@pytest.mark.parametrize("n,m,g", [(2, 4, 4), (1, 4, 4)])
def test_encoder_layer_vs_fp64_reference(n, m, g):
    batch, seq = 2, 32
    wts = encoder.random_layer_weights(7, "cpu")
    layer = encoder.SparseBertLayer({k: v.cuda() for k, v in wts.items()}, n, m, g)
    x = synthetic.activations(768, batch * seq, seed=9)
    y = layer(torch.from_numpy(x).cuda(), batch, seq)
    torch.cuda.synchronize()
    ref = _reference_layer({k: v.numpy() for k, v in wts.items()}, x, batch, seq, n, m, g)
    err = float(np.max(np.abs(y.cpu().numpy().astype(np.float64) - ref)))
    assert err <= 2e-4, err                     # post-LN values are O(1); fp32 chain vs fp64
    # the dense reference layer on densify(W) agrees too (same masked weights, cuBLAS GEMMs; TF32 off)
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        dense = encoder.DenseBertLayer(layer.dense_weights(), layer)
        yd = dense(torch.from_numpy(x).cuda(), batch, seq)
        torch.cuda.synchronize()
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev
    assert float(np.max(np.abs(yd.cpu().numpy().astype(np.float64) - ref))) <= 2e-4


def test_encoder_graph_replay_equals_eager():
    batch, seq = 2, 32
    layers = [encoder.SparseBertLayer(encoder.random_layer_weights(s, "cuda"), 2, 4, 4) for s in range(2)]
    enc = encoder.Encoder(layers)
    x = torch.from_numpy(synthetic.activations(768, batch * seq, seed=3)).cuda()
    eager = enc(x, batch, seq).clone()
    xs = x.clone()
    enc.capture(xs, batch, seq)
    out = enc.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, eager)


@pytest.mark.parametrize("act", [0, 1])
@pytest.mark.parametrize("tile", [1, 6])
def test_sp24_epilogue(act, tile):
    """The fused bias / GELU / residual epilogue of K6 against the oracle (bf16 in, fp32 out)."""
    n, m, g, M, K, N = 2, 4, 4, 384, 2048, 300
    W = synthetic.weights(M, K, seed=51, dtype="bf16")
    B = synthetic.activations(K, N, seed=52, dtype="bf16")
    R = synthetic.activations(M, N, seed=53)
    bias = (np.random.default_rng(54).standard_normal(M) * 0.1).astype(np.float32)
    v, i = sten.sparsify_grouped_nm(dev(W, "bf16"), n, m, g)
    v24, meta = sten.sp24_pack(v, i, n, m, g, K)
    C = sten.spmm_sp24_epilogue(v24, meta, M, K, dev(B, "bf16"), bias=torch.from_numpy(bias).cuda(), act=act,
                                residual=dev(R, "f32"), out_dtype=torch.float32, tile=tile)
    torch.cuda.synchronize()
    v_ref, i_ref = oracle.sparsify(W, n, m, g)
    C_ref, Bound = oracle.spmm(v_ref, i_ref, B, n, m, g)
    ref = oracle.bias_act(C_ref, bias, act) + R.astype(np.float64)
    err = np.abs(C.cpu().numpy().astype(np.float64) - ref)
    assert (err <= 1.13 * 1e-5 * Bound + 1e-5 * (np.abs(ref) + 1)).all()


def test_encoder_layer_bf16_sp24_vs_fp64_reference():
    """The bf16 encoder layer on the 2:4 sparse tensor cores vs the fp64 reference (bf16 tolerance)."""
    batch, seq, n, m, g = 2, 32, 2, 4, 4
    wts = encoder.random_layer_weights(8, "cpu")
    layer = encoder.SparseBertLayer({k: v.cuda() for k, v in wts.items()}, n, m, g, dtype=torch.bfloat16)
    assert layer.backend == "sp24"
    x = synthetic.activations(768, batch * seq, seed=10, dtype="bf16")
    y = layer(torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).cuda(), batch, seq)
    torch.cuda.synchronize()
    wb = {k: synthetic.bf16_bits_to_f32(synthetic.f32_to_bf16_bits(v.numpy())) if k in ("qkv", "o", "w1", "w2")
          else v.numpy() for k, v in wts.items()}
    ref = _reference_layer(wb, synthetic.bf16_bits_to_f32(x), batch, seq, n, m, g)
    err = float(np.max(np.abs(y.float().cpu().numpy().astype(np.float64) - ref)))
    assert err <= 0.15, err                     # bf16 activations between layers; post-LN values are O(1)
