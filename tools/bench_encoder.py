"""NEXT-3 latency: a 12-layer BERT-base encoder (C4: batch 256 x seq 128) with every linear in
grouped n:m on the library's SpMM (fused bias / GELU / residual epilogues) vs the same encoder
with dense cuBLAS GEMMs on densify(W) -- each captured as ONE CUDA graph, CUDA events around the
replay, median of 5 (the GPU analogue of the paper's 3.2x "vs dense PyTorch").
   python tools/bench_encoder.py [--batch 256] [--seq 128] [--layers 12] [--nm 2:4] [--g 4]"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2304_07613_b200 import encoder  # noqa: E402


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sorted(ts)[len(ts) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--seq", type=int, default=128)
    ap.add_argument("--layers", type=int, default=12)
    ap.add_argument("--nm", default="2:4")
    ap.add_argument("--g", type=int, default=4)
    ap.add_argument("--dtype", choices=["f32", "bf16"], default="f32")
    args = ap.parse_args()
    n, m = (int(x) for x in args.nm.split(":"))
    torch.backends.cuda.matmul.allow_tf32 = False
    N = args.batch * args.seq
    dt = torch.float32 if args.dtype == "f32" else torch.bfloat16
    layers = [encoder.SparseBertLayer(encoder.random_layer_weights(s, "cuda"), n, m, args.g, dtype=dt)
              for s in range(args.layers)]
    x = torch.randn(encoder.HIDDEN, N, device="cuda").to(dt)
    sp = encoder.Encoder(layers)
    sp.capture(x, args.batch, args.seq)
    t_sparse = timed(sp.replay)
    dense = encoder.Encoder([encoder.DenseBertLayer(l.dense_weights(), l) for l in layers])
    dense.capture(x, args.batch, args.seq)
    t_dense = timed(dense.replay)
    diff = float((sp.replay().float() - dense.replay().float()).abs().max())
    torch.backends.cuda.matmul.allow_tf32 = True
    dense_tf32 = encoder.Encoder([encoder.DenseBertLayer(l.dense_weights(), l) for l in layers])
    dense_tf32.capture(x, args.batch, args.seq)
    t_tf32 = timed(dense_tf32.replay)
    torch.backends.cuda.matmul.allow_tf32 = False
    # the linears alone (the 4 of every layer, in sequence, same shapes and epilogues), for the breakdown
    def linears_only(layer_objs, sparse):
        xs = x
        hs = torch.empty(encoder.HIDDEN, N, device="cuda", dtype=dt)
        fs = torch.empty(encoder.FFN, N, device="cuda", dtype=dt)

        def run():
            for l in layer_objs:
                if sparse:
                    l._linear("qkv", xs, l.bias["bqkv"])
                    l._linear("o", xs, l.bias["bo"], residual=hs)
                    l._linear("w1", xs, l.bias["b1"], act=1)
                    l._linear("w2", fs, l.bias["b2"], residual=hs)
                else:
                    torch.addmm(l.bias["bqkv"][:, None], l.w["qkv"], xs)
                    torch.addmm(l.bias["bo"][:, None], l.w["o"], xs).add_(hs)
                    torch.nn.functional.gelu(torch.addmm(l.bias["b1"][:, None], l.w["w1"], xs))
                    torch.addmm(l.bias["b2"][:, None], l.w["w2"], fs).add_(hs)
        run()
        torch.cuda.synchronize()
        gph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gph):
            run()
        return timed(gph.replay)
    t_lin_sparse = linears_only(layers, True)
    t_lin_dense = linears_only(dense.layers, False)
    lin = encoder.linear_flops(N) * args.layers
    out = {"what": "12-layer BERT-base encoder forward, batch %d x seq %d (%d tokens), %s, %s:g%d linears (%s)"
                   % (args.batch, args.seq, N, args.dtype, args.nm, args.g, layers[0].backend),
           "sparse_ms": round(t_sparse, 3), "dense_cublas_ms": round(t_dense, 3),
           "dense_cublas_tf32_ms": round(t_tf32, 3) if args.dtype == "f32" else None,
           "speedup_vs_dense": round(t_dense / t_sparse, 3),
           "linears_only_sparse_ms": round(t_lin_sparse, 3), "linears_only_dense_ms": round(t_lin_dense, 3),
           "linears_only_speedup": round(t_lin_dense / t_lin_sparse, 3),
           "linear_eff_tflops_sparse_incl_attention": round(lin / (t_sparse * 1e-3) / 1e12, 2),
           "max_abs_diff_sparse_vs_dense": diff,
           "how": "each encoder captured as one CUDA graph; CUDA events around the replay, median of 5; dense = "
                  "torch.addmm on densify(W) (same masked weights), attention = torch SDPA, LN = torch ops"}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
