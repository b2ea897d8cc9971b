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
    args = ap.parse_args()
    n, m = (int(x) for x in args.nm.split(":"))
    torch.backends.cuda.matmul.allow_tf32 = False
    N = args.batch * args.seq
    layers = [encoder.SparseBertLayer(encoder.random_layer_weights(s, "cuda"), n, m, args.g)
              for s in range(args.layers)]
    x = torch.randn(encoder.HIDDEN, N, device="cuda")
    sp = encoder.Encoder(layers)
    sp.capture(x, args.batch, args.seq)
    t_sparse = timed(sp.replay)
    dense = encoder.Encoder([encoder.DenseBertLayer(l.dense_weights(), l) for l in layers])
    dense.capture(x, args.batch, args.seq)
    t_dense = timed(dense.replay)
    diff = float((sp.replay() - dense.replay()).abs().max())
    torch.backends.cuda.matmul.allow_tf32 = True
    dense_tf32 = encoder.Encoder([encoder.DenseBertLayer(l.dense_weights(), l) for l in layers])
    dense_tf32.capture(x, args.batch, args.seq)
    t_tf32 = timed(dense_tf32.replay)
    torch.backends.cuda.matmul.allow_tf32 = False
    # attention + LN alone (the non-linear part both encoders share), for the breakdown
    lin = encoder.linear_flops(N) * args.layers
    out = {"what": "12-layer BERT-base encoder forward, batch %d x seq %d (%d tokens), fp32, %s:g%d linears"
                   % (args.batch, args.seq, N, args.nm, args.g),
           "sparse_ms": round(t_sparse, 3), "dense_fp32_cublas_ms": round(t_dense, 3),
           "dense_tf32_cublas_ms": round(t_tf32, 3),
           "speedup_vs_dense_fp32": round(t_dense / t_sparse, 3), "speedup_vs_dense_tf32": round(t_tf32 / t_sparse, 3),
           "linear_eff_tflops_sparse_incl_attention": round(lin / (t_sparse * 1e-3) / 1e12, 2),
           "max_abs_diff_sparse_vs_dense": diff,
           "how": "each encoder captured as one CUDA graph; CUDA events around the replay, median of 5; dense = "
                  "torch.addmm on densify(W) (same masked weights), attention = torch SDPA, LN = torch ops"}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
