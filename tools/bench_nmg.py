"""Measurement of the chunked n:m:g path (the paper's own format, NEXT-1) on the C2 BERT-base
shapes: per case, sparsify (greedy conversion) and SpMM each timed as a CUDA graph of R
launches over rotating input copies (> L2), CUDA events, median of 5 replays.  Also the energy
(kept L1 mass fraction) of n:m:g vs grouped n:m (A) at the same n, m, g.

python tools/bench_nmg.py [--g 4] [--out FILE]      (prints one JSON line)
"""
import argparse
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import synthetic
from paper_2304_07613_b200 import sten

FFMA_PEAK_TF = 148 * 128 * 2 * 1.965e9 / 1e12      # DESIGN.md section 6 (derived)


def graph_time_us(fn, R, reps=5):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for i in range(2):
            fn(i)
    torch.cuda.synchronize()
    gph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gph, stream=s):
        for i in range(R):
            fn(i)
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        gph.replay()                  # replays on the current stream
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / R)
    return float(np.median(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--g", type=int, default=4)
    ap.add_argument("--N", type=int, default=1024)
    ap.add_argument("--dtype", default="f32")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    g, N = args.g, args.N
    tdt = torch.float32 if args.dtype == "f32" else torch.bfloat16
    s = 4 if args.dtype == "f32" else 2
    rows = []
    for (M, K) in [(768, 768), (768, 3072), (3072, 768)]:
        for (n, m) in [(2, 4), (1, 4), (1, 8)]:
            L = math.comb(m, n) * g
            if K % L or M % m:
                continue
            W = torch.from_numpy(synthetic.weights(M, K, seed=1234)).to(tdt)
            Bh = torch.from_numpy(synthetic.activations(K, N, seed=1235)).to(tdt)
            R = max(4, int(3 * 126e6 // (M * K * s + K * N * s + M * N * s)) + 1)
            Ws = [W.cuda() for _ in range(R)]
            Bs = [Bh.cuda() for _ in range(R)]
            vals = [torch.empty((M // m, K // L, L, n), dtype=tdt, device="cuda") for _ in range(R)]
            idxs = [torch.empty((M // m, K // L, L), dtype=torch.int16, device="cuda") for _ in range(R)]
            Cs = [torch.empty((M, N), dtype=tdt, device="cuda") for _ in range(R)]
            for r in range(R):
                sten.nmg_sparsify(Ws[r], n, m, g, values=vals[r], idx=idxs[r])
            t_sp = graph_time_us(lambda i: sten.nmg_sparsify(Ws[i % R], n, m, g, values=vals[i % R],
                                                             idx=idxs[i % R]), R)
            t_mm = graph_time_us(lambda i: sten.nmg_spmm(vals[i % R], idxs[i % R], Bs[i % R], n, m, g,
                                                         out=Cs[i % R]), R)
            # energy: chunked n:m:g vs grouped n:m (A) with the same n, m, g (fp32 weights)
            Dn = sten.nmg_densify(vals[0], idxs[0], n, m, g, K).float()
            va, ia = sten.sparsify_grouped_nm(Ws[0].t().contiguous(), n, m, g)   # (A) on W^T: m-blocks along M
            Da = sten.densify(va, ia, n, m, g, M).float().t()
            den = Ws[0].float().abs().sum().item()
            e_nmg = Dn.abs().sum().item() / den
            e_a = Da.abs().sum().item() / den
            nz = 2.0 * M * K * n / m * N
            rows.append({"case": "%dx%dx%d %d:%d:%d %s" % (M, K, N, n, m, g, args.dtype),
                         "sparsify_us": round(t_sp, 2), "spmm_us": round(t_mm, 2),
                         "spmm_eff_gflops": round(2.0 * M * K * N / (t_mm * 1e-6) / 1e9, 1),
                         "spmm_nz_tflops": round(nz / (t_mm * 1e-6) / 1e12, 3),
                         "spmm_frac_ffma": round(nz / (t_mm * 1e-6) / 1e12 / FFMA_PEAK_TF, 4),
                         "energy_nmg": round(e_nmg, 5), "energy_grouped_A_same_g": round(e_a, 5)})
            print(json.dumps(rows[-1]), flush=True)
    tot_nz = sum(2.0 * int(r["case"].split("x")[0]) * int(r["case"].split("x")[1]) * N *
                 int(r["case"].split()[1].split(":")[0]) / int(r["case"].split()[1].split(":")[1]) for r in rows)
    tot_t = sum(r["spmm_us"] for r in rows) * 1e-6
    out = {"what": "chunked n:m:g (paper format) on C2 shapes, one B200", "g": g, "N": N, "dtype": args.dtype,
           "spmm_nz_tflops_all": round(tot_nz / tot_t / 1e12, 3),
           "spmm_frac_ffma_all": round(tot_nz / tot_t / 1e12 / FFMA_PEAK_TF, 4),
           "ffma_peak_tflops": round(FFMA_PEAK_TF, 2), "cases": rows}
    line = json.dumps(out)
    print(line)
    if args.out:
        with open(args.out, "a") as f:
            f.write(line + "\n")


if __name__ == "__main__":
    main()
