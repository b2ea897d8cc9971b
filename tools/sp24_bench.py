"""K6 (2:4 sparse tcgen05) timing probe on the C3 / C4 / C5 bf16 shapes: every tile variant,
the pack, and dense cuBLAS on densify(W) (context).  Prints one JSON line per case.
   python tools/sp24_bench.py [--config 2|3|4] [--g 4] [--reps 20]"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synthetic  # noqa: E402
from paper_2304_07613_b200 import sten  # noqa: E402


def timed(fn, reps, rot):
    for i in range(3):
        fn(i % rot)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    ts = []
    for r in range(reps):
        e0.record()
        fn(r % rot)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--g", type=int, default=4)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--tiles", default="1,2,3,4,5")
    args = ap.parse_args()
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    cases = synthetic.config_cases(args.config, g=args.g, dtype="bf16")
    for c in cases:
        if not sten.sp24_compatible(c.n, c.m):
            continue
        K = c.K + synthetic.pad_for(c.K, c.m, 1) if c.K % c.m else c.K
        W = torch.randn(c.M, K, device="cuda").mul_(0.02).bfloat16()
        # rotate input copies so the timed working set exceeds L2 (126 MB)
        bbytes = K * c.N * 2
        rot = max(2, int(3 * 126e6 // bbytes) + 1)
        Bs = [torch.randn(K, c.N, device="cuda").bfloat16() for _ in range(rot)]
        v, i = sten.sparsify_grouped_nm(W, c.n, c.m, c.g)
        v24, meta = sten.sp24_pack(v, i, c.n, c.m, c.g, K)
        Cout = torch.empty(c.M, c.N, device="cuda", dtype=torch.bfloat16)
        flops = 2.0 * c.M * c.K * c.N
        nz = flops * c.n / c.m
        row = {"case": "%dx%dx%d %d:%d:g%d bf16" % (c.M, c.K, c.N, c.n, c.m, c.g)}
        t_pack = timed(lambda r: sten.sp24_pack(v, i, c.n, c.m, c.g, K), args.reps, 1)
        row["pack_us"] = round(t_pack, 2)
        for tile in [int(x) for x in args.tiles.split(",")]:
            t = timed(lambda r: sten.spmm_sp24(v24, meta, c.M, K, Bs[r], out=Cout, tile=tile), args.reps, rot)
            row["tile%d_us" % tile] = round(t, 2)
            row["tile%d_eff_tflops" % tile] = round(flops / t / 1e6, 1)
        D = sten.densify(v, i, c.n, c.m, c.g, K)
        td = timed(lambda r: torch.matmul(D, Bs[r], out=Cout), args.reps, rot)
        row["dense_cublas_us"] = round(td, 2)
        row["dense_cublas_eff_tflops"] = round(flops / td / 1e6, 1)
        best = min(row["tile%d_us" % t] for t in [int(x) for x in args.tiles.split(",")])
        hbm = peaks.get("hbm_gbs", 6537.0)
        byts = c.M * K * c.n / c.m * 2 + c.M // c.g * K // c.m * c.n + K * c.N * 2 + c.M * c.N * 2
        tf = peaks.get("bf16_tflops", 1664.9)
        t_roof = max(nz / tf / 1e6, byts / hbm / 1e3)
        row["roofline_frac_best"] = round(t_roof / best, 3)
        row["speedup_vs_dense"] = round(td / best, 2)
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
