"""Plan sweep for one SpMM shape (GPU): times every (tile, split) variant with CUDA events.

    python tools/sweep.py --M 768 --K 3072 --N 1024 --n 2 --m 4 --g 4 [--dtype f32]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2304_07613_b200 import sten  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    for k, v in dict(M=768, K=3072, N=1024, n=2, m=4, g=4).items():
        p.add_argument("--" + k, type=int, default=v)
    p.add_argument("--dtype", default="f32")
    p.add_argument("--algo", type=int, default=1)
    p.add_argument("--tiles", default="1,2,3")
    p.add_argument("--splits", default="1,2,3,4,6,8")
    p.add_argument("--reps", type=int, default=20)
    a = p.parse_args()
    dt = torch.float32 if a.dtype == "f32" else torch.bfloat16
    W = (torch.randn(a.M, a.K, device="cuda") * 0.02).to(dt)
    B = torch.randn(a.K, a.N, device="cuda").to(dt)
    v, i = sten.sparsify_grouped_nm(W, a.n, a.m, a.g)
    C = torch.empty(a.M, a.N, device="cuda", dtype=dt)
    nz = 2.0 * a.M * (a.K // a.m * a.n) * a.N
    auto = sten.spmm_plan(a.n, a.m, a.g, a.M, a.K, a.N, ab_dtype=dt, c_dtype=dt).as_dict()
    flush = torch.empty(256 * 2 ** 20 // 4, device="cuda")
    res = []
    for tile in [int(x) for x in a.tiles.split(",")]:
        for split in [int(x) for x in a.splits.split(",")]:
            plan = sten.make_plan(a.algo, split_k=split, tile=tile)
            try:
                sten.spmm_grouped_nm(v, i, B, a.n, a.m, a.g, out=C, plan=plan)
                torch.cuda.synchronize()
            except Exception as e:  # unsupported variant
                res.append({"tile": tile, "split": split, "err": str(e)[:60]})
                continue
            ts = []
            for _ in range(a.reps):
                flush.zero_()
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record()
                sten.spmm_grouped_nm(v, i, B, a.n, a.m, a.g, out=C, plan=plan)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            ts.sort()
            t = ts[len(ts) // 2]
            res.append({"tile": tile, "split": split, "us": round(t * 1e3, 2), "nz_tflops": round(nz / (t * 1e-3) / 1e12, 2)})
    print(json.dumps({"shape": vars(a), "auto": auto, "results": res}))


if __name__ == "__main__":
    main()
