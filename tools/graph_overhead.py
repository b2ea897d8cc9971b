"""Diagnose per-kernel overhead inside CUDA graphs for the C2 step (GPU).

Times graph replays of: 9 sparsify launches, 9 SpMM launches, the full step,
and the step with 9 extra empty kernels, to separate launch/ramp overhead from work.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import json  # noqa: E402

import torch  # noqa: E402

import synthetic  # noqa: E402
from paper_2304_07613_b200 import sten  # noqa: E402


def timed(fn, reps=20):
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn()
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s):
        fn()
    torch.cuda.synchronize()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    return round(ts[len(ts) // 2], 1)


def main():
    cases = synthetic.config_cases(1, g=4)
    data = []
    for c in cases:
        W = torch.randn(c.M, c.Kp, device="cuda") * 0.02
        B = torch.randn(c.Kp, c.N, device="cuda")
        v, i = sten.sparsify_grouped_nm(W, c.n, c.m, c.g)
        C = torch.empty(c.M, c.N, device="cuda")
        plan = sten.spmm_plan(c.n, c.m, c.g, c.M, c.Kp, c.N)
        data.append((c, W, B, v, i, C, plan))
    dummy = torch.empty(1, device="cuda")

    def sparsify_all():
        for c, W, B, v, i, C, plan in data:
            sten.sparsify_grouped_nm(W, c.n, c.m, c.g, values=v, idx=i)

    def spmm_all():
        for c, W, B, v, i, C, plan in data:
            sten.spmm_grouped_nm(v, i, B, c.n, c.m, c.g, out=C, plan=plan)

    def step():
        for c, W, B, v, i, C, plan in data:
            sten.sparsify_grouped_nm(W, c.n, c.m, c.g, values=v, idx=i)
            sten.spmm_grouped_nm(v, i, B, c.n, c.m, c.g, out=C, plan=plan)

    def empties():
        for _ in data:
            dummy.add_(1.0)

    def spmm_nosplit():
        for c, W, B, v, i, C, plan in data:
            sten.spmm_grouped_nm(v, i, B, c.n, c.m, c.g, out=C, plan=sten.make_plan(1, 1, plan.tile))

    res = {"sparsify_x9_us": timed(sparsify_all), "spmm_x9_us": timed(spmm_all), "step_us": timed(step),
           "empty_x9_us": timed(empties), "spmm_x9_split1_us": timed(spmm_nosplit)}
    for k, (c, W, B, v, i, C, plan) in enumerate(data):
        res["spmm_%d_us" % k] = timed(lambda: sten.spmm_grouped_nm(v, i, B, c.n, c.m, c.g, out=C, plan=plan))
        res["sparsify_%d_us" % k] = timed(lambda: sten.sparsify_grouped_nm(W, c.n, c.m, c.g, values=v, idx=i))
    print(json.dumps(res))


if __name__ == "__main__":
    main()
