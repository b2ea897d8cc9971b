"""Grouped sparsify of the C2 step's 9 weights: ONE mixed launch vs one launch per (m, n) class vs one
launch per weight (tools only).  R rotating input sets (R x bytes > 3 x L2), each variant as R
back-to-back launches in one CUDA graph, CUDA events around the replay; prints us per step and GB/s
of the algorithmic bytes (read W, write values + idx)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import synthetic
from paper_2304_07613_b200 import sten

cfg = int(os.environ.get("CFG", "1"))
dtype = os.environ.get("DT", "f32")
g = int(os.environ.get("G", "4"))
cases = synthetic.config_cases(cfg, g=g, dtype=dtype)
tdt = torch.float32 if dtype == "f32" else torch.bfloat16
s = 4 if dtype == "f32" else 2
nbytes = sum(c.M * c.Kp * s + c.M * c.kept * s + (c.M // c.g) * (c.Kp // c.m) * c.n for c in cases)
R = max(2, -(-3 * 126 * 2 ** 20 // nbytes))
sets = []
for r in range(R):
    data = []
    for k, c in enumerate(cases):
        W = synthetic.weights(c.M, c.K, seed=k, dtype=dtype, k_pad=c.k_pad)
        Wt = torch.from_numpy(W.view("int16") if dtype == "bf16" else W)
        Wt = (Wt.view(torch.bfloat16) if dtype == "bf16" else Wt).cuda()
        data.append((Wt, c.n, c.m, c.g, torch.empty((c.M, c.kept), dtype=tdt, device="cuda"),
                     torch.empty((c.M // c.g, c.Kp // c.m, c.n), dtype=torch.uint8, device="cuda")))
    sets.append(data)
classes = sorted({(c.m, c.n) for c in cases})


def mixed(r):
    sten.sparsify_grouped_nm_batched(sets[r])


def per_class(r):
    for cl in classes:
        sten.sparsify_grouped_nm_batched([p for p in sets[r] if (p[2], p[1]) == cl])


def per_weight(r):
    for (W, n, m, gg, v, i) in sets[r]:
        sten.sparsify_grouped_nm(W, n, m, gg, values=v, idx=i)


out = {"config": cfg, "dtype": dtype, "g": g, "bytes_per_step": nbytes, "R": R}
st = torch.cuda.Stream()
variants = (("mixed", mixed), ("per_class", per_class), ("per_weight", per_weight))
if os.environ.get("ONLY"):
    variants = [v for v in variants if v[0] == os.environ["ONLY"]]
for name, fn in variants:
    with torch.cuda.stream(st):
        for r in range(R):
            fn(r)
    torch.cuda.synchronize()
    gph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gph, stream=st):
        for r in range(R):
            fn(r)
    gph.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        gph.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / R)
    t = sorted(ts)[2]
    out[name] = {"us": round(t * 1e3, 2), "gbs": round(nbytes / (t * 1e-3) / 1e9, 1)}
    del gph
# the mixed launch's results equal the per-weight launches (same bits)
mixed(0)
ref = [(v.clone(), i.clone()) for (_, _, _, _, v, i) in sets[0]]
per_weight(0)
torch.cuda.synchronize()
out["same_bits"] = all(torch.equal(a[0].view(torch.int16 if dtype == "bf16" else torch.int32),
                                   p[4].view(torch.int16 if dtype == "bf16" else torch.int32)) and torch.equal(a[1], p[5])
                       for a, p in zip(ref, sets[0]))
print(json.dumps(out))
