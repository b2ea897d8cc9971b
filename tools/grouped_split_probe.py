"""Grouped split-K launch over subsets of the C2 problems (per sparsity), tile 2 vs others, to see
where the grouped step's time goes (tools only)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synthetic
from paper_2304_07613_b200 import sten

cases = synthetic.config_cases(1, g=4, dtype="f32")
R = 4
sets = []
for r in range(R):
    d = []
    for k, c in enumerate(cases):
        W = torch.from_numpy(synthetic.weights(c.M, c.K, seed=k, k_pad=c.k_pad)).cuda()
        B = torch.from_numpy(synthetic.activations(c.K, c.N, seed=100 + k, k_pad=c.k_pad)).cuda()
        v, i = sten.sparsify_grouped_nm(W, c.n, c.m, c.g)
        d.append((v, i, B, c.n, c.m, c.g, torch.empty((c.M, c.N), device="cuda")))
    sets.append(d)


def graph_us(fn, reps=5):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for r in range(R):
            fn(r)
    torch.cuda.synchronize()
    gph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gph, stream=s):
        for r in range(R):
            fn(r)
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); gph.replay(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / R)
    return sorted(ts)[len(ts) // 2]


out = {}
for label, sel in [("all", range(9)), ("2:4", [0, 3, 6]), ("1:4", [1, 4, 7]), ("1:10", [2, 5, 8]),
                   ("2:4+1:4", [0, 1, 3, 4, 6, 7])]:
    sel = list(sel)
    nz = sum(2.0 * cases[k].M * cases[k].kept * cases[k].N for k in sel)
    for tile in (0, 2):
        probs = [[sets[r][k] for k in sel] for r in range(R)]
        nb = sten.batched_workspace_size(probs[0], None, tile)
        wss = [torch.zeros(max(nb, 16) // 4 + 4, device="cuda") for _ in range(R)]
        t = graph_us(lambda r: sten.spmm_grouped_nm_batched_ex(probs[r], wss[r], None, tile))
        out["%s_tile%d_us" % (label, tile)] = round(t, 2)
        out["%s_tile%d_frac" % (label, tile)] = round(nz / (t * 1e-6) / 74.45e12, 3)
print(json.dumps(out))
