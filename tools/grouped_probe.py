"""C2 SpMMs: one grouped launch (sten_spmm_grouped_nm_batched) vs the 9 per-case launches (tuned
plans, one stream) vs the 9 launches on 9 streams; R rotating input sets (> L2), CUDA graphs,
CUDA events on the replaying stream, median of 5."""
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
plans = [sten.spmm_autotune(v, i, B, n, m, g, out=C, reps=5) for (v, i, B, n, m, g, C) in sets[0]]
lanes = [torch.cuda.Stream() for _ in cases]


def graph_us(fn, reps=5):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for r in range(R):
            fn(r, s)
    torch.cuda.synchronize()
    gph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gph, stream=s):
        for r in range(R):
            fn(r, s)
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); gph.replay(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / R)
    return sorted(ts)[len(ts) // 2]


def single(r, s):
    for (v, i, B, n, m, g, C), p in zip(sets[r], plans):
        sten.spmm_grouped_nm(v, i, B, n, m, g, out=C, plan=p)


def multi(r, s):
    fork = torch.cuda.Event(); fork.record(s)
    for ls, (v, i, B, n, m, g, C), p in zip(lanes, sets[r], plans):
        ls.wait_event(fork)
        with torch.cuda.stream(ls):
            sten.spmm_grouped_nm(v, i, B, n, m, g, out=C, plan=p)
    for ls in lanes:
        s.wait_stream(ls)


def grouped(tile):
    def f(r, s):
        sten.spmm_grouped_nm_batched(sets[r], tile=tile)
    return f


wss = {}


def grouped_split(tile, splits=None):
    key = (tile, None if splits is None else tuple(splits))
    nb = sten.batched_workspace_size(sets[0], splits, tile)
    wss[key] = [torch.zeros(max(nb, 16) // 4 + 4, device="cuda") for _ in range(R)]

    def f(r, s):
        sten.spmm_grouped_nm_batched_ex(sets[r], wss[key][r], splits, tile)
    return f


nz = sum(2.0 * c.M * c.kept * c.N for c in cases)
out = {"single_stream_us": graph_us(single), "nine_streams_us": graph_us(multi),
       "grouped_tile1_us": graph_us(grouped(1)), "grouped_tile2_us": graph_us(grouped(2)),
       "grouped_split_auto_tile1_us": graph_us(grouped_split(1)),
       "grouped_split_auto_tile2_us": graph_us(grouped_split(2))}
for f in (1, 2, 4):
    for tile in (1, 2):
        # splits proportional to K' with the factor f (K' = 1536 -> 4 f ... clipped at 8)
        sp = [max(1, min(8, round(f * c.kept / 384))) for c in cases]
        out["grouped_split_x%d_tile%d_us" % (f, tile)] = graph_us(grouped_split(tile, sp))
out = {k: round(v, 2) for k, v in out.items()}
out["nz_tflops"] = {k: round(nz / (v * 1e-6) / 1e12, 2) for k, v in out.items()}
print(json.dumps(out))
