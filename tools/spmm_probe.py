"""Per-launch SpMM time of the C2 cases: R back-to-back launches (rotating input copies) in one
CUDA graph, CUDA events around the replay on the replaying stream (diagnostic tool; compares with
the event-node-bracketed times of bench.py)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synthetic
from paper_2304_07613_b200 import sten


def graph_us(fn, R, reps=5):
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
        e0.record(); gph.replay(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / R)
    return sorted(ts)[len(ts) // 2]


for c in synthetic.config_cases(1, g=4, dtype="f32"):
    R = 8
    Ws = [torch.from_numpy(synthetic.weights(c.M, c.K, seed=1, k_pad=c.k_pad)).cuda() for _ in range(R)]
    Bs = [torch.from_numpy(synthetic.activations(c.K, c.N, seed=2, k_pad=c.k_pad)).cuda() for _ in range(R)]
    vi = [sten.sparsify_grouped_nm(W, c.n, c.m, c.g) for W in Ws]
    Cs = [torch.empty((c.M, c.N), device="cuda") for _ in range(R)]
    plan = sten.spmm_autotune(vi[0][0], vi[0][1], Bs[0], c.n, c.m, c.g, out=Cs[0], reps=5)
    t = graph_us(lambda i: sten.spmm_grouped_nm(vi[i % R][0], vi[i % R][1], Bs[i % R], c.n, c.m, c.g,
                                                out=Cs[i % R], plan=plan), R)
    nz = 2.0 * c.M * c.kept * c.N
    print(json.dumps({"case": c.label(), "plan": plan.as_dict(), "spmm_us_b2b": round(t, 2),
                      "nz_tflops": round(nz / t / 1e6, 2)}), flush=True)
