"""NEXT-3 measurement: SpMM with bias + GELU fused into the epilogue vs the SpMM followed by
torch's bias add and GELU (BERT-base FFN1 shapes).  Per-launch device time of R back-to-back
steps in a CUDA graph over rotating inputs (> L2), CUDA events, median of 5."""
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


rows = []
for (M, K, N, n, m, g) in [(3072, 768, 1024, 2, 4, 4), (3072, 768, 4096, 2, 4, 4), (3072, 768, 4096, 1, 4, 4)]:
    R = 8
    W = torch.from_numpy(synthetic.weights(M, K, seed=1)).cuda()
    Bs = [torch.from_numpy(synthetic.activations(K, N, seed=2 + r)).cuda() for r in range(R)]
    bias = (torch.randn(M, device="cuda") * 0.02).contiguous()
    v, i = sten.sparsify_grouped_nm(W, n, m, g)
    Cs = [torch.empty((M, N), device="cuda") for _ in range(R)]
    plan = sten.spmm_autotune(v, i, Bs[0], n, m, g, out=Cs[0], reps=5)
    plan.algo = sten.ALGO_SIMT

    def unfused(k):
        C = sten.spmm_grouped_nm(v, i, Bs[k % R], n, m, g, out=Cs[k % R], plan=plan)
        C.add_(bias[:, None])
        torch.nn.functional.gelu(C, approximate="none")
    def fused(k):
        sten.spmm_grouped_nm_bias_act(v, i, Bs[k % R], n, m, g, bias=bias, act=sten.ACT_GELU, out=Cs[k % R], plan=plan)
    t_u, t_f = graph_us(unfused, R), graph_us(fused, R)
    rows.append({"case": "%dx%dx%d %d:%d:%d" % (M, K, N, n, m, g), "plan": plan.as_dict(),
                 "spmm+torch_bias_gelu_us": round(t_u, 2), "fused_us": round(t_f, 2), "speedup": round(t_u / t_f, 3)})
    print(json.dumps(rows[-1]), flush=True)
