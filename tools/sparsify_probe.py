"""Time sten_sparsify_grouped_nm alone (events, back-to-back launches) against a plain
device copy of the same bytes, warm (one W) and cold (rotating Ws > L2).  Diagnostic tool."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2304_07613_b200 import sten

def timeit(fn, reps=40):
    """per-launch device time of `reps` launches captured in one CUDA graph (no host overhead)"""
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3): fn(0)
    torch.cuda.synchronize()
    gph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gph, stream=s):
        for i in range(reps): fn(i)
    gph.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); gph.replay(); e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3

out = []
for (M, K, n, m, g) in [(768, 768, 2, 4, 4), (768, 3072, 2, 4, 4), (3072, 768, 1, 4, 4), (768, 800, 1, 10, 4),
                        (8192, 8192, 1, 8, 4)]:
    R = max(2, int(3 * 126e6 // (M * K * 4)) + 1)
    Ws = [torch.randn(M, K, device="cuda") * 0.02 for _ in range(R)]
    vals = torch.empty(M, K // m * n, device="cuda")
    idx = torch.empty(M // g, K // m, n, dtype=torch.uint8, device="cuda")
    dst = torch.empty(M, K // m * n, device="cuda")
    f = lambda i: sten.sparsify_grouped_nm(Ws[i % R], n, m, g, values=vals, idx=idx)
    warm = timeit(lambda i: sten.sparsify_grouped_nm(Ws[0], n, m, g, values=vals, idx=idx))
    cold = timeit(f)
    cp = timeit(lambda i: dst.copy_(Ws[i % R][:, : K // m * n]))
    sf = timeit(lambda i: sten.resparsify_same_format(Ws[i % R], idx, n, m, g, values=vals))
    byts = M * K * 4 + M * K // m * n * 4 + M // g * K // m * n
    out.append(dict(shape=[M, K, n, m, g], warm_us=round(warm, 2), cold_us=round(cold, 2), copy_us=round(cp, 2), same_format_us=round(sf, 2),
                    cold_gbs=round(byts / cold / 1e3, 1)))
    print(json.dumps(out[-1]), flush=True)
