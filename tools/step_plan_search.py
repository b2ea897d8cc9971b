"""Coordinate search of the per-case SpMM plans for the CONCURRENT C2 step (9 lanes, sparsify +
SpMM per lane, one CUDA graph per input set, R rotating sets > L2): start from the plan cache,
try alternatives case by case, keep a change only if the step improves by > 1 %.  Writes the
best plan set to --out.  (Tuning tool; the bench reads the result as its plan cache.)"""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synthetic
from paper_2304_07613_b200 import sten

ap = argparse.ArgumentParser()
ap.add_argument("--start", default="paper_2304_07613_b200/plans/c2_f32_g4_step.json")
ap.add_argument("--out", default="gpurun_out/c2_plans_searched.json")
args = ap.parse_args()
cases = synthetic.config_cases(1, g=4, dtype="f32")
R = 4
sets = []
for r in range(R):
    d = []
    for k, c in enumerate(cases):
        W = torch.from_numpy(synthetic.weights(c.M, c.K, seed=k, k_pad=c.k_pad)).cuda()
        B = torch.from_numpy(synthetic.activations(c.K, c.N, seed=100 + k, k_pad=c.k_pad)).cuda()
        v = torch.empty((c.M, c.kept), device="cuda")
        i = torch.empty((c.M // c.g, c.Kp // c.m, c.n), dtype=torch.uint8, device="cuda")
        d.append(dict(W=W, B=B, v=v, i=i, C=torch.empty((c.M, c.N), device="cuda")))
    sets.append(d)
lanes = [torch.cuda.Stream() for _ in cases]
start = json.load(open(args.start))
plans = {c.label(): start[c.label()] for c in cases}


def step_us(plans, reps=5):
    pl = [sten.make_plan(plans[c.label()]["algo"], plans[c.label()]["split_k"], plans[c.label()]["tile"]) for c in cases]
    s = torch.cuda.Stream()
    graphs = []
    for r in range(R):
        def run():
            fork = torch.cuda.Event(); fork.record(s)
            for ls, c, d, p in zip(lanes, cases, sets[r], pl):
                ls.wait_event(fork)
                with torch.cuda.stream(ls):
                    sten.sparsify_grouped_nm(d["W"], c.n, c.m, c.g, values=d["v"], idx=d["i"])
                    sten.spmm_grouped_nm(d["v"], d["i"], d["B"], c.n, c.m, c.g, out=d["C"], plan=p)
            for ls in lanes:
                s.wait_stream(ls)
        with torch.cuda.stream(s):
            run()
        torch.cuda.synchronize()
        gph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gph, stream=s):
            run()
        graphs.append(gph)
    for gph in graphs:
        gph.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            for gph in graphs:
                gph.replay()
        e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / (5 * R))
    return sorted(ts)[len(ts) // 2]


cands = [(t, s) for t in (1, 4, 5, 6, 7) for s in (1, 2, 3, 4, 5)]
best = step_us(plans)
print("start", round(best, 2), flush=True)
for c in cases:
    lab = c.label()
    cur = plans[lab]
    for (t, sp) in cands:
        if t == cur["tile"] and sp == cur["split_k"]:
            continue
        trial = dict(plans)
        trial[lab] = {"algo": 1, "split_k": sp, "tile": t}
        try:
            u = step_us(trial, reps=3)
        except Exception:
            continue
        if u < best * 0.99:
            u2 = step_us(trial)                                   # confirm
            if u2 < best * 0.99:
                best, plans = u2, trial
                print("improved", lab, t, sp, round(best, 2), flush=True)
print("final", round(best, 2))
json.dump(plans, open(args.out, "w"), indent=1)
