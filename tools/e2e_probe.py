"""End-to-end (host buffers) schedules of the C2 step (tools only): per-case sten_sparse_linear_host_async
on L lanes vs the pipelined call (one copy-in / compute / copy-out stream triple, or two triples on
alternating cases).  Prints ms per step for each."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import synthetic
from paper_2304_07613_b200 import sten

cases = synthetic.config_cases(1, g=4, dtype="f32")
bufs = []
for k, c in enumerate(cases):
    W = synthetic.weights(c.M, c.K, seed=k, k_pad=c.k_pad)
    B = synthetic.activations(c.K, c.N, seed=100 + k, k_pad=c.k_pad)
    Wh, Bh = torch.from_numpy(W).pin_memory(), torch.from_numpy(B).pin_memory()
    Ch = torch.empty((c.M, c.N)).pin_memory()
    ws = torch.empty(sten.sparse_linear_host_workspace_size(c.n, c.m, c.g, c.M, c.Kp, c.N), dtype=torch.uint8,
                     device="cuda")
    bufs.append((Wh, Bh, c.n, c.m, c.g, Ch, ws))
main = torch.cuda.current_stream()


def timed(step, n=10):
    for _ in range(2):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        step()
    e1.record()
    torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) / n, 4)


def forked(streams, body):
    def step():
        ev = torch.cuda.Event()
        ev.record(main)
        for s in streams:
            s.wait_event(ev)
        body()
        for s in streams:
            main.wait_stream(s)
    return step


out = {}
for L in (3, 9):
    lanes = [torch.cuda.Stream() for _ in range(L)]
    out["lanes%d" % L] = timed(forked(lanes, lambda: [sten.sparse_linear_host_async(p[0], p[1], p[2], p[3], p[4], p[5], p[6],
                                                                                      stream=lanes[k % L])
                                                     for k, p in enumerate(bufs)]))
by_c = sorted(range(9), key=lambda k: -(cases[k].M * cases[k].N))
by_in = sorted(range(9), key=lambda k: cases[k].M * cases[k].Kp + cases[k].Kp * cases[k].N)
tri = [torch.cuda.Stream() for _ in range(3)]
for name, order in (("pipe_largestC_first", by_c), ("pipe_smallest_in_first", by_in), ("pipe_given", list(range(9)))):
    probs = [bufs[k] for k in order]
    out[name] = timed(forked(tri, lambda: sten.sparse_linear_host_pipelined_async(probs, *tri)))
tri2 = [torch.cuda.Stream() for _ in range(3)]
probs = [bufs[k] for k in by_c]
out["pipe_two_triples"] = timed(forked(tri + tri2, lambda: (sten.sparse_linear_host_pipelined_async(probs[0::2], *tri),
                                                            sten.sparse_linear_host_pipelined_async(probs[1::2], *tri2))))
print(json.dumps(out))
# the same copies as the pipelined call without the kernels (copy-in stream, copy-out stream)
dev_in = [(torch.empty(p[0].shape, device="cuda"), torch.empty(p[1].shape, device="cuda"),
           torch.empty(p[5].shape, device="cuda")) for p in bufs]


def copies_only():
    ev = torch.cuda.Event()
    ev.record(main)
    tri[0].wait_event(ev)
    tri[2].wait_event(ev)
    for k in by_in:
        with torch.cuda.stream(tri[0]):
            dev_in[k][0].copy_(bufs[k][0], non_blocking=True)
            dev_in[k][1].copy_(bufs[k][1], non_blocking=True)
        with torch.cuda.stream(tri[2]):
            bufs[k][5].copy_(dev_in[k][2], non_blocking=True)
    main.wait_stream(tri[0])
    main.wait_stream(tri[2])


print(json.dumps({"copies_only_27": timed(copies_only)}))
