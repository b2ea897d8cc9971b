"""Host link probe: pinned H2D of the C2 step's input bytes, D2H of its output bytes, and both at once (tools only)."""
import torch, json
h = torch.empty(121 * 2**20, dtype=torch.uint8).pin_memory()
d = torch.empty_like(h, device="cuda")
ho = torch.empty(57 * 2**20, dtype=torch.uint8).pin_memory()
do = torch.empty_like(ho, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, n=5):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); 
    for _ in range(n): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n
def h2d():
    d.copy_(h, non_blocking=True)
def d2h():
    ho.copy_(do, non_blocking=True)
def both():
    cur = torch.cuda.current_stream()
    ev = torch.cuda.Event(); ev.record(cur)
    s1.wait_event(ev); s2.wait_event(ev)
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): ho.copy_(do, non_blocking=True)
    cur.wait_stream(s1); cur.wait_stream(s2)
a, b, c = t(h2d), t(d2h), t(both)
print(json.dumps({"h2d_121MB_ms": round(a, 3), "h2d_GBs": round(121 * 2**20 / a / 1e6, 1), "d2h_57MB_ms": round(b, 3),
                  "d2h_GBs": round(57 * 2**20 / b / 1e6, 1), "both_ms": round(c, 3)}))
