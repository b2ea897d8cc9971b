"""Per-CTA timeline of the C2 grouped split-K SpMM launch (instrumented -DSTEN_TIMING build; tools only).
Stamps per CTA: 0 start, 1 setup done, 2 first slab ready, 3 main loop done, 4 partial parked,
5 reduction done (last part only), 7 = smid + 1.  Reports the launch span, per-SM busy time (sum of
its CTAs' start..end), the idle fraction, and where the time of an average CTA goes."""
import ctypes, json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("STEN_LIB_PATH", os.path.join(ROOT, "build", "libsten_timing.so"))
import numpy as np
import torch
import synthetic
from paper_2304_07613_b200 import sten

tile = int(os.environ.get("TILE", "2"))
cases = synthetic.config_cases(1, g=4, dtype="f32")
probs = []
for k, c in enumerate(cases):
    W = torch.from_numpy(synthetic.weights(c.M, c.K, seed=k, k_pad=c.k_pad)).cuda()
    B = torch.from_numpy(synthetic.activations(c.K, c.N, seed=100 + k, k_pad=c.k_pad)).cuda()
    v, i = sten.sparsify_grouped_nm(W, c.n, c.m, c.g)
    probs.append((v, i, B, c.n, c.m, c.g, torch.empty((c.M, c.N), device="cuda")))
nb = sten.batched_workspace_size(probs, None, tile)
ws = torch.zeros(max(nb, 16) // 4 + 4, device="cuda")
lib = sten.load()
lib.sten_debug_timing.argtypes = [ctypes.c_void_p, ctypes.c_int]
flush = torch.empty(256 * 2 ** 20, dtype=torch.uint8, device="cuda")
for _ in range(3):
    flush.fill_(1)
    sten.spmm_grouped_nm_batched_ex(probs, ws, None, tile)
torch.cuda.synchronize()
buf = np.zeros((16384, 8), dtype=np.uint64)
lib.sten_debug_timing(buf.ctypes.data, 16384)
rows = buf[buf[:, 0] > 0].astype(np.int64)
t0 = rows[:, 0].min()
st = rows[:, :7].copy()
st[:, 1:7][st[:, 1:7] < st[:, [0]]] = 0          # stamps left over from an earlier launch
end = st[:, 1:7].max(axis=1)
span = (end.max() - t0) / 1e3
sm = rows[:, 7] - 1
busy = np.zeros(int(sm.max()) + 1)
for s_, a_, e_ in zip(sm, st[:, 0], end):
    busy[s_] += (e_ - a_) / 1e3


def mean_gap(a, b):
    ok = (st[:, a] > 0) & (st[:, b] > 0)
    return round(float(((st[ok, b] - st[ok, a]) / 1e3).mean()), 2) if ok.any() else None


out = {"tile": tile, "ctas": int(len(rows)), "span_us": round(span, 2),
       "sm_busy_mean_us": round(float(busy.mean()), 2), "sm_busy_min_us": round(float(busy.min()), 2),
       "idle_frac": round(1 - float(busy.mean()) / span, 4),
       "cta_mean_us": {"setup": mean_gap(0, 1), "first_slab": mean_gap(1, 2), "main_loop": mean_gap(2, 3),
                       "park": mean_gap(3, 4), "reduce_last": mean_gap(4, 5),
                       "total": round(float(((end - st[:, 0]) / 1e3).mean()), 2)},
       "last_start_us": round((rows[:, 0].max() - t0) / 1e3, 2)}
# end-time distribution of the SMs (tail)
sm_end = np.zeros(int(sm.max()) + 1)
for s_, e_ in zip(sm, end):
    sm_end[s_] = max(sm_end[s_], (e_ - t0) / 1e3)
out["sm_end_us_pct"] = {p: round(float(np.percentile(sm_end, p)), 2) for p in (0, 10, 50, 90, 100)}
print(json.dumps(out))
