"""Fig.-6 analogue: kept-magnitude energy of grouped n:m (A) and chunked
n:m:g (B) over g on seeded N(0, 0.02^2) weights (CPU oracle; the pinned statistical claims are
tests/test_energy_sweep.py).  Writes profiles/energy_sweep_r02.json."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import synthetic  # noqa: E402

M, K = 768, 3072          # the BERT-base FFN2 weight shape (C2)
rows = []
for (n, m) in [(2, 4), (1, 4), (1, 8), (2, 8), (3, 6)]:
    for g in (1, 2, 4, 8, 16, 32):
        W = synthetic.weights(M, K, seed=1234)
        r = {"n": n, "m": m, "g": g}
        if K % m == 0 and M % g == 0:
            v, i = oracle.sparsify(W, n, m, g)
            r["grouped_A"] = round(oracle.energy(oracle.densify(v, i, n, m, g, K), W), 5)
        L = oracle.nmg_chunk(n, m, g)
        if K % L == 0 and M % m == 0:
            v, i = oracle.nmg_sparsify(W, n, m, g)
            r["chunked_B"] = round(oracle.energy(oracle.nmg_densify(v, i, n, m, g, K), W), 5)
        print(r, flush=True)
        rows.append(r)
out = {"_what": "energy ||X^||_1/||X||_1 (PAPER.md:648) of one seeded %dx%d N(0,0.02^2) weight" % (M, K),
       "rows": rows}
with open(os.path.join(ROOT, "profiles", "energy_sweep_r02.json"), "w") as f:
    json.dump(out, f, indent=1)
