"""One grouped split-K launch over the 9 C2 SpMMs (for ncu; tools only)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
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
for _ in range(3):
    sten.spmm_grouped_nm_batched_ex(probs, ws, None, tile)
torch.cuda.synchronize()
print("ok")
