"""One SpMM of a given shape and plan (for ncu captures):
python tools/spmm_one.py M K N n m g algo split tile [bf16]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2304_07613_b200 import sten
M, K, N, n, m, g, algo, split, tile = map(int, sys.argv[1:10])
dt = torch.bfloat16 if len(sys.argv) > 10 and sys.argv[10] == "bf16" else torch.float32
W = (torch.randn(M, K, device="cuda") * 0.02).to(dt)
B = torch.randn(K, N, device="cuda").to(dt)
v, i = sten.sparsify_grouped_nm(W, n, m, g)
plan = sten.make_plan(algo, split_k=split, tile=tile)
for _ in range(2):
    C = sten.spmm_grouped_nm(v, i, B, n, m, g, plan=plan)
torch.cuda.synchronize()
