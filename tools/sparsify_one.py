"""One sparsify launch of a given shape (for ncu captures): python tools/sparsify_one.py M K n m g [bf16]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2304_07613_b200 import sten
M, K, n, m, g = map(int, sys.argv[1:6])
dt = torch.bfloat16 if len(sys.argv) > 6 and sys.argv[6] == "bf16" else torch.float32
W = (torch.randn(M, K, device="cuda") * 0.02).to(dt)
for _ in range(2):
    sten.sparsify_grouped_nm(W, n, m, g)
torch.cuda.synchronize()
