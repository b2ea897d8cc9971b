"""One chunked n:m:g conversion + SpMM of a given shape (for ncu captures):
python tools/nmg_one.py M K N n m g"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2304_07613_b200 import sten
M, K, N, n, m, g = map(int, sys.argv[1:7])
W = torch.randn(M, K, device="cuda") * 0.02
B = torch.randn(K, N, device="cuda")
for _ in range(2):
    v, i = sten.nmg_sparsify(W, n, m, g)
    C = sten.nmg_spmm(v, i, B, n, m, g)
torch.cuda.synchronize()
