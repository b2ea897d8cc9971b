"""One-rank NCCL smoke of parallel.FusedAllGatherSpmm (symmetric memory + fused-epilogue SpMM)."""
import os, sys, torch, torch.distributed as dist
sys.path.insert(0, os.getcwd())
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29533")  # tests pass a free port
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
import synthetic
from paper_2304_07613_b200 import sten, parallel
n, m, g, M, K, N = 2, 4, 4, 96, 256, 300
W = torch.from_numpy(synthetic.weights(M, K, seed=1)).cuda(); B = torch.from_numpy(synthetic.activations(K, N, seed=2)).cuda()
v, i = sten.sparsify_grouped_nm(W, n, m, g)
f = parallel.FusedAllGatherSpmm(v, i, n, m, g, K, N)
C = f.forward(B)
ref = sten.spmm_grouped_nm(v, i, B, n, m, g, plan=f.plan)
torch.cuda.synchronize()
print("fused world=1 equal:", torch.equal(C, ref))
dist.destroy_process_group()
