"""World-size-1 NCCL run of every partition class of paper_2304_07613_b200.parallel with the
real CUDA compute (the C-ABI SpMM), checked element by element against the CPU oracle.

Run as a subprocess by tests/test_gpu_parity.py::test_partitions_nccl_world1_vs_oracle
(MASTER_ADDR / MASTER_PORT from the environment); prints one "CASE <name> ok|FAIL ..." line
per check and "ALL OK" at the end.  Test infrastructure: it may import oracle/.
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import synthetic  # noqa: E402
from paper_2304_07613_b200 import parallel, sten  # noqa: E402


def rel(C: torch.Tensor, C_ref: np.ndarray, Bound: np.ndarray) -> float:
    c = C.float().cpu().numpy().astype(np.float64)
    return float(np.max(np.abs(c - C_ref) / np.maximum(Bound, 1e-30)))


def main():
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    torch.cuda.set_device(0)
    ok_all = True

    def report(name, ok, extra=""):
        nonlocal ok_all
        ok_all &= bool(ok)
        print("CASE %s %s %s" % (name, "ok" if ok else "FAIL", extra), flush=True)

    for (dtype, n, m, g, M, K, N) in [("f32", 2, 4, 4, 200, 384, 1000), ("f32", 1, 10, 4, 96, 400, 333),
                                      ("bf16", 1, 4, 16, 256, 512, 520), ("bf16", 2, 4, 64, 256, 256, 300)]:
        tol = 1e-5 if dtype == "f32" else 2e-2
        tdt = torch.float32 if dtype == "f32" else torch.bfloat16
        W = synthetic.weights(M, K, seed=M + K, dtype=dtype)
        B = synthetic.activations(K, N, seed=N, dtype=dtype)
        Wt = torch.from_numpy(W.view(np.int16) if dtype == "bf16" else W)
        Bt = torch.from_numpy(B.view(np.int16) if dtype == "bf16" else B)
        if dtype == "bf16":
            Wt, Bt = Wt.view(torch.bfloat16), Bt.view(torch.bfloat16)
        Wd, Bd = Wt.cuda(), parallel.aligned_rows(Bt.cuda())   # 16-byte row pitch (TMA contract)
        v, i = sten.sparsify_grouped_nm(Wd, n, m, g)
        v_ref, i_ref = oracle.sparsify(W, n, m, g)
        C_ref, Bound = oracle.spmm(v_ref, i_ref, B, n, m, g)
        label = "%s %d:%d:g%d %dx%dx%d" % (dtype, n, m, g, M, K, N)
        report("sparsify " + label, np.array_equal(i.cpu().numpy(), i_ref))

        # token sharding, NCCL all-gather on the side stream, 3 chunks
        ts = parallel.TokenShardedSpmm.from_sten(v, i, n, m, g, K, N, out_dtype=torch.float32, chunks=3)
        c0, c1 = ts.local_range()
        C = ts.forward_allgather(Bd[:, c0:c1])
        torch.cuda.synchronize()
        e = rel(C, C_ref, Bound)
        report("token " + label, C.shape == (M, N) and e <= tol, "rel %.2e" % e)
        # P11: the sharded product equals the unsharded one with the global plan, bit for bit
        plan = sten.spmm_plan(n, m, g, M, K, N, ab_dtype=tdt, c_dtype=torch.float32)
        C1 = sten.spmm_grouped_nm(v, i, Bd, n, m, g, out_dtype=torch.float32, plan=plan)
        torch.cuda.synchronize()
        report("token-p11 " + label, torch.equal(C, C1))

        # row sharding: this rank's groups, B replicated, all-gather along M
        r0, r1 = parallel.group_range(M, g, 1, 0)
        rs = parallel.RowShardedSpmm(M, g, N, torch.float32, "cuda",
                                     parallel.sten_compute(v[r0:r1], i[r0 // g:r1 // g], n, m, g, plan,
                                                           torch.float32))
        C = rs.forward_allgather(Bd)
        torch.cuda.synchronize()
        e = rel(C, C_ref, Bound)
        report("row " + label, C.shape == (M, N) and e <= tol, "rel %.2e" % e)

        # all-gather fused into the SpMM epilogue over symmetric memory (peer stores)
        fz = parallel.FusedAllGatherSpmm(v, i, n, m, g, K, N, out_dtype=torch.float32)
        for rep in range(2):                     # twice: the pre-barrier path on buffer reuse
            C = fz.forward(Bd, copy=True)
        torch.cuda.synchronize()
        e = rel(C, C_ref, Bound)
        report("fused " + label, C.shape == (M, N) and e <= tol, "rel %.2e" % e)
        Cf = sten.spmm_grouped_nm(v, i, Bd, n, m, g, out_dtype=torch.float32, plan=fz.plan)
        torch.cuda.synchronize()
        report("fused-p11 " + label, torch.equal(C, Cf))
    dist.destroy_process_group()
    print("ALL OK" if ok_all else "SOME FAILED", flush=True)


if __name__ == "__main__":
    main()
