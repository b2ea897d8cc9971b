"""Multi-process (gloo, world size 2, CPU) tests of the partition / gather logic of
paper_2304_07613_b200.parallel.  The compute step is the CPU oracle (test
infrastructure), injected through the `compute=` hook; on GPUs the same classes
run the C-ABI SpMM (covered by tests/test_gpu_parity.py::test_p11_*)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2304_07613_b200 import parallel


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _oracle_compute(values, idx, n, m, g):
    import oracle

    def fn(B_cols, out):
        C = oracle.spmm(values, idx, np.ascontiguousarray(B_cols.numpy()), n, m, g, with_bound=False)
        out.copy_(torch.from_numpy(C.astype(np.float32)))
        return out
    return fn


def _worker(rank, world, port, mode, result_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import synthetic
        n, m, g, M, K, N = 2, 4, 4, 48, 64, 100
        W = synthetic.weights(M, K, seed=3)
        B = synthetic.activations(K, N, seed=3)
        values, idx = oracle.sparsify(W, n, m, g)
        if mode == "token":
            sh = parallel.TokenShardedSpmm(M, N, torch.float32, "cpu", _oracle_compute(values, idx, n, m, g),
                                           chunks=3)
            c0, c1 = sh.local_range()
            C = sh.forward_allgather(torch.from_numpy(B[:, c0:c1].copy()))
        else:
            r0, r1 = parallel.group_range(M, g, world, rank)
            sh = parallel.RowShardedSpmm(M, g, N, torch.float32, "cpu",
                                         _oracle_compute(values[r0:r1], idx[r0 // g:r1 // g], n, m, g))
            C = sh.forward_allgather(torch.from_numpy(B))
        ref = oracle.spmm(values, idx, B, n, m, g, with_bound=False).astype(np.float32)
        ok = C.shape == (M, N) and np.array_equal(C.numpy(), ref)
        with open(result_path + ".%d" % rank, "w") as f:
            f.write("ok" if ok else "mismatch %s" % (C.shape,))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["token", "row"])
def test_sharded_equals_unsharded_gloo(tmp_path, mode):
    world = 2
    path = str(tmp_path / "res")
    mp.start_processes(_worker, args=(world, _free_port(), mode, path), nprocs=world, join=True,
                       start_method="spawn")
    for r in range(world):
        assert open(path + ".%d" % r).read() == "ok"


def test_shard_ranges_cover_and_align():
    for N in [1, 7, 8, 100, 1024, 65536, 65537]:
        for world in [1, 2, 3, 4, 8]:
            ranges = [parallel.shard_range(N, world, r) for r in range(world)]
            covered = [c for (a, b) in ranges for c in range(a, b)]
            assert covered == list(range(N))
            assert all(a % 8 == 0 for a, b in ranges if b > a)
    for M, g in [(768, 4), (8192, 128), (64, 16)]:
        for world in [1, 2, 4, 8]:
            rows = [parallel.group_range(M, g, world, r) for r in range(world)]
            assert rows[0][0] == 0 and rows[-1][1] == M
            assert all(r0 % g == 0 and r1 % g == 0 for r0, r1 in rows)
            assert all(rows[i][1] == rows[i + 1][0] for i in range(world - 1))
