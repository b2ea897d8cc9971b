"""Multi-GPU partition of the grouped n:m SpMM.

One process per GPU (torchrun), torch.distributed over NCCL for the plumbing.
Two partitions, both with no collective inside the product itself:

* token (column) sharding -- the sparse weight (values, idx) is replicated,
  rank p owns the dense-operand columns [c0_p, c1_p) and computes C[:, c0_p:c1_p];
  an all-gather of the C shards follows only when a consumer needs all of C;
* row sharding -- rank p owns whole groups [p*G/P, (p+1)*G/P) of the weight,
  B is replicated, and the all-gather runs along M (contiguous in C).

Every rank uses the plan of the GLOBAL problem (sten_spmm_plan_query on the
full shape), so the per-column summation order is the same as on one GPU and
the gathered result equals the single-GPU product bit for bit (pin P11).

The all-gather is chunk-pipelined on a side stream: the local column range is
cut into `chunks` pieces; after piece i is computed on the compute stream its
gather is enqueued on the comm stream while piece i+1 computes.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from . import sten


def shard_range(n_total: int, world: int, rank: int, align: int = 8) -> tuple[int, int]:
    """Contiguous, `align`-multiple shard boundaries (the last shard takes the rest)."""
    per = -(-n_total // world)
    per = -(-per // align) * align
    c0 = min(n_total, rank * per)
    c1 = min(n_total, (rank + 1) * per)
    return c0, c1


def group_range(M: int, g: int, world: int, rank: int) -> tuple[int, int]:
    G = M // g
    return (rank * G // world) * g, ((rank + 1) * G // world) * g


class TokenShardedSpmm:
    """C[:, shard] = densify(values, idx) @ B[:, shard] on every rank (+ optional all-gather)."""

    def __init__(self, values, idx, n, m, g, K, N_global, out_dtype=None, chunks: int = 1, group=None):
        self.values, self.idx = values, idx
        self.n, self.m, self.g, self.K = n, m, g, K
        self.M = values.shape[0]
        self.N_global = N_global
        self.out_dtype = out_dtype or values.dtype
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.group = group
        self.plan = sten.spmm_plan(n, m, g, self.M, K, N_global, ab_dtype=values.dtype, c_dtype=self.out_dtype)
        per = -(-N_global // self.world)
        self.n_local = -(-per // 8) * 8
        self.chunks = max(1, chunks)
        self.comm_stream = torch.cuda.Stream() if values.is_cuda else None

    def local_range(self):
        return shard_range(self.N_global, self.world, self.rank)

    def forward_local(self, B_local: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        return sten.spmm_grouped_nm(self.values, self.idx, B_local, self.n, self.m, self.g, out=out,
                                    out_dtype=self.out_dtype, plan=self.plan)

    def forward_allgather(self, B_local: torch.Tensor, gathered: torch.Tensor | None = None) -> torch.Tensor:
        """Compute the local shard chunk by chunk and all-gather each chunk as soon as
        it is done.  Returns [world][M][n_local]; column j of rank p is global column
        p*n_local + j (use `assemble` for a [M][N] view/copy)."""
        M, nl = self.M, self.n_local
        if gathered is None:
            gathered = torch.empty((self.world, M, nl), dtype=self.out_dtype, device=B_local.device)
        n_have = B_local.shape[1]
        local = torch.zeros((M, nl), dtype=self.out_dtype, device=B_local.device)
        step = -(-nl // self.chunks)
        step = -(-step // 8) * 8
        compute = torch.cuda.current_stream()
        # gather chunk-wise into [world][chunk][M][step] staging, then scatter to layout
        bounds = [(c, min(nl, c + step)) for c in range(0, nl, step)]
        stage = [torch.empty((self.world, M, c1 - c0), dtype=self.out_dtype, device=B_local.device)
                 for (c0, c1) in bounds]
        for (c0, c1), st in zip(bounds, stage):
            hi = min(c1, n_have)
            piece = torch.empty((M, c1 - c0), dtype=self.out_dtype, device=B_local.device)
            if hi > c0:
                sten.spmm_grouped_nm(self.values, self.idx, B_local[:, c0:hi], self.n, self.m, self.g,
                                     out=piece[:, : hi - c0], plan=self.plan)
            if hi < c1:
                piece[:, max(0, hi - c0):].zero_()
            ev = torch.cuda.Event()
            ev.record(compute)
            with torch.cuda.stream(self.comm_stream):
                self.comm_stream.wait_event(ev)
                dist.all_gather_into_tensor(st, piece, group=self.group)
                piece.record_stream(self.comm_stream)
        compute.wait_stream(self.comm_stream)
        for (c0, c1), st in zip(bounds, stage):
            gathered[:, :, c0:c1].copy_(st)
        del local
        return gathered

    def assemble(self, gathered: torch.Tensor) -> torch.Tensor:
        """[world][M][n_local] -> [M][N_global] (copy)."""
        full = gathered.permute(1, 0, 2).reshape(self.M, self.world * self.n_local)
        return full[:, : self.N_global].contiguous()


class RowShardedSpmm:
    """Rank p owns groups [p*G/P, (p+1)*G/P): C[rows_p, :] = W_p x B, then all-gather along M."""

    def __init__(self, values_local, idx_local, n, m, g, K, M_global, N, out_dtype=None, group=None):
        self.values, self.idx = values_local, idx_local
        self.n, self.m, self.g, self.K = n, m, g, K
        self.M_global, self.N = M_global, N
        self.out_dtype = out_dtype or values_local.dtype
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        # plan of the global shape: same per-column K order on every rank
        self.plan = sten.spmm_plan(n, m, g, M_global, K, N, ab_dtype=values_local.dtype, c_dtype=self.out_dtype)

    def forward_local(self, B: torch.Tensor, out=None) -> torch.Tensor:
        return sten.spmm_grouped_nm(self.values, self.idx, B, self.n, self.m, self.g, out=out,
                                    out_dtype=self.out_dtype, plan=self.plan)

    def forward_allgather(self, B: torch.Tensor) -> torch.Tensor:
        local = self.forward_local(B)
        rows = local.shape[0]
        full = torch.empty((rows * self.world, self.N), dtype=self.out_dtype, device=B.device)
        dist.all_gather_into_tensor(full, local.contiguous(), group=self.group)
        return full
